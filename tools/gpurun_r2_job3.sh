python -m pytest tests/test_gpu_c2.py tests/test_gpu_adapter.py tests/test_gpu_wide.py -q -x > gpurun_out/t3.log 2>&1; tail -40 gpurun_out/t3.log
./paper_1712_05878_b200/_build/adapter_roles_selftest > gpurun_out/roles.log 2>&1; tail -30 gpurun_out/roles.log
