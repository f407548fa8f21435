# round-2 validation: new GPU tests first, then the full GPU suite, then the bench
python -m pytest tests/test_gpu_c2.py -x -q > gpurun_out/t_c2.log 2>&1; tail -30 gpurun_out/t_c2.log
python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; tail -15 gpurun_out/t_all.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench20.json 2>gpurun_out/bench20.err; tail -c 3000 gpurun_out/bench20.json; tail -5 gpurun_out/bench20.err
