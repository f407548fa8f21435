# register-block transpose: tests, bandwidth vs the previous build, wide round
python -m pytest tests/test_gpu_dense.py -q -x -k transpose 2>&1 | tail -2
python tools/transpose_bench.py > gpurun_out/transpose_new.json 2>&1; cat gpurun_out/transpose_new.json | tr -d '\n '; echo
GHC_LIB_PATH=_ab/libghc_head.so python tools/transpose_bench.py > gpurun_out/transpose_head.json 2>&1; cat gpurun_out/transpose_head.json | tr -d '\n '; echo
python tools/wide_bench.py 2>&1 | tail -1
GHC_LIB_PATH=_ab/libghc_head.so python tools/wide_bench.py 2>&1 | tail -1
