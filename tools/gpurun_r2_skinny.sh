# SIMT partials for narrow split-K products (N <= 32): GEMM accuracy tests,
# wide / generic parity, wide round time, launch list (vs GHC_SKINNY=tc)
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_wide.py tests/test_gpu_generic.py -q -x -m gpu 2>&1 | tail -2
python tools/wide_bench.py 2>&1 | tail -1
GHC_SKINNY=tc python tools/wide_bench.py 2>&1 | tail -1
python tools/wide_bench.py 2>&1 | tail -1
ROUNDS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/wide_bench.py > gpurun_out/rl_wide3.csv 2>/dev/null; python tools/rooflines_agg.py "wide=gpurun_out/rl_wide3.csv" | grep -i "skinny\|splitk\|tma_kernel<32>\|path"
