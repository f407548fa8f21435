# CTA-pair GEMM: correctness vs f64, speed vs the single-CTA kernel, wide round
timeout 300 python -m pytest tests/test_gpu_dense.py -x -q -m gpu 2>&1 | tail -5
timeout 200 python tools/gemm_bench.py 2>&1 | tail -3
GHC_GEMM=single timeout 200 python tools/gemm_bench.py 2>&1 | tail -3
timeout 300 python tools/wide_bench.py 2>&1 | tail -2
