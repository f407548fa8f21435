# one-launch column sums (colsum4_kernel) in the wide round: layered-path parity, round time, launch list
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_generic.py -q -x -m gpu 2>&1 | tail -2
python tools/wide_bench.py 2>&1 | tail -1
python tools/wide_bench.py 2>&1 | tail -1
ROUNDS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/wide_bench.py > gpurun_out/rl_wide2.csv 2>/dev/null; python tools/rooflines_agg.py "wide=gpurun_out/rl_wide2.csv" | grep -i "colsum\|total\|path"
