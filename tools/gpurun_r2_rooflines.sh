# ncu launch list of every kernel of every product path (cold caches,
# serialised), aggregated into one table: profiles/r02_kernel_rooflines.md
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
run() { timeout 900 ncu --metrics $M --clock-control none --csv $2 > gpurun_out/rl_$1.csv 2> gpurun_out/rl_$1.err; echo "$1 rc $?"; }
run paths "python tools/all_kernels.py"
run update "python tools/update_bench.py --once"
ROUNDS=1 run wide "python tools/wide_bench.py"
run codec "python tools/codec_bench.py"
python tools/rooflines_agg.py "c2 / worker / session / p2p=gpurun_out/rl_paths.csv" "master update=gpurun_out/rl_update.csv" \
  "wide round (c5 net)=gpurun_out/rl_wide.csv" "codec=gpurun_out/rl_codec.csv" > gpurun_out/kernel_rooflines.md
cat gpurun_out/kernel_rooflines.md
