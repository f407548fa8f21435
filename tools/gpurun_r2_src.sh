# source-level stall sampling of the current ordinary round kernel (CS=4)
export GHC_NO_COOP=1
ncu --section SourceCounters --section WarpStateStats --section LaunchStats --clock-control none --import-source on \
  -k regex:lstm_round_kernel -s 2 -c 1 -o gpurun_out/r02_src python bench.py --gpus 1 --steps 400 --warmup 5 --no-cpu --e2e-steps 20 > gpurun_out/ncu_src.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/r02_src.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_src_cs.csv 2>gpurun_out/src_err.log; echo "export rc $?"; head -c 600 gpurun_out/r02_src_cs.csv
