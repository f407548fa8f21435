# the wide net's LSTM trunk (flat kernel, TRUNK_FWD / TRUNK_GRAD): where 19 us go
export GHC_NO_COOP=1
ROUNDS=2 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section SpeedOfLight --clock-control none --import-source on \
  -k regex:lstm_softmax_step_kernel -s 2 -c 2 -o gpurun_out/r02_trunk python tools/wide_bench.py > gpurun_out/ncu_trunk.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/r02_trunk.ncu-rep --page details --csv > gpurun_out/r02_trunk_details.csv 2>/dev/null
ncu -i gpurun_out/r02_trunk.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_trunk_src.csv 2>/dev/null
