#!/bin/bash
# ncu full capture (SASS-level warp-state sampling) of one multi-round launch
# of the fused round kernel (launch #2 of bench.py = the timed launch).
# usage: bash tools/gpu_prof_tc.sh [name] [env...]
mkdir -p gpurun_out
NAME=${1:-prof_tc}
export GHC_NO_COOP=1  # ncu cannot replay cooperative cluster launches
CMD="python bench.py --steps 300 --warmup 3 --no-cpu --e2e-steps 5"
timeout 300 $CMD > gpurun_out/bench_small.log 2>&1; echo "plain rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lstm_round -s 1 -c 1 -o gpurun_out/$NAME $CMD > gpurun_out/ncu_$NAME.log 2>&1; echo "ncu rc $?"
tail -2 gpurun_out/ncu_$NAME.log | cut -c1-300
