#!/bin/bash
# ncu launch list (per-launch durations) of a short bench run; plain run first
mkdir -p gpurun_out
export GHC_NO_COOP=1  # ncu cannot replay cooperative cluster launches
CMD="python bench.py --steps 200 --warmup 3 --no-cpu --e2e-steps 20"
timeout 300 $CMD > gpurun_out/bench_small.log 2>&1; echo "plain rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc $?"
