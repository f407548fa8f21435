#!/bin/bash
# bench (plain) + ncu launch list + ncu full capture of the fused round kernel
mkdir -p gpurun_out
export GHC_NO_COOP=1  # ncu cannot replay cooperative cluster launches
CMD="python bench.py --steps 200 --warmup 3 --no-cpu --e2e-steps 20"
timeout 300 $CMD > gpurun_out/bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lstm_round -s 2 -c 1 -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc $?"
timeout 600 ncu --set full --clock-control none -k regex:sgd_apply -s 5 -c 1 -o gpurun_out/prof_sgd $CMD > gpurun_out/ncu_sgd.log 2>&1; echo "ncu3 rc $?"
