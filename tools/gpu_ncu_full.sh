#!/bin/bash
# ncu --set full of ONE launch of a kernel (regex $1, skip $2 launches) in a short bench run
mkdir -p gpurun_out
export GHC_NO_COOP=1
CMD="python bench.py --steps 200 --warmup 3 --no-cpu --e2e-steps 20"
timeout 300 $CMD > gpurun_out/bench_small.log 2>&1; echo "plain rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-1} -c 1 -o gpurun_out/${3:-prof} $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
