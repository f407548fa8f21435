bash tools/gpurun_r2_mps.sh 2>&1 | head -30
bash tools/gpurun_r2_mps_bench.sh 2>&1 | grep -v "^ref\|impl" | head -20
