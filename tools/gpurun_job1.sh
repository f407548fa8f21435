#!/bin/bash
# GPU job: smoke, gpu tests, bench, ncu launch list + full capture of the fused kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as e; e.build(); e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?"
CMD="python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 20"
timeout 300 $CMD > gpurun_out/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lstm_softmax -s 2 -c 2 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc $?"
tail -3 gpurun_out/pytest_gpu.log
