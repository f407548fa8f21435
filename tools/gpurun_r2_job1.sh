set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/fixed_cost.py > gpurun_out/fixed_cost.json 2> gpurun_out/fixed_cost.err
cat gpurun_out/fixed_cost.json
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench20.json 2>gpurun_out/bench20.err; tail -c 600 gpurun_out/bench20.json
