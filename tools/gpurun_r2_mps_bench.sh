# bench.py's N > 1 path (torchrun, one rank per process, fused NVLink-path
# exchange) end to end with all ranks on ONE GPU under MPS — validates the
# SCALE run's code path (the numbers are not a scaling measurement: the ranks
# share one device)
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export GHC_BENCH_DEVICE=0
for N in 2 4 8; do
GHC_MAX_CTAS=$((128 / N)) timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $((29700 + N)) bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/mps_bench_n$N.json 2> gpurun_out/mps_bench_n$N.err
echo "N=$N rc $?"; tail -c 400 gpurun_out/mps_bench_n$N.json; echo
GHC_MAX_CTAS=$((128 / N)) timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $((29710 + N)) bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/mps_ref_n$N.json 2> gpurun_out/mps_ref_n$N.err
echo "ref N=$N rc $?"; tail -c 200 gpurun_out/mps_ref_n$N.json; echo
done
echo quit | nvidia-cuda-mps-control; echo "mps down"
