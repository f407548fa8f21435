# W processes (one rank each) through the fused cross-rank round on one GPU
# under MPS (the multi-GPU code path with one device standing in for the
# peers); the grids are capped (GHC_MAX_CTAS) so all ranks' persistent
# kernels are co-resident; every step bounded by timeout, MPS shut down at
# the end.  run W cta_cap B samples_per_file
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
run() {
  GHC_MAX_CTAS=$2 MPS_B=$3 MPS_SPF=$4 timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port $((29500 + $1)) tools/mps_ranks.py > gpurun_out/mps_w$1_b$3.log 2>&1
  echo "W=$1 ctas<=$2 B=$3 rc $?"; grep -h "{" gpurun_out/mps_w$1_b$3.log; grep -h "CudaError" gpurun_out/mps_w$1_b$3.log | head -1
}
run 2 64 100 300
run 2 64 1000 2000
run 2 64 256 2000
run 4 32 100 300
run 4 32 500 2000
run 8 16 64 300
run 8 16 250 2000
echo quit | nvidia-cuda-mps-control; echo "mps down"
