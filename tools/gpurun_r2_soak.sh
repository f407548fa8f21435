# soak: 1,000,000 fused rounds in one launch (no hang, finite losses, weights
# replica check vs a split run), resident stress, and the N = 8 bench under
# MPS three times (the SCALE run's code path)
python - <<'PY'
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1712_05878_b200 as g
ctx = g.Context(0)
arch = g.Architecture(ctx, "lstm(5,20,10),softmax(20,3)")
x, y = g.generate(g.data_spec(20, 5000))
B, R = 1000, 1_000_000
dx = g.pack_dataset(ctx, ctx.upload(x), ctx.upload(y))
m = g.Master(arch, g.init_weights(arch, 7), 0.001, 0.9)
loss = ctx.array(R)
t0 = time.time()
m.sync_rounds(dx, None, None, 0, B, R, loss_out=loss)  # rows 0..999 every round (no index stream)
ctx.sync()
dt = time.time() - t0
l = loss.numpy() / B
w, v, ver, rej = m.read()
print({"rounds": R, "wall_s": round(dt, 2), "us_per_round": round(dt / R * 1e6, 3), "version": int(ver),
       "rejected": int(rej), "loss_first": float(l[0]), "loss_last": float(l[-1]),
       "all_finite": bool(np.isfinite(l).all() and np.isfinite(w).all())})
PY
python tools/res_stress.py 2>&1 | tail -1
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export GHC_BENCH_DEVICE=0
for i in 1 2 3; do
GHC_MAX_CTAS=16 timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port $((29800 + i)) bench.py --gpus 8 --steps 20 --warmup 5 > gpurun_out/soak_n8_$i.json 2> gpurun_out/soak_n8_$i.err
echo "N=8 run $i rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/soak_n8_$i.json').read().splitlines()[-1]); print(d['n_gpus'], round(d['ms_per_step']*1e3,2), d['training'])"
done
echo quit | nvidia-cuda-mps-control; echo "mps down"
