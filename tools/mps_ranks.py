"""PROCESSES (one rank each, 2..8), running the fused cross-rank sync round
(ghc_p2p_sync_rounds) against each other on ONE GPU under MPS — the
multi-process code path of a multi-GPU run (CUDA-IPC-mapped receive rows,
system-scope tagged stores and polls, the xepoch hand-over between launches)
with the same device standing in for the peer.  Each process's persistent
grid is capped (GHC_MAX_CLUSTERS) so both fit side by side.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mps_ranks.py

Checks: the two ranks' master replicas are bit-identical; both match the
oracle's 2-worker sync Downpour (BASELINE.md bound 1e-5); versions exact;
splitting the rounds over several launches gives the same bits."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import torch.distributed as tdist  # noqa: E402

import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import dist as gd  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
tdist.init_process_group("gloo")
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
W, B, epochs, nf, spf = world, int(os.environ.get("MPS_B", "100")), 1, 8, int(os.environ.get("MPS_SPF", "300"))
spec = g.data_spec(nf, spf)
x, y = g.generate(spec)  # the shared dataset (every rank holds all of it here)
plans = [gd.plan_worker(spec, W, k, B, epochs, 99) for k in range(W)]
counts = gd.round_counts(spec, W, B, epochs, 99)
R = counts.shape[0]
if os.environ.get("MPS_R"):  # first MPS_R rounds only (diagnostics)
    R = min(R, int(os.environ["MPS_R"]))
    counts = np.ascontiguousarray(counts[:R])
p = plans[rank]
idx = np.zeros(R * B, np.int32)
nr = min(p.rounds, R)
idx[: nr * B] = (p.idx_local + p.row0)[: nr * B]
dx, dy, di, dc = ctx.upload(x), ctx.upload(y), ctx.upload(idx), ctx.upload(counts)
res = {}
for split in ((R,) if os.environ.get("MPS_R") else (R, 7)):
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    ex = gd.P2PExchange(arch, rank, world, dist=tdist)
    loss = ctx.array(R)
    for r0 in range(0, R, split):
        n = min(split, R - r0)
        ex.device_barrier()  # ghc_p2p_barrier across the processes (start alignment)
        ex.sync_rounds(m, dx, dy, di, B, 0, dc, B, n, loss_out=loss, idx_offset=r0 * B,
                       counts_offset=r0 * world, loss_offset=r0)
    ctx.sync()
    w, v, ver, rej = m.read()
    ex.close()
    res[split] = (w, ver, rej, loss.numpy())
    tdist.barrier()
allw = [None] * world
tdist.all_gather_object(allw, res[R][0].tobytes())
out = {"rank": rank, "rounds": int(R), "version": int(res[R][1]), "rejected": int(res[R][2]),
       "replicas_bit_identical": all(a == allw[0] for a in allw),
       "split_launches_bit_identical": bool(np.array_equal(res[R][0], res[7][0])) if 7 in res else None}
if rank == 0:
    from oracle import oracle  # the checker (test infrastructure only)
    oracle.lib()
    so = oracle.data_spec(nf, spf)
    xo, yo = oracle.generate(so)
    r = oracle.run_sync(oracle.parse_arch(ARCH), so, xo, yo,
                        oracle.train_cfg(n_workers=W, batch_size=B, epochs=epochs, max_updates=R))
    w = res[R][0]
    out["oracle_updates"] = int(r.stats.updates)
    out["rel_err_vs_oracle"] = float(np.linalg.norm(w.astype(np.float64) - r.w) / np.linalg.norm(r.w))
    out["max_abs_err_vs_oracle"] = float(np.max(np.abs(w - r.w)))
    ok = (out["replicas_bit_identical"] and out["split_launches_bit_identical"] is not False and
          out["version"] == r.stats.updates == R and out["rel_err_vs_oracle"] <= 1e-5 and
          out["max_abs_err_vs_oracle"] <= 1e-5)
    out["ok"] = bool(ok)
    print(json.dumps(out), flush=True)
tdist.barrier()
