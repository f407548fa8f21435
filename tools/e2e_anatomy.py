"""Where the e2e (host-dataset) round time goes beyond the device-timed one.

Same master, same rounds, CUDA events on the context stream:
  dev_gate   packed dataset + indices in HBM, launch queued behind the gate
             kernel (the bench's `value`)
  dev        the same without the gate (host call inside the events)
  host_gate  packed dataset + indices in pinned host memory (zero-copy
             gather over PCIe), loss to host memory, gate
  host       the same without the gate (the bench's `e2e`)
for K = 20 and 200 rounds per call, medians of 5 calls each; plus the host
wall time of the sync_rounds call itself.
"""
import json
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
B = 1000
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
rng = np.random.default_rng(0)
KMAX = 200
idx = rng.integers(0, len(y), size=KMAX * B).astype(np.int32)
dx = g.pack_dataset(ctx, ctx.upload(x), ctx.upload(y))
di = ctx.upload(idx)
dl = ctx.array(KMAX)
xp = g.pack_rows(x, y)
hX = ctx.host_array(xp.shape)
hX.np[:] = xp
hI = ctx.host_array(KMAX * B, np.int32)
hI.np[:] = idx
hl = ctx.host_array(KMAX)
w0 = g.init_weights(arch, 7)
m = g.Master(arch, w0, 0.01, 0.9)
for _ in range(10):
    m.sync_rounds(dx, None, di, B, B, KMAX)
ctx.sync()
out = {}
for K in (20, KMAX):
    for name, (X, I, L, gate) in {"dev_gate": (dx, di, dl, True), "dev": (dx, di, dl, False),
                                  "host_gate": (hX, hI, hl, True), "host": (hX, hI, hl, False)}.items():
        ts, calls = [], []
        for rep in range(6):
            ctx.sync()
            if gate:
                ctx.hold()
            ctx.timer_start()
            t0 = time.perf_counter()
            m.sync_rounds(X, None, I, B, B, K, loss_out=L)
            calls.append((time.perf_counter() - t0) * 1e6)
            if gate:
                ctx.release()
            ms = ctx.timer_stop()
            ctx.sync()
            if rep:
                ts.append(ms * 1e3 / K)
        out[f"K{K}_{name}"] = {"us_per_round": statistics.median(ts), "host_call_us": statistics.median(calls[1:])}
print(json.dumps(out, indent=1))

# per-phase probe of one gated K = 20 call on each dataset placement
maxc = int(ctx.lib.ghc_plan_max_clusters(arch.h))
cs = int(ctx.lib.ghc_plan_cluster_size(arch.h))
warps = min(8, max(1, -(-B // (maxc * cs))))
ctas = min(maxc, -(-(-(-B // warps)) // cs)) * cs
R = 20
probe_out = {}
for name, (X, I, L) in {"dev": (dx, di, dl), "host": (hX, hI, hl)}.items():
    probe = ctx.array(R * ctas * 16, np.uint64)
    probe.zero()
    ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
    ctx.sync()
    ctx.hold()
    ctx.timer_start()
    m.sync_rounds(X, None, I, B, B, R, loss_out=L)
    ctx.release()
    ms = ctx.timer_stop()
    ctx.sync()
    ctx.lib.ghc_plan_set_probe(arch.h, None)
    pr = probe.numpy().reshape(R, ctas, 16).astype(np.int64)
    start, end = pr[0, :, 0].min(), pr[R - 1, :, 13].max()
    entry, exit_ = pr[0, :, 14].min(), pr[R - 1, :, 15].max()
    probe_out[name] = {"event_us": ms * 1e3, "in_kernel_span_us": (end - start) / 1e3,
                       "entry_to_round0_us": (start - entry) / 1e3,
                       "last_commit_to_exit_us": (exit_ - end) / 1e3,
                       "outside_kernel_body_us": ms * 1e3 - (exit_ - entry) / 1e3,
                       "round_us": [(pr[r, :, 13].max() - pr[r, :, 0].min()) / 1e3 for r in range(R)],
                       "round0_input_wait_us": float(np.median(pr[0, :, 8] - pr[0, :, 0])) / 1e3,
                       "round1_input_wait_us": float(np.median(pr[1, :, 8] - pr[1, :, 0])) / 1e3}
print(json.dumps(probe_out, indent=1))
