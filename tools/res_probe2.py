"""Resident service, queued 1-round host commands: where a command's time goes
(probe: round start / phases / commit per CTA, tlog: doorbell seen / done)."""
import ctypes as C
import os
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
B = 1000
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
idx = np.random.default_rng(0).integers(0, len(y), size=300 * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
G = 128
probe = ctx.array(1 * G * 16, np.uint64)
probe.zero()
ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
res = g.Resident(m, B, idle_seconds=30.0)
ctx.lib.ghc_plan_set_probe(arch.h, None)
import time  # noqa: E402
HOST = "--host" in sys.argv
if HOST:  # per-call batches in pinned host memory (packed rows), as the bench's per_call
    xp = g.pack_rows(x[idx[:40 * B]], y[idx[:40 * B]])
    hx = ctx.host_array(xp.shape)
    hx.np[:] = xp
DEPTH = int(os.environ.get("DEPTH", "3"))
seqs = []
t0 = time.perf_counter()
for k in range(30):
    if HOST:
        seqs.append(res.submit(hx.sub(k * B), None, None, 0, 1))
    else:
        seqs.append(res.submit(dx, dy, di, B, 1, idx_offset=k * B))
    if k >= DEPTH - 1:
        res.wait(seqs[k - DEPTH + 1])
res.wait(seqs[-1])
wall = (time.perf_counter() - t0) * 1e6 / 30
t = (C.c_uint64 * 133)()
ctx.lib.ghc_resident_times(res.h, t)
t = [int(v) for v in t]
res.stop()
s = seqs[-1]
bell, done = t[5 + 2 * (s % 64)], t[6 + 2 * (s % 64)]
prev_done = t[6 + 2 * ((s - 1) % 64)]
pr = probe.numpy().reshape(G, 16).astype(np.int64)
bells = [t[5 + 2 * (q % 64)] for q in seqs[10:29]]
dones = [t[6 + 2 * (q % 64)] for q in seqs[10:29]]
out = {"host_batches": HOST, "wall_us_per_call": wall,
       "prev_done_to_bell_seen_us": (bell - prev_done) / 1e3,
       "bell_seen_to_first_round_start_us": (pr[:, 0].min() - bell) / 1e3,
       "round_start_spread_us": (pr[:, 0].max() - pr[:, 0].min()) / 1e3,
       "round_us": (pr[:, 13].max() - pr[:, 0].min()) / 1e3,
       "x_wait_us": float(np.median(pr[:, 8] - pr[:, 0])) / 1e3,
       "samples_us": float(np.median(pr[:, 2] - pr[:, 0])) / 1e3,
       "last_commit_to_done_us": (done - pr[:, 13].max()) / 1e3,
       "bell_seen_to_done_us": (done - bell) / 1e3,
       "bell_to_bell_us_median": float(np.median(np.diff(bells))) / 1e3,
       "done_to_done_us_median": float(np.median(np.diff(dones))) / 1e3}
print(json.dumps(out, indent=1))
