"""Resident service, queued 1-round commands: per command (all of them), the
round span (first CTA start → last commit) and the gap from the previous
command's last commit to this command's first round start, from the
%globaltimer probe (indexed by the launch's round counter in the resident
kernel).  DEPTH commands in flight; --host: batches in pinned host memory."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
B, NCMD = 1000, 40
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
idx = np.random.default_rng(0).integers(0, len(y), size=300 * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
G = 128
probe = ctx.array((NCMD + 8) * G * 16, np.uint64)
probe.zero()
ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
res = g.Resident(m, B, idle_seconds=30.0)
HOST = "--host" in sys.argv
LOSS = "--loss" in sys.argv
if HOST:
    xp = g.pack_rows(x[idx[:NCMD * B]], y[idx[:NCMD * B]])
    hx = ctx.host_array(xp.shape)
    hx.np[:] = xp
hl = ctx.host_array(NCMD) if LOSS else None
DEPTH = int(os.environ.get("DEPTH", "3"))
seqs = []
t0 = time.perf_counter()
for k in range(NCMD):
    lo = hl.sub(k) if LOSS else None
    if HOST:
        seqs.append(res.submit(hx.sub(k * B), None, None, 0, 1, loss_out=lo))
    else:
        seqs.append(res.submit(dx, dy, di, B, 1, idx_offset=k * B, loss_out=lo))
    if k >= DEPTH - 1:
        res.wait(seqs[k - DEPTH + 1])
res.wait(seqs[-1])
wall = (time.perf_counter() - t0) * 1e6 / NCMD
res.stop()
ctx.lib.ghc_plan_set_probe(arch.h, None)
pr = probe.numpy().reshape(-1, G, 16).astype(np.int64)[:NCMD]
start = pr[:, :, 0].min(axis=1)
commit = pr[:, :, 13].max(axis=1)
xw = np.median(pr[:, :, 8] - pr[:, :, 0], axis=1)
done_arr = np.median(pr[:, :, 14] - pr[:, :, 13], axis=1)   # commit → arrival issued (per CTA)
next_cmd = np.median(pr[:, :, 15] - pr[:, :, 14], axis=1)   # arrival → next command in hand
to_start = np.median(pr[1:, :, 0] - pr[:-1, :, 15], axis=1)  # next command → its round start
span = (commit - start) / 1e3
gap = (start[1:] - commit[:-1]) / 1e3
sl = slice(10, NCMD - 2)
out = {"host_batches": HOST, "loss_to_host": LOSS, "depth": DEPTH, "wall_us_per_call": wall,
       "round_span_us_median": float(np.median(span[sl])),
       "gap_prev_commit_to_start_us_median": float(np.median(gap[10:NCMD - 2])),
       "gap_us_p90": float(np.percentile(gap[10:NCMD - 2], 90)),
       "x_wait_us_median": float(np.median(xw[sl])) / 1e3,
       "start_to_start_us_median": float(np.median(np.diff(start)[10:NCMD - 2])) / 1e3,
       "cta_commit_to_arrival_us": float(np.median(done_arr[sl])) / 1e3,
       "cta_arrival_to_next_cmd_us": float(np.median(next_cmd[sl])) / 1e3,
       "cta_next_cmd_to_round_start_us": float(np.median(to_start[10:NCMD - 2])) / 1e3,
       "cta_commit_spread_us": float(np.median(pr[sl, :, 13].max(axis=1) - pr[sl, :, 13].min(axis=1))) / 1e3,
       "phase_us_from_round_start": {nm: float(np.median(np.median(pr[sl, :, i] - pr[sl, :, 0], axis=1))) / 1e3
                                     for nm, i in (("x_in", 8), ("fwd", 9), ("softmax", 10), ("bptt", 11),
                                                   ("dW", 12), ("samples", 2), ("push_wait", 4),
                                                   ("row_store", 5), ("subslice_sgd", 6), ("gather_push", 7),
                                                   ("commit", 13))},
       "phase_us_from_round_start_max_cta": {nm: float(np.median(np.max(pr[sl, :, i] - pr[sl, :, 0], axis=1))) / 1e3
                                             for nm, i in (("x_in", 8), ("fwd", 9), ("samples", 2), ("push_wait", 4),
                                                           ("subslice_sgd", 6), ("gather_push", 7), ("commit", 13))},
       "round_start_spread_us": float(np.median(pr[sl, :, 0].max(axis=1) - pr[sl, :, 0].min(axis=1))) / 1e3}
print(json.dumps(out, indent=1))
