"""Rounds reading their batches from pinned HOST memory (the e2e path: packed
dataset rows + shuffled indices in host memory, the kernel gathers over PCIe
one round ahead) vs the same from device memory: per-phase probe medians."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
B, R = 1000, 200
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
idx = np.random.default_rng(0).integers(0, len(y), size=R * B).astype(np.int32)
xp = g.pack_rows(x, y)
hX = ctx.host_array(xp.shape)
hX.np[:] = xp
hI = ctx.host_array(R * B, np.int32)
hI.np[:] = idx
dX = ctx.upload(xp)
dI = ctx.upload(idx)
G = 128
out = {}
for name, (X, I) in {"device": (dX, dI), "host": (hX, hI)}.items():
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    m.sync_rounds(X, None, I, B, B, 5)
    ctx.sync()
    probe = ctx.array(R * G * 16, np.uint64)
    probe.zero()
    ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
    ctx.timer_start()
    m.sync_rounds(X, None, I, B, B, R)
    ms = ctx.timer_stop()
    ctx.lib.ghc_plan_set_probe(arch.h, None)
    pr = probe.numpy().reshape(R, G, 16).astype(np.int64)[10:R - 2]
    med = lambda a: float(np.median(a)) / 1e3  # noqa: E731
    out[name] = {"us_per_round_event": 1e3 * ms / R,
                 "round_span_us": med(pr[:, :, 13].max(axis=1) - pr[:, :, 0].min(axis=1)),
                 "x_wait_us": med(np.median(pr[:, :, 8] - pr[:, :, 0], axis=1)),
                 "x_wait_max_us": med(np.max(pr[:, :, 8] - pr[:, :, 0], axis=1)),
                 "samples_us": med(np.median(pr[:, :, 2] - pr[:, :, 0], axis=1)),
                 "samples_max_us": med(np.max(pr[:, :, 2] - pr[:, :, 0], axis=1)),
                 "start_spread_us": med(pr[:, :, 0].max(axis=1) - pr[:, :, 0].min(axis=1))}
print(json.dumps(out, indent=1))
