"""Fixed per-call cost of the persistent sync-round launch (VERDICT r1 'weak #4').

Times ONE ghc_master_sync_rounds call of R rounds for several R (CUDA events,
median of repeats) after a given amount of warm-up, and fits t(R) = a + b*R:
`a` is the fixed cost of a call (launch, cold first round, state load/publish),
`b` the steady-state round.  Also times the driver's bench shape (5 warm-up
rounds in one call, then 20 timed rounds in one call) with and without a
longer GPU warm-up before it, to separate clock ramp-up from per-call cost.
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
RMAX = 20000
idx = rng.integers(0, len(y), size=RMAX * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
w0 = g.init_weights(arch, 7)
out = {}


def once(m, R, off=0):
    ctx.timer_start()
    m.sync_rounds(dx, dy, di, B, B, R, idx_offset=off * B)
    return ctx.timer_stop()


# (1) the driver's shape on a cold process: 5 warm-up rounds, then 20 timed
m = g.Master(arch, w0, 0.01, 0.9)
m.sync_rounds(dx, dy, di, B, B, 5)
ctx.sync()
out["driver_shape_cold_us_per_round"] = 1e3 * once(m, 20, 5) / 20
out["driver_shape_cold_2nd_us_per_round"] = 1e3 * once(m, 20, 25) / 20

# (2) after ~1 s of continuous rounds (clocks up, caches warm)
t0 = time.time()
while time.time() - t0 < 1.0:
    m.sync_rounds(dx, dy, di, B, B, 2000)
    ctx.sync()
out["driver_shape_warm_us_per_round"] = 1e3 * once(m, 20, 5) / 20

# (3) fit t(R) = a + b R
rows = {}
for R in (1, 2, 5, 10, 20, 50, 100, 200, 1000, 5000):
    ts = [once(m, R) for _ in range(15)]
    rows[R] = statistics.median(ts) * 1e3  # µs
Rs = np.array(list(rows.keys()), float)
ts = np.array(list(rows.values()), float)
b, a = np.polyfit(Rs, ts, 1)
out["call_us_by_rounds"] = rows
out["fit_fixed_us"] = a
out["fit_round_us"] = b

# (4) back-to-back 1-round calls (launch queue full): per-call throughput
ctx.sync()
ctx.timer_start()
for k in range(200):
    m.sync_rounds(dx, dy, di, B, B, 1, idx_offset=k * B)
out["b2b_1round_us"] = 1e3 * ctx.timer_stop() / 200
print(json.dumps(out, indent=1))
