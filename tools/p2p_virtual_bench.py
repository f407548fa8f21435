"""µs per sync round of the fused cross-rank exchange with G virtual ranks on
one GPU (total batch fixed at 1000: 1000/G per rank, the grid split between
ranks) vs the single-rank round — the exchange's added cost, measured with
local memory standing in for NVLink peer memory."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import dist as gd  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
R = 2000
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
dx, dy = ctx.upload(x), ctx.upload(y)
rng = np.random.default_rng(0)
out = {}
for G in (1, 2, 4):
    B = 1000 // G
    idx = rng.integers(0, len(y), size=(G, R * B)).astype(np.int32)
    di = ctx.upload(idx)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    if G == 1:
        run = lambda n: m.sync_rounds(dx, dy, di, B, B, n)  # noqa: E731
    else:
        ex = gd.P2PExchange(arch, 0, G, virtual=True)
        dc = ctx.upload(np.full((R, G), B, np.int32))
        run = lambda n: ex.sync_rounds(m, dx, dy, di, B, R * B, dc, B, n)  # noqa: E731
    run(20)
    ctx.sync()
    ctx.timer_start()
    run(R)
    ms = ctx.timer_stop()
    out[G] = 1e3 * ms / R
print(json.dumps({"us_per_round_by_virtual_ranks": out}))
