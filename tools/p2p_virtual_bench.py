"""µs per sync round of the fused cross-rank exchange with G virtual ranks on
one GPU (all ranks' CTAs in ONE grid, peer pointers into one allocation —
the multi-GPU kernel code with local memory standing in for NVLink peer
memory), two ways:

  strong : total batch fixed at 1000 (1000/G per rank), the grid split
           between the ranks — the exchange's added cost per round;
  weak   : B = 1000 per rank (c2's shape: G × 1000 samples per round), the
           SAME grid serving all G ranks, so a rank gets 1/G of the SMs —
           the compute grows G× here, unlike on G real GPUs.

Per round and rank the hop moves EP 8-byte (value, epoch-tag) elements to
every rank (incl. itself): G·EP·8 B pushed, G·EP·8 B polled.  The NVLink
roofline of that hop (900 GB/s per direction per B200) is reported next to
the measured time: the hop is latency-bound, not bandwidth-bound.
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import dist as gd  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
R = 1000
NVLINK_GBS = 900.0
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
dx, dy = ctx.upload(x), ctx.upload(y)
rng = np.random.default_rng(0)
EP = None
out = {"rounds": R, "strong_us_per_round": {}, "weak_us_per_round": {}}


def run(G, B):
    global EP
    idx = rng.integers(0, len(y), size=(G, R * B)).astype(np.int32)
    di = ctx.upload(idx)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    if G == 1:
        fn = lambda n: m.sync_rounds(dx, dy, di, B, B, n)  # noqa: E731
        ex = None
    else:
        ex = gd.P2PExchange(arch, 0, G, virtual=True)
        EP = int(ctx.lib.ghc_p2p_row_elems(ex.h))
        dc = ctx.upload(np.full((R, G), B, np.int32))
        fn = lambda n: ex.sync_rounds(m, dx, dy, di, B, R * B, dc, B, n)  # noqa: E731
    fn(20)
    ctx.sync()
    ctx.hold()
    ctx.timer_start()
    fn(R)
    ctx.release()
    ms = ctx.timer_stop()
    if ex is not None:
        ex.close()
    return 1e3 * ms / R


for G in (1, 2, 4, 8):
    out["strong_us_per_round"][G] = run(G, 1000 // G)
for G in (1, 2, 4, 8):
    out["weak_us_per_round"][G] = run(G, 1000)
out["hop_bytes_per_rank_per_round"] = {G: 2 * G * EP * 8 for G in (2, 4, 8)}
out["hop_nvlink_time_us_at_900GBs"] = {G: 2 * G * EP * 8 / (NVLINK_GBS * 1e3) for G in (2, 4, 8)}
out["EP"] = EP
print(json.dumps(out, indent=1))
