"""Bit-level A/B of two builds of libghc (GHC_LIB_PATH): 50 sync rounds of
the c2 bench net (B = 1000, shuffled batches) from the same init; prints a
hash of the final weights, velocity and per-round losses.  Used to confirm
that an instruction-level change (e.g. FFMA → FFMA2 pairs) is bit-identical."""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

B, R = 1000, 50
ctx = g.Context(0)
arch = g.Architecture(ctx, "lstm(5,20,10),softmax(20,3)")
x, y = g.generate(g.data_spec(96, 9500))
idx = np.random.default_rng(5).integers(0, len(y), size=R * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
loss = ctx.array(R)
m.sync_rounds(dx, dy, di, B, B, R, loss_out=loss)
ctx.sync()
w, v, ver, rej = m.read()
h = hashlib.sha256(w.tobytes() + v.tobytes() + loss.numpy().tobytes()).hexdigest()[:16]
print(g._lib.LIB_PATH, h, ver, rej, float(loss.numpy()[-1]) / B)
