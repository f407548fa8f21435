"""Long randomised resident command stream (the test's stress, many more
commands): random lengths 1..4, queue depths 1..6, short host pauses,
device / pinned-host batches; final weights and every loss compared bit for
bit with one ordinary launch over the same rounds.  python tools/res_stress.py [n_cmds]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

NC = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
B = 1000
ctx = g.Context(0)
arch = g.Architecture(ctx, "lstm(5,20,10),softmax(20,3)")
rng = np.random.default_rng(11)
lens = rng.integers(1, 5, size=NC)
R = int(lens.sum())
spec = g.data_spec(8, 5000)
x, y = g.generate(spec)
idx = rng.integers(0, len(y), size=R * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
dp = g.pack_dataset(ctx, dx, dy)
w0 = g.init_weights(arch, 7)
ref = g.Master(arch, w0, 0.01, 0.9)
lref = ctx.array(R)
ref.sync_rounds(dp, None, di, B, B, R, loss_out=lref)
hx = ctx.host_array((R * B, 64))
hx.np[:] = g.pack_rows(x[idx], y[idx])
m = g.Master(arch, w0, 0.01, 0.9)
loss = ctx.array(R)
res = g.Resident(m, B, idle_seconds=30.0)
t0 = time.time()
seqs, r0 = [], 0
for k in range(NC):
    n = int(lens[k])
    if rng.random() < 0.5:
        seqs.append(res.submit(dp, None, di, B, n, loss_out=loss, idx_offset=r0 * B, loss_offset=r0))
    else:
        seqs.append(res.submit(hx.sub(r0 * B), None, None, B, n, loss_out=loss, loss_offset=r0))
    r0 += n
    depth = int(rng.integers(1, 7))
    while len(seqs) >= depth:
        res.wait(seqs.pop(0))
    if rng.random() < 0.05:
        time.sleep(float(rng.uniform(0, 5e-4)))
for s in seqs:
    res.wait(s)
res.stop()
wall = time.time() - t0
ok_w = bool(np.array_equal(m.read()[0], ref.read()[0]))
ok_l = bool(np.array_equal(loss.numpy(), lref.numpy()))
print(json.dumps({"commands": NC, "rounds": R, "wall_s": wall, "weights_bit_identical": ok_w,
                  "losses_bit_identical": ok_l, "version": int(m.read()[2])}))
sys.exit(0 if ok_w and ok_l else 1)
