"""One short invocation of every product path, for an ncu launch list of
every kernel the library launches (tools/gpurun_r2_rooflines.sh aggregates
the lists into profiles/r02_kernel_rooflines.md):
  c2 fused sync rounds (packed rows, B = 1000), worker grad / forward /
  validate (bench net), the generic LSTM path (lstm(5,40,10)), the SPEC
  session roles (c3 EASGD, c4 replayed async, c5 hierarchical; 8 virtual
  workers, B = 1000), the virtual-rank fused exchange (4 ranks).
The update kernels, the wide round and the codec have their own drivers
(tools/update_bench.py --once, tools/wide_bench.py, tools/codec_bench.py)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import dist as gd  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
B = 1000
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(16, 2000)
x, y = g.generate(spec)
idx = np.random.default_rng(0).integers(0, len(y), size=8 * B).astype(np.int32)
dxr, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
dx = g.pack_dataset(ctx, dxr, dy)
w0 = g.init_weights(arch, 7)
m = g.Master(arch, w0, 0.01, 0.9)
m.sync_rounds(dx, None, di, B, B, 3)                       # c2 fused rounds
dw = ctx.upload(w0)
gr, ls = ctx.array(arch.n_params), ctx.array(1)
g.worker_grad_device(arch, dw, dxr, dy, B, gr, ls, idx=di)  # worker step
g.forward(w0, arch, x[:B], y[:B])
g.validate(w0, arch, x[:2000], y[:2000])
m.apply(gr)                                                # master apply (bench net)
ga = g.Architecture(ctx, "lstm(5,40,10),softmax(40,3)")    # generic LSTM path
gm = g.Master(ga, g.init_weights(ga, 7), 0.01, 0.9)
gm.sync_rounds(dxr, dy, di, B, B, 2)
ex = gd.P2PExchange(arch, 0, 4, virtual=True)              # virtual-rank fused exchange
dc = ctx.upload(np.full((2, 4), 250, np.int32))
ex.sync_rounds(m, dx, None, di, 250, 0, dc, 250, 2)
ex.close()
sspec = g.data_spec(16, 1000)
for kw, order in [
    (dict(algo=g.EASGD, n_workers=8, batch_size=B, epochs=1, alpha=0.5, tau=2, lr=0.05), None),
    (dict(n_workers=8, batch_size=B, epochs=1, mode=g.REPLAY),
     np.random.default_rng(7).permutation(np.repeat(np.arange(8, dtype=np.int32), 2))),
    (dict(n_workers=8, batch_size=B, epochs=1, groups=2, flush_k=2), None),
]:
    s = g.Session(arch, g.train_config(**kw), sspec)
    s.run(order)
ctx.sync()
print("ok")
