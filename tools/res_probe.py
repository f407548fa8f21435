import json, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1712_05878_b200 as g
ARCH = "lstm(5,20,10),softmax(20,3)"; B = 1000
ctx = g.Context(0); arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500); x, y = g.generate(spec)
idx = np.random.default_rng(0).integers(0, len(y), size=300 * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
R = 20; G = 128
probe = ctx.array(R * G * 16, np.uint64); probe.zero()
ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
res = g.Resident(m, B, idle_seconds=30.0)
res.submit_stream(dx, dy, di, B, 5); ctx.sync()
res.submit_stream(dx, dy, di, B, R); ctx.sync()
res.stop()
ctx.lib.ghc_plan_set_probe(arch.h, None)
pr = probe.numpy().reshape(R, G, 16).astype(np.int64)
names = {(0,2):"samples",(2,3):"cta_partial",(3,4):"push_wait",(4,5):"row_store",(5,6):"subslice_sgd",(6,7):"gather_push",(7,13):"w_wait"}
for r in (0, 1, 10):
    d = {nm: float(np.median(pr[r,:,b]-pr[r,:,a])) for (a,b),nm in names.items()}
    d["round"] = float(pr[r,:,13].max() - pr[r,:,0].min())
    d["x_wait_s0"] = float(np.median(pr[r,:,8]-pr[r,:,0]))
    d["start_spread"] = float(pr[r,:,0].max()-pr[r,:,0].min())
    print(r, json.dumps(d))
