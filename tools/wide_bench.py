"""Wide variant (lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),
softmax(4096,3), P = 16.9 M) sync rounds on one GPU: samples/s and the
per-kernel time split (CUDA events per launch are not available inside
ghc_master_sync_rounds, so the split comes from an ncu launch list)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

WIDE = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"
B, R = 1000, int(os.environ.get("ROUNDS", "20"))
ctx = g.Context(0)
arch = g.Architecture(ctx, WIDE)
spec = g.data_spec(8, 5000)
x, y = g.generate(spec)
idx = np.random.default_rng(0).integers(0, len(y), size=(R + 3) * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
m.sync_rounds(dx, dy, di, B, B, 3)
ctx.sync()
ctx.timer_start()
m.sync_rounds(dx, dy, di, B, B, R, idx_offset=3 * B)
ms = ctx.timer_stop()
print(json.dumps({"arch": WIDE, "batch": B, "rounds": R, "ms_per_round": ms / R,
                  "samples_per_s": B * R / (ms / 1e3),
                  "tflops_fp32_effective": 101_330_944 * B * R / (ms / 1e3) / 1e12,
                  "kernel_name": arch.kernel_name, "gemm": os.environ.get("GHC_GEMM", "tma")}))
