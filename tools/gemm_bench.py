"""Dense-layer GEMM (ghc_gemm_nt, tcgen05 kind::tf32 3xTF32) on the wide
variant's shapes: effective fp32 TFLOP/s (2·M·N·K / time) and rel-L2 error vs
an fp64 product, for the TMA warp-specialised kernel (default) and the
register-staged one (GHC_GEMM=legacy, run as a second process)."""
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import _lib  # noqa: E402

ctx = g.Context(0)
out = {"kernel": os.environ.get("GHC_GEMM", "tma")}
for (M, N, K) in [(1000, 4096, 4096), (4096, 4096, 1000), (1000, 4096, 20), (1000, 20, 4096)]:
    rng = np.random.default_rng(1)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    dA, dB, dC = ctx.upload(A), ctx.upload(B), ctx.array((M, N))
    ts = []
    for it in range(8):
        ctx.timer_start()
        _lib.check(ctx.lib.ghc_gemm_nt(ctx.h, dA.ptr, dB.ptr, dC.ptr, M, N, K, K, K, N, 0, 2, None,
                                       None, N, 1.0))
        t = ctx.timer_stop()
        if it >= 2:
            ts.append(t)
    ms = statistics.median(ts)
    Cg = dC.numpy()
    Cr = A.astype(np.float64) @ B.astype(np.float64).T
    out[f"{M}x{N}x{K}"] = {"ms": ms, "tflops_fp32_effective": 2.0 * M * N * K / ms / 1e9,
                            "rel_l2": float(np.linalg.norm(Cg - Cr) / np.linalg.norm(Cr))}
print(json.dumps(out))
