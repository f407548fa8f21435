"""ghc_transpose bandwidth (CUDA events, median of 20 after warm-up):
the wide round's transposes — W1ᵀ (4096×4096), dZᵀ (1000×4096), W0ᵀ
(4096×20).  GB/s = (read + write bytes) / time; a 256 MB L2 flush before
each timed launch (cold) and back-to-back (warm)."""
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import _lib  # noqa: E402

ctx = g.Context(0)
flush = ctx.array(64 * 1024 * 1024)
out = {}
for rows, cols in [(4096, 4096), (1000, 4096), (4096, 20)]:
    x = ctx.upload(np.random.default_rng(0).normal(size=(rows, cols)).astype(np.float32))
    t = ctx.array((cols, rows))
    for mode in ("cold", "warm"):
        ts = []
        for i in range(25):
            if mode == "cold":
                flush.zero()
            ctx.timer_start()
            _lib.check(ctx.lib.ghc_transpose(ctx.h, t.ptr, x.ptr, rows, cols, cols, rows))
            ms = ctx.timer_stop()
            if i >= 5:
                ts.append(ms)
        ms = statistics.median(ts)
        out[f"{rows}x{cols}_{mode}"] = {"us": ms * 1e3, "GBps": 2 * 4 * rows * cols / (ms * 1e-3) / 1e9}
print(json.dumps(out, indent=1))
