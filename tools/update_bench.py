"""HBM roofline of every master-update / exchange-combine kernel (SURVEY §8(d):
SGD-momentum 20 B/param, EASGD center 12 B/param, pull 12 B/param, weighted
mean (W+1)·4 B/param) at the wide variant's P = 16,881,699, each launch
preceded by a 256 MB L2 write-flush, CUDA events on the context stream.

    python tools/update_bench.py            # JSON line per kernel
    python tools/update_bench.py --once     # one launch each (for ncu -k regex:...)
"""
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_05878_b200 as g  # noqa: E402
from paper_1712_05878_b200 import gradhub  # noqa: E402

WIDE = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"
P = 16_881_699
W = 8


def peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if k in d:
                return float(d[k]), "measured"
        for v in d.values():
            if isinstance(v, dict) and "hbm_gbs" in v:
                return float(v["hbm_gbs"]), "measured"
    except (OSError, ValueError):
        pass
    return 6532.5, "fallback"


def main():
    once = "--once" in sys.argv
    ctx = g.Context(0)
    rng = np.random.default_rng(0)
    w0 = rng.normal(size=P).astype(np.float32)
    w, v, c = ctx.upload(w0), ctx.upload(np.zeros(P, np.float32)), ctx.upload(w0 * 0.5)
    gr = ctx.upload((rng.normal(size=P) * 1e-3).astype(np.float32))
    slots = ctx.upload(np.tile((rng.normal(size=P) * 1e-3).astype(np.float32), W))
    out = ctx.array(P)
    st = ctx.array(1, np.int32)
    ver = ctx.array(2, np.int32)  # uint64 version
    flush = ctx.array(64 << 20)
    counts_arr = (C.c_double * W)(*[1000.0 + k for k in range(W)])
    counts = C.cast(counts_arr, C.c_void_p)
    lib = ctx.lib
    arch = g.Architecture(ctx, WIDE)
    m = g.Master(arch, w0, 0.01, 0.9)
    ck = gradhub.check
    cases = [
        ("sgd_db_kernel", "ghc_master_apply (one pass, double-buffered)", 20,
         lambda: m.apply(gr)),
        ("sgd_apply_kernel", "ghc_sgd_apply (in place)", 20,
         lambda: ck(lib.ghc_sgd_apply(ctx.h, w.ptr, v.ptr, gr.ptr, P, 0.01, 0.9, st.ptr, None))),
        ("easgd_worker_kernel", "ghc_easgd_worker_step, pull round (batch_index % tau == 0)", 16,
         lambda: ck(lib.ghc_easgd_worker_step(ctx.h, w.ptr, c.ptr, gr.ptr, P, 0.01, 0.5, 10, 0,
                                              st.ptr))),
        ("elastic_kernel", "ghc_elastic_pull", 12,
         lambda: ck(lib.ghc_elastic_pull(ctx.h, w.ptr, c.ptr, P, 0.5))),
        ("elastic_kernel", "ghc_easgd_center_step", 12,
         lambda: ck(lib.ghc_easgd_center_step(ctx.h, c.ptr, w.ptr, P, 0.5, ver.ptr))),
        ("weighted_mean_kernel", f"ghc_weighted_mean, {W} slots", 4 * (W + 1),
         lambda: ck(lib.ghc_weighted_mean(ctx.h, out.ptr, slots.ptr, counts, W, P))),
    ]
    pk, kind = peak_gbs()
    for kernel, api, bpp, fn in cases:
        times = []
        for it in range(1 if once else 23):
            flush.zero()
            ctx.timer_start()
            fn()
            t = ctx.timer_stop()
            if it >= 3 or once:
                times.append(t)
        t = statistics.median(times)
        gbs = bpp * P / (t / 1e3) / 1e9
        print(json.dumps({"kernel": kernel, "api": api, "P": P, "bytes_per_param": bpp,
                          "ms": t, "achieved_gbs": gbs, "peak_gbs": pk, "peak_kind": kind,
                          "frac": gbs / pk, "l2": "256 MB write-flush before every launch"}),
              flush=True)


if __name__ == "__main__":
    main()
