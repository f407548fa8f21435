"""HBM roofline of every master-update / exchange-combine kernel (SURVEY §8(d):
SGD-momentum 20 B/param, EASGD center 12 B/param, pull 12 B/param, weighted
mean (W+1)·4 B/param) at the wide variant's P = 16,881,699.

Steady-state streaming: each kernel runs back to back over NSET = 8 distinct
buffer sets (8 × the working set ≫ the 126 MB L2), so no launch reuses L2
data and every launch pays the write-back of its predecessor's dirty lines;
the CUDA-event time of the NSET launches / NSET is one launch.

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
NSET = 8


def peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6532.5, "fallback"


def main():
    once = "--once" in sys.argv
    nset = 1 if once else NSET
    ctx = g.Context(0)
    rng = np.random.default_rng(0)
    w0 = rng.normal(size=P).astype(np.float32)
    sets = []
    for _ in range(nset):
        sets.append(dict(w=ctx.upload(w0), v=ctx.upload(np.zeros(P, np.float32)),
                         c=ctx.upload(w0 * 0.5),
                         g=ctx.upload((rng.normal(size=P) * 1e-3).astype(np.float32)),
                         slots=ctx.upload(np.tile((rng.normal(size=P) * 1e-3).astype(np.float32), W)),
                         out=ctx.array(P), w2=ctx.array(P), v2=ctx.array(P)))
    st = ctx.array(1, np.int32)
    ver = ctx.array(2, np.int32)  # uint64 version
    counts_arr = (C.c_double * W)(*[1000.0 + k for k in range(W)])
    counts = C.cast(counts_arr, C.c_void_p)
    lib = ctx.lib
    arch = g.Architecture(ctx, WIDE)
    masters = [g.Master(arch, w0, 0.01, 0.9) for _ in range(nset)]
    ck = gradhub.check
    cases = [
        ("sgd_db_kernel", "ghc_master_apply (one pass, double-buffered)", 20,
         lambda i, s: masters[i].apply(s["g"])),
        ("sgd_apply_kernel", "ghc_sgd_apply (in place)", 20,
         lambda i, s: ck(lib.ghc_sgd_apply(ctx.h, s["w"].ptr, s["v"].ptr, s["g"].ptr, P, 0.01, 0.9,
                                           st.ptr, None))),
        ("sgd_out_kernel", "ghc_sgd_step_out (value semantics, one pass)", 20,
         lambda i, s: ck(lib.ghc_sgd_step_out(ctx.h, s["w"].ptr, s["v"].ptr, s["g"].ptr, s["w2"].ptr,
                                              s["v2"].ptr, P, 0.01, 0.9, st.ptr, None))),
        ("easgd_worker_out_kernel", "ghc_easgd_worker_step_out, pull round (one pass)", 16,
         lambda i, s: ck(lib.ghc_easgd_worker_step_out(ctx.h, s["w"].ptr, s["c"].ptr, s["g"].ptr,
                                                       s["w2"].ptr, P, 0.01, 0.5, 10, 0, st.ptr))),
        ("easgd_worker_kernel", "ghc_easgd_worker_step, pull round (batch_index % tau == 0)", 16,
         lambda i, s: ck(lib.ghc_easgd_worker_step(ctx.h, s["w"].ptr, s["c"].ptr, s["g"].ptr, P, 0.01,
                                                   0.5, 10, 0, st.ptr))),
        ("elastic_kernel", "ghc_elastic_pull", 12,
         lambda i, s: ck(lib.ghc_elastic_pull(ctx.h, s["w"].ptr, s["c"].ptr, P, 0.5))),
        ("elastic_kernel", "ghc_easgd_center_step", 12,
         lambda i, s: ck(lib.ghc_easgd_center_step(ctx.h, s["c"].ptr, s["w"].ptr, P, 0.5, ver.ptr))),
        ("weighted_mean_kernel", f"ghc_weighted_mean, {W} slots", 4 * (W + 1),
         lambda i, s: ck(lib.ghc_weighted_mean(ctx.h, s["out"].ptr, s["slots"].ptr, counts, W, P))),
    ]
    pk, kind = peak_gbs()
    for kernel, api, bpp, fn in cases:
        times = []
        for it in range(1 if once else 8):
            ctx.sync()
            ctx.timer_start()
            for i, s in enumerate(sets):
                fn(i, s)
            t = ctx.timer_stop() / nset
            if it >= 2 or once:
                times.append(t)
        t = statistics.median(times)
        gbs = bpp * P / (t / 1e3) / 1e9
        print(json.dumps({"kernel": kernel, "api": api, "P": P, "bytes_per_param": bpp,
                          "ms": t, "achieved_gbs": gbs, "peak_gbs": pk, "peak_kind": kind,
                          "frac": gbs / pk,
                          "l2": f"steady-state streaming over {nset} distinct buffer sets"}),
              flush=True)


if __name__ == "__main__":
    main()
