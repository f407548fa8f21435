"""HBM roofline of the device wire codec (codec.cu) on the wide variant's
GRADIENT frame (P = 16,881,699 → 67.5 MB f32 / 135 MB f64): algorithmic
bytes = parameters read + frame written (pack), frame read + parameters
written (unpack); a 256 MB buffer is cleared before every launch (L2 flush)."""
import ctypes as C
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

WIDE = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"
ctx = g.Context(0)
arch = g.Architecture(ctx, WIDE)
P = arch.n_params
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6532.5)
w = ctx.upload((np.random.default_rng(0).normal(size=P) * 0.1).astype(np.float32))
flush = ctx.array(64 << 20)
out = {}
for f64 in (0, 1):
    n = C.c_int64(0)
    ctx.lib.ghc_frame_size(arch.h, 2, f64, C.byref(n))
    fr = ctx.array(n.value, np.uint8)
    w2 = ctx.array(P)
    ln = C.c_int64(0)
    tp, tu = [], []
    for it in range(13):
        flush.zero()
        ctx.timer_start()
        g.gradhub.check(ctx.lib.ghc_encode_frame(arch.h, 2, f64, w.ptr, 1, 1, fr.ptr, n.value, C.byref(ln)))
        t = ctx.timer_stop()
        flush.zero()
        k, f, st = C.c_int32(), C.c_int32(), C.c_int32()
        v, c = C.c_uint64(), C.c_uint64()
        ctx.timer_start()
        g.gradhub.check(ctx.lib.ghc_decode_frame(arch.h, fr.ptr, n.value, C.byref(k), w2.ptr, C.byref(v),
                                         C.byref(c), C.byref(f), C.byref(st)))
        u = ctx.timer_stop()
        if it >= 3:
            tp.append(t)
            tu.append(u)
    bytes_ = 4 * P + n.value
    tpm, tum = statistics.median(tp), statistics.median(tu)
    out["f64" if f64 else "f32"] = {
        "frame_bytes": n.value, "algorithmic_bytes": bytes_,
        "pack_ms": tpm, "pack_gbs": bytes_ / tpm / 1e6, "pack_frac": bytes_ / tpm / 1e6 / peak,
        "unpack_ms_incl_host_header_parse": tum, "unpack_gbs": bytes_ / tum / 1e6,
        "round_trip_exact": bool(np.array_equal(w2.numpy(), w.numpy())) if not f64 else None}
out["peak_gbs"] = peak
print(json.dumps(out, indent=1))
