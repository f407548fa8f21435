"""Phase timing of the fused sync-round kernel (diagnostics, GPU only).

    python -m paper_1712_05878_b200.diag [--rounds 200] [--batch 1000]

Enables the %globaltimer probe of ghc_plan_set_probe and prints, per phase,
the median / max over CTAs and rounds (ns): weight load, samples
(forward+backward), partial store, barrier 1, slice reduce + SGD, barrier 2,
and the gap to the next round.
"""
from __future__ import annotations

import argparse
import os
import json

import numpy as np

from . import gradhub as g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=200)
    ap.add_argument("--batch", type=int, default=1000)
    ap.add_argument("--arch", default="lstm(5,20,10),softmax(20,3)")
    ap.add_argument("--barriers", action="store_true", help="grid-barrier micro-benchmark")
    ap.add_argument("--dump", default=None, help="save the raw probe array [rounds][ctas][16] (.npy)")
    ap.add_argument("--p2p", type=int, default=1,
                    help="G > 1: fused cross-rank exchange with G virtual ranks (batch per rank)")
    args = ap.parse_args()
    ctx = g.Context(0)
    if args.barriers:
        import ctypes as C
        res = {}
        for impl, name in enumerate(["atomic_counter", "flag_gather_bcast", "flag_all_poll",
                                     "cluster8_hw", "all_poll_nofence", "column16",
                                     "all_poll_acquire"]):
            for ctas in (128, 144):
                ns = C.c_double()
                rc = ctx.lib.ghc_diag_barrier_bench(ctx.h, impl, ctas, 224, 2000, C.byref(ns))
                res[f"{name}@{ctas}"] = ns.value if rc == 0 else g._lib.load().ghc_last_error().decode()
        print(json.dumps(res, indent=1))
        return
    arch = g.Architecture(ctx, args.arch)
    B, R = args.batch, args.rounds
    spec = g.data_spec(20, 5000)
    x, y = g.generate(spec)
    idx = np.concatenate(g.batches(spec, 1, 0, B, 3, 99)[:R]).astype(np.int32)
    dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    G = args.p2p
    if G > 1:
        from . import dist as gd
        ex = gd.P2PExchange(arch, 0, G, virtual=True)
        idx = np.concatenate([idx] * G)
        di = ctx.upload(idx)
        dc = ctx.upload(np.full((R, G), B, np.int32))
        run = lambda n: ex.sync_rounds(m, dx, dy, di, B, R * B, dc, B, n)  # noqa: E731
    else:
        run = lambda n: m.sync_rounds(dx, dy, di, B, B, n)  # noqa: E731
    run(5)
    maxc = int(ctx.lib.ghc_plan_max_clusters(arch.h))
    cs = int(ctx.lib.ghc_plan_cluster_size(arch.h))
    if maxc > 0:  # = launch_step() in ghc_internal.cuh (cluster variant)
        spw = int(os.environ.get("GHC_SPW_DIAG", "1"))
        mc = maxc // G
        warps = min(8, max(1, -(-B // (mc * cs * spw))))
        ctas = min(mc, -(-(-(-B // (warps * spw))) // cs)) * cs * G
        # ClusterRS (st.async pushes + tagged L2 rows; G > 1 adds the NVLink hop in (c))
        bounds = [(0, 2, "samples"), (2, 3, "cta_partial"), (3, 4, "push_partials_wait"),
                  (4, 5, "cluster_row_store"), (5, 6, "subslice_poll_sgd_store"),
                  (6, 7, "weights_gather_push"), (7, 13, "weights_wait")]
        last = 13
    else:          # = step_geometry()
        sms = ctx.num_sms
        warps = min(8, max(1, -(-B // sms)))
        ctas = -(-B // warps)
        bounds = [(0, 1, "weights"), (1, 2, "samples"), (2, 3, "store_partial"),
                  (3, 4, "barrier1"), (4, 5, "reduce_sgd"), (5, 6, "barrier2")]
        last = 6
    probe = ctx.array(R * ctas * 16, np.uint64)
    probe.zero()
    ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
    ctx.timer_start()
    run(R)
    ms = ctx.timer_stop()
    ctx.lib.ghc_plan_set_probe(arch.h, None)
    pr = probe.numpy().reshape(R, ctas, 16).astype(np.int64)
    used = int((pr[0, :, 0] != 0).sum())
    pr = pr[:, :used, :]
    if args.dump:
        np.save(args.dump, pr)
    out = {"kernel": arch.kernel_name, "max_clusters": maxc, "cluster_size": cs, "warps": warps,
           "rounds": R,
           "ctas": used, "us_per_round": 1e3 * ms / R, "phases_ns": {}}
    for a0, a1, nm in bounds:
        d = pr[:, :, a1] - pr[:, :, a0]
        out["phases_ns"][nm] = {"median": float(np.median(d)), "max": float(d.max())}
    gap = pr[1:, :, 0] - pr[:-1, :, last]
    out["phases_ns"]["next_round_gap"] = {"median": float(np.median(gap)), "max": float(gap.max())}
    inner = ["x_wait", "forward", "softmax", "bptt_chain", "weight_grads"]
    prev = pr[:, :, 0]
    for i, nm in enumerate(inner):
        cur = pr[:, :, 8 + i]
        d = cur - prev
        out["phases_ns"]["sample0_" + nm] = {"median": float(np.median(d)), "max": float(d.max())}
        prev = cur
    # critical path: slowest CTA to finish samples vs fastest
    done = pr[:, :, 3]
    out["samples_done_spread_ns"] = float(np.median(done.max(1) - done.min(1)))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
