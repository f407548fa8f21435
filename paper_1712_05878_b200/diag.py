"""Phase timing of the fused sync-round kernel (diagnostics, GPU only).

    python -m paper_1712_05878_b200.diag [--rounds 200] [--batch 1000]

Enables the %globaltimer probe of ghc_plan_set_probe and prints, per phase,
the median / max over CTAs and rounds (ns): weight load, samples
(forward+backward), partial store, barrier 1, slice reduce + SGD, barrier 2,
and the gap to the next round.
"""
from __future__ import annotations

import argparse
import json

import numpy as np

from . import gradhub as g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=200)
    ap.add_argument("--batch", type=int, default=1000)
    ap.add_argument("--arch", default="lstm(5,20,10),softmax(20,3)")
    args = ap.parse_args()
    ctx = g.Context(0)
    arch = g.Architecture(ctx, args.arch)
    B, R = args.batch, args.rounds
    spec = g.data_spec(20, 5000)
    x, y = g.generate(spec)
    idx = np.concatenate(g.batches(spec, 1, 0, B, 3, 99)[:R]).astype(np.int32)
    dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    m.sync_rounds(dx, dy, di, B, B, 5)
    sms = ctx.num_sms
    warps = min(8, max(1, -(-B // sms)))
    ctas = -(-B // warps)  # = step_geometry() in ghc_internal.cuh
    probe = ctx.array(R * ctas * 8, np.uint64)
    probe.zero()
    ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
    ctx.timer_start()
    m.sync_rounds(dx, dy, di, B, B, R)
    ms = ctx.timer_stop()
    ctx.lib.ghc_plan_set_probe(arch.h, None)
    pr = probe.numpy().reshape(R, ctas, 8).astype(np.int64)
    used = (pr[0, :, 0] != 0).sum()
    pr = pr[:, :used, :]
    names = ["weights", "samples", "store_partial", "barrier1", "reduce_sgd", "barrier2"]
    out = {"rounds": R, "ctas": int(used), "us_per_round": 1e3 * ms / R, "phases_ns": {}}
    for i, nm in enumerate(names):
        d = pr[:, :, i + 1] - pr[:, :, i]
        out["phases_ns"][nm] = {"median": float(np.median(d)), "max": float(d.max()),
                                "mean": float(d.mean())}
    gap = pr[1:, :, 0] - pr[:-1, :, 6]
    out["phases_ns"]["next_round_gap"] = {"median": float(np.median(gap)), "max": float(gap.max())}
    # critical path: slowest CTA to finish samples vs fastest
    done = pr[:, :, 3]
    out["samples_done_spread_ns"] = float(np.median(done.max(1) - done.min(1)))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
