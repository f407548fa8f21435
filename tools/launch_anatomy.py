"""Where the fixed per-call cost of the persistent round launch goes.

For launches of R rounds (CUDA events around each call) with the %globaltimer
phase probe on: event time vs the in-kernel span (first CTA's round-0 start →
last CTA's last-round commit), the first round's duration vs the steady
rounds, and the same for back-to-back launches.  Also the driver-shaped bench
(20 timed rounds) with and without an nvidia-smi sampler running, to separate
the sampler's perturbation from the launch cost.
"""
import json
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
B = 1000
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(96, 9500)
x, y = g.generate(spec)
rng = np.random.default_rng(0)
idx = rng.integers(0, len(y), size=4000 * B).astype(np.int32)
dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
out = {}
for _ in range(3):  # warm
    m.sync_rounds(dx, dy, di, B, B, 2000)
ctx.sync()

maxc = int(ctx.lib.ghc_plan_max_clusters(arch.h))
cs = int(ctx.lib.ghc_plan_cluster_size(arch.h))
warps = min(8, max(1, -(-B // (maxc * cs))))
ctas = min(maxc, -(-(-(-B // warps)) // cs)) * cs
for R in (1, 2, 20):
    probe = ctx.array(R * ctas * 16, np.uint64)
    probe.zero()
    ctx.lib.ghc_plan_set_probe(arch.h, probe.ptr)
    ctx.sync()
    ctx.timer_start()
    m.sync_rounds(dx, dy, di, B, B, R)
    ms = ctx.timer_stop()
    ctx.lib.ghc_plan_set_probe(arch.h, None)
    pr = probe.numpy().reshape(R, ctas, 16).astype(np.int64)
    start = pr[0, :, 0].min()
    end = pr[R - 1, :, 13].max()
    r_dur = [(pr[r, :, 13].max() - pr[r, :, 0].min()) / 1e3 for r in range(R)]
    entry, exit_ = pr[0, :, 14].min(), pr[R - 1, :, 15].max()
    out[f"R{R}"] = {"event_us": ms * 1e3, "in_kernel_span_us": (end - start) / 1e3,
                    "entry_to_round0_us": (start - entry) / 1e3,
                    "last_commit_to_exit_us": (exit_ - end) / 1e3,
                    "entry_spread_us": float(pr[0, :, 14].max() - entry) / 1e3,
                    "outside_rounds_us": ms * 1e3 - (end - start) / 1e3,
                    "round_us": r_dur[:3] + ([float(np.median(r_dur[3:]))] if R > 3 else []),
                    "round0_input_wait_us": float(np.median(pr[0, :, 8] - pr[0, :, 0])) / 1e3,
                    "cta_start_spread_us": float(pr[0, :, 0].max() - pr[0, :, 0].min()) / 1e3}


def driver_shape():
    mm = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    mm.sync_rounds(dx, dy, di, B, B, 5)
    for _ in range(50):
        mm.sync_rounds(dx, dy, di, B, B, 25)
    ctx.sync()
    ctx.timer_start()
    mm.sync_rounds(dx, dy, di, B, B, 20, idx_offset=5 * B)
    return ctx.timer_stop() * 1e3 / 20


def gated(R):
    mm = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    mm.sync_rounds(dx, dy, di, B, B, 5)
    ctx.sync()
    ctx.hold()
    ctx.timer_start()
    mm.sync_rounds(dx, dy, di, B, B, R, idx_offset=5 * B)
    ctx.release()
    return ctx.timer_stop() * 1e3


out["gated_event_us"] = {R: gated(R) for R in (1, 2, 20, 200)}
out["driver_shape_us_per_round_no_sampler"] = [driver_shape() for _ in range(5)]
p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.DEVNULL)
time.sleep(1.0)
out["driver_shape_us_per_round_with_sampler"] = [driver_shape() for _ in range(5)]
p.terminate()
p.wait()
import ctypes as C  # noqa: E402
lb = {}
smem = 200 * 1024
for v in range(8):
    s1, s2 = C.c_double(), C.c_double()
    rc = ctx.lib.ghc_diag_launch_bench(ctx.h, v, 128, 256, smem, C.byref(s1), C.byref(s2))
    lb[f"coop{v & 1}_cluster{(v >> 1) & 1}_smem{(v >> 2) & 1}"] = (s1.value, s2.value) if rc == 0 else \
        ctx.lib.ghc_last_error().decode()
out["empty_kernel_launch_us_single_b2b"] = lb
print(json.dumps(out, indent=1))
