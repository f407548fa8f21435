"""The SPEC roles on one GPU with virtual workers (session.cu) at the
benchmark batch: samples/s and µs per master update for c2-shaped sync
Downpour (8 workers), c3 EASGD (8 workers, α = 0.5, τ = 10), c4 replayed
async Downpour (8 workers) and c5 hierarchical (2 × 4), B = 1000 per worker.
One session run each after a warm-up run; wall clock around Session.run
(synchronising).  These are the c3-c5 configs of BASELINE.json measured on
one device — the reference's threaded CPU roles are the comparison point
(bench.py --impl reference runs c2)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_05878_b200 as g  # noqa: E402

ARCH = "lstm(5,20,10),softmax(20,3)"
W, B = 8, 1000
ctx = g.Context(0)
arch = g.Architecture(ctx, ARCH)
spec = g.data_spec(16, 8000)  # 2 files x 8000 per worker: 16 batches per worker per epoch
out = {}


def timed(cfg, order=None, epochs_samples=None):
    s = g.Session(arch, cfg, spec)
    s.run(order)  # warm-up (module loads, allocations)
    s = g.Session(arch, cfg, spec)
    ctx.sync()
    t0 = time.perf_counter()
    s.run(order)
    ctx.sync()
    dt = time.perf_counter() - t0
    r = s.read()
    return dt, r


for name, kw, order_fn in [
    ("c2_sync_downpour_8w", dict(n_workers=W, batch_size=B, epochs=2), None),
    ("c3_easgd_8w", dict(algo=g.EASGD, n_workers=W, batch_size=B, epochs=2, alpha=0.5, tau=10, lr=0.05), None),
    ("c4_async_replay_8w", dict(n_workers=W, batch_size=B, epochs=2, mode=g.REPLAY),
     lambda: np.random.default_rng(7).permutation(np.repeat(np.arange(W, dtype=np.int32), 32))),
    ("c5_hierarchical_2x4", dict(n_workers=W, batch_size=B, epochs=2, groups=2, flush_k=2), None),
]:
    order = order_fn() if order_fn else None
    dt, r = timed(g.train_config(**kw), order)
    samples = int(r["samples"]) if "samples" in r else None
    upd = int(r["version"])
    out[name] = {"wall_s": dt, "master_updates": upd, "samples": samples,
                 "samples_per_s": (samples / dt) if samples else None,
                 "us_per_update": 1e6 * dt / max(upd, 1)}
print(json.dumps(out, indent=1))
