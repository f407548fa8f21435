"""GPU: the SPEC roles on device vs the CPU oracle runners.

Configs from BASELINE.json: c2-shaped sync Downpour with W workers, c3 EASGD
(8 workers, α=0.5, τ=10, round-robin "sync" and a replayed async order), c4
async Downpour (8 workers, replayed arrival order), c5 hierarchical 2×4.
Tolerance: ‖Δw‖₂/‖w‖₂ ≤ 1e-5 and max|Δw| ≤ 1e-5 after the
whole run (fp32 device vs f64 reference with the f32 wire); integer
accounting (versions, samples, staleness) exact.
"""
import numpy as np
import pytest

from conftest import BENCH_ARCH

import paper_1712_05878_b200 as g

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def close(w, wo, tol=1e-5):
    r, m = rel(w, wo), float(np.max(np.abs(np.asarray(w, np.float64) - wo)))
    assert r <= tol and m <= tol, (r, m)


def oracle_data(oracle, nf, spf):
    spec = oracle.data_spec(nf, spf)
    x, y = oracle.generate(spec)
    return spec, x, y


@pytest.mark.parametrize("W,B,epochs", [(1, 100, 1), (4, 50, 1), (8, 64, 2), (3, 70, 1)])
def test_sync_downpour_virtual_workers(ctx, oracle, W, B, epochs):
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(n_workers=W, batch_size=B, epochs=epochs),
                  g.data_spec(8, 300))
    loss, _ = s.run()
    out = s.read()
    spec, x, y = oracle_data(oracle, 8, 300)
    r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), spec, x, y,
                        oracle.train_cfg(n_workers=W, batch_size=B, epochs=epochs))
    assert out["version"] == r.stats.updates and out["samples"] == r.stats.samples
    close(out["w"], r.w)
    assert np.max(np.abs(loss[: len(r.loss)] - r.loss) / r.loss) <= 1e-4


def test_async_downpour_replay_c4(ctx, oracle):
    W = 8
    arch = g.Architecture(ctx, BENCH_ARCH)
    cfg = g.train_config(n_workers=W, batch_size=40, epochs=1, mode=g.REPLAY)
    s = g.Session(arch, cfg, g.data_spec(16, 200))
    rng = np.random.default_rng(3)
    # a feasible arrival order: each worker has 5 batches
    order = np.repeat(np.arange(W, dtype=np.int32), 5)
    rng.shuffle(order)
    loss, stale = s.run(order)
    out = s.read()
    spec, x, y = oracle_data(oracle, 16, 200)
    r = oracle.run_replay(oracle.parse_arch(BENCH_ARCH), spec, x, y,
                          oracle.train_cfg(n_workers=W, batch_size=40, epochs=1), order)
    assert np.array_equal(stale, r.extra["staleness"])
    assert out["version"] == r.stats.updates == len(order)
    close(out["w"], r.w)
    for k in range(W):  # each worker holds the weights of its last reply
        close(out["worker_w"][k], r.extra["worker_w"][k])


@pytest.mark.parametrize("replay", [False, True])
def test_easgd_c3(ctx, oracle, replay):
    W = 8
    arch = g.Architecture(ctx, BENCH_ARCH)
    kw = dict(algo=g.EASGD, n_workers=W, batch_size=25, epochs=2, alpha=0.5, tau=10, lr=0.05)
    s = g.Session(arch, g.train_config(mode=g.REPLAY if replay else g.SYNC, **kw),
                  g.data_spec(16, 200))
    n_batches = 2 * (400 // 25)
    if replay:
        order = np.repeat(np.arange(W, dtype=np.int32), n_batches)
        np.random.default_rng(11).shuffle(order)
    else:
        order = np.tile(np.arange(W, dtype=np.int32), n_batches)
    loss, _ = s.run(order if replay else None)
    out = s.read()
    spec, x, y = oracle_data(oracle, 16, 200)
    r = oracle.run_replay(oracle.parse_arch(BENCH_ARCH), spec, x, y,
                          oracle.train_cfg(algo=oracle.EASGD, n_workers=W, batch_size=25,
                                           epochs=2, alpha=0.5, tau=10, lr=0.05), order)
    assert out["version"] == r.stats.updates  # center version = exchanges
    close(out["w"], r.w)
    for k in range(W):
        close(out["worker_w"][k], r.extra["worker_w"][k])


def test_hierarchical_c5_shape(ctx, oracle):
    """2 sub-masters × 4 workers → top master (flush K=2, pass-through parent)."""
    arch = g.Architecture(ctx, BENCH_ARCH)
    kw = dict(n_workers=8, batch_size=40, epochs=1, groups=2, flush_k=2)
    s = g.Session(arch, g.train_config(**kw), g.data_spec(16, 200))
    s.run()
    out = s.read()
    spec, x, y = oracle_data(oracle, 16, 200)
    r = oracle.run_hier(oracle.parse_arch(BENCH_ARCH), spec, x, y, oracle.train_cfg(**kw))
    assert out["version"] == r.stats.updates and out["samples"] == r.stats.samples
    close(out["w"], r.w)
    for q in range(2):
        close(out["group_w"][q], r.extra["group_w"][q])


def test_hierarchical_pass_through_equals_flat(ctx):
    """AC11 on device: 1 group × 1 worker, K=1, parent (η=1, μ=0) ≡ flat."""
    arch = g.Architecture(ctx, BENCH_ARCH)
    flat = g.Session(arch, g.train_config(n_workers=1, batch_size=50, epochs=1),
                     g.data_spec(2, 200))
    flat.run()
    hier = g.Session(arch, g.train_config(n_workers=1, batch_size=50, epochs=1, groups=1,
                                          flush_k=1), g.data_spec(2, 200))
    hier.run()
    assert np.max(np.abs(flat.read()["w"] - hier.read()["w"])) <= 1e-6


def test_session_config_errors(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    with pytest.raises(g.ConfigError):
        g.Session(arch, g.train_config(n_workers=5), g.data_spec(4, 10))  # more workers than files
    with pytest.raises(g.ConfigError):
        g.Session(arch, g.train_config(algo=g.EASGD, alpha=1.0), g.data_spec(4, 10))
    with pytest.raises(g.ShapeError):
        g.Session(arch, g.train_config(), g.data_spec(4, 10, n_classes=4))
    s = g.Session(arch, g.train_config(n_workers=2, mode=g.REPLAY), g.data_spec(4, 10))
    with pytest.raises(g.ConfigError):
        s.run()  # replay needs an order
    with pytest.raises(g.ProtocolError):
        g.Session(arch, g.train_config(n_workers=2, mode=g.REPLAY, batch_size=10),
                  g.data_spec(4, 10)).run(np.zeros(3, np.int32))  # worker 0 has 2 batches


def test_validate_vs_oracle(ctx, oracle):
    """ghc_validate: correct count exact, mean loss ≤ 1e-5."""
    arch = g.Architecture(ctx, BENCH_ARCH)
    spec, x, y = oracle_data(oracle, 4, 500)
    a = oracle.parse_arch(BENCH_ARCH)
    for w in (g.init_weights(arch, 7), np.zeros(arch.n_params)):
        acc, lo, ok = g.validate(w, arch, x.astype(np.float32), y)
        oko, loo = oracle.validate(a, np.asarray(w, np.float32).astype(np.float64), x, y)
        assert ok == oko and acc == oko / len(y)
        assert abs(lo - loo) / loo <= 1e-5
    with pytest.raises(g.ConfigError):
        g.validate(g.init_weights(arch, 7), arch, x[:0].astype(np.float32), y[:0])


@pytest.mark.parametrize("mode", ["sync", "replay"])
def test_session_validation_cadence(ctx, oracle, mode):
    """Validation every V master updates and once at the end (SPEC.md:378,
    384); each record equals ghc_validate of the weights at that version, and
    V = 0 leaves only the final record."""
    W, B, V = 4, 50, 5
    arch = g.Architecture(ctx, BENCH_ARCH)
    spec, x, y = oracle_data(oracle, 8, 300)
    hx, hy = x[:400].astype(np.float32), y[:400]
    kw = dict(n_workers=W, batch_size=B, epochs=1)
    if mode == "replay":
        kw["mode"] = g.REPLAY
    order = np.repeat(np.arange(W, dtype=np.int32), 12) if mode == "replay" else None
    recs = {}
    for every in (V, 0):
        s = g.Session(arch, g.train_config(**kw), g.data_spec(8, 300))
        s.set_validation(hx, hy, every)
        s.run(order)
        recs[every] = s.validations()
        out = s.read()
    n_upd = out["version"]
    assert [r[0] for r in recs[V]] == list(range(V, n_upd + 1, V)) + \
        ([n_upd] if n_upd % V else [])
    assert len(recs[0]) == 1 and recs[0][0][0] == n_upd
    acc, lo, _ = g.validate(out["w"], arch, hx, hy)
    assert recs[V][-1][1] == acc == recs[0][0][1] and abs(recs[V][-1][2] - lo) <= 1e-6 * lo


@pytest.mark.parametrize("delta,lo,hi", [(5.0, 0.90, 1.0), (0.0, 0.0, 0.45)])
def test_end_to_end_learning_ac10(ctx, delta, lo, hi):
    """SPEC.md:629 (AC10): on the synthetic dataset at desk scale (10 files ×
    500 samples), a W = 4 async Downpour run (replayed arrival order) for
    E = 10 epochs reaches held-out accuracy ≥ 0.90 at δ = 5; at δ = 0 the
    classes are indistinguishable and accuracy stays near chance (1/3)."""
    W, B, E = 4, 100, 10
    arch = g.Architecture(ctx, BENCH_ARCH)
    spec = g.data_spec(10, 500, delta=delta)
    n_b = [len(g.batches(spec, W, k, B, E, 99)) for k in range(W)]
    order = np.concatenate([np.full(n, k, np.int32) for k, n in enumerate(n_b)])
    np.random.default_rng(5).shuffle(order)
    s = g.Session(arch, g.train_config(n_workers=W, batch_size=B, epochs=E, mode=g.REPLAY), spec)
    # held-out set: files 10, 11 of the same dataset (same class trajectories,
    # fresh samples; generation is determined by (spec, file index))
    hx, hy = g.generate(g.data_spec(12, 500, delta=delta), 10, 2)
    s.set_validation(hx, hy, 0)
    loss, _ = s.run(order)
    (ver, acc, vloss), = s.validations()
    assert ver == len(order) and lo <= acc <= hi, (acc, vloss)


def test_async_downpour_c4_b1000(ctx, oracle):
    """c4 at the benchmark batch: 8 workers × B = 1000, 64 replayed arrivals."""
    W, B = 8, 1000
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(n_workers=W, batch_size=B, epochs=1, mode=g.REPLAY),
                  g.data_spec(16, 4000))
    order = np.repeat(np.arange(W, dtype=np.int32), 8)  # 8 batches per worker
    np.random.default_rng(7).shuffle(order)
    loss, stale = s.run(order)
    out = s.read()
    spec, x, y = oracle_data(oracle, 16, 4000)
    r = oracle.run_replay(oracle.parse_arch(BENCH_ARCH), spec, x, y,
                          oracle.train_cfg(n_workers=W, batch_size=B, epochs=1), order)
    assert np.array_equal(stale, r.extra["staleness"])
    assert out["version"] == r.stats.updates == len(order) and out["samples"] == r.stats.samples
    close(out["w"], r.w)


def test_easgd_c3_b1000(ctx, oracle):
    """c3 at the benchmark batch: 8 workers, α = 0.5, τ = 10, B = 1000, 2 epochs."""
    W, B = 8, 1000
    kw = dict(algo=g.EASGD, n_workers=W, batch_size=B, epochs=2, alpha=0.5, tau=10, lr=0.05)
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(mode=g.SYNC, **kw), g.data_spec(16, 4000))
    s.run(None)
    out = s.read()
    order = np.tile(np.arange(W, dtype=np.int32), 2 * 8)
    spec, x, y = oracle_data(oracle, 16, 4000)
    r = oracle.run_replay(oracle.parse_arch(BENCH_ARCH), spec, x, y,
                          oracle.train_cfg(algo=oracle.EASGD, n_workers=W, batch_size=B, epochs=2,
                                           alpha=0.5, tau=10, lr=0.05), order)
    assert out["version"] == r.stats.updates
    close(out["w"], r.w)
    for k in range(W):
        close(out["worker_w"][k], r.extra["worker_w"][k])


def test_hierarchical_c5_b1000(ctx, oracle):
    """c5's topology at the benchmark batch: 2 sub-masters × 4 workers,
    B = 1000 per worker, flush K = 2 into the pass-through top master."""
    kw = dict(n_workers=8, batch_size=1000, epochs=1, groups=2, flush_k=2)
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(**kw), g.data_spec(16, 4000))
    s.run()
    out = s.read()
    spec, x, y = oracle_data(oracle, 16, 4000)
    r = oracle.run_hier(oracle.parse_arch(BENCH_ARCH), spec, x, y, oracle.train_cfg(**kw))
    assert out["version"] == r.stats.updates and out["samples"] == r.stats.samples
    close(out["w"], r.w)
    for q in range(2):
        close(out["group_w"][q], r.extra["group_w"][q])
