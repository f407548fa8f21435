"""CPU: the oracle (gh_oracle.c) pinned against the reference's golden vectors
and, where oracle/_ref was built, against the reference library itself
(bit-exact).  Mirrors SPEC.md's ACCEPTANCE CRITERIA where the oracle can
check them on CPU (AC1, AC2, AC3, AC8, AC11)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import BENCH_ARCH

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def unhex(v):
    return np.array([float.fromhex(s) for s in v])


def test_mix_seed_and_mt19937_64(oracle):
    L = oracle.lib()
    # std::mt19937_64 with the default seed 5489: 10000th draw is
    # 9981545732273789042 (C++11 [rand.predef]).
    r = (C.c_uint8 * C.sizeof(C.c_uint64 * 320))()
    L.gho_rng_seed(C.byref(r), 5489)
    v = 0
    for _ in range(10000):
        v = L.gho_rng_u64(C.byref(r))
    assert v == 9981545732273789042
    assert L.gho_mix_seed(0, 0) == L.gho_mix_seed(0, 0)
    assert L.gho_mix_seed(7, 0) != L.gho_mix_seed(7, 1)


def test_spec_examples_match_golden(oracle):
    # sgd μ=0, η=0.1, w=1, g=2 → 0.8
    rc, w, v = oracle.sgd_step([1.0], [0.0], [2.0], 0.1, 0.0)
    assert rc == oracle.OK and w[0] == GOLD["sgd_mu0"]["w1"] == 0.8
    # two steps μ=0.9, g=1
    w, v = np.array([1.0]), np.array([0.0])
    for _ in range(2):
        _, w, v = oracle.sgd_step(w, v, [1.0], 0.1, 0.9)
    assert w[0] == GOLD["sgd_two_steps"]["w_after"]
    # NaN rejects the whole update, w untouched (optim.cpp:49-51)
    rc, w, _ = oracle.sgd_step([1.0, 1.0], [0.0, 0.0], [0.0, np.nan], 0.1, 0.0)
    assert rc == GOLD["sgd_nan_rc"] == oracle.NONFINITE and list(w) == [1.0, 1.0]
    assert oracle.sgd_step([1.0], [0.0], [0.0], 0.0, 0.0)[0] == GOLD["sgd_lr0_rc"]
    assert oracle.sgd_step([1.0], [0.0], [0.0], 0.1, 1.0)[0] == GOLD["sgd_mu1_rc"]
    L = oracle.lib()
    w = np.array([2.0]); c = np.array([0.0])
    L.gho_easgd_worker_step(oracle._p(w), oracle._p(c), oracle._p(np.zeros(1)), 1, 0.01, 0.5, 1, 0)
    assert w[0] == GOLD["easgd_pull_half"]
    w = np.array([8.0])
    out = []
    for bi in range(2):
        L.gho_easgd_worker_step(oracle._p(w), oracle._p(c), oracle._p(np.zeros(1)), 1, 0.01, 0.25, 1, bi)
        out.append(w[0])
    assert out == GOLD["easgd_pull_quarter_twice"]
    c = np.array([0.0])
    assert L.gho_easgd_center_step(oracle._p(c), oracle._p(np.array([4.0])), 1, 0.5) == oracle.OK
    assert c[0] == GOLD["easgd_center_mid"]["c"]
    # α = 1 is rejected by the code (SPEC.md:164 disagrees; the code wins)
    assert L.gho_easgd_center_step(oracle._p(c), oracle._p(np.array([4.0])), 1, 1.0) == \
        GOLD["easgd_center_alpha1_rc"] == oracle.CONFIG


def test_zero_weights_uniform(oracle):
    a = oracle.parse_arch(BENCH_ARCH)
    x = np.random.default_rng(0).normal(size=(6, 50))
    y = np.array([0, 1, 2, 0, 1, 2], np.int32)
    g, p, lo = oracle.forward_backward(a, np.zeros(oracle.n_params(a)), x, y)
    assert np.array_equal(p.ravel(), unhex(GOLD["zero_weights"]["probs"]))
    assert lo == float.fromhex(GOLD["zero_weights"]["loss"])
    assert abs(lo - np.log(3)) < 1e-15
    # code gives 1/K - freq for the output bias (SPEC.md:85 states the opposite sign)
    assert np.array_equal(g[-3:], unhex(GOLD["zero_weights"]["bias_grad"]))


@pytest.mark.parametrize("name", ["bench", "small"])
def test_nn_golden_bitexact(oracle, name):
    d = GOLD[f"nn_{name}"]
    a = oracle.parse_arch(d["arch"])
    w = oracle.init_weights(a, d["seed"])
    assert np.array_equal(w, unhex(d["w"]))
    assert str(oracle.lib().gho_weights_checksum(C.byref(a), oracle._p(w))) == d["checksum"]
    x = unhex(d["x"]).reshape(9, -1)
    g, p, lo = oracle.forward_backward(a, w, x, np.array(d["y"], np.int32))
    assert np.array_equal(g, unhex(d["grad"]))
    assert np.array_equal(p.ravel(), unhex(d["probs"]))
    assert lo == float.fromhex(d["loss"])


def test_data_golden(oracle):
    spec = oracle.data_spec(10, 500)
    x, y = oracle.generate(spec)
    d = GOLD["data_desk"]
    assert np.array_equal(x[0], unhex(d["x_first_row"]))
    assert float(x.sum()) == float.fromhex(d["x_sum"])
    assert np.bincount(y).tolist() == d["label_counts"]
    idx = oracle.epoch_indices(spec, 2, 1, 3, 99)
    assert idx[:40].tolist() == GOLD["epoch_indices_w2_k1_e3"]


def test_sync_c1_golden(oracle):
    spec = oracle.data_spec(10, 500)
    x, y = oracle.generate(spec)
    a = oracle.parse_arch(BENCH_ARCH)
    cfg = oracle.train_cfg(n_workers=2, batch_size=100, epochs=1, max_updates=20)
    r = oracle.run_sync(a, spec, x, y, cfg)
    assert np.array_equal(r.w, unhex(GOLD["sync_c1_20"]["w"]))
    assert np.array_equal(r.loss, unhex(GOLD["sync_c1_20"]["loss"]))


def test_shard_files_partition(oracle):
    L = oracle.lib()
    for n_files, W in [(100, 10), (5, 1), (7, 3), (96, 8), (13, 5)]:
        sizes, seen = [], []
        for k in range(W):
            f0, nf = C.c_int32(), C.c_int32()
            assert L.gho_shard_files(n_files, W, k, C.byref(f0), C.byref(nf)) == 0
            sizes.append(nf.value)
            seen.extend(range(f0.value, f0.value + nf.value))
        assert seen == list(range(n_files))
        assert max(sizes) - min(sizes) <= 1
    assert L.gho_shard_files(3, 4, 0, C.byref(C.c_int32()), C.byref(C.c_int32())) == oracle.CONFIG
    f0, nf = C.c_int32(), C.c_int32()
    L.gho_shard_files(7, 3, 0, C.byref(f0), C.byref(nf))
    assert nf.value == 3  # SPEC.md:439 (7,3) → {3,2,2}


def test_epoch_is_permutation(oracle):
    spec = oracle.data_spec(7, 33)
    for k in range(3):
        a = oracle.epoch_indices(spec, 3, k, 0, 5)
        b = oracle.epoch_indices(spec, 3, k, 0, 5, shuffle=False)
        assert sorted(a.tolist()) == b.tolist()
        assert not np.array_equal(a, b)
        assert not np.array_equal(a, oracle.epoch_indices(spec, 3, k, 1, 5))


@pytest.mark.parametrize("arch", ["dense(50,6,tanh),softmax(6,3)",
                                  "dense(50,5,relu),dense(5,4,identity),softmax(4,3)",
                                  "lstm(5,4,10),softmax(4,3)", "lstm(5,3,10),dense(3,4,tanh),softmax(4,3)"])
def test_gradcheck_ac1(oracle, arch):
    """AC1: backward vs central differences, eps=1e-5, 1e-4."""
    a = oracle.parse_arch(arch)
    w = oracle.init_weights(a, 11)
    x, y = oracle.generate(oracle.data_spec(1, 12))
    g, _, _ = oracle.forward_backward(a, w, x, y)
    fd = oracle.finite_diff(a, w, x, y, 1e-5)
    assert np.max(np.abs(g - fd) / np.maximum(1.0, np.abs(g))) < 1e-4


def test_serial_equivalence_ac2(oracle):
    """AC2: 1 worker, async, f64 wire ≡ a serial sgd loop on the same stream."""
    a = oracle.parse_arch(BENCH_ARCH)
    spec = oracle.data_spec(2, 300)
    x, y = oracle.generate(spec)
    cfg = oracle.train_cfg(n_workers=1, batch_size=50, epochs=2, wire_f64=1, mu=0.5)
    steps = 24
    r = oracle.run_replay(a, spec, x, y, cfg, np.zeros(steps, np.int32))
    w = oracle.init_weights(a, 7); v = np.zeros_like(w)
    for b in oracle_batches(oracle, spec, 1, 0, 50, 2, 99)[:steps]:
        g, _, _ = oracle.forward_backward(a, w, x[b], y[b])
        _, w, v = oracle.sgd_step(w, v, g, 0.01, 0.5)
    assert np.max(np.abs(r.w - w) / np.maximum(1e-300, np.abs(w))) <= 1e-12
    assert np.all(r.extra["staleness"] == 0)


def oracle_batches(O, spec, W, k, B, epochs, seed):
    out = []
    for e in range(epochs):
        idx = O.epoch_indices(spec, W, k, e, seed)
        out.extend(idx[i:i + B] for i in range(0, len(idx), B))
    return out


def test_sync_equals_weighted_serial_ac3(oracle):
    """AC3: sync W=4 ≡ serial SGD on the 4-way sample-weighted mean (f64 wire)."""
    a = oracle.parse_arch(BENCH_ARCH)
    spec = oracle.data_spec(8, 100)
    x, y = oracle.generate(spec)
    cfg = oracle.train_cfg(n_workers=4, batch_size=30, epochs=1, wire_f64=1)
    r = oracle.run_sync(a, spec, x, y, cfg)
    w = oracle.init_weights(a, 7); v = np.zeros_like(w)
    streams = [oracle_batches(oracle, spec, 4, k, 30, 1, 99) for k in range(4)]
    for rnd in range(len(streams[0])):
        acc = np.zeros_like(w); tot = 0.0
        for k in range(4):
            b = streams[k][rnd]
            g, _, _ = oracle.forward_backward(a, w, x[b], y[b])
            acc += len(b) * g
            tot += len(b)
        _, w, v = oracle.sgd_step(w, v, acc / tot, 0.01, 0.9)
    assert np.array_equal(r.w, w)
    r2 = oracle.run_sync(a, spec, x, y, cfg)
    assert np.array_equal(r.w, r2.w)  # bit-deterministic across repeats


@pytest.mark.parametrize("alpha", [0.1, 0.5, 0.9])
def test_easgd_contraction_ac8(oracle, alpha):
    """AC8: zero gradients; after each exchange the gap shrinks by (1-α)^2
    (documented updated-center ordering)."""
    L = oracle.lib()
    P = 5
    w = np.full(P, 2.0); c = np.zeros(P)
    for _ in range(3):
        gap0 = w - c
        w1 = w.copy()  # local step with g = 0
        L.gho_easgd_center_step(oracle._p(c), oracle._p(w1), P, alpha)
        L.gho_easgd_worker_step(oracle._p(w), oracle._p(c), oracle._p(np.zeros(P)), P, 0.01, alpha, 1, 0)
        assert np.allclose(w - c, (1 - alpha) ** 2 * gap0, rtol=0, atol=1e-12)


def test_hierarchical_equivalence_ac11(oracle):
    """AC11: 1 group × 1 worker, K=1, pass-through parent ≡ flat 1 worker."""
    a = oracle.parse_arch(BENCH_ARCH)
    spec = oracle.data_spec(2, 200)
    x, y = oracle.generate(spec)
    flat = oracle.run_sync(a, spec, x, y, oracle.train_cfg(n_workers=1, batch_size=40, wire_f64=1))
    hier = oracle.run_hier(a, spec, x, y, oracle.train_cfg(n_workers=1, batch_size=40, wire_f64=1,
                                                          groups=1, flush_k=1, parent_lr=1.0,
                                                          parent_mu=0.0))
    assert np.max(np.abs(flat.w - hier.w)) <= 1e-9
    # 2 × 2 completes with full sample accounting
    spec4 = oracle.data_spec(4, 100)
    x4, y4 = oracle.generate(spec4)
    h2 = oracle.run_hier(a, spec4, x4, y4, oracle.train_cfg(n_workers=4, batch_size=25, groups=2,
                                                           flush_k=2))
    assert h2.stats.samples == 400


def test_async_replay_staleness(oracle):
    a = oracle.parse_arch(BENCH_ARCH)
    spec = oracle.data_spec(4, 100)
    x, y = oracle.generate(spec)
    cfg = oracle.train_cfg(n_workers=4, batch_size=25, epochs=1)
    order = np.tile(np.arange(4, dtype=np.int32), 4)
    r = oracle.run_replay(a, spec, x, y, cfg, order)
    # round-robin: first gradients of workers 1..3 are stale by 1..3, then 3
    assert r.extra["staleness"].tolist() == [0, 1, 2, 3] + [3] * 12
    assert r.stats.updates == 16


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle",
                                                    "_ref", "libghref.so")),
                    reason="oracle/_ref not built (needs /root/reference)")
class TestAgainstReferenceBuild:
    def test_frame_codec_bitexact(self, oracle):
        """gho_encode_frame == the reference encoder (proto.cpp encode) byte for
        byte; gho_decode_frame inverts it and reports DecodeStatus like decode."""
        for arch in [BENCH_ARCH, "dense(50,8,tanh),dense(8,6,relu),softmax(6,3)"]:
            a = oracle.parse_arch(arch)
            w = oracle.init_weights(a, 3)
            for kind in (1, 2):
                for f64 in (0, 1):
                    fr = oracle.encode_frame(a, kind, w, 99, 17, f64)
                    assert fr == oracle.ref_encode(arch, kind, w, 99, 17, f64)
                    rc, st, k, w2, ver, cnt, ff = oracle.decode_frame(a, fr)
                    assert (rc, st, k, ver, ff) == (0, 0, kind, 99, f64)
                    want = w if f64 else w.astype(np.float32).astype(np.float64)
                    assert np.array_equal(w2, want) and cnt == (17 if kind == 2 else 0)
        assert oracle.encode_frame(a, 0, None) == oracle.ref_encode(None, 0, None)
        fr = oracle.encode_frame(oracle.parse_arch(BENCH_ARCH), 2, oracle.init_weights(
            oracle.parse_arch(BENCH_ARCH), 1), 1, 5, 0)
        for bad, st in [(b"XHUB" + fr[4:], 1), (fr[:4] + b"\x02\x00" + fr[6:], 2), (fr[:-3], 3),
                         (fr[:6] + b"\x09" + fr[7:], 5), (fr[:3], 3),
                         (fr[:7] + (int.from_bytes(fr[7:15], "little") + 1).to_bytes(8, "little")
                          + fr[15:] + b"\x00", 6)]:
            assert oracle.decode_frame(oracle.parse_arch(BENCH_ARCH), bad)[:2] == (6, st)

    def test_forward_backward_bitexact(self, oracle):
        for arch in [BENCH_ARCH, "dense(50,8,tanh),dense(8,6,relu),softmax(6,3)",
                     "lstm(5,7,10),dense(7,4,identity),softmax(4,3)"]:
            a = oracle.parse_arch(arch)
            w = oracle.init_weights(a, 5)
            x, y = oracle.generate(oracle.data_spec(1, 40))
            g, p, lo = oracle.forward_backward(a, w, x, y)
            gr, pr, lor = oracle.ref_forward_backward(arch, w, x, y)
            assert np.array_equal(g, gr) and np.array_equal(p, pr) and lo == lor

    def test_sync_threads_bitexact(self, oracle):
        a = oracle.parse_arch(BENCH_ARCH)
        spec = oracle.data_spec(6, 150)
        x, y = oracle.generate(spec)
        for W, B in [(1, 64), (3, 50), (4, 33)]:
            cfg = oracle.train_cfg(n_workers=W, batch_size=B, epochs=2)
            r1 = oracle.run_sync(a, spec, x, y, cfg)
            r2 = oracle.ref_run_sync(BENCH_ARCH, spec, x, y, cfg)
            assert np.array_equal(r1.w, r2.w) and np.array_equal(r1.v, r2.v)
            assert r1.stats.updates == r2.stats.updates


def test_validate_oracle_pins(oracle):
    """validate pins: zero weights → uniform p, argmax 0 on
    the tie, so accuracy = share of label 0 and loss = ln K; the count equals
    an independent numpy argmax over the oracle's probabilities."""
    a = oracle.parse_arch("lstm(5,20,10),softmax(20,3)")
    s = oracle.data_spec(2, 150)
    x, y = oracle.generate(s)
    ok, lo = oracle.validate(a, np.zeros(oracle.n_params(a)), x, y)
    assert ok == int((y == 0).sum()) and abs(lo - np.log(3)) < 1e-12
    w = oracle.init_weights(a, 7)
    ok, lo = oracle.validate(a, w, x, y)
    _, probs, loo = oracle.forward_backward(a, w, x, y, want_grad=False)
    assert ok == int((np.argmax(probs, 1) == y).sum()) and lo == loo
