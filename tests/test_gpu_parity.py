"""GPU parity: the sm_100a kernels through the C ABI vs the CPU oracle (f64
restatement pinned bit-exactly to the reference).

Tolerances (stated here): the device computes in fp32 with
MUFU-based sigmoid/tanh while the reference computes in f64, so
  * a single worker gradient:  ‖Δg‖₂/‖g‖₂ ≤ 2e-5, loss rel ≤ 1e-5;
  * probabilities:            max |Δp| ≤ 2e-6;
  * optimiser kernels:        max |Δ| ≤ 1e-6·max(1,|x|) (pure fp32 arithmetic);
  * 100 sync Downpour rounds: ‖Δw‖₂/‖w‖₂ ≤ 1e-5 and max|Δw| ≤ 1e-5
    (BASELINE.md §4 target);
  * everything integer (indices, versions, reject counts) is exact.
"""
import numpy as np
import pytest

from conftest import BENCH_ARCH, WIDE_ARCH

import paper_1712_05878_b200 as g

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["simt", "tc", "flat"])
def step_variant(request, monkeypatch):
    """Every parity case runs on all three fused-step variants: the SIMT
    cluster kernel with the reduce-scatter exchange (default, lstm_round.cuh),
    the tensor-core kernel (GHC_STEP=tc, lstm_tc.cuh) and the flat
    grid-barrier kernel (GHC_STEP=flat, lstm_step.cuh).  The variant is fixed
    when a plan is created."""
    if request.param == "simt":
        monkeypatch.delenv("GHC_STEP", raising=False)
    else:
        monkeypatch.setenv("GHC_STEP", request.param)
    return request.param

SHAPES = [BENCH_ARCH, "lstm(5,8,10),softmax(8,3)", "lstm(3,4,5),softmax(4,3)",
          "lstm(2,16,3),softmax(16,4)", "lstm(5,32,10),softmax(32,3)",
          "lstm(4,12,6),softmax(12,5)"]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def dataset(arch_text, n, seed=1234):
    n_p, width, K = g.arch_info(arch_text)
    import re
    D, H, T = map(int, re.match(r"lstm\((\d+),(\d+),(\d+)\)", arch_text).groups())
    spec = g.data_spec(1, n, seq_len=T, input_dim=D, n_classes=K, delta=1.0, seed=seed)
    return g.generate(spec)


@pytest.mark.parametrize("arch_text", SHAPES)
@pytest.mark.parametrize("n", [1, 7, 100, 1000, 5000])
def test_worker_grad_vs_oracle(ctx, oracle, arch_text, n):
    arch = g.Architecture(ctx, arch_text)
    w = g.init_weights(arch, 7)
    x, y = dataset(arch_text, n)
    gg, lo = g.forward_backward(w.astype(np.float32), arch, x, y)
    a = oracle.parse_arch(arch_text)
    go, _, loo = oracle.forward_backward(a, w.astype(np.float32).astype(np.float64),
                                         x.astype(np.float64), y)
    assert rel(gg, go) <= 2e-5, rel(gg, go)
    assert abs(lo - loo) / loo <= 1e-5


def test_forward_probs(ctx, oracle):
    arch = g.Architecture(ctx, BENCH_ARCH)
    w = g.init_weights(arch, 3).astype(np.float32)
    x, y = dataset(BENCH_ARCH, 333)
    p, lo = g.forward(w, arch, x, y)
    _, po, loo = oracle.forward_backward(oracle.parse_arch(BENCH_ARCH), w.astype(np.float64),
                                         x.astype(np.float64), y, want_grad=False)
    assert np.max(np.abs(p - po)) <= 2e-6
    assert np.allclose(p.sum(1), 1.0, atol=1e-6)
    assert abs(lo - loo) / loo <= 1e-5


def test_zero_weights_uniform(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    x, y = dataset(BENCH_ARCH, 50)
    p, lo = g.forward(np.zeros(arch.n_params, np.float32), arch, x, y)
    assert np.allclose(p, 1 / 3, atol=1e-7)
    assert abs(lo - np.log(3)) < 1e-6


def test_grad_deterministic_and_gather(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    x, y = dataset(BENCH_ARCH, 4000)
    w = ctx.upload(g.init_weights(arch, 7).astype(np.float32))
    dx, dy = ctx.upload(x), ctx.upload(y)
    perm = np.random.default_rng(5).permutation(4000)[:1000].astype(np.int32)
    didx = ctx.upload(perm)
    g1, g2, g3 = (ctx.array(arch.n_params) for _ in range(3))
    l1, l2, l3 = (ctx.array(1) for _ in range(3))
    g.worker_grad_device(arch, w, dx, dy, 1000, g1, l1, idx=didx)
    g.worker_grad_device(arch, w, dx, dy, 1000, g2, l2, idx=didx)
    assert np.array_equal(g1.numpy(), g2.numpy()) and np.array_equal(l1.numpy(), l2.numpy())
    bx, by = ctx.upload(x[perm]), ctx.upload(y[perm])
    g.worker_grad_device(arch, w, bx, by, 1000, g3, l3)
    assert np.array_equal(g1.numpy(), g3.numpy())


def test_label_out_of_range(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    x, y = dataset(BENCH_ARCH, 10)
    y[3] = 3
    with pytest.raises(g.ShapeError):
        g.forward_backward(np.zeros(arch.n_params, np.float32), arch, x, y)


def test_empty_batch_and_negative_label(ctx):
    """nn.cpp:104 (n_samples >= 1) and nn.cpp:242/290 (labels in [0, K)) on
    every device entry: the fused worker step, the master's sync rounds and
    the resident service."""
    arch = g.Architecture(ctx, BENCH_ARCH)
    x, y = dataset(BENCH_ARCH, 10)
    w = np.zeros(arch.n_params, np.float32)
    with pytest.raises(g.ShapeError):
        g.forward_backward(w, arch, x[:0], y[:0])
    yn = y.copy()
    yn[0] = -1
    with pytest.raises(g.ShapeError):
        g.forward_backward(w, arch, x, yn)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    dx, dy = ctx.upload(x), ctx.upload(y)
    with pytest.raises(g.ShapeError):
        m.sync_rounds(dx, dy, None, 10, 0, 1)
    with pytest.raises(g.ShapeError):
        g.Resident(m, 0)
    # the label K-1 is valid, K is not (checked on the device, raised at the next sync point)
    yk = y.copy()
    yk[:] = 2
    g.forward_backward(w, arch, x, yk)


def test_invalid_arch_is_config_error(ctx):
    """ConfigError only where the reference rejects too (arch.cpp:26-73);
    shapes outside the fused table run on the generic path (test_gpu_generic)."""
    with pytest.raises(g.ConfigError):
        g.Architecture(ctx, "softmax(3,3),dense(3,3,tanh)")
    with pytest.raises(g.ConfigError):
        g.Architecture(ctx, "lstm(5,20,10),softmax(21,3)")
    assert "lstm_gemm" in g.Architecture(ctx, "lstm(5,40,10),softmax(40,3)").kernel_name


@pytest.mark.parametrize("P", [1, 2143, 4097, 16_881_699])
def test_sgd_apply_vs_oracle(ctx, oracle, P):
    rng = np.random.default_rng(P)
    w, v, gr = (rng.normal(size=P).astype(np.float32) for _ in range(3))
    w2, s2 = g.sgd_step(ctx, w, gr, g.OptimState(v, 0.01, 0.9))
    rc, wo, vo = oracle.sgd_step(w.astype(np.float64), v.astype(np.float64),
                                 gr.astype(np.float64), 0.01, 0.9)
    assert rc == 0
    assert np.max(np.abs(w2 - wo) / np.maximum(1, np.abs(wo))) <= 1e-6
    assert np.max(np.abs(s2.velocity - vo) / np.maximum(1, np.abs(vo))) <= 1e-6


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_sgd_rejects_nonfinite_whole_update(ctx, bad):
    P = 100_003
    w = np.ones(P, np.float32); v = np.zeros(P, np.float32); gr = np.ones(P, np.float32)
    gr[P - 7] = bad
    with pytest.raises(g.NonFiniteGradientError):
        g.sgd_step(ctx, w, gr, g.OptimState(v, 0.1, 0.5))
    # the next (finite) update goes through — the flag was reset on device
    w2, _ = g.sgd_step(ctx, w, np.ones(P, np.float32), g.OptimState(v, 0.1, 0.0))
    assert np.allclose(w2, 0.9)


@pytest.mark.parametrize("P", [1, 4097, 1_000_003])
def test_sgd_in_place_equals_one_pass(ctx, P):
    """ghc_sgd_apply (in place, check pass + update pass) and ghc_sgd_step_out
    (value semantics, one pass) give the same bits; a rejected in-place update
    leaves w, v untouched; overlapping outputs are refused."""
    rng = np.random.default_rng(P + 1)
    w, v, gr = (rng.normal(size=P).astype(np.float32) for _ in range(3))
    lib = ctx.lib
    dw, dv, dg = ctx.upload(w), ctx.upload(v), ctx.upload(gr)
    w2, v2, st = ctx.array(P), ctx.array(P), ctx.upload(np.full(1, 7, np.int32))
    ver = ctx.upload(np.zeros(1, np.uint64))
    g.gradhub.check(lib.ghc_sgd_step_out(ctx.h, dw.ptr, dv.ptr, dg.ptr, w2.ptr, v2.ptr, P, 0.01, 0.9,
                                         st.ptr, ver.ptr), "sgd_step_out")
    assert int(st.numpy()[0]) == 0 and int(ver.numpy()[0]) == 1
    np.testing.assert_array_equal(dw.numpy(), w)  # inputs untouched
    g.gradhub.check(lib.ghc_sgd_apply(ctx.h, dw.ptr, dv.ptr, dg.ptr, P, 0.01, 0.9, st.ptr, ver.ptr),
                    "sgd_apply")
    assert int(st.numpy()[0]) == 0 and int(ver.numpy()[0]) == 2
    np.testing.assert_array_equal(dw.numpy(), w2.numpy())
    np.testing.assert_array_equal(dv.numpy(), v2.numpy())
    gb = gr.copy(); gb[P // 2] = np.nan
    dgb = ctx.upload(gb)
    before_w, before_v = dw.numpy(), dv.numpy()
    g.gradhub.check(lib.ghc_sgd_apply(ctx.h, dw.ptr, dv.ptr, dgb.ptr, P, 0.01, 0.9, st.ptr, ver.ptr),
                    "sgd_apply")
    assert int(st.numpy()[0]) == 2 and int(ver.numpy()[0]) == 2
    np.testing.assert_array_equal(dw.numpy(), before_w)
    np.testing.assert_array_equal(dv.numpy(), before_v)
    g.gradhub.check(lib.ghc_sgd_step_out(ctx.h, dw.ptr, dv.ptr, dgb.ptr, w2.ptr, v2.ptr, P, 0.01, 0.9,
                                         st.ptr, ver.ptr), "sgd_step_out")
    assert int(st.numpy()[0]) == 2 and int(ver.numpy()[0]) == 2
    np.testing.assert_array_equal(dw.numpy(), before_w)
    with pytest.raises(g.ConfigError):
        g.gradhub.check(lib.ghc_sgd_step_out(ctx.h, dw.ptr, dv.ptr, dg.ptr, dw.ptr, v2.ptr, P, 0.01, 0.9,
                                             st.ptr, None), "sgd_step_out")


def test_easgd_worker_in_place_equals_one_pass(ctx):
    P = 300_007
    rng = np.random.default_rng(5)
    w, c, gr = (rng.normal(size=P).astype(np.float32) for _ in range(3))
    lib = ctx.lib
    for bi in (0, 3):
        dw, dc, dg = ctx.upload(w), ctx.upload(c), ctx.upload(gr)
        w2, st = ctx.array(P), ctx.upload(np.full(1, 7, np.int32))
        g.gradhub.check(lib.ghc_easgd_worker_step_out(ctx.h, dw.ptr, dc.ptr, dg.ptr, w2.ptr, P, 0.05,
                                                      0.5, 3, bi, st.ptr), "easgd_out")
        assert int(st.numpy()[0]) == 0
        g.gradhub.check(lib.ghc_easgd_worker_step(ctx.h, dw.ptr, dc.ptr, dg.ptr, P, 0.05, 0.5, 3, bi,
                                                  st.ptr), "easgd")
        np.testing.assert_array_equal(dw.numpy(), w2.numpy())


def test_sgd_spec_examples(ctx):
    w, _ = g.sgd_step(ctx, np.array([1.0], np.float32), np.array([2.0], np.float32),
                      g.OptimState(np.zeros(1, np.float32), 0.1, 0.0))
    assert abs(w[0] - 0.8) < 1e-7
    s = g.OptimState(np.zeros(1, np.float32), 0.1, 0.9)
    w = np.array([1.0], np.float32)
    for _ in range(2):
        w, s = g.sgd_step(ctx, w, np.ones(1, np.float32), s)
    assert abs(w[0] - (1.0 - 0.1 - 0.19)) < 1e-6
    with pytest.raises(g.ConfigError):
        g.sgd_step(ctx, w, np.ones(1, np.float32), g.OptimState(np.zeros(1, np.float32), 0.1, 1.0))


def test_easgd_ops(ctx, oracle):
    P = 10_001
    rng = np.random.default_rng(1)
    w, c, gr = (rng.normal(size=P).astype(np.float32) for _ in range(3))
    L = oracle.lib()
    for bi, tau in [(0, 10), (3, 10), (20, 10)]:
        out = g.easgd_worker_step(ctx, w, c, gr, g.OptimState(None, 0.05), 0.5, tau, bi)
        wo = w.astype(np.float64).copy()
        L.gho_easgd_worker_step(oracle._p(wo), oracle._p(c.astype(np.float64)),
                                oracle._p(gr.astype(np.float64)), P, 0.05, 0.5, tau, bi)
        assert np.max(np.abs(out - wo)) <= 1e-6
    cn, ver = g.easgd_center_step(ctx, c, w, 0.5, 41)
    assert ver == 42 and np.max(np.abs(cn - (c + 0.5 * (w.astype(np.float64) - c)))) <= 1e-6
    pulled = g.elastic_pull(ctx, w, c, 0.25)
    assert np.max(np.abs(pulled - (w - 0.25 * (w.astype(np.float64) - c)))) <= 1e-6
    with pytest.raises(g.ConfigError):
        g.easgd_center_step(ctx, c, w, 1.0)
    gbad = gr.copy(); gbad[5] = np.nan
    with pytest.raises(g.NonFiniteGradientError):
        g.easgd_worker_step(ctx, w, c, gbad, g.OptimState(None, 0.05), 0.5, 10, 0)


def test_master_sync_rounds_vs_oracle(ctx, oracle):
    """c2-shaped sync Downpour (1 master + 1 colocated worker, B=1000), 100
    rounds in ONE persistent launch vs the oracle's f32-wire run."""
    B, R = 1000, 100
    spec = g.data_spec(20, 5000)
    x, y = g.generate(spec)
    arch = g.Architecture(ctx, BENCH_ARCH)
    w0 = g.init_weights(arch, 7)
    stream = g.batches(spec, 1, 0, B, 1, 99)[:R]
    idx = np.concatenate(stream).astype(np.int32)
    m = g.Master(arch, w0, 0.01, 0.9)
    dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(idx)
    loss = ctx.array(R)
    m.sync_rounds(dx, dy, di, B, B, R, loss_out=loss)
    w, v, ver, rej = m.read()
    assert ver == R and rej == 0
    so = oracle.data_spec(20, 5000)
    xo, yo = oracle.generate(so)
    r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), so, xo, yo,
                        oracle.train_cfg(n_workers=1, batch_size=B, epochs=1, max_updates=R))
    assert r.stats.updates == R
    assert rel(w, r.w) <= 1e-5 and np.max(np.abs(w - r.w)) <= 1e-5, (rel(w, r.w),
                                                                      np.max(np.abs(w - r.w)))
    lo = loss.numpy() / B
    assert np.max(np.abs(lo - r.loss) / r.loss) <= 1e-4
    # split into several launches: same bits as one launch (device commit state carries)
    m2 = g.Master(arch, w0, 0.01, 0.9)
    for k in range(0, R, 25):
        m2.sync_rounds(dx, dy, di, B, B, 25, idx_offset=k * B)
    w2, v2, ver2, _ = m2.read()
    assert ver2 == R and np.array_equal(w, w2) and np.array_equal(v, v2)


def test_master_rejects_nonfinite_round(ctx):
    B = 200
    spec = g.data_spec(2, 1000)
    x, y = g.generate(spec)
    x_bad = x.copy()
    x_bad[5, 3] = np.nan  # sample 5 poisons round 0's gradient
    arch = g.Architecture(ctx, BENCH_ARCH)
    w0 = g.init_weights(arch, 7)
    m = g.Master(arch, w0, 0.01, 0.9)
    idx = np.arange(3 * B, dtype=np.int32)
    m.sync_rounds(ctx.upload(x_bad), ctx.upload(y), ctx.upload(idx), B, B, 1)
    w, v, ver, rej = m.read()
    assert ver == 0 and rej == 1
    assert np.array_equal(w, w0.astype(np.float32)) and not v.any()
    m.sync_rounds(ctx.upload(x_bad), ctx.upload(y), ctx.upload(idx), B, B, 2, idx_offset=B)
    w, v, ver, rej = m.read()
    assert ver == 2 and rej == 1 and np.isfinite(w).all()


@pytest.mark.parametrize("arch_text", [BENCH_ARCH, WIDE_ARCH])
def test_master_apply_vs_oracle(ctx, oracle, arch_text):
    """ghc_master_apply (one-pass double-buffered sgd_db_kernel, optim.cpp:
    39-65): each accepted update flips the current buffer on device; a
    non-finite gradient is rejected whole (optim.cpp:49-51) and leaves the
    current buffer and version untouched; it composes with sync_rounds."""
    arch = g.Architecture(ctx, arch_text)
    P = arch.n_params
    rng = np.random.default_rng(P)
    w0 = g.init_weights(arch, 3)
    m = g.Master(arch, w0, 0.01, 0.9)
    w, v = w0.astype(np.float64), np.zeros(P)
    for k in range(3):
        gr = (rng.normal(size=P) * 0.1).astype(np.float32)
        m.apply(ctx.upload(gr))
        rc, w, v = oracle.sgd_step(w, v, gr.astype(np.float64), 0.01, 0.9)
        assert rc == 0
        wd, vd, ver, rej = m.read()
        assert ver == k + 1 and rej == 0
        assert np.max(np.abs(wd - w) / np.maximum(1, np.abs(w))) <= 1e-6
        assert np.max(np.abs(vd - v) / np.maximum(1, np.abs(v))) <= 1e-6
        w, v = wd.astype(np.float64), vd.astype(np.float64)  # continue from the f32 state
    gbad = np.ones(P, np.float32)
    gbad[P // 2] = np.nan
    m.apply(ctx.upload(gbad))
    wd, vd, ver, rej = m.read()
    assert ver == 3 and rej == 1
    assert np.array_equal(wd, w.astype(np.float32)) and np.array_equal(vd, v.astype(np.float32))
    if arch_text != BENCH_ARCH:
        return
    # sync_rounds picks up the applied buffer, and apply picks up sync_rounds'
    spec = g.data_spec(2, 500)
    x, y = g.generate(spec)
    m.sync_rounds(ctx.upload(x), ctx.upload(y), ctx.upload(np.arange(200, dtype=np.int32)), 200,
                  200, 1)
    w1, v1, ver, _ = m.read()
    assert ver == 4 and not np.array_equal(w1, wd)
    gr = (rng.normal(size=P) * 0.1).astype(np.float32)
    m.apply(ctx.upload(gr))
    _, wo, vo = oracle.sgd_step(w1.astype(np.float64), v1.astype(np.float64),
                                gr.astype(np.float64), 0.01, 0.9)
    w2, v2, ver, _ = m.read()
    assert ver == 5 and np.max(np.abs(w2 - wo) / np.maximum(1, np.abs(wo))) <= 1e-6


@pytest.mark.parametrize("B", [1000, 3000])
def test_master_streams_host_batches(ctx, B):
    """Zero-copy end-to-end path: batches in pinned host memory (HostArray,
    no gather table → round r reads rows r*B ..), losses stored to host
    memory.  Same bits as gathering the same rows from a device-resident
    dataset, and as staging them contiguously on the device.  B = 3000 takes
    the kernel's non-prefetching path (more samples than warp slots)."""
    R = 12
    spec = g.data_spec(20, 5000)
    x, y = g.generate(spec)
    arch = g.Architecture(ctx, BENCH_ARCH)
    w0 = g.init_weights(arch, 7)
    idx = np.random.default_rng(3).permutation(len(y))[: R * B].astype(np.int32)
    m1 = g.Master(arch, w0, 0.01, 0.9)
    l1 = ctx.array(R)
    m1.sync_rounds(ctx.upload(x), ctx.upload(y), ctx.upload(idx), B, B, R, loss_out=l1)
    hx = ctx.host_array((R * B, x.shape[1]))
    hy = ctx.host_array(R * B, np.int32)
    hl = ctx.host_array(R)
    hx.np[:] = x[idx]
    hy.np[:] = y[idx]
    hl.np[:] = np.nan
    m2 = g.Master(arch, w0, 0.01, 0.9)
    m2.sync_rounds(hx, hy, None, B, B, R, loss_out=hl)
    ctx.sync()
    m3 = g.Master(arch, w0, 0.01, 0.9)
    m3.sync_rounds(ctx.upload(x[idx]), ctx.upload(y[idx]), None, B, B, R)
    (w1, v1, ver1, _), (w2, v2, ver2, _), (w3, _, _, _) = m1.read(), m2.read(), m3.read()
    assert ver1 == ver2 == R
    assert np.array_equal(w1, w2) and np.array_equal(v1, v2) and np.array_equal(w1, w3)
    assert np.array_equal(l1.numpy(), hl.np)


@pytest.mark.parametrize("W,ns", [(8, [1000] * 8), (8, [1000, 999, 37, 1, 500, 1000, 64, 200]), (3, [250, 17, 1000])])
def test_worker_grads_one_launch(ctx, W, ns):
    """ghc_worker_grads (W workers' gradients in one launch, per-worker
    weights and batches) vs W ghc_worker_grad calls: same values to fp32
    rounding (the per-worker reduction order differs), loss sums likewise;
    repeat → same bits."""
    arch = g.Architecture(ctx, BENCH_ARCH)
    P = arch.n_params
    x, y = g.generate(g.data_spec(8, 1000))
    rng = np.random.default_rng(W + sum(ns))
    ws = np.stack([g.init_weights(arch, 7 + k) for k in range(W)]).astype(np.float32)
    idxs = [rng.integers(0, len(y), size=n).astype(np.int32) for n in ns]
    dx, dy, dw = ctx.upload(x), ctx.upload(y), ctx.upload(ws)
    di = [ctx.upload(i) for i in idxs]
    grad, loss = ctx.array((W, P)), ctx.array(W)
    g.worker_grads_device(arch, dw, dx, dy, di, ns, grad, loss)
    G, L = grad.numpy(), loss.numpy()
    for k in range(W):
        gk, lk = ctx.array(P), ctx.array(1)
        g.worker_grad_device(arch, ctx.upload(ws[k]), dx, dy, ns[k], gk, lk, idx=di[k])
        ref = gk.numpy()
        assert np.linalg.norm(G[k] - ref) / np.linalg.norm(ref) <= 1e-6, k
        assert abs(L[k] - lk.numpy()[0]) <= 1e-5 * abs(lk.numpy()[0]), k
    g.worker_grads_device(arch, dw, dx, dy, di, ns, grad, loss)
    assert np.array_equal(grad.numpy(), G)
