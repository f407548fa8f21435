"""GPU: architectures with dense layers (layered path: LSTM trunk kernel +
tcgen05 3×TF32 dense GEMMs + softmax-CE head) vs the CPU oracle, including
the wide-layer variant of config c5:
lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3).
Tolerances: gradient ‖Δg‖/‖g‖ ≤ 5e-5 (3×TF32 GEMMs with K up to 4096 measure
≤ 7e-6, the rest is fp32), loss ≤ 1e-5; training weights ‖Δw‖/‖w‖ ≤ 1e-5 and,
for the 4096-wide model, max|Δw| ≤ 1e-4 (its LSTM-trunk gradients pass through
two K=4096 tensor-core GEMMs; the bench net keeps the 1e-5 max bound)."""
import numpy as np
import pytest

import paper_1712_05878_b200 as g

pytestmark = pytest.mark.gpu

WIDE = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"
ARCHS = ["dense(50,64,relu),softmax(64,3)",
         "dense(50,40,tanh),dense(40,24,identity),softmax(24,3)",
         "lstm(5,8,10),dense(8,64,relu),dense(64,48,tanh),softmax(48,3)",
         "lstm(3,4,5),dense(4,16,identity),softmax(16,3)"]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def data(arch_text, n, seed=5):
    _, width, K = g.arch_info(arch_text)
    T, D = (5, 3) if width == 15 else (10, 5)
    return g.generate(g.data_spec(1, n, seq_len=T, input_dim=D, n_classes=K, delta=1.0, seed=seed))


@pytest.mark.parametrize("arch_text", ARCHS)
@pytest.mark.parametrize("n", [1, 37, 300])
def test_layered_grad_vs_oracle(ctx, oracle, arch_text, n):
    arch = g.Architecture(ctx, arch_text)
    w = g.init_weights(arch, 11).astype(np.float32)
    x, y = data(arch_text, n)
    gg, lo = g.forward_backward(w, arch, x, y)
    go, _, loo = oracle.forward_backward(oracle.parse_arch(arch_text), w.astype(np.float64),
                                         x.astype(np.float64), y)
    assert rel(gg, go) <= 5e-5, rel(gg, go)
    assert abs(lo - loo) / loo <= 1e-5
    p, lf = g.forward(w, arch, x, y)
    _, po, _ = oracle.forward_backward(oracle.parse_arch(arch_text), w.astype(np.float64),
                                       x.astype(np.float64), y, want_grad=False)
    assert np.max(np.abs(p - po)) <= 2e-6 and abs(lf - loo) / loo <= 1e-5


def test_wide_variant_grad_vs_oracle(ctx, oracle):
    arch = g.Architecture(ctx, WIDE)
    assert arch.n_params == 16_881_699  # SURVEY §8 wide variant
    w = g.init_weights(arch, 7).astype(np.float32)
    x, y = g.generate(g.data_spec(1, 12, seed=3))
    gg, lo = g.forward_backward(w, arch, x, y)
    go, _, loo = oracle.forward_backward(oracle.parse_arch(WIDE), w.astype(np.float64),
                                         x.astype(np.float64), y)
    assert rel(gg, go) <= 5e-5, rel(gg, go)
    assert abs(lo - loo) / loo <= 1e-5


def test_wide_sync_rounds_vs_oracle(ctx, oracle):
    B, R = 16, 6
    spec = g.data_spec(2, 64)
    x, y = g.generate(spec)
    arch = g.Architecture(ctx, WIDE)
    w0 = g.init_weights(arch, 7)
    m = g.Master(arch, w0, 0.01, 0.9)
    idx = np.concatenate(g.batches(spec, 1, 0, B, 1, 99)[:R]).astype(np.int32)
    m.sync_rounds(ctx.upload(x), ctx.upload(y), ctx.upload(idx), B, B, R)
    w, v, ver, rej = m.read()
    so = oracle.data_spec(2, 64)
    xo, yo = oracle.generate(so)
    r = oracle.run_sync(oracle.parse_arch(WIDE), so, xo, yo,
                        oracle.train_cfg(n_workers=1, batch_size=B, epochs=1, max_updates=R))
    assert ver == R and rej == 0
    assert rel(w, r.w) <= 1e-5 and np.max(np.abs(w - r.w)) <= 1e-4


def test_hierarchical_c5_wide(ctx, oracle):
    """Config c5: 2 sub-masters × 4 workers → top master, wide-layer model."""
    kw = dict(n_workers=8, batch_size=4, epochs=1, groups=2, flush_k=1, max_updates=3)
    arch = g.Architecture(ctx, WIDE)
    s = g.Session(arch, g.train_config(**kw), g.data_spec(8, 16))
    s.run()
    out = s.read()
    spec = oracle.data_spec(8, 16)
    x, y = oracle.generate(spec)
    r = oracle.run_hier(oracle.parse_arch(WIDE), spec, x, y, oracle.train_cfg(**kw))
    assert out["version"] == r.stats.updates
    assert rel(out["w"], r.w) <= 1e-5 and np.max(np.abs(out["w"] - r.w)) <= 1e-4
