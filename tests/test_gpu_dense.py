"""GPU: tcgen05 3×TF32 GEMM (dense layers, nn.cpp:129-145 / 312-334) vs an
f64 numpy reference.  Tolerance: max |ΔC| ≤ 1e-5·√K for unit-normal operands —
3×TF32 is fp32-class (a plain TF32 product would be ~1e-3)."""
import ctypes as C

import numpy as np
import pytest

import paper_1712_05878_b200 as g
from paper_1712_05878_b200 import _lib

pytestmark = pytest.mark.gpu


def gemm(ctx, A, B, epi=0, act=2, bias=None, Y=None, alpha=1.0):
    M, K = A.shape
    N = B.shape[0]
    dA, dB = ctx.upload(A.astype(np.float32)), ctx.upload(B.astype(np.float32))
    dC = ctx.array((M, N))
    db = ctx.upload(bias.astype(np.float32)) if bias is not None else None
    dY = ctx.upload(Y.astype(np.float32)) if Y is not None else None
    _lib.check(ctx.lib.ghc_gemm_nt(ctx.h, dA.ptr, dB.ptr, dC.ptr, M, N, K, K, K, N, epi, act,
                                   db.ptr if db else None, dY.ptr if dY else None, N, alpha))
    return dC.numpy()


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (128, 32, 8), (1000, 4096, 20), (250, 300, 77),
                                   (1000, 4096, 4096), (4096, 20, 1000), (20, 64, 1000),
                                   # narrow N, long K → split-K (partials + ordered combine)
                                   (1000, 20, 4096), (130, 3, 2048), (1000, 20, 300), (1, 7, 999)])
def test_gemm_nt_vs_f64(ctx, M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    Cg = gemm(ctx, A, B)
    Cr = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.sqrt(K)  # |A|,|B| ~ 1
    err = np.max(np.abs(Cg - Cr)) / scale
    assert np.linalg.norm(Cg - Cr) / np.linalg.norm(Cr) <= 1e-5  # plain TF32 ~1e-3


@pytest.mark.parametrize("act", [0, 1, 2])
def test_gemm_epilogues(ctx, act):
    rng = np.random.default_rng(act)
    A = rng.normal(size=(200, 64)).astype(np.float32)
    B = rng.normal(size=(96, 64)).astype(np.float32) * 0.1
    bias = rng.normal(size=96)
    Z = A.astype(np.float64) @ B.astype(np.float64).T + bias
    ref = np.tanh(Z) if act == 0 else (np.maximum(Z, 0) if act == 1 else Z)
    assert np.max(np.abs(gemm(ctx, A, B, epi=1, act=act, bias=bias) - ref)) <= 1e-5
    Y = ref.astype(np.float32)
    D = A.astype(np.float64) @ B.astype(np.float64).T
    d = (1 - Y.astype(np.float64) ** 2) if act == 0 else ((Y > 0) * 1.0 if act == 1 else 1.0)
    assert np.max(np.abs(gemm(ctx, A, B, epi=2, act=act, Y=Y) - D * d)) <= 1e-5
    assert np.max(np.abs(gemm(ctx, A, B, alpha=0.25) - 0.25 * D)) <= 1e-5


@pytest.mark.parametrize("act", [0, 1, 2])
def test_gemm_splitk_epilogues(ctx, act):
    """The split-K path applies the same epilogues after the ordered combine,
    and is deterministic (repeat → same bits)."""
    rng = np.random.default_rng(10 + act)
    A = rng.normal(size=(300, 2048)).astype(np.float32) * 0.05
    B = rng.normal(size=(20, 2048)).astype(np.float32) * 0.05
    bias = rng.normal(size=20)
    D = A.astype(np.float64) @ B.astype(np.float64).T
    Z = D + bias
    ref = np.tanh(Z) if act == 0 else (np.maximum(Z, 0) if act == 1 else Z)
    out = gemm(ctx, A, B, epi=1, act=act, bias=bias)
    assert np.max(np.abs(out - ref)) <= 1e-5
    assert np.array_equal(out, gemm(ctx, A, B, epi=1, act=act, bias=bias))
    Y = ref.astype(np.float32)
    d = (1 - Y.astype(np.float64) ** 2) if act == 0 else ((Y > 0) * 1.0 if act == 1 else 1.0)
    assert np.max(np.abs(gemm(ctx, A, B, epi=2, act=act, Y=Y) - D * d)) <= 1e-5
    assert np.max(np.abs(gemm(ctx, A, B, alpha=0.25) - 0.25 * D)) <= 1e-5


@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (300, 260, 77), (1000, 4096, 4100), (513, 700, 1000)])
def test_gemm_pair_shapes(ctx, M, N, K):
    """CTA-pair kernel (M, N ≥ 256): ragged M / N / K edges (TMA zero-fill),
    several accumulator segments (K > 512), and repeat → same bits."""
    rng = np.random.default_rng(M + N + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    Cg = gemm(ctx, A, B)
    Cr = A.astype(np.float64) @ B.astype(np.float64).T
    assert np.linalg.norm(Cg - Cr) / np.linalg.norm(Cr) <= 1e-5
    assert np.array_equal(Cg, gemm(ctx, A, B))


@pytest.mark.parametrize("act", [0, 1, 2])
def test_gemm_pair_epilogues(ctx, act):
    rng = np.random.default_rng(20 + act)
    M, N, K = 520, 384, 640
    A = rng.normal(size=(M, K)).astype(np.float32) * 0.05
    B = rng.normal(size=(N, K)).astype(np.float32) * 0.05
    bias = rng.normal(size=N)
    D = A.astype(np.float64) @ B.astype(np.float64).T
    Z = D + bias
    ref = np.tanh(Z) if act == 0 else (np.maximum(Z, 0) if act == 1 else Z)
    assert np.max(np.abs(gemm(ctx, A, B, epi=1, act=act, bias=bias) - ref)) <= 1e-5
    Y = ref.astype(np.float32)
    d = (1 - Y.astype(np.float64) ** 2) if act == 0 else ((Y > 0) * 1.0 if act == 1 else 1.0)
    assert np.max(np.abs(gemm(ctx, A, B, epi=2, act=act, Y=Y) - D * d)) <= 1e-5
    assert np.max(np.abs(gemm(ctx, A, B, alpha=0.25) - 0.25 * D)) <= 1e-5


@pytest.mark.parametrize("rows,cols", [(1000, 4096), (4096, 20), (20, 4096), (257, 132), (1, 256), (300, 300)])
def test_transpose_vec(ctx, rows, cols):
    """The float4 register-block transpose (rows·cols ≥ 2^16 or aligned
    shapes): ragged 64-tiles and partial 4×4 blocks at the edges."""
    x = np.random.default_rng(rows + cols).normal(size=(rows, cols)).astype(np.float32)
    dx = ctx.upload(x)
    dt = ctx.array((cols, rows))
    _lib.check(ctx.lib.ghc_transpose(ctx.h, dt.ptr, dx.ptr, rows, cols, cols, rows))
    assert np.array_equal(dt.numpy(), x.T)


def test_transpose(ctx):
    x = np.random.default_rng(0).normal(size=(1000, 77)).astype(np.float32)
    dx = ctx.upload(x)
    dt = ctx.array((77, 1000))
    _lib.check(ctx.lib.ghc_transpose(ctx.h, dt.ptr, dx.ptr, 1000, 77, 77, 1000))
    assert np.array_equal(dt.numpy(), x.T)
