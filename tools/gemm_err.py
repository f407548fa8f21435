import numpy as np, paper_1712_05878_b200 as g
from paper_1712_05878_b200 import _lib
ctx = g.Context(0)
for (M,N,K) in [(128,128,32),(128,128,64),(128,128,96),(128,128,128),(128,128,256),(1000,4096,4096),(4096,20,1000),(20,64,1000)]:
    rng = np.random.default_rng(1)
    A = rng.normal(size=(M,K)).astype(np.float32); B = rng.normal(size=(N,K)).astype(np.float32)
    dA, dB = ctx.upload(A), ctx.upload(B); dC = ctx.array((M,N))
    _lib.check(ctx.lib.ghc_gemm_nt(ctx.h, dA.ptr, dB.ptr, dC.ptr, M, N, K, K, K, N, 0, 2, None, None, N, 1.0))
    Cg = dC.numpy(); Cr = A.astype(np.float64) @ B.astype(np.float64).T; C32 = A @ B.T
    e = np.abs(Cg-Cr); e32 = np.abs(C32-Cr)
    i = np.unravel_index(np.argmax(e), e.shape)
    print(M,N,K, "gpu max", e.max(), "fp32 numpy max", e32.max(), "rel_l2", np.linalg.norm(Cg-Cr)/np.linalg.norm(Cr), "argmax", i, Cg[i], Cr[i], "frac_bad", np.mean(e > 10*e32.max()))
