# the K = 20 forward GEMM of the wide net (1000x4096x20): why 40 us
cat > /tmp/one_gemm.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, paper_1712_05878_b200 as g
from paper_1712_05878_b200 import _lib
ctx = g.Context(0)
M, N, K = [int(v) for v in sys.argv[1:4]]
rng = np.random.default_rng(1)
A = rng.normal(size=(M, K)).astype(np.float32); B = rng.normal(size=(N, K)).astype(np.float32)
dA, dB, dC = ctx.upload(A), ctx.upload(B), ctx.array((M, N))
for _ in range(2):
    _lib.check(ctx.lib.ghc_gemm_nt(ctx.h, dA.ptr, dB.ptr, dC.ptr, M, N, K, K, K, N, 0, 2, None, None, N, 1.0))
ctx.sync()
PY
ncu --set full --import-source on --clock-control none -k regex:gemm -s 1 -c 1 -o gpurun_out/r02_k20 python /tmp/one_gemm.py 1000 4096 20 > gpurun_out/ncu_k20.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/r02_k20.ncu-rep --page details --csv > gpurun_out/r02_k20_details.csv 2>/dev/null
ncu -i gpurun_out/r02_k20.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_k20_src.csv 2>/dev/null
