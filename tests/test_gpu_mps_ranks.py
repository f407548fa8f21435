"""GPU: the fused cross-rank sync round across PROCESSES (one rank each),
on one GPU under MPS — the multi-GPU code path (CUDA-IPC-mapped receive
rows, system-scope tagged stores / polls, the xepoch hand-over between
launches) with one device standing in for the peers.  The ranks' master
replicas must be bit-identical, splitting the rounds over launches must not
change a bit, and the result must match the oracle's W-worker sync Downpour
(BASELINE.md bound).  Skipped where MPS is not installed."""
import json
import os
import shutil
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvidia-cuda-mps-control") is None, reason="MPS not installed")
@pytest.mark.parametrize("world,cta_cap,batch", [(2, 64, 100), (4, 32, 100)])
def test_fused_exchange_across_processes(world, cta_cap, batch):
    tmp = tempfile.mkdtemp(prefix="ghc_mps_")
    env = dict(os.environ, CUDA_MPS_PIPE_DIRECTORY=os.path.join(tmp, "pipe"),
               CUDA_MPS_LOG_DIRECTORY=os.path.join(tmp, "log"))
    os.makedirs(env["CUDA_MPS_PIPE_DIRECTORY"])
    os.makedirs(env["CUDA_MPS_LOG_DIRECTORY"])
    if subprocess.run(["nvidia-cuda-mps-control", "-d"], env=env, timeout=30).returncode != 0:
        pytest.skip("MPS daemon did not start")
    try:
        run_env = dict(env, GHC_MAX_CTAS=str(cta_cap), MPS_B=str(batch), MPS_SPF="300")
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
                            "--nproc-per-node", str(world), "--master-addr", "127.0.0.1",
                            "--master-port", str(29600 + world), "tools/mps_ranks.py"],
                           cwd=ROOT, env=run_env, capture_output=True, text=True, timeout=300)
    finally:
        subprocess.run(["nvidia-cuda-mps-control"], input="quit\n", env=env, text=True, timeout=60)
        shutil.rmtree(tmp, ignore_errors=True)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-2000:]
    out = json.loads(lines[-1])
    assert out["ok"], out
    assert out["replicas_bit_identical"] and out["split_launches_bit_identical"]
    assert out["version"] == out["oracle_updates"] and out["rejected"] == 0
