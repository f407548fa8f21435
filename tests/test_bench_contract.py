"""CPU: the bench.py JSON contract (keys, types, per-GPU roofline) for the
N = 1 and N > 1 lines, and the reference arm's argument handling — no GPU
needed (result_line only formats measured numbers)."""
import argparse
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
            "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _args(**kw):
    a = argparse.Namespace(batch=1000, steps=1000, warmup=50, exchange="p2p",
                           traffic=bench.TRAFFIC_PER_ROUND)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("world", [1, 8])
def test_result_line_contract(world):
    ms = 12.5  # 1000 rounds × 12.5 µs
    e2e = {"value": 7.9e7, "unit": bench.UNIT, "h2d_bytes_per_step": 204000,
           "d2h_bytes_per_step": 4}
    line = bench.result_line(_args(), world, ms, None, 1000, e2e, None, 1,
                             {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []},
                             1000, 0, [1.0, 0.1], 0.5, "lstm_round", None)
    assert REQUIRED <= set(line)
    assert line["n_gpus"] == world and line["scaling"] == "weak" and line["warmup"] >= 3
    assert line["value"] == pytest.approx(world * 1000 * 1000 / (ms / 1e3))
    assert line["config"]["workload"] and "model" not in line["config"]
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "TFLOP/s"
    # per-GPU (per launch) achieved rate; the fraction is the same at any N
    assert r["achieved"] == pytest.approx(bench.FLOP_PER_SAMPLE * 1000 * 1000 / (ms / 1e3) / 1e12)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["traffic"] == pytest.approx(bench.TRAFFIC_PER_ROUND * 1000)
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["gpu_launches"] >= 1


def test_gpus_n_spawns_n_ranks(monkeypatch):
    """`bench.py --gpus N` with no launcher re-runs itself as N ranks under
    torch.distributed.run on 127.0.0.1 (the driver's plain
    `python bench.py --gpus 8` must measure 8 GPUs)."""
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3"])
    assert bench.main() == 0
    (cmd,) = calls
    assert "torch.distributed.run" in cmd and "--nproc-per-node=2" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-6:] == ["--gpus", "2", "--steps", "5",
                                                             "--warmup", "3"]


def test_world_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    assert bench.main() == 2


def test_spawned_ranks_run_the_reference_arm(tmp_path):
    """End to end on CPU: --impl reference --gpus 2 spawns 2 ranks; rank 0
    alone prints the reference line, the other rank exits 0 without work."""
    import json
    import subprocess
    from oracle import oracle as O
    if not O.has_ref():
        pytest.skip("oracle/_ref not built")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "3", "--warmup", "3", "--ref-rounds", "1",
                          "--ref-workers", "2"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=str(tmp_path))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(s) for s in out.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
