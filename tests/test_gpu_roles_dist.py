"""GPU: async Downpour and EASGD across PROCESSES (roles_dist.py) — gradient
and weight exchange as CUDA-IPC device-to-device copies, gloo control tokens,
replayed arrival order — vs the oracle's replay runner.

The W ranks share GPU 0 here: the protocol synchronises on host tokens and no
kernel waits on another process's kernel, so this exercises the multi-process
path honestly; on an 8-GPU box the same copies go over NVLink.
Tolerance as in test_gpu_roles.py: ‖Δw‖₂/‖w‖₂ ≤ 1e-5 and max|Δw| ≤ 1e-5;
staleness and versions exact.
"""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARCH = "lstm(5,20,10),softmax(20,3)"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, outdir, algo, order, spec_args, cfg_kw):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1712_05878_b200 as g
    from paper_1712_05878_b200 import roles_dist as rd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = g.Context(0)
    arch = g.Architecture(ctx, ARCH)
    cfg = g.train_config(**cfg_kw)
    spec = g.data_spec(*spec_args)
    if algo == "hier":
        out = rd.run_hierarchical(arch, spec, cfg, rank, world, dist)
    else:
        fn = rd.run_async_downpour if algo == "async" else rd.run_easgd
        out = fn(arch, spec, cfg, order, rank, world, dist)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **{k: np.asarray(v) for k, v in out.items()})
    dist.destroy_process_group()


def _spawn(tmp_path, world, algo, order, spec_args, cfg_kw):
    import torch.multiprocessing as mp
    mp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path), algo, order, spec_args, cfg_kw),
             nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"r{k}.npz")) for k in range(world)]


def _close(w, wo, tol=1e-5):
    r = float(np.linalg.norm(np.asarray(w, np.float64) - wo) / np.linalg.norm(wo))
    m = float(np.max(np.abs(np.asarray(w, np.float64) - wo)))
    assert r <= tol and m <= tol, (r, m)


@pytest.mark.parametrize("W", [2, 4])
def test_async_downpour_p2p_vs_oracle(tmp_path, oracle, W):
    B, spec_args = 40, (8, 200)
    n_b = 8 * 200 // W // B
    order = np.repeat(np.arange(W, dtype=np.int32), n_b)
    np.random.default_rng(3).shuffle(order)
    outs = _spawn(tmp_path, W, "async", order, spec_args,
                  dict(n_workers=W, batch_size=B, epochs=1))
    spec = oracle.data_spec(*spec_args)
    x, y = oracle.generate(spec)
    r = oracle.run_replay(oracle.parse_arch(ARCH), spec, x, y,
                          oracle.train_cfg(n_workers=W, batch_size=B, epochs=1), order)
    assert int(outs[0]["version"]) == r.stats.updates == len(order)
    assert np.array_equal(outs[0]["staleness"], r.extra["staleness"])
    _close(outs[0]["w"], r.w)
    for k in range(W):  # each worker holds the weights of its last reply
        _close(outs[k]["worker_w"], r.extra["worker_w"][k])


@pytest.mark.parametrize("replay", [False, True])
def test_easgd_p2p_vs_oracle(tmp_path, oracle, replay):
    W, B, spec_args = 4, 25, (8, 200)
    kw = dict(n_workers=W, batch_size=B, epochs=2, alpha=0.5, tau=10, lr=0.05)
    n_b = 2 * (8 * 200 // W // B)
    if replay:
        order = np.repeat(np.arange(W, dtype=np.int32), n_b)
        np.random.default_rng(11).shuffle(order)
    else:
        order = np.tile(np.arange(W, dtype=np.int32), n_b)  # round-robin = sync EASGD
    outs = _spawn(tmp_path, W, "easgd", order, spec_args, dict(algo=1, **kw))
    spec = oracle.data_spec(*spec_args)
    x, y = oracle.generate(spec)
    r = oracle.run_replay(oracle.parse_arch(ARCH), spec, x, y,
                          oracle.train_cfg(algo=oracle.EASGD, **kw), order)
    assert int(outs[0]["version"]) == r.stats.updates  # center version = exchanges
    _close(outs[0]["center"], r.w)
    for k in range(W):
        _close(outs[k]["worker_w"], r.extra["worker_w"][k])


@pytest.mark.parametrize("W,K", [(4, 2), (8, 2), (4, 3)])
def test_hierarchical_p2p_vs_oracle(tmp_path, oracle, W, K):
    """2 sub-masters × W/2 workers → top master (pass-through parent), every
    transfer a device-to-device IPC copy; flushes every K group updates and at
    data end."""
    spec_args = (16, 200)
    kw = dict(n_workers=W, batch_size=40, epochs=1, groups=2, flush_k=K)
    outs = _spawn(tmp_path, W, "hier", None, spec_args, kw)
    spec = oracle.data_spec(*spec_args)
    x, y = oracle.generate(spec)
    r = oracle.run_hier(oracle.parse_arch(ARCH), spec, x, y, oracle.train_cfg(**kw))
    _close(outs[0]["w"], r.w)
    for q in range(2):
        _close(outs[q * (W // 2)]["group_w"], r.extra["group_w"][q])
