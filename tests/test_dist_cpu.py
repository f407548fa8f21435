"""CPU, world size 2 over gloo: the host side of the multi-GPU sync round.

Each process is one worker rank (as under torchrun on the GPU box).  The
device compute is replaced by the CPU oracle (f64) — the test checks the
protocol around it that ghc_dist_sync_rounds relies on:
  * shard planning and the global→local index streams (bit-exact vs the
    single-process oracle's streams),
  * round counts known on every rank without communication,
  * the exchange math: each worker pre-scales its summed gradient by 1/Σc,
    one SUM collective, every rank applies sgd_step on identical bits
    (the ALLREDUCE mode) — must equal the oracle's W=2 sync Downpour run,
  * the unique-id rendezvous (bytes from rank 0 reach every rank).
"""
import os
import socket

import numpy as np
import pytest

from conftest import BENCH_ARCH, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1712_05878_b200 as g
    from paper_1712_05878_b200 import dist as gd
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = gd.rendezvous(dist, rank, lambda: bytes(range(128)))
    assert uid == bytes(range(128))
    # P2PExchange bootstrap: every rank's 64-byte IPC handle, in rank order
    hs = gd.allgather_bytes(dist, bytes([rank + 1]) * gd.P2PExchange.HANDLE_BYTES)
    assert hs == [bytes([q + 1]) * 64 for q in range(world)]
    # collective success check (P2PExchange's fallback to NCCL): every rank
    # sees the same verdict, with the failing ranks' messages
    ok, pay = gd.agree(dist, True, bytes([rank]))
    assert ok and pay == [bytes([q]) for q in range(world)]
    ok, bad = gd.agree(dist, rank != 1, b"no peer access" if rank == 1 else b"")
    assert not ok and bad == [(1, "no peer access")]

    B, epochs, seed = 70, 1, 99
    spec = g.data_spec(6, 110)
    plan = gd.plan_worker(spec, world, rank, B, epochs, seed)
    counts = gd.round_counts(spec, world, B, epochs, seed)
    assert np.array_equal(counts[: plan.rounds, rank], plan.counts)
    # local rows of this worker's shard only
    xs, ys = g.generate(spec, plan.first_file, plan.n_files)
    a = O.parse_arch(BENCH_ARCH)
    w = O.init_weights(a, 7)
    v = np.zeros_like(w)
    for r in range(counts.shape[0]):
        C = float(counts[r].sum())
        mine = int(counts[r, rank])
        gsum = np.zeros(len(w) + 1)
        if mine:
            sel = plan.idx_local[r * B: r * B + mine]
            gr, _, lo = O.forward_backward(a, w.astype(np.float32).astype(np.float64),
                                           xs[sel].astype(np.float64), ys[sel])
            gr = gr.astype(np.float32).astype(np.float64)  # f32 wire
            gsum[:-1] = gr * (mine / C)
            gsum[-1] = lo * mine
        t = torch.from_numpy(gsum)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        rc, w, v = O.sgd_step(w, v, t.numpy()[:-1], 0.01, 0.9)
        assert rc == 0
    np.save(os.path.join(outdir, f"w{rank}.npy"), w)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sync_round_matches_oracle(tmp_path, oracle):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    w0 = np.load(tmp_path / "w0.npy")
    w1 = np.load(tmp_path / "w1.npy")
    assert np.array_equal(w0, w1)  # replicated master: identical bits on every rank
    spec = oracle.data_spec(6, 110)
    x, y = oracle.generate(spec)
    r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), spec, x, y,
                        oracle.train_cfg(n_workers=2, batch_size=70, epochs=1))
    assert np.max(np.abs(w0 - r.w)) <= 1e-12 * max(1.0, np.max(np.abs(r.w))) * 100


def test_plan_streams_equal_oracle_streams(oracle):
    import paper_1712_05878_b200 as g
    from paper_1712_05878_b200 import dist as gd
    spec = g.data_spec(17, 23)
    so = oracle.data_spec(17, 23)
    for world in (1, 2, 3, 8):
        counts = gd.round_counts(spec, world, 10, 2, 5)
        for k in range(world):
            p = gd.plan_worker(spec, world, k, 10, 2, 5)
            glob = []
            for e in range(2):
                glob.extend(oracle.epoch_indices(so, world, k, e, 5).tolist())
            got = []
            for r in range(p.rounds):
                got.extend((p.idx_local[r * 10: r * 10 + p.counts[r]] + p.row0).tolist())
            assert got == glob
            assert counts[: p.rounds, k].tolist() == p.counts.tolist()
            assert not counts[p.rounds:, k].any()


def test_hierarchical_group_colors():
    """Topology::hierarchical(2,4) (transport.cpp:520-531) → ncclCommSplit
    colors: GPU r in group r // 4, group leaders {0, 4} form the uplink."""
    groups, wpg = 2, 4
    colors = [r // wpg for r in range(groups * wpg)]
    leaders = [r for r in range(groups * wpg) if r % wpg == 0]
    assert colors == [0, 0, 0, 0, 1, 1, 1, 1] and leaders == [0, 4]
