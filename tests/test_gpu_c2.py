"""GPU: BASELINE.json config c2 at its stated size, the NCCL exchange path,
the cross-process NVLink hop, and the error paths the reference defines.

* c2 = sync Downpour, 8 workers × B = 1000 on the benchmark dataset
  (96 files × 9,500 samples), 100 rounds: the fused exchange with 8 virtual
  ranks in one grid (the multi-GPU kernel code, peer pointers into one
  allocation) vs the reference's own threaded sync run (oracle/_ref, which
  the C restatement matches bit for bit) — BASELINE.md §4: ‖Δw‖₂/‖w‖₂ ≤ 1e-5,
  max|Δw| ≤ 1e-5, versions exact.
* ghc_dist_sync_rounds (NCCL reduce/broadcast and all-reduce) at world 1,
  including a non-finite round (whole-update rejection, optim.cpp:49-51).
* Two processes on one GPU map each other's receive rows with
  ghc_p2p_export/import and exchange one tagged row each way through the
  IPC mapping (the cross-rank hop of the fused kernel; no round kernels wait
  on each other, so no co-residency is needed).
* Non-finite gradients in the replayed async / hierarchical / EASGD roles:
  version, staleness and sample accounting follow only ACCEPTED updates and
  EASGD stops at the failing step (oracle gho_run_replay / gho_run_hier).
* Labels outside [0,K) on the asynchronous device path → ShapeError at the
  next synchronising call (nn.cpp:241-244).
"""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import BENCH_ARCH

import paper_1712_05878_b200 as g
from paper_1712_05878_b200 import dist as gd

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def close(w, wo, tol=1e-5):
    r, m = rel(w, wo), float(np.max(np.abs(np.asarray(w, np.float64) - wo)))
    assert r <= tol and m <= tol, (r, m)


def streams(spec, W, B, epochs, seed=99):
    plans = [gd.plan_worker(spec, W, k, B, epochs, seed) for k in range(W)]
    counts = gd.round_counts(spec, W, B, epochs, seed)
    R = counts.shape[0]
    idx = np.zeros((W, R * B), np.int32)
    for k, p in enumerate(plans):
        idx[k, : p.rounds * B] = p.idx_local + p.row0
    return idx, counts, R


def test_c2_eight_workers_b1000_100_rounds(ctx, oracle):
    """c2 at its size: 8 workers × 1000 samples, 100 sync rounds."""
    W, B, R = 8, 1000, 100
    spec = g.data_spec(96, 9500)
    x, y = g.generate(spec)
    idx, counts, Rall = streams(spec, W, B, 1)
    assert Rall >= R
    idx = np.ascontiguousarray(idx[:, : R * B])
    counts = np.ascontiguousarray(counts[:R])
    arch = g.Architecture(ctx, BENCH_ARCH)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    ex = gd.P2PExchange(arch, 0, W, virtual=True)
    loss = ctx.array(R)
    ex.sync_rounds(m, ctx.upload(x), ctx.upload(y), ctx.upload(idx), B, R * B, ctx.upload(counts),
                   B, R, loss_out=loss)
    w, _, ver, rej = m.read()
    ex.close()
    so = oracle.data_spec(96, 9500)
    cfg = oracle.train_cfg(n_workers=W, batch_size=B, epochs=1, max_updates=R)
    if oracle.has_ref():  # the reference itself, threaded (bit-identical to the restatement)
        r = oracle.ref_run_sync(BENCH_ARCH, so, x.astype(np.float64), y, cfg)
    else:
        r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), so, x.astype(np.float64), y, cfg)
    assert ver == r.stats.updates == R and rej == 0
    close(w, r.w)
    lo = loss.numpy() / (W * B)
    assert np.max(np.abs(lo - r.loss[:R]) / r.loss[:R]) <= 1e-4


def _poison(x, spec, W, k, batch, B, epochs=1, pos=5):
    """NaN into the row worker k reads at `pos` of its `batch`-th batch."""
    rows = g.batches(spec, W, k, B, epochs, 99)[batch]
    x = x.copy()
    x[int(rows[pos])] = np.nan
    return x


@pytest.mark.parametrize("mode", [gd.REDUCE_BCAST, gd.ALLREDUCE])
def test_dist_sync_rounds_world1(ctx, oracle, mode):
    """NCCL exchange path (dist.cu) on a 1-rank communicator vs the oracle's
    sync Downpour with one worker, one poisoned round rejected whole."""
    B, nf, spf = 100, 8, 300
    spec = g.data_spec(nf, spf)
    x, y = g.generate(spec)
    x = _poison(x, spec, 1, 0, 3, B)
    plan = gd.plan_worker(spec, 1, 0, B, 1, 99)
    arch = g.Architecture(ctx, BENCH_ARCH)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    comm = gd.Comm(ctx, gd.nccl_unique_id(), 0, 1)
    R = plan.rounds
    loss = ctx.array(R)
    counts = plan.counts.reshape(R, 1)
    dx, dy, di = ctx.upload(x), ctx.upload(y), ctx.upload(plan.idx_local)
    comm.device_barrier()  # the bench's start alignment (reduce + broadcast of one float)
    gd.dist_sync_rounds(m, comm, mode, dx, dy, di, B, counts[:5], 5, loss)  # two calls: the
    gd.dist_sync_rounds(m, comm, mode, dx, dy, di, B, counts[5:], R - 5, ctx.array(R),
                        idx_offset=5 * B)  # cached buffer index must stay right
    w, _, ver, rej = m.read()
    so = oracle.data_spec(nf, spf)
    r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), so, x.astype(np.float64), y,
                        oracle.train_cfg(n_workers=1, batch_size=B, epochs=1))
    assert r.stats.rejected == 1
    assert ver == r.stats.updates and rej == r.stats.rejected
    close(w, r.w)


def _p2p_rank(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1712_05878_b200 as gg
    from paper_1712_05878_b200 import dist as gdd
    import ctypes as C

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = gg.Context(0)
    arch = gg.Architecture(ctx, BENCH_ARCH)
    ex = gdd.P2PExchange(arch, rank, world, dist=dist)  # export / import through torch.distributed
    lib = ctx.lib
    n = int(lib.ghc_p2p_row_elems(ex.h))
    res = []
    for tag in (1, 2, 3):  # both parities, epochs advancing
        for dst in range(world):
            gg.gradhub.check(lib.ghc_p2p_diag_push(ex.h, dst, tag, n), "diag_push")
        dist.barrier()  # every rank's stores done (each push ends with a stream sync)
        for src in range(world):
            bad = C.c_int32(-1)
            gg.gradhub.check(lib.ghc_p2p_diag_check(ex.h, src, tag, n, C.byref(bad)), "diag_check")
            res.append(bad.value)
        dist.barrier()
    np.save(os.path.join(outdir, f"p2p{rank}.npy"), np.array(res + [n]))
    ex.close()
    dist.destroy_process_group()


def test_p2p_two_process_tagged_hop(tmp_path):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_p2p_rank, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for k in range(2):
        r = np.load(tmp_path / f"p2p{k}.npy")
        assert r[-1] > 2000  # a full gradient row (P + loss slot, padded)
        assert np.all(r[:-1] == 0), r


def test_labels_out_of_range_device_path(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    spec = g.data_spec(2, 200)
    x, y = g.generate(spec)
    y = y.copy()
    y[17] = 7
    w = ctx.upload(g.init_weights(arch, 7).astype(np.float32))
    dx, dy = ctx.upload(x), ctx.upload(y)
    gr, ls = ctx.array(arch.n_params), ctx.array(1)
    g.worker_grad_device(arch, w, dx, dy, 100, gr, ls)  # rows 0..99 include row 17
    with pytest.raises(g.ShapeError):
        arch.check_error()
    arch.check_error()  # cleared
    g.worker_grad_device(arch, w, dx, dy, 10, gr, ls)  # rows 0..9: clean
    arch.check_error()
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    m.sync_rounds(dx, dy, None, 100, 100, 2)  # round 0 reads rows 0..99
    with pytest.raises(g.ShapeError):
        m.read()


def _oracle_xy(oracle, nf, spf):
    so = oracle.data_spec(nf, spf)
    x, y = oracle.generate(so)
    return so, x, y


def test_sync_session_nonfinite_round(ctx, oracle):
    W, B, nf, spf = 2, 100, 8, 300
    spec = g.data_spec(nf, spf)
    so, x, y = _oracle_xy(oracle, nf, spf)
    x = _poison(x, spec, W, 1, 2, B)
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(n_workers=W, batch_size=B, epochs=1), spec)
    s.load_data(x, y)
    s.run()
    out = s.read()
    r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), so, x, y,
                        oracle.train_cfg(n_workers=W, batch_size=B, epochs=1))
    assert r.stats.rejected == 1
    assert (out["version"], out["rejected"], out["samples"]) == \
        (r.stats.updates, r.stats.rejected, r.stats.samples)
    close(out["w"], r.w)


def test_async_replay_nonfinite_accounting(ctx, oracle):
    """a rejected gradient advances neither version, basis nor
    samples; staleness and weights match the oracle's replay."""
    W, B, nf, spf = 4, 40, 8, 200
    spec = g.data_spec(nf, spf)
    so, x, y = _oracle_xy(oracle, nf, spf)
    x = _poison(x, spec, W, 2, 1, B)
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(n_workers=W, batch_size=B, epochs=1, mode=g.REPLAY), spec)
    s.load_data(x, y)
    order = np.repeat(np.arange(W, dtype=np.int32), (nf // W) * spf // B)
    np.random.default_rng(5).shuffle(order)
    _, stale = s.run(order)
    out = s.read()
    r = oracle.run_replay(oracle.parse_arch(BENCH_ARCH), so, x, y,
                          oracle.train_cfg(n_workers=W, batch_size=B, epochs=1), order)
    assert r.stats.rejected == 1
    assert np.array_equal(stale, r.extra["staleness"])
    assert (out["version"], out["samples"]) == (r.stats.updates, r.stats.samples)
    close(out["w"], r.w)
    for k in range(W):
        close(out["worker_w"][k], r.extra["worker_w"][k])


def test_hierarchical_nonfinite_group_update(ctx, oracle):
    nf, spf = 16, 200
    kw = dict(n_workers=4, batch_size=40, epochs=1, groups=2, flush_k=2)
    spec = g.data_spec(nf, spf)
    so, x, y = _oracle_xy(oracle, nf, spf)
    x = _poison(x, spec, 4, 3, 2, 40)
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(**kw), spec)
    s.load_data(x, y)
    s.run()
    out = s.read()
    r = oracle.run_hier(oracle.parse_arch(BENCH_ARCH), so, x, y, oracle.train_cfg(**kw))
    assert r.stats.rejected >= 1
    assert (out["version"], out["rejected"], out["samples"]) == \
        (r.stats.updates, r.stats.rejected, r.stats.samples)
    close(out["w"], r.w)
    for q in range(2):
        close(out["group_w"][q], r.extra["group_w"][q])


def test_easgd_replay_stops_at_nonfinite(ctx, oracle):
    """the EASGD worker aborts at the first non-finite gradient
    (optim.cpp:90-92); nothing after it changes the center or any worker."""
    W, B, nf, spf = 4, 25, 8, 200
    spec = g.data_spec(nf, spf)
    so, x, y = _oracle_xy(oracle, nf, spf)
    x = _poison(x, spec, W, 1, 3, B)
    kw = dict(algo=g.EASGD, n_workers=W, batch_size=B, epochs=1, alpha=0.5, tau=2, lr=0.05)
    arch = g.Architecture(ctx, BENCH_ARCH)
    s = g.Session(arch, g.train_config(mode=g.REPLAY, **kw), spec)
    s.load_data(x, y)
    order = np.repeat(np.arange(W, dtype=np.int32), (nf // W) * spf // B)
    np.random.default_rng(2).shuffle(order)
    with pytest.raises(g.NonFiniteGradientError):
        s.run(order)
    out = s.read()
    okw = dict(kw)
    okw["algo"] = oracle.EASGD
    r = oracle.run_replay(oracle.parse_arch(BENCH_ARCH), so, x, y, oracle.train_cfg(**okw), order,
                          allow_error=True)
    assert r.extra["rc"] == oracle.NONFINITE
    close(out["w"], r.w)
    for k in range(W):
        close(out["worker_w"][k], r.extra["worker_w"][k])
