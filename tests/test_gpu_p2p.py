"""GPU: the fused NVLink exchange (p2p.cu + lstm_round.cuh ClusterXchg 4x)
with all ranks as virtual ranks sharing one grid on one GPU — the same kernel
code the multi-process path runs, peer pointers into one allocation.

Each rank trains on its own shard's shuffled batches (dist.plan_worker, the
SPEC data layer); the result must match the oracle's sync Downpour with W
workers (sample-weighted mean) to the BASELINE.md bound
‖Δw‖₂/‖w‖₂ ≤ 1e-5, max|Δw| ≤ 1e-5; versions exact.
"""
import numpy as np
import pytest

from conftest import BENCH_ARCH

import paper_1712_05878_b200 as g
from paper_1712_05878_b200 import dist as gd

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def streams(spec, W, B, epochs, seed=99):
    plans = [gd.plan_worker(spec, W, k, B, epochs, seed) for k in range(W)]
    counts = gd.round_counts(spec, W, B, epochs, seed)
    R = counts.shape[0]
    idx = np.zeros((W, R * B), np.int32)
    for k, p in enumerate(plans):
        idx[k, : p.rounds * B] = p.idx_local + p.row0  # global rows of the shared dataset
    return idx, counts, R


@pytest.mark.parametrize("W,B,epochs,nf,spf", [(2, 100, 1, 8, 300), (4, 50, 1, 8, 300),
                                               (8, 64, 2, 8, 300), (3, 70, 1, 8, 300),
                                               (2, 500, 1, 20, 1000)])
def test_p2p_virtual_ranks_vs_oracle(ctx, oracle, W, B, epochs, nf, spf):
    spec = g.data_spec(nf, spf)
    x, y = g.generate(spec)
    idx, counts, R = streams(spec, W, B, epochs)
    arch = g.Architecture(ctx, BENCH_ARCH)
    w0 = g.init_weights(arch, 7)
    m = g.Master(arch, w0, 0.01, 0.9)
    ex = gd.P2PExchange(arch, 0, W, virtual=True)
    loss = ctx.array(R)
    ex.sync_rounds(m, ctx.upload(x), ctx.upload(y), ctx.upload(idx), B, R * B,
                   ctx.upload(counts), B, R, loss_out=loss)
    w, v, ver, rej = m.read()
    so = oracle.data_spec(nf, spf)
    xo, yo = oracle.generate(so)
    r = oracle.run_sync(oracle.parse_arch(BENCH_ARCH), so, xo, yo,
                        oracle.train_cfg(n_workers=W, batch_size=B, epochs=epochs))
    assert ver == r.stats.updates == R and rej == 0
    rr, mm = rel(w, r.w), float(np.max(np.abs(w - r.w)))
    assert rr <= 1e-5 and mm <= 1e-5, (rr, mm)
    lo = loss.numpy()
    assert np.max(np.abs(lo[: len(r.loss)] / counts.sum(1)[: len(r.loss)] - r.loss) / r.loss) <= 1e-4
    ex.close()


def test_p2p_split_launches_same_bits(ctx):
    """Rounds split over launches (arrival counters and the exchange epoch
    persist) give the same bits as one launch; repeated runs are identical."""
    W, B = 4, 50
    spec = g.data_spec(8, 300)
    x, y = g.generate(spec)
    idx, counts, R = streams(spec, W, B, 1)
    arch = g.Architecture(ctx, BENCH_ARCH)
    w0 = g.init_weights(arch, 7)
    dx, dy, di, dc = ctx.upload(x), ctx.upload(y), ctx.upload(idx), ctx.upload(counts)
    outs = []
    for split in (R, 3, R):
        m = g.Master(arch, w0, 0.01, 0.9)
        ex = gd.P2PExchange(arch, 0, W, virtual=True)
        for r0 in range(0, R, split):
            n = min(split, R - r0)
            ex.device_barrier()  # ghc_p2p_barrier: a no-op for virtual ranks
            ex.sync_rounds(m, dx, dy, di, B, R * B, dc, B, n, idx_offset=r0 * B,
                           counts_offset=r0 * W)
        outs.append(m.read()[0])
        ex.close()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_p2p_config_errors(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    with pytest.raises(g.ConfigError):
        gd.P2PExchange(arch, 0, 1, virtual=True)
    with pytest.raises(g.ConfigError):
        gd.P2PExchange(arch, 0, 9, virtual=True)
