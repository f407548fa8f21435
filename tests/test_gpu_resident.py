"""GPU: the resident round service (ghc_resident_*, resident.cu) — the
persistent sync-round kernel launched once and fed commands through
doorbells.  It runs the same kernel code as ghc_master_sync_rounds, so the
result of any split of rounds into commands is BIT-identical to one
ordinary launch over the same rounds (weights, velocity, version, losses);
both submission paths; idle expiry ends the kernel by itself."""
import time

import numpy as np
import pytest

from conftest import BENCH_ARCH

import paper_1712_05878_b200 as g

pytestmark = pytest.mark.gpu


def _setup(ctx, R, B=1000):
    arch = g.Architecture(ctx, BENCH_ARCH)
    spec = g.data_spec(8, 5000)
    x, y = g.generate(spec)
    idx = np.random.default_rng(3).integers(0, len(y), size=R * B).astype(np.int32)
    return arch, x, y, idx, ctx.upload(x), ctx.upload(y), ctx.upload(idx)


def test_resident_matches_one_launch_bit_exact(ctx):
    R, B = 30, 1000
    arch, x, y, idx, dx, dy, di = _setup(ctx, R, B)
    w0 = g.init_weights(arch, 7)
    ref = g.Master(arch, w0, 0.01, 0.9)
    lref = ctx.array(R)
    ref.sync_rounds(dx, dy, di, B, B, R, loss_out=lref)
    wr, vr, ver_r, rej_r = ref.read()

    m = g.Master(arch, w0, 0.01, 0.9)
    loss = ctx.array(R)
    res = g.Resident(m, B)
    res.submit_stream(dx, dy, di, B, 7, loss_out=loss)                       # device doorbell
    res.submit_stream(dx, dy, di, B, 3, loss_out=loss, idx_offset=7 * B, loss_offset=7)
    ctx.sync()
    res.check()
    s = res.submit(dx, dy, di, B, 12, loss_out=loss, idx_offset=10 * B, loss_offset=10)  # host ring
    res.wait(s)
    s = res.submit(dx, dy, di, B, 8, loss_out=loss, idx_offset=22 * B, loss_offset=22)
    res.wait(s)
    res.stop()
    w, v, ver, rej = m.read()
    assert ver == ver_r == R and rej == rej_r == 0
    assert np.array_equal(w, wr) and np.array_equal(v, vr)
    assert np.array_equal(loss.numpy(), lref.numpy())


def test_resident_host_batches_per_call(ctx):
    """The per-call API: each command's batch in pinned host memory, its loss
    written straight to pinned host memory, submit + wait per batch."""
    R, B = 12, 1000
    arch, x, y, idx, dx, dy, di = _setup(ctx, R, B)
    w0 = g.init_weights(arch, 7)
    hx = ctx.host_array((R * B, x.shape[1]))
    hy = ctx.host_array(R * B, np.int32)
    hl = ctx.host_array(R)
    hx.np[:] = x[idx]
    hy.np[:] = y[idx]
    hl.np[:] = np.nan
    m = g.Master(arch, w0, 0.01, 0.9)
    res = g.Resident(m, B)
    for k in range(R):
        res.wait(res.submit(hx.sub(k * B), hy.sub(k * B), None, 0, 1, loss_out=hl.sub(k)))
        assert np.isfinite(hl.np[k])  # the loss is in host memory when wait returns
    res.stop()
    ref = g.Master(arch, w0, 0.01, 0.9)
    lref = ctx.array(R)
    ref.sync_rounds(dx, dy, di, B, B, R, loss_out=lref)
    assert np.array_equal(m.read()[0], ref.read()[0])
    assert np.array_equal(hl.np, lref.numpy())


def test_resident_queued_commands_prefetch(ctx):
    """Commands queued ahead (submit k+1 before waiting for k): the kernel
    fetches the next command's first batch during the current command's last
    round; results bit-identical to one launch, ragged command lengths."""
    R, B = 24, 1000
    arch, x, y, idx, dx, dy, di = _setup(ctx, R, B)
    w0 = g.init_weights(arch, 7)
    ref = g.Master(arch, w0, 0.01, 0.9)
    lref = ctx.array(R)
    ref.sync_rounds(dx, dy, di, B, B, R, loss_out=lref)
    m = g.Master(arch, w0, 0.01, 0.9)
    loss = ctx.array(R)
    res = g.Resident(m, B)
    seqs, r0 = [], 0
    for n in (1, 1, 3, 1, 5, 2, 1, 1, 4, 1, 1, 3):  # 24 rounds
        seqs.append(res.submit(dx, dy, di, B, n, loss_out=loss, idx_offset=r0 * B, loss_offset=r0))
        r0 += n
        if len(seqs) > 2:
            res.wait(seqs[-3])
    res.wait(seqs[-1])
    res.stop()
    assert r0 == R
    assert np.array_equal(m.read()[0], ref.read()[0])
    assert np.array_equal(loss.numpy(), lref.numpy())


def test_resident_idle_expiry(ctx):
    R, B = 4, 1000
    arch, x, y, idx, dx, dy, di = _setup(ctx, R, B)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    res = g.Resident(m, B, idle_seconds=0.2)
    res.wait(res.submit(dx, dy, di, B, 2))
    time.sleep(0.6)
    with pytest.raises(g.CudaError):
        res.wait(res.submit(dx, dy, di, B, 2, idx_offset=2 * B))
    res.stop()
    _, _, ver, _ = m.read()
    assert ver == 2  # the state of the served commands was published at the idle stop


def test_resident_config_errors(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    with pytest.raises(g.ConfigError):
        g.Resident(m, 100_000)  # more samples than warp slots: not servable resident
    wide = g.Architecture(ctx, "lstm(5,20,10),dense(20,64,relu),softmax(64,3)")
    mw = g.Master(wide, g.init_weights(wide, 7), 0.01, 0.9)
    with pytest.raises(g.ConfigError):
        g.Resident(mw, 100)


def test_packed_rows_bit_identical(ctx, monkeypatch):
    """Packed dataset rows (x | label | pad to 32 B, labels == NULL): the same
    rounds, bit for bit, with fewer DRAM sectors per gathered sample."""
    R, B = 20, 1000
    arch, x, y, idx, dx, dy, di = _setup(ctx, R, B)
    w0 = g.init_weights(arch, 7)
    dp = g.pack_dataset(ctx, dx, dy)
    hp = g.pack_rows(x, y)
    assert dp.shape[1] == 64 and np.array_equal(dp.numpy(), hp)
    outs = []
    for xs, ys in ((dx, dy), (dp, None)):
        m = g.Master(arch, w0, 0.01, 0.9)
        loss = ctx.array(R)
        m.sync_rounds(xs, ys, di, B, B, R, loss_out=loss)
        outs.append((m.read()[0], loss.numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    m = g.Master(arch, w0, 0.01, 0.9)  # resident service on packed rows
    res = g.Resident(m, B)
    res.wait(res.submit(dp, None, di, B, R))
    res.stop()
    assert np.array_equal(m.read()[0], outs[0][0])
    monkeypatch.setenv("GHC_STEP", "tc")
    atc = g.Architecture(ctx, BENCH_ARCH)
    mt = g.Master(atc, w0, 0.01, 0.9)
    with pytest.raises(g.ConfigError):
        mt.sync_rounds(dp, None, di, B, B, 1)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_resident_randomised_command_stream(ctx, seed):
    """Stress of the command protocol (the peeked-command fast path, the early
    and late next-batch fetch, the slot ring): random command lengths, queue
    depths 1..6 and host-side pauses between submissions, batches alternating
    between device and pinned host memory — always bit-identical to one
    ordinary launch over the same rounds."""
    rng = np.random.default_rng(seed)
    B = 1000
    lens = rng.integers(1, 5, size=40)
    R = int(lens.sum())
    arch, x, y, idx, dx, dy, di = _setup(ctx, R, B)
    w0 = g.init_weights(arch, 7)
    # packed rows (x | label | pad) for both paths; host copies of each round's batch
    dp = g.pack_dataset(ctx, dx, dy)
    ref = g.Master(arch, w0, 0.01, 0.9)
    lref = ctx.array(R)
    ref.sync_rounds(dp, None, di, B, B, R, loss_out=lref)
    xp = g.pack_rows(x[idx], y[idx])  # round r's batch = rows r*B .. r*B+B-1
    hx = ctx.host_array(xp.shape)
    hx.np[:] = xp
    m = g.Master(arch, w0, 0.01, 0.9)
    loss = ctx.array(R)
    res = g.Resident(m, B)
    seqs, r0, k = [], 0, 0
    while r0 < R:
        n = int(lens[k])
        if rng.random() < 0.5:  # device dataset + index stream
            seqs.append(res.submit(dp, None, di, B, n, loss_out=loss, idx_offset=r0 * B, loss_offset=r0))
        else:  # contiguous batches in pinned host memory
            seqs.append(res.submit(hx.sub(r0 * B), None, None, B, n, loss_out=loss, loss_offset=r0))
        r0 += n
        k += 1
        depth = int(rng.integers(1, 7))
        while len(seqs) >= depth and seqs:
            res.wait(seqs.pop(0))
        if rng.random() < 0.2:
            time.sleep(float(rng.uniform(0, 2e-4)))
    for s in seqs:
        res.wait(s)
    res.stop()
    assert np.array_equal(m.read()[0], ref.read()[0])
    assert np.array_equal(loss.numpy(), lref.numpy())
