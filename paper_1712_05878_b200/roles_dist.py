"""Asynchronous Downpour, EASGD and hierarchical masters across processes
(one per GPU): the SPEC roles with the exchange over NVLink
P2P copies (the sync Downpour round has its own fused path, p2p.cu).

BASELINE north_star: "gradient send and weight broadcast move over NVLink ...
P2P copies in async mode".  Rank k is worker k; rank 0 also runs the master.
Data moves device→device through CUDA-IPC-mapped buffers (`ghc_ipc_*` +
`ghc_memcpy_d2d`): a worker copies its gradient (Downpour) or its stepped
weights (EASGD) straight into its slot of the master's mailbox on GPU 0, and
the master copies the reply into the worker's inbox.  Only 4-byte control
tokens travel through torch.distributed (gloo), so the master can process
messages in a REPLAYED arrival order — the oracle comparison of SURVEY §8(c):

* async Downpour: order[i] = worker whose next gradient the
  master applies (sgd_step, reject on non-finite); the worker then receives
  the new weights and computes its next gradient from them (strict Fig.-1
  cycle, so staleness = version − basis_version arises only from interleaving);
* EASGD (optim.cpp:82-123, oracle decision 1): order[i] = worker whose next
  local batch runs; workers step locally (w1 = w − η·g) without talking to
  anyone; when batch_index % τ == 0 the worker sends w1, the master applies
  c' = c + α(w1 − c) (exchanges in order) and replies c', the worker pulls
  w = w1 − α(w1 − c').

No kernel ever waits on another process's kernel (the ranks synchronise on
host tokens), so the protocol is exercised honestly with several processes
sharing one GPU (tests/test_gpu_roles_dist.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import dist as gd
from . import gradhub as g

HANDLE_BYTES = 64


class _Ipc:
    """IPC view of this rank's buffers and the mapped buffers of its peers."""

    def __init__(self, ctx: g.Context):
        self.ctx = ctx
        self.opened = []

    def handle(self, arr: g.DeviceArray) -> bytes:
        buf = (C.c_uint8 * HANDLE_BYTES)()
        g.check(self.ctx.lib.ghc_ipc_handle(self.ctx.h, arr.ptr, buf), "ipc_handle")
        return bytes(buf)

    def open(self, h: bytes) -> int:
        p = C.c_void_p()
        buf = (C.c_uint8 * HANDLE_BYTES).from_buffer_copy(h)
        g.check(self.ctx.lib.ghc_ipc_open(self.ctx.h, buf, C.byref(p)), "ipc_open")
        self.opened.append(p.value)
        return p.value

    def close(self):
        for p in self.opened:
            self.ctx.lib.ghc_ipc_close(self.ctx.h, C.c_void_p(p))
        self.opened = []


def _copy(ctx, dst: int, src: int, nbytes: int):
    g.check(ctx.lib.ghc_memcpy_d2d(ctx.h, C.c_void_p(dst), C.c_void_p(src), nbytes), "memcpy_d2d")


class _Worker:
    """This rank's shard, batch stream and weights."""

    def __init__(self, arch: g.Architecture, spec, cfg, world: int, rank: int):
        ctx = self.ctx = arch.ctx
        self.arch, self.cfg = arch, cfg
        self.plan = gd.plan_worker(spec, world, rank, cfg.batch_size, cfg.epochs, cfg.shuffle_seed,
                                   bool(cfg.shuffle))
        x, y = g.generate(spec, self.plan.first_file, self.plan.n_files)
        self.dx, self.dy = ctx.upload(x), ctx.upload(y)
        idx = self.plan.idx_local if len(self.plan.idx_local) else np.zeros(1, np.int32)
        self.didx = ctx.upload(idx)
        P = arch.n_params
        self.w = ctx.upload(g.init_weights(arch, cfg.weight_seed).astype(np.float32))
        self.gl = ctx.array(P + 4)  # gradient [P] + loss sum at [P]
        self.status = ctx.array(1, np.int32)
        self.j = 0                  # next batch

    def grad(self, dst_ptr: int | None = None):
        """Mean gradient of the next batch at the current weights → gl (or dst)."""
        B = self.cfg.batch_size
        n = int(self.plan.counts[self.j])
        out = dst_ptr if dst_ptr is not None else self.gl.ptr.value
        lib = self.ctx.lib
        g.check(lib.ghc_worker_grad(self.arch.h, self.w.ptr, self.dx.ptr, self.dy.ptr,
                                    self.didx.offset(self.j * B), n, 1.0 / n, C.c_void_p(out),
                                    C.c_void_p(out + 4 * self.arch.n_params)), "worker_grad")
        self.j += 1


def _tok(dist, peer: int, send: bool, payload=(0,)):
    """Control token (gloo); returns the received payload (int64 values)."""
    import torch
    t = torch.tensor(list(payload), dtype=torch.int64)
    if send:
        dist.send(t, dst=peer)
    else:
        dist.recv(t, src=peer)
    return t.tolist()


def run_async_downpour(arch: g.Architecture, spec, cfg, order, rank: int, world: int, dist):
    """Async Downpour over P2P copies with a replayed arrival order.
    Returns dict(worker_w) on every rank, plus master w, v, version,
    staleness on rank 0."""
    ctx = arch.ctx
    P = arch.n_params
    order = np.asarray(order, np.int32)
    wk = _Worker(arch, spec, cfg, world, rank)
    ipc = _Ipc(ctx)
    slot = 4 * (P + 4)
    if rank == 0:
        mailbox = ctx.array(world * (P + 4))
        mw = ctx.upload(g.init_weights(arch, cfg.weight_seed).astype(np.float32))
        mv = ctx.array(P)
        mv.zero()
        st = ctx.array(1, np.int32)
    handles = gd.allgather_bytes(dist, ipc.handle(wk.w))          # every worker's inbox
    mail_h = gd.allgather_bytes(dist, ipc.handle(mailbox) if rank == 0 else b"")[0]
    out = {}
    if rank == 0:
        inbox = [None] + [ipc.open(h) for h in handles[1:]]
        version, basis, stale = 0, [0] * world, []
        for k in order.tolist():
            dst = mailbox.ptr.value + k * slot
            if k == 0:
                wk.grad(dst)
            else:
                _tok(dist, k, send=False)  # worker k's gradient landed in its slot
            stale.append(version - basis[k])
            g.check(ctx.lib.ghc_sgd_apply(ctx.h, mw.ptr, mv.ptr, C.c_void_p(dst), P, cfg.lr,
                                          cfg.mu, st.ptr, None), "sgd_apply")
            # only an accepted update advances the version (optim.cpp:49-51,
            # oracle gho_run_replay): the rejecting kernel leaves its status
            version += int(st.numpy()[0]) == 0
            if k == 0:
                _copy(ctx, wk.w.ptr.value, mw.ptr.value, 4 * P)
            else:
                _copy(ctx, inbox[k], mw.ptr.value, 4 * P)  # reply over NVLink
                ctx.sync()
                _tok(dist, k, send=True)
            basis[k] = version
        ctx.sync()
        out.update(w=mw.numpy(), v=mv.numpy(), version=version, staleness=np.array(stale))
    else:
        mail = ipc.open(mail_h) + rank * slot
        for _ in range(int((order == rank).sum())):
            wk.grad()
            _copy(ctx, mail, wk.gl.ptr.value, 4 * (P + 1))  # gradient → master mailbox (NVLink)
            ctx.sync()
            _tok(dist, 0, send=True)
            _tok(dist, 0, send=False)  # the reply landed in wk.w
    ctx.sync()
    out["worker_w"] = wk.w.numpy()
    dist.barrier()
    ipc.close()
    return out


def run_easgd(arch: g.Architecture, spec, cfg, order, rank: int, world: int, dist):
    """EASGD over P2P copies; order[i] = worker whose next local batch runs
    (round-robin = the sync mode).  Returns worker_w on every rank and the
    center + its version on rank 0."""
    ctx = arch.ctx
    P = arch.n_params
    order = np.asarray(order, np.int32)
    tau = cfg.tau
    wk = _Worker(arch, spec, cfg, world, rank)
    cbuf = ctx.array(P)  # the center of my last exchange (reply inbox)
    ipc = _Ipc(ctx)
    if rank == 0:
        mailbox = ctx.array(world * P)
        center = ctx.upload(g.init_weights(arch, cfg.weight_seed).astype(np.float32))
        cver = ctx.array(1, np.uint64)
        cver.zero()
    handles = gd.allgather_bytes(dist, ipc.handle(cbuf))
    mail_h = gd.allgather_bytes(dist, ipc.handle(mailbox) if rank == 0 else b"")[0]
    never = (1 << 63)  # tau for a local step without pull: w1 = w − η·g

    def local_step():
        wk.grad()
        g.check(ctx.lib.ghc_easgd_worker_step(ctx.h, wk.w.ptr, wk.w.ptr, wk.gl.ptr, P, cfg.lr,
                                              cfg.alpha, never, 1, wk.status.ptr), "easgd_worker")

    out = {}
    if rank == 0:
        inbox = [None] + [ipc.open(h) for h in handles[1:]]
        bidx = [0] * world
        for k in order.tolist():
            exch = bidx[k] % tau == 0
            bidx[k] += 1
            if k == 0:
                local_step()
                src = wk.w.ptr.value
            elif exch:
                _tok(dist, k, send=False)  # worker k's w1 landed in its slot
                src = mailbox.ptr.value + 4 * k * P
            else:
                continue  # a local step of another worker: nothing for the master
            if not exch:
                continue
            g.check(ctx.lib.ghc_easgd_center_step(ctx.h, center.ptr, C.c_void_p(src), P,
                                                  cfg.alpha, cver.ptr), "easgd_center")
            if k == 0:
                g.check(ctx.lib.ghc_elastic_pull(ctx.h, wk.w.ptr, center.ptr, P, cfg.alpha),
                        "elastic_pull")
            else:
                _copy(ctx, inbox[k], center.ptr.value, 4 * P)  # reply c' over NVLink
                ctx.sync()
                _tok(dist, k, send=True)
        ctx.sync()
        out.update(center=center.numpy(), version=int(cver.numpy()[0]))
    else:
        mail = ipc.open(mail_h) + 4 * rank * P
        for j in range(int((order == rank).sum())):
            local_step()
            if j % tau == 0:
                _copy(ctx, mail, wk.w.ptr.value, 4 * P)  # w1 → master mailbox
                ctx.sync()
                _tok(dist, 0, send=True)
                _tok(dist, 0, send=False)  # c' landed in cbuf
                g.check(ctx.lib.ghc_elastic_pull(ctx.h, wk.w.ptr, cbuf.ptr, P, cfg.alpha),
                        "elastic_pull")
    ctx.sync()
    out["worker_w"] = wk.w.numpy()
    dist.barrier()
    ipc.close()
    return out


def run_hierarchical(arch: g.Architecture, spec, cfg, rank: int, world: int, dist):
    """Hierarchical masters (Topology::hierarchical
    transport.cpp:520-531, oracle decision 2) across processes: cfg.groups
    groups of world/groups workers; the sub-master of group q runs on the
    group's first rank, the top master on rank 0.  Per round every group does
    a sync Downpour step (workers → sub-master mailbox, sample-weighted combine
    in rank order SPEC.md:358-366, sgd_step(lr, mu)); a group flushes after
    flush_k updates (or when its data ends) by sending snapshot − current,
    weighted by the samples it absorbed, to the top master, which combines the
    flushing groups in group order, applies sgd_step(parent_lr, parent_mu) and
    replies; the group adopts the reply as weights and snapshot.  All
    transfers are CUDA-IPC device-to-device copies.  Returns worker_w on every
    rank, group_w on sub-masters, top w on rank 0."""
    ctx = arch.ctx
    lib = ctx.lib
    P = arch.n_params
    G = cfg.groups
    Wg = world // G
    q, sub = rank // Wg, (rank // Wg) * Wg
    wk = _Worker(arch, spec, cfg, world, rank)
    counts = gd.round_counts(spec, world, cfg.batch_size, cfg.epochs, cfg.shuffle_seed)
    R = counts.shape[0]
    # flush schedule: kept by each sub-master from its group's ACCEPTED
    # updates (a rejected group step absorbs nothing, oracle gho_run_hier) and
    # reported to the top master with one token per round
    absorbed_q, since_q = 0, 0
    ipc = _Ipc(ctx)
    w0 = g.init_weights(arch, cfg.weight_seed).astype(np.float32)
    if rank == sub:
        mail = ctx.array(Wg * P)                # gradient slot of each group worker
        stage = ctx.array(Wg * P)               # active slots, compacted in rank order
        wg, vg, snap = ctx.upload(w0), ctx.array(P), ctx.upload(w0)
        vg.zero()
        comb, psd, vd = ctx.array(P), ctx.array(P), ctx.array(P)
        st = ctx.array(1, np.int32)
    if rank == 0:
        tmail = ctx.array(G * P)                # pseudo-gradient slot of each group
        tstage = ctx.array(G * P)
        tw, tv, tcomb = ctx.upload(w0), ctx.array(P), ctx.array(P)
        tv.zero()
        tst = ctx.array(1, np.int32)
    inbox_h = gd.allgather_bytes(dist, ipc.handle(wk.w))
    mail_h = gd.allgather_bytes(dist, ipc.handle(mail) if rank == sub else b"")
    wg_h = gd.allgather_bytes(dist, ipc.handle(wg) if rank == sub else b"")
    tmail_h = gd.allgather_bytes(dist, ipc.handle(tmail) if rank == 0 else b"")[0]
    if rank != sub:
        my_slot = ipc.open(mail_h[sub]) + 4 * (rank - sub) * P
    else:
        inbox = {k: ipc.open(inbox_h[k]) for k in range(sub + 1, sub + Wg)}
        top_slot = (tmail.ptr.value if rank == 0 else ipc.open(tmail_h)) + 4 * q * P
    if rank == 0:
        sub_wg = {qq: (wg.ptr.value if qq == 0 else ipc.open(wg_h[qq * Wg])) for qq in range(G)}

    def sgd(w, v, gp, lr, mu, stat):
        g.check(lib.ghc_sgd_apply(ctx.h, w.ptr, v.ptr, C.c_void_p(gp), P, lr, mu, stat.ptr, None),
                "sgd_apply")

    def combine(out, slots, stage_buf, weights):
        """Σ c_i slot_i / Σ c_i over the slots with c_i > 0, in slot order."""
        act = [i for i, c in enumerate(weights) if c > 0]
        for n, i in enumerate(act):
            _copy(ctx, stage_buf.ptr.value + 4 * n * P, slots.ptr.value + 4 * i * P, 4 * P)
        wts = (C.c_double * len(act))(*[float(weights[i]) for i in act])
        g.check(lib.ghc_weighted_mean(ctx.h, out.ptr, stage_buf.ptr, wts, len(act), P),
                "weighted_mean")

    for r in range(R + 1):  # round R: data exhausted, final flushes only
        cnt = counts[r] if r < R else np.zeros(world, np.int32)
        gcnt = cnt[sub:sub + Wg]
        flushing, absorbed = [0] * G, [0] * G
        # ---- worker: mean gradient of its next batch at the group weights ----
        if cnt[rank]:
            if rank == sub:
                wk.grad()
                _copy(ctx, mail.ptr.value, wk.gl.ptr.value, 4 * P)
            else:
                wk.grad()
                _copy(ctx, my_slot, wk.gl.ptr.value, 4 * P)
                ctx.sync()
                _tok(dist, sub, send=True)
        if rank == sub:
            # ---- sub-master: sync combine + sgd_step (lr, mu) ----
            if gcnt.sum() > 0:
                for j in range(1, Wg):
                    if gcnt[j]:
                        _tok(dist, sub + j, send=False)
                combine(comb, mail, stage, gcnt)
                sgd(wg, vg, comb.ptr.value, cfg.lr, cfg.mu, st)
                if int(st.numpy()[0]) == 0:  # accepted
                    absorbed_q += int(gcnt.sum())
                    since_q += 1
                flushing[q] = int(since_q >= cfg.flush_k)
            else:
                flushing[q] = int(absorbed_q > 0)  # final flush of a finished group
            absorbed[q] = absorbed_q
            if flushing[q]:
                absorbed_q = since_q = 0
            if rank != 0:
                _tok(dist, 0, send=True, payload=(flushing[q], absorbed[q]))
            else:
                for qq in range(1, G):
                    flushing[qq], absorbed[qq] = _tok(dist, qq * Wg, send=False, payload=(0, 0))
            if flushing[q]:
                # pseudo-gradient snapshot − current (oracle decision 2) → top master
                _copy(ctx, psd.ptr.value, snap.ptr.value, 4 * P)
                vd.zero()
                sgd(psd, vd, wg.ptr.value, 1.0, 0.0, st)  # psd + (−1·wg): exactly snap − wg
                _copy(ctx, top_slot, psd.ptr.value, 4 * P)
                ctx.sync()
                if rank != 0:
                    _tok(dist, 0, send=True)
        if rank == 0 and any(flushing):
            # ---- top master: combine the flushing groups (group order), sgd_step ----
            for qq in range(1, G):
                if flushing[qq]:
                    _tok(dist, qq * Wg, send=False)
            combine(tcomb, tmail, tstage, [absorbed[qq] if flushing[qq] else 0 for qq in range(G)])
            sgd(tw, tv, tcomb.ptr.value, cfg.parent_lr, cfg.parent_mu, tst)
            for qq in range(G):
                if flushing[qq]:
                    _copy(ctx, sub_wg[qq], tw.ptr.value, 4 * P)  # reply → the group's weights
            ctx.sync()
            for qq in range(1, G):
                if flushing[qq]:
                    _tok(dist, qq * Wg, send=True)
        if rank == sub:
            if flushing[q]:
                if rank != 0:
                    _tok(dist, 0, send=False)  # the top weights landed in wg
                _copy(ctx, snap.ptr.value, wg.ptr.value, 4 * P)
            if r < R:  # ---- the group's weights → every worker of the group ----
                _copy(ctx, wk.w.ptr.value, wg.ptr.value, 4 * P)
                for p in inbox.values():
                    _copy(ctx, p, wg.ptr.value, 4 * P)
                ctx.sync()
                for k in inbox:
                    _tok(dist, k, send=True)
        elif r < R:
            _tok(dist, sub, send=False)  # the group weights landed in wk.w
    ctx.sync()
    out = {"worker_w": wk.w.numpy()}
    if rank == sub:
        out["group_w"] = wg.numpy()
    if rank == 0:
        out["w"] = tw.numpy()
    dist.barrier()
    ipc.close()
    return out
