"""Asynchronous Downpour and EASGD across processes (one per GPU): the SPEC
roles with the exchange over NVLink P2P copies.

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


def _tok(dist, peer: int, send: bool):
    import torch
    t = torch.zeros(1, dtype=torch.int32)
    if send:
        dist.send(t, dst=peer)
    else:
        dist.recv(t, src=peer)


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
            version += 1
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
