"""Multi-GPU host plumbing for the sync Downpour round (one process per GPU).

The reference runs its ranks as threads over `establish(Topology, backend)`
(transport.cpp:533-586); here each GPU is a worker process launched by
torchrun and this module does the host-side parts of the new "nvlink" backend:

* `plan_worker` — the worker's shard (shard_files), the local
  rows it must generate, and its per-round global→local index stream
  (batches);
* `round_counts` — every worker's sample count in every round, computed
  identically on every rank from the deterministic data layer, so the
  sample-weighted mean needs no extra exchange (ghc_dist_sync_rounds);
* `rendezvous` — moves the 128-byte NCCL unique id from rank 0 to every rank
  through torch.distributed (plumbing only; the exchange itself is NCCL over
  NVLink inside libghc);
* `P2PExchange` — the fused NVLink exchange (p2p.cu): every rank's cudaIpc
  handle is all-gathered through torch.distributed (`allgather_bytes`), then
  the persistent round kernels of all ranks reduce the gradient through peer
  memory themselves (no NCCL call per round).  `virtual=True` runs all ranks
  in one grid on one GPU (same kernel code) — the single-GPU test of the path.

Everything here is pure host logic and is covered by world-size-2 gloo tests on
CPU (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import gradhub as g


@dataclass
class WorkerPlan:
    rank: int
    world: int
    first_file: int
    n_files: int
    row0: int            # global row index of the shard's first sample
    rows: int            # samples in the shard
    rounds: int          # rounds this worker participates in
    idx_local: np.ndarray  # [rounds*B] int32 local row indices (padded)
    counts: np.ndarray     # [rounds] samples per round for this worker


def plan_worker(spec, world: int, rank: int, batch: int, epochs: int, shuffle_seed: int,
                shuffle: bool = True) -> WorkerPlan:
    f0, nf = g.shard_files(spec.n_files, world, rank)
    row0 = f0 * spec.samples_per_file
    rows = nf * spec.samples_per_file
    stream, counts = [], []
    for e in range(epochs):
        idx = g.epoch_indices(spec, world, rank, e, shuffle_seed, shuffle) - row0
        for i in range(0, len(idx), batch):
            b = idx[i:i + batch]
            pad = np.zeros(batch, np.int64)
            pad[:len(b)] = b
            stream.append(pad)
            counts.append(len(b))
    idx_local = (np.concatenate(stream) if stream else np.zeros(0)).astype(np.int32)
    return WorkerPlan(rank, world, f0, nf, row0, rows, len(counts), idx_local,
                      np.asarray(counts, np.int32))


def round_counts(spec, world: int, batch: int, epochs: int, shuffle_seed: int) -> np.ndarray:
    """[rounds][world] samples of each worker per round (0 once it is DONE);
    identical on every rank without communication."""
    per = []
    for k in range(world):
        f0, nf = g.shard_files(spec.n_files, world, k)
        rows = nf * spec.samples_per_file
        c = []
        for _ in range(epochs):
            c.extend(min(batch, rows - i) for i in range(0, rows, batch))
        per.append(c)
    R = max(len(c) for c in per)
    out = np.zeros((R, world), np.int32)
    for k, c in enumerate(per):
        out[: len(c), k] = c
    return out


def rendezvous(dist, rank: int, make_id) -> bytes:
    """Broadcast rank 0's unique id (bytes) to every rank via torch.distributed."""
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def nccl_unique_id() -> bytes:
    from . import _lib
    buf = (C.c_uint8 * 128)()
    _lib.check(_lib.load().ghc_comm_unique_id(buf), "ncclGetUniqueId")
    return bytes(buf)


class Comm:
    """ghc_comm: NCCL communicator over the node's GPUs (NVLink/NVSwitch)."""

    def __init__(self, ctx: g.Context, uid: bytes, rank: int, world: int):
        self.ctx = ctx
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        g.check(ctx.lib.ghc_comm_init(ctx.h, buf, rank, world, C.byref(h)), "ncclCommInitRank")
        self.h = h

    def device_barrier(self):
        """A barrier on the context stream: a 1-element reduce to rank 0 and
        a broadcast back (NCCL), so work queued after it starts on all ranks
        together — the start alignment of a timed multi-rank region."""
        if getattr(self, "_one", None) is None:
            self._one = self.ctx.array(1)
            self._one.zero()
        g.check(self.ctx.lib.ghc_comm_reduce_sum(self.h, self._one.ptr, self._one.ptr, 1, 0), "reduce_sum")
        g.check(self.ctx.lib.ghc_comm_broadcast(self.h, self._one.ptr, 1, 0), "broadcast")

    def split(self, color: int, key: int) -> "Comm | None":
        h = C.c_void_p()
        g.check(self.ctx.lib.ghc_comm_split(self.h, color, key, C.byref(h)), "ncclCommSplit")
        if not h.value:
            return None
        c = Comm.__new__(Comm)
        c.ctx, c.h = self.ctx, h
        return c


REDUCE_BCAST, ALLREDUCE = 0, 1


def dist_sync_rounds(master: g.Master, comm: Comm, exchange: int, x, y, idx, stride: int,
                     counts: np.ndarray, rounds: int, loss_out=None, idx_offset: int = 0):
    """ghc_dist_sync_rounds: `rounds` sync Downpour rounds across the comm."""
    counts = np.ascontiguousarray(counts, np.int32)
    g.check(master.ctx.lib.ghc_dist_sync_rounds(
        master.h, comm.h, exchange, x.ptr, y.ptr, idx.offset(idx_offset), stride,
        C.c_void_p(counts.ctypes.data), rounds,
        loss_out.ptr if loss_out is not None else None), "dist_sync_rounds")


def allgather_bytes(dist, payload: bytes) -> list:
    """Every rank's payload, in rank order, on every rank (torch.distributed)."""
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, payload)
    return out


def agree(dist, ok: bool, payload: bytes = b""):
    """Collective success check: every rank contributes (ok, payload).
    Returns (True, [payload of every rank, rank order]) when all ranks
    succeeded, else (False, [(rank, payload) of the failed ranks]) — the same
    answer on every rank, so no rank is left waiting in a later collective."""
    allp = allgather_bytes(dist, bytes([1 if ok else 0]) + bytes(payload))
    if all(p[0] for p in allp):
        return True, [p[1:] for p in allp]
    return False, [(k, p[1:].decode(errors="replace")) for k, p in enumerate(allp) if not p[0]]


class P2PUnavailable(RuntimeError):
    """Peer memory could not be exported/mapped on some rank (raised on every
    rank alike)."""


class P2PExchange:
    """ghc_p2p: fused NVLink exchange of the sync round (p2p.cu)."""

    HANDLE_BYTES = 64

    def __init__(self, arch: g.Architecture, rank: int, world: int, dist=None,
                 virtual: bool = False):
        self.ctx = arch.ctx
        self.world = world
        lib = self.ctx.lib
        h = C.c_void_p()
        self.h = None
        if virtual:
            g.check(lib.ghc_p2p_create_virtual(arch.h, world, C.byref(h)), "p2p_create_virtual")
            self.h = h
        else:
            # Every rank takes part in every agreement even when its own step
            # failed, so a rank that cannot create, export or map the peer
            # memory makes ALL ranks raise P2PUnavailable (callers fall back to
            # NCCL) instead of leaving the others blocked in a collective.
            rc = lib.ghc_p2p_create(arch.h, rank, world, C.byref(h))
            why = b"" if rc == 0 else lib.ghc_last_error()[:200]
            if rc == 0:
                self.h = h
            ok, bad = agree(dist, rc == 0, why)
            if not ok:
                self.close()
                raise P2PUnavailable(f"ghc_p2p_create failed: {bad}")
            mine = (C.c_uint8 * self.HANDLE_BYTES)()
            rc = lib.ghc_p2p_export(h, mine)
            ok, allh = agree(dist, rc == 0, bytes(mine))
            if not ok:
                self.close()
                raise P2PUnavailable(f"ghc_p2p_export failed: {allh}")
            buf = (C.c_uint8 * (self.HANDLE_BYTES * world)).from_buffer_copy(b"".join(allh))
            rc = lib.ghc_p2p_import(h, buf)
            why = b"" if rc == 0 else lib.ghc_last_error()[:200]
            ok, bad = agree(dist, rc == 0, why)
            if not ok:
                self.close()
                raise P2PUnavailable(f"ghc_p2p_import failed: {bad}")

    def sync_rounds(self, master: g.Master, x, y, idx, stride: int, idx_vstride: int, counts,
                    n_max: int, rounds: int, loss_out=None, idx_offset: int = 0,
                    counts_offset: int = 0, loss_offset: int = 0):
        """ghc_p2p_sync_rounds; counts: device int32 [rounds][world] or None."""
        g.check(self.ctx.lib.ghc_p2p_sync_rounds(
            master.h, self.h, x.ptr, y.ptr if y is not None else None,
            idx.offset(idx_offset) if idx is not None else None,
            stride, idx_vstride, counts.offset(counts_offset) if counts is not None else None,
            n_max, rounds, loss_out.offset(loss_offset) if loss_out is not None else None),
            "p2p_sync_rounds")

    def device_barrier(self):
        """ghc_p2p_barrier: queue a device-side barrier of all ranks on the
        context stream (aligns the ranks' next launch without host skew)."""
        g.check(self.ctx.lib.ghc_p2p_barrier(self.h), "p2p_barrier")

    def close(self):
        if self.h is not None and self.ctx.h and not g._SHUTDOWN[0]:
            self.ctx.lib.ghc_p2p_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
