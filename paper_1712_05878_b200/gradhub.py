"""Python mirror of the reference's Model / Algo / Data interface over libghc.

Names and argument meaning follow /root/reference/proj/include/gradhub/*.hpp so
tests read like the reference's own: `Architecture`, `init_weights`,
`forward`, `backward`-as-`forward_backward`, `loss`, `sgd_step`,
`elastic_pull`, `easgd_worker_step`, `easgd_center_step`, `shard_files`,
`batches`; errors are the reference exception classes.  Host-array calls are
copy-in/copy-out through the C ABI (the drop-in path); `DeviceArray`-based
calls keep everything resident in HBM (the fast path).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (CacheMismatchError, ConfigError, CudaError, DataSpec, GradhubError,  # noqa: F401
                   NcclError, NonFiniteGradientError, ProtocolError, ShapeError,
                   TransportError, check)

_SHUTDOWN = [False]


def _at_exit():
    # the process is going away: the driver reclaims device memory; finalizers
    # must not touch library objects whose owners may already be gone
    _SHUTDOWN[0] = True


import atexit  # noqa: E402

atexit.register(_at_exit)


def _vp(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class Context:
    """ghc_ctx: one CUDA device + stream (one per GPU per host thread)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.ghc_ctx_create(device, C.byref(h)), "ghc_ctx_create")
        self.h = h
        self.device = device

    def close(self):
        """Explicit teardown (all plans/arrays/sessions of this context must be
        released first).  Not called from a finalizer: GC order is arbitrary."""
        if self.h:
            self.lib.ghc_ctx_destroy(self.h)
            self.h = None

    @property
    def num_sms(self) -> int:
        return self.lib.ghc_ctx_num_sms(self.h)

    @property
    def launches(self) -> int:
        return int(self.lib.ghc_ctx_launch_count(self.h))

    def sync(self):
        check(self.lib.ghc_ctx_sync(self.h), "ghc_ctx_sync")

    def hold(self):
        """ghc_stream_hold: queue work behind a gate (device timing without
        the host's launch calls); release() lets it run."""
        check(self.lib.ghc_stream_hold(self.h))

    def release(self):
        check(self.lib.ghc_stream_release(self.h))

    def timer_start(self):
        check(self.lib.ghc_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_float()
        check(self.lib.ghc_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def host_array(self, shape, dtype=np.float32) -> "HostArray":
        return HostArray(self, shape, dtype)

    def array(self, shape, dtype=np.float32) -> "DeviceArray":
        return DeviceArray(self, shape, dtype)

    def upload(self, a: np.ndarray) -> "DeviceArray":
        a = np.ascontiguousarray(a)
        d = DeviceArray(self, a.shape, a.dtype)
        d.copy_from(a)
        return d


class DeviceArray:
    """A device buffer owned through the C ABI (ghc_malloc / ghc_free)."""

    def __init__(self, ctx: Context, shape, dtype=np.float32):
        self.ctx = ctx
        self.shape = tuple(shape) if isinstance(shape, (tuple, list)) else (int(shape),)
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(ctx.lib.ghc_malloc(ctx.h, self.nbytes, C.byref(p)), "ghc_malloc")
        self.ptr = p

    def free(self):
        if self.ptr is not None and self.ctx.h and not _SHUTDOWN[0]:
            self.ctx.lib.ghc_free(self.ctx.h, self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def offset(self, elements: int) -> C.c_void_p:
        return C.c_void_p(self.ptr.value + elements * self.dtype.itemsize)

    def copy_from(self, a: np.ndarray):
        a = np.ascontiguousarray(a, self.dtype)
        assert a.nbytes <= self.nbytes
        check(self.ctx.lib.ghc_memcpy_h2d(self.ctx.h, self.ptr, _vp(a), a.nbytes), "h2d")
        self.ctx.sync()

    def zero(self):
        check(self.ctx.lib.ghc_memset(self.ctx.h, self.ptr, 0, self.nbytes))

    def numpy(self) -> np.ndarray:
        out = np.empty(self.shape, self.dtype)
        check(self.ctx.lib.ghc_memcpy_d2h(self.ctx.h, _vp(out), self.ptr, self.nbytes), "d2h")
        self.ctx.sync()
        return out


class HostArray:
    """Pinned host buffer (ghc_host_alloc) exposed as a numpy view.  It is
    device-accessible (UVA), so it can stand in for a DeviceArray where the C
    ABI reads batches or writes losses: Master.sync_rounds then streams the
    rows from host memory inside the persistent round kernel (zero-copy)."""

    def __init__(self, ctx: Context, shape, dtype=np.float32):
        self.ctx = ctx
        self.shape = tuple(shape) if isinstance(shape, (tuple, list)) else (int(shape),)
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(ctx.lib.ghc_host_alloc(self.nbytes, C.byref(p)), "ghc_host_alloc")
        self.ptr = p
        n = int(np.prod(self.shape))
        buf = (C.c_char * self.nbytes).from_address(p.value)
        self.np = np.frombuffer(buf, dtype=self.dtype, count=n).reshape(self.shape)

    def free(self):
        if self.ptr is not None and not _SHUTDOWN[0]:
            self.np = None
            self.ctx.lib.ghc_host_free(self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def offset(self, elements: int) -> C.c_void_p:
        return C.c_void_p(self.ptr.value + elements * self.dtype.itemsize)

    def sub(self, row: int) -> "_View":
        """View starting at `row` (first-axis index): pass to the C ABI like
        the array itself (e.g. one batch of a pinned host batch stream)."""
        step = int(np.prod(self.shape[1:])) if len(self.shape) > 1 else 1
        return _View(self.offset(row * step))


class _View:
    """A raw pointer that stands in for an array in the C-ABI wrappers."""

    def __init__(self, ptr: C.c_void_p):
        self.ptr = ptr

    def offset(self, elements: int) -> C.c_void_p:
        assert elements == 0, "offset into a view"
        return self.ptr


class Architecture:
    """Architecture (arch.hpp:36-57) compiled to a device plan (ghc_plan)."""

    def __init__(self, ctx: Context, text: str):
        self.ctx = ctx
        self.text = text
        h = C.c_void_p()
        check(ctx.lib.ghc_plan_create(ctx.h, text.encode(), C.byref(h)), "parse_architecture")
        self.h = h

    def __del__(self):
        try:
            if self.h and self.ctx.h and not _SHUTDOWN[0]:
                self.ctx.lib.ghc_plan_destroy(self.h)
            self.h = None
        except Exception:
            pass

    @property
    def n_params(self) -> int:
        return int(self.ctx.lib.ghc_plan_n_params(self.h))

    @property
    def input_width(self) -> int:
        return int(self.ctx.lib.ghc_plan_input_width(self.h))

    @property
    def n_classes(self) -> int:
        return int(self.ctx.lib.ghc_plan_n_classes(self.h))

    def check_error(self):
        """ghc_plan_check_error: raise ShapeError if a launch of this plan met a
        label outside [0,K) since the last check (nn.cpp:241-244)."""
        check(self.ctx.lib.ghc_plan_check_error(self.h), "loss")

    @property
    def kernel_name(self) -> str:
        return self.ctx.lib.ghc_plan_kernel_name(self.h).decode()

    def tensors(self):
        cap = 64
        off = np.zeros(cap, np.int64); d0 = np.zeros(cap, np.int64); d1 = np.zeros(cap, np.int64)
        nt = C.c_int()
        check(self.ctx.lib.ghc_plan_tensors(self.h, _vp(off), _vp(d0), _vp(d1), cap, C.byref(nt)))
        return [(int(off[i]), int(d0[i]), int(d1[i])) for i in range(nt.value)]


def arch_info(text: str):
    """Host-only parse + validate (arch.cpp:26-73,173-214): (n_params,
    input_width, n_classes); raises ConfigError like the reference."""
    n = C.c_int64(); wdt = C.c_int64(); k = C.c_int32()
    check(_lib.load().ghc_arch_info(text.encode(), C.byref(n), C.byref(wdt), C.byref(k)),
          "parse_architecture")
    return n.value, wdt.value, k.value


def init_weights(arch, seed: int) -> np.ndarray:
    """nn.cpp:83-98 (host, f64, bit-identical to the reference).  `arch` is an
    Architecture or the architecture text."""
    if isinstance(arch, str):
        w = np.zeros(arch_info(arch)[0], np.float64)
        check(_lib.load().ghc_init_weights_text(arch.encode(), seed, _vp(w)), "init_weights")
        return w
    w = np.zeros(arch.n_params, np.float64)
    check(arch.ctx.lib.ghc_init_weights(arch.h, seed, _vp(w)), "init_weights")
    return w


def worker_grad_device(arch: Architecture, w: DeviceArray, x: DeviceArray, y: DeviceArray, n: int,
                       grad: DeviceArray, loss_sum: DeviceArray, grad_scale: float | None = None,
                       idx: DeviceArray | None = None):
    """Fused forward+loss+backward on device buffers (ghc_worker_grad)."""
    scale = 1.0 / n if grad_scale is None else grad_scale
    check(arch.ctx.lib.ghc_worker_grad(arch.h, w.ptr, x.ptr, y.ptr,
                                       idx.ptr if idx is not None else None, n, scale,
                                       grad.ptr, loss_sum.ptr), "worker_grad")


def worker_grads_device(arch: Architecture, w: DeviceArray, x: DeviceArray, y: DeviceArray | None,
                        idx: list, n: list, grad: DeviceArray, loss: DeviceArray | None = None):
    """ghc_worker_grads: len(n) independent worker gradients in one launch;
    worker k at w[k] (rows of w = P each), rows idx[k] (a DeviceArray or None)
    of x, scaled by 1/n[k], into grad[k]; loss sums into loss[k]."""
    W = len(n)
    P = arch.n_params
    ptrs = (C.c_void_p * W)(*[i.ptr.value if i is not None else None for i in idx])
    ns = (C.c_int32 * W)(*[int(v) for v in n])
    check(arch.ctx.lib.ghc_worker_grads(arch.h, W, w.ptr, w.shape[1] if len(w.shape) > 1 else P, x.ptr,
                                        y.ptr if y is not None else None, ptrs, ns, grad.ptr,
                                        grad.shape[1] if len(grad.shape) > 1 else P,
                                        loss.ptr if loss is not None else None), "worker_grads")


def forward_backward(w: np.ndarray, arch: Architecture, x: np.ndarray, y: np.ndarray):
    """forward (nn.cpp:100) + loss (nn.cpp:234) + backward (nn.cpp:250) with
    host arrays: returns (mean gradient f32[P], loss).  Copy-in/copy-out."""
    ctx = arch.ctx
    x = np.ascontiguousarray(x, np.float32).reshape(-1, arch.input_width)
    y = np.ascontiguousarray(y, np.int32)
    n = y.shape[0]
    if n < 1:
        raise ShapeError("batch: n_samples must be >= 1")
    if x.shape[0] != n:
        raise ShapeError("batch: inputs size != n_samples*width")
    if y.min() < 0 or y.max() >= arch.n_classes:
        raise ShapeError(f"loss: label out of range [0,{arch.n_classes})")
    dw = ctx.upload(np.asarray(w, np.float32))
    dx = ctx.upload(x)
    dy = ctx.upload(y)
    g = ctx.array(arch.n_params)
    ls = ctx.array(1)
    worker_grad_device(arch, dw, dx, dy, n, g, ls)
    arch.check_error()
    return g.numpy(), float(ls.numpy()[0]) / n


def forward(w: np.ndarray, arch: Architecture, x: np.ndarray, y: np.ndarray):
    """forward + loss: returns (probs[n×K], loss)."""
    ctx = arch.ctx
    x = np.ascontiguousarray(x, np.float32).reshape(-1, arch.input_width)
    y = np.ascontiguousarray(y, np.int32)
    n = y.shape[0]
    dw = ctx.upload(np.asarray(w, np.float32))
    dx = ctx.upload(x)
    dy = ctx.upload(y)
    probs = ctx.array((n, arch.n_classes))
    ls = ctx.array(1)
    check(ctx.lib.ghc_forward(arch.h, dw.ptr, dx.ptr, dy.ptr, None, n, probs.ptr, ls.ptr),
          "forward")
    arch.check_error()
    return probs.numpy(), float(ls.numpy()[0]) / n


@dataclass
class OptimState:
    """OptimState (optim.hpp:11-19)."""
    velocity: np.ndarray
    learning_rate: float = 0.01
    momentum: float = 0.0


def sgd_step(ctx: Context, w: np.ndarray, g: np.ndarray, s: OptimState):
    """sgd_step (optim.cpp:39-65): returns (w', OptimState'); raises
    NonFiniteGradientError (caller keeps its weights) on a non-finite g."""
    w = np.asarray(w, np.float32)
    if np.shape(g) != w.shape or s.velocity.shape != w.shape:
        raise ShapeError("sgd_step: gradient/velocity shape does not match weights")
    dw = ctx.upload(w); dv = ctx.upload(np.asarray(s.velocity, np.float32))
    dg = ctx.upload(np.asarray(g, np.float32))
    w2, v2 = ctx.array(w.shape), ctx.array(w.shape)
    st = ctx.upload(np.zeros(1, np.int32))
    # value semantics → the one-pass out-of-place kernel (ghc_sgd_step_out)
    check(ctx.lib.ghc_sgd_step_out(ctx.h, dw.ptr, dv.ptr, dg.ptr, w2.ptr, v2.ptr, w.size,
                                   s.learning_rate, s.momentum, st.ptr, None), "sgd_step")
    if int(st.numpy()[0]) == 2:
        raise NonFiniteGradientError("sgd_step: gradient has NaN/Inf entries; update rejected")
    return w2.numpy(), OptimState(v2.numpy(), s.learning_rate, s.momentum)


def elastic_pull(ctx: Context, w: np.ndarray, center: np.ndarray, alpha: float) -> np.ndarray:
    """elastic_pull (optim.cpp:67-80)."""
    dw = ctx.upload(np.asarray(w, np.float32)); dc = ctx.upload(np.asarray(center, np.float32))
    check(ctx.lib.ghc_elastic_pull(ctx.h, dw.ptr, dc.ptr, dw.shape[0], alpha), "elastic_pull")
    return dw.numpy()


def easgd_worker_step(ctx: Context, w, center, g, s: OptimState, alpha: float, tau: int,
                      batch_index: int) -> np.ndarray:
    """easgd_worker_step (optim.cpp:82-105)."""
    dw = ctx.upload(np.asarray(w, np.float32)); dc = ctx.upload(np.asarray(center, np.float32))
    dg = ctx.upload(np.asarray(g, np.float32)); st = ctx.upload(np.zeros(1, np.int32))
    w2 = ctx.array(dw.shape)
    check(ctx.lib.ghc_easgd_worker_step_out(ctx.h, dw.ptr, dc.ptr, dg.ptr, w2.ptr, dw.shape[0],
                                            s.learning_rate, alpha, tau, batch_index, st.ptr),
          "easgd_worker_step")
    if int(st.numpy()[0]) == 2:
        raise NonFiniteGradientError("easgd_worker_step: gradient has NaN/Inf entries")
    return w2.numpy()


def easgd_center_step(ctx: Context, center, worker, alpha: float, version: int = 0):
    """easgd_center_step (optim.cpp:107-123): returns (c', version+1)."""
    dc = ctx.upload(np.asarray(center, np.float32)); dw = ctx.upload(np.asarray(worker, np.float32))
    ver = ctx.upload(np.array([version], np.uint64))
    check(ctx.lib.ghc_easgd_center_step(ctx.h, dc.ptr, dw.ptr, dc.shape[0], alpha, ver.ptr),
          "easgd_center_step")
    return dc.numpy(), int(ver.numpy()[0])


class Master:
    """Device-resident Downpour master (ghc_master): w/v in HBM, version,
    on-device commit/reject.  `sync_rounds` runs whole sync rounds of the
    colocated worker in one persistent launch."""

    def __init__(self, arch: Architecture, w0: np.ndarray, lr: float, mu: float):
        self.arch = arch
        self.ctx = arch.ctx
        w0 = np.ascontiguousarray(w0, np.float64)
        h = C.c_void_p()
        check(self.ctx.lib.ghc_master_create(arch.h, _vp(w0), lr, mu, C.byref(h)), "master_create")
        self.h = h

    def __del__(self):
        try:
            if self.h and self.arch.h and self.ctx.h and not _SHUTDOWN[0]:
                self.ctx.lib.ghc_master_destroy(self.h)
            self.h = None
        except Exception:
            pass

    def sync_rounds(self, x: DeviceArray, y: DeviceArray, idx: DeviceArray | None, stride: int,
                    n: int, rounds: int, counts: DeviceArray | None = None,
                    loss_out: DeviceArray | None = None, idx_offset: int = 0,
                    loss_offset: int = 0, counts_offset: int = 0):
        check(self.ctx.lib.ghc_master_sync_rounds(
            self.h, x.ptr, y.ptr if y is not None else None,
            idx.offset(idx_offset) if idx is not None else None, stride,
            counts.offset(counts_offset) if counts is not None else None, n, rounds,
            loss_out.offset(loss_offset) if loss_out is not None else None), "sync_rounds")

    def apply(self, g: DeviceArray):
        check(self.ctx.lib.ghc_master_apply(self.h, g.ptr), "master_apply")

    def read(self):
        P = self.arch.n_params
        w = np.zeros(P, np.float32); v = np.zeros(P, np.float32)
        ver = C.c_uint64(); rej = C.c_uint64()
        check(self.ctx.lib.ghc_master_read(self.h, _vp(w), _vp(v), C.byref(ver), C.byref(rej)))
        return w, v, ver.value, rej.value

    def weights_ptr(self) -> C.c_void_p:
        wp = C.c_void_p()
        check(self.ctx.lib.ghc_master_weights(self.h, C.byref(wp), None))
        return wp


def pack_rows(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Packed dataset rows on the host (ghc_dataset_pack's layout): x, the
    label's int32 bits, zero pad to a multiple of 32 floats (128-byte rows)."""
    x = np.ascontiguousarray(x, np.float32)
    n, width = x.shape
    stride = (width + 1 + 31) & ~31
    out = np.zeros((n, stride), np.float32)
    out[:, :width] = x
    out[:, width] = np.ascontiguousarray(y, np.int32).view(np.float32)
    return out


def pack_dataset(ctx: Context, dx: DeviceArray, dy: DeviceArray) -> DeviceArray:
    """ghc_dataset_pack on the device; pass the result as x with y=None."""
    n, width = dx.shape
    stride = int(ctx.lib.ghc_packed_row_floats(width))
    out = DeviceArray(ctx, (n, stride))
    check(ctx.lib.ghc_dataset_pack(ctx.h, dx.ptr, dy.ptr, n, width, out.ptr), "dataset_pack")
    return out


class Resident:
    """ghc_resident: the persistent sync-round kernel launched once for
    `master` (n samples per round) and fed commands through doorbells.
    `submit` / `wait` use the pinned host ring (the per-call API: returns once
    the command's rounds are committed and their losses are in loss_out);
    `submit_stream` queues a submit + wait kernel pair on the context stream
    (device-timed with the context's CUDA events).  `stop` publishes the
    master state (required before reading the master)."""

    def __init__(self, master: "Master", n: int, idle_seconds: float = 2.0):
        self.master, self.ctx = master, master.ctx
        h = C.c_void_p()
        check(self.ctx.lib.ghc_resident_start(master.h, n, idle_seconds, C.byref(h)), "resident_start")
        self.h = h

    @staticmethod
    def _args(x, y, idx, idx_offset, loss_out, loss_offset):
        return (x.ptr, y.ptr if y is not None else None,
                idx.offset(idx_offset) if idx is not None else None,
                loss_out.offset(loss_offset) if loss_out is not None else None)

    def submit(self, x, y, idx, stride: int, rounds: int, loss_out=None, idx_offset: int = 0,
               loss_offset: int = 0) -> int:
        px, py, pi, pl = self._args(x, y, idx, idx_offset, loss_out, loss_offset)
        seq = C.c_uint64()
        check(self.ctx.lib.ghc_resident_submit(self.h, px, py, pi, stride, rounds, pl, C.byref(seq)),
              "resident_submit")
        return seq.value

    def wait(self, seq: int):
        check(self.ctx.lib.ghc_resident_wait(self.h, seq), "resident_wait")

    def submit_stream(self, x, y, idx, stride: int, rounds: int, loss_out=None, idx_offset: int = 0,
                      loss_offset: int = 0) -> int:
        px, py, pi, pl = self._args(x, y, idx, idx_offset, loss_out, loss_offset)
        seq = C.c_uint64()
        check(self.ctx.lib.ghc_resident_submit_stream(self.h, self.ctx.h, px, py, pi, stride, rounds,
                                                      pl, C.byref(seq)), "resident_submit_stream")
        return seq.value

    def check(self):
        check(self.ctx.lib.ghc_resident_check(self.h), "resident")

    def stop(self):
        if self.h is not None:
            h, self.h = self.h, None
            check(self.ctx.lib.ghc_resident_stop(h), "resident_stop")

    def __del__(self):
        try:
            if self.h is not None and not _SHUTDOWN[0]:
                self.stop()
        except Exception:
            pass


def validate(w, arch: Architecture, x, y):
    """validate: (accuracy, mean loss, correct count) of
    weights w over a held-out set, one fused forward on the device."""
    ctx = arch.ctx
    dw = ctx.upload(np.ascontiguousarray(w, np.float32))
    dx = ctx.upload(np.ascontiguousarray(x, np.float32))
    dy = ctx.upload(np.ascontiguousarray(y, np.int32))
    ok = C.c_int64(0)
    lo = C.c_double(0.0)
    check(ctx.lib.ghc_validate(arch.h, dw.ptr, dx.ptr, dy.ptr, len(y), C.byref(ok), C.byref(lo)),
          "validate")
    return ok.value / len(y), lo.value, ok.value


# ---------------------------------------------------------------- wire frames
FRAME_SHUTDOWN, FRAME_WEIGHTS, FRAME_GRADIENT = 0, 1, 2


def encode_frame(arch: Architecture, kind: int, w=None, version: int = 0, sample_count: int = 1,
                 wire_f64: bool = False) -> bytes:
    """GHUB frame (proto.cpp:214-272) packed on the device (ghc_encode_frame)."""
    ctx = arch.ctx
    n = C.c_int64(0)
    check(ctx.lib.ghc_frame_size(arch.h, kind, int(wire_f64), C.byref(n)), "frame_size")
    out = ctx.array(max(n.value, 16), np.uint8)
    dw = ctx.upload(np.ascontiguousarray(w, np.float32)) if w is not None else None
    ln = C.c_int64(0)
    check(ctx.lib.ghc_encode_frame(arch.h, kind, int(wire_f64), dw.ptr if dw else None, version,
                                   sample_count, out.ptr, out.nbytes, C.byref(ln)), "encode")
    return out.numpy()[: ln.value].tobytes()


def decode_frame(arch: Architecture, frame: bytes):
    """ghc_decode_frame → (kind, w f32[P] or None, version, sample_count, wire_f64);
    raises ProtocolError (with .decode_status) / ShapeError like the reference."""
    ctx = arch.ctx
    buf = np.frombuffer(frame, np.uint8) if len(frame) else np.zeros(1, np.uint8)
    d = ctx.upload(np.ascontiguousarray(buf))
    w = ctx.array(arch.n_params)
    kind, f64, st = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    ver, cnt = C.c_uint64(0), C.c_uint64(0)
    rc = ctx.lib.ghc_decode_frame(arch.h, d.ptr, len(frame), C.byref(kind), w.ptr, C.byref(ver),
                                  C.byref(cnt), C.byref(f64), C.byref(st))
    try:
        check(rc, "decode")
    except GradhubError as e:
        e.decode_status = st.value
        raise
    wv = w.numpy() if kind.value in (FRAME_WEIGHTS, FRAME_GRADIENT) else None
    return kind.value, wv, ver.value, cnt.value, bool(f64.value)


# ---------------------------------------------------------------- data layer
def data_spec(n_files, samples_per_file, seq_len=10, input_dim=5, n_classes=3, delta=5.0,
              seed=1234) -> DataSpec:
    return DataSpec(n_files, samples_per_file, seq_len, input_dim, n_classes, 0, delta, seed)


def generate(spec: DataSpec, f0: int = 0, nf: int | None = None):
    """generate_synthetic for files [f0, f0+nf): f32 rows."""
    nf = spec.n_files - f0 if nf is None else nf
    n = nf * spec.samples_per_file
    x = np.zeros((n, spec.seq_len * spec.input_dim), np.float32)
    y = np.zeros(n, np.int32)
    check(_lib.load().ghc_data_generate(C.byref(spec), f0, nf, _vp(x), _vp(y)), "generate")
    return x, y


def shard_files(n_files: int, n_workers: int, worker: int):
    """shard_files: (first_file, n_files) of `worker`."""
    f0 = C.c_int32(); nf = C.c_int32()
    check(_lib.load().ghc_data_shard(n_files, n_workers, worker, C.byref(f0), C.byref(nf)),
          "shard_files")
    return f0.value, nf.value


def epoch_indices(spec: DataSpec, n_workers: int, worker: int, epoch: int, shuffle_seed: int,
                  shuffle: bool = True) -> np.ndarray:
    """The worker's shard permutation for `epoch` (global sample indices)."""
    f0, nf = shard_files(spec.n_files, n_workers, worker)
    out = np.zeros(nf * spec.samples_per_file, np.int64)
    cnt = C.c_int64()
    check(_lib.load().ghc_data_epoch_indices(C.byref(spec), n_workers, worker, epoch,
                                             shuffle_seed, int(shuffle), _vp(out), C.byref(cnt)),
          "epoch_indices")
    return out[: cnt.value]


def batches(spec: DataSpec, n_workers: int, worker: int, batch_size: int, epochs: int,
            shuffle_seed: int, shuffle: bool = True):
    """batches over `epochs`: list of global-index arrays
    (short final batch of each epoch kept with its true size)."""
    out = []
    for e in range(epochs):
        idx = epoch_indices(spec, n_workers, worker, e, shuffle_seed, shuffle)
        out.extend(idx[i:i + batch_size] for i in range(0, len(idx), batch_size))
    return out


# ---------------------------------------------------------------- roles
DOWNPOUR, EASGD = 0, 1
SYNC, REPLAY = 0, 1


def train_config(**kw) -> "_lib.TrainConfig":
    """TrainConfig with the bench/test defaults."""
    d = dict(algo=DOWNPOUR, mode=SYNC, n_workers=2, batch_size=100, epochs=1, tau=10, lr=0.01,
             mu=0.9, alpha=0.5, shuffle=1, weight_seed=7, shuffle_seed=99, groups=0, flush_k=1,
             parent_lr=1.0, parent_mu=0.0, max_updates=0, pad_=0)
    d.update(kw)
    c = _lib.TrainConfig()
    for k, v in d.items():
        setattr(c, k, v)
    return c


class Session:
    """A training session (ghc_session): the SPEC master/worker roles with
    W workers on this GPU — sync / replayed-async Downpour, EASGD,
    hierarchical masters."""

    def __init__(self, arch: Architecture, cfg, spec: DataSpec):
        self.arch, self.cfg, self.spec = arch, cfg, spec
        self.ctx = arch.ctx
        h = C.c_void_p()
        check(self.ctx.lib.ghc_session_create(arch.h, C.byref(cfg), C.byref(spec), C.byref(h)),
              "session_create")
        self.h = h

    def __del__(self):
        try:
            if self.h and self.arch.h and self.ctx.h and not _SHUTDOWN[0]:
                self.ctx.lib.ghc_session_destroy(self.h)
            self.h = None
        except Exception:
            pass

    def run(self, order=None, max_trace=1 << 16):
        n = 0 if order is None else len(order)
        o = None if order is None else np.ascontiguousarray(order, np.int32)
        cap = max(n, max_trace)
        loss = np.full(cap, np.nan, np.float32)
        stale = np.zeros(cap, np.int64)
        check(self.ctx.lib.ghc_session_run(self.h, None if o is None else _vp(o), n, _vp(loss),
                                           _vp(stale), cap), "session_run")
        return loss, stale[:n]

    def load_data(self, x: np.ndarray, y: np.ndarray):
        """Replace the session's dataset rows (same shape as the spec's)."""
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        check(self.ctx.lib.ghc_session_load_data(self.h, _vp(x), _vp(y), len(y)), "load_data")

    def set_validation(self, x: np.ndarray, y: np.ndarray, every: int = 0):
        """Held-out set of the master's serial validation:
        every `every` master updates (0: only at the end) and once at the end."""
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        check(self.ctx.lib.ghc_session_set_validation(self.h, _vp(x), _vp(y), len(y), every),
              "set_validation")

    def validations(self):
        """VALIDATE_RESULT records: list of (version, accuracy, mean loss)."""
        n = C.c_int64(0)
        check(self.ctx.lib.ghc_session_validations(self.h, 0, None, None, None, C.byref(n)))
        ver = np.zeros(n.value, np.uint64)
        acc = np.zeros(n.value, np.float64)
        lo = np.zeros(n.value, np.float64)
        check(self.ctx.lib.ghc_session_validations(self.h, n.value, _vp(ver), _vp(acc), _vp(lo),
                                                   C.byref(n)))
        return [(int(a), float(b), float(c)) for a, b, c in zip(ver, acc, lo)]

    def read(self):
        P = self.arch.n_params
        W = self.cfg.n_workers
        G = max(self.cfg.groups, 1)
        w = np.zeros(P, np.float32); v = np.zeros(P, np.float32)
        ww = np.zeros((W, P), np.float32); gw = np.zeros((G, P), np.float32)
        st = np.zeros(4, np.uint64)
        check(self.ctx.lib.ghc_session_read(self.h, _vp(w), _vp(v), _vp(ww), _vp(gw), _vp(st)),
              "session_read")
        return {"w": w, "v": v, "worker_w": ww, "group_w": gw[: self.cfg.groups],
                "version": int(st[0]), "rejected": int(st[1]), "samples": int(st[2]),
                "rounds": int(st[3])}
