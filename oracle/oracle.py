"""CPU ORACLE — ctypes wrapper (TEST INFRASTRUCTURE ONLY).

Loads oracle/_build/libgh_oracle.so (the C restatement, gh_oracle.c) and, when
present, oracle/_ref/libghref.so (the reference's own sources + SPEC roles,
ref_roles.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm may import this module; the product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "_build", "libgh_oracle.so")
_REF = os.path.join(HERE, "_ref", "libghref.so")

OK, SHAPE, NONFINITE, CACHE_MISMATCH, CONFIG, TRANSPORT, PROTOCOL = range(7)
DOWNPOUR, EASGD = 0, 1
MAX_LAYERS = 16


class Arch(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("kind", C.c_int32 * MAX_LAYERS),
                ("a", C.c_int32 * MAX_LAYERS), ("b", C.c_int32 * MAX_LAYERS),
                ("c", C.c_int32 * MAX_LAYERS)]


class DataSpec(C.Structure):
    _fields_ = [("n_files", C.c_int32), ("samples_per_file", C.c_int32),
                ("seq_len", C.c_int32), ("input_dim", C.c_int32),
                ("n_classes", C.c_int32), ("pad_", C.c_int32),
                ("delta", C.c_double), ("seed", C.c_uint64)]


class TrainCfg(C.Structure):
    _fields_ = [("algo", C.c_int32), ("n_workers", C.c_int32),
                ("batch_size", C.c_int32), ("epochs", C.c_int32),
                ("lr", C.c_double), ("mu", C.c_double), ("alpha", C.c_double),
                ("tau", C.c_int32), ("shuffle", C.c_int32),
                ("weight_seed", C.c_uint64), ("shuffle_seed", C.c_uint64),
                ("wire_f64", C.c_int32), ("max_updates", C.c_int32),
                ("groups", C.c_int32), ("flush_k", C.c_int32),
                ("parent_lr", C.c_double), ("parent_mu", C.c_double)]


class RunStats(C.Structure):
    _fields_ = [("updates", C.c_int64), ("rejected", C.c_int64),
                ("samples", C.c_int64), ("version", C.c_uint64)]


def _p(a, t=C.c_double):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


_lib = None
_ref = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.gho_weights_checksum.restype = C.c_uint64
        _lib.gho_arch_n_params.restype = C.c_int64
        _lib.gho_arch_input_width.restype = C.c_int64
        _lib.gho_epoch_indices.restype = C.c_int64
        _lib.gho_mix_seed.restype = C.c_uint64
        _lib.gho_frame_size.restype = C.c_int64
        _lib.gho_frame_size.argtypes = [C.c_void_p, C.c_int, C.c_int]
        _lib.gho_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        _lib.gho_rng_u64.restype = C.c_uint64
        _lib.gho_rng_normal.restype = C.c_double
        _lib.gho_rng_uniform01.restype = C.c_double
        _lib.gho_rng_below.restype = C.c_uint64
        _lib.gho_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        _lib.gho_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        _lib.gho_init_weights.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        _lib.gho_sgd_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                      C.c_double, C.c_double]
        _lib.gho_elastic_pull.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_double]
        _lib.gho_easgd_worker_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                               C.c_double, C.c_double, C.c_uint64, C.c_uint64]
        _lib.gho_easgd_center_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_double]
        _lib.gho_forward_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.gho_finite_diff.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int64, C.c_double, C.c_void_p]
        _lib.gho_epoch_indices.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_uint64, C.c_int32, C.c_void_p]
        _lib.gho_generate_files.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                            C.c_void_p]
    return _lib


def has_ref() -> bool:
    return os.path.exists(_REF)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            raise FileNotFoundError(f"{_REF} not built (needs /root/reference at build time)")
        _ref = C.CDLL(_REF)
        _ref.ghr_last_error.restype = C.c_char_p
        _ref.ghr_init_weights.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p]
        _ref.ghr_sgd_step.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_double, C.c_double, C.c_void_p]
        _ref.ghr_elastic_pull.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_double]
        _ref.ghr_easgd_worker_step.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_double, C.c_double, C.c_uint64, C.c_uint64]
        _ref.ghr_easgd_center_step.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_double,
                                               C.c_void_p]
        _ref.ghr_forward_backward.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        _ref.ghr_stale_cache_probe.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_int64]
        _ref.ghr_finite_diff.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int64, C.c_double, C.c_void_p]
        _ref.ghr_checksum.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p]
        _ref.ghr_encode.argtypes = [C.c_int, C.c_char_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                    C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
        _ref.ghr_epoch_indices.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p]
        _ref.ghr_bench_sync.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int32,
                                        C.c_int32, C.c_void_p, C.c_void_p]
        _ref.ghr_bench_fwd_bwd.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.c_void_p]
    return _ref


# --------------------------------------------------------------------------
# Python-facing helpers
# --------------------------------------------------------------------------

def parse_arch(text: str) -> Arch:
    a = Arch()
    rc = lib().gho_arch_parse(text.encode(), C.byref(a))
    if rc != OK:
        raise ValueError(f"bad architecture {text!r} (status {rc})")
    return a


def n_params(arch: Arch) -> int:
    return int(lib().gho_arch_n_params(C.byref(arch)))


def tensor_table(arch: Arch):
    cap = 48
    off = np.zeros(cap, np.int64); sz = np.zeros(cap, np.int64)
    d0 = np.zeros(cap, np.int64); d1 = np.zeros(cap, np.int64)
    nt = lib().gho_arch_tensors(C.byref(arch), _p(off, C.c_int64), _p(sz, C.c_int64),
                                _p(d0, C.c_int64), _p(d1, C.c_int64), cap)
    return [(int(off[i]), int(sz[i]), int(d0[i]), int(d1[i])) for i in range(nt)]


def init_weights(arch: Arch, seed: int) -> np.ndarray:
    w = np.zeros(n_params(arch), np.float64)
    lib().gho_init_weights(C.byref(arch), seed, _p(w))
    return w


def forward_backward(arch: Arch, w, x, y, want_grad=True):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.int32)
    n = y.shape[0]
    K = lib().gho_arch_n_classes(C.byref(arch))
    g = np.zeros(n_params(arch), np.float64) if want_grad else None
    probs = np.zeros((n, K), np.float64)
    lo = C.c_double(0.0)
    rc = lib().gho_forward_backward(C.byref(arch), _p(np.ascontiguousarray(w, np.float64)),
                                    _p(x), _p(y, C.c_int32), n, _p(g), _p(probs), C.byref(lo))
    if rc != OK:
        raise RuntimeError(f"gho_forward_backward status {rc}")
    return g, probs, lo.value


def validate(arch: Arch, w, x, y):
    """gho_validate: (correct count, mean loss) over a held-out set."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.int32)
    ok = C.c_int64(0)
    lo = C.c_double(0.0)
    rc = lib().gho_validate(C.byref(arch), _p(np.ascontiguousarray(w, np.float64)), _p(x),
                            _p(y, C.c_int32), C.c_int64(len(y)), C.byref(ok), C.byref(lo))
    if rc != OK:
        raise RuntimeError(f"gho_validate status {rc}")
    return ok.value, lo.value


def encode_frame(arch: Arch, kind: int, w, version=0, sample_count=1, wire_f64=0) -> bytes:
    """gho_encode_frame: kind 0 SHUTDOWN, 1 WEIGHTS, 2 GRADIENT."""
    n = lib().gho_frame_size(C.byref(arch), kind, wire_f64)
    buf = np.zeros(n, np.uint8)
    ln = C.c_int64(0)
    wv = None if w is None else np.ascontiguousarray(w, np.float64)
    rc = lib().gho_encode_frame(C.byref(arch), kind, _p(wv), C.c_uint64(version),
                                C.c_uint64(sample_count), wire_f64, _p(buf, C.c_uint8),
                                C.c_int64(n), C.byref(ln))
    if rc != OK:
        raise RuntimeError(f"gho_encode_frame status {rc}")
    return bytes(buf[: ln.value])


def decode_frame(arch: Arch, frame: bytes):
    """gho_decode_frame → (rc, decode_status, kind, w, version, sample_count, f64)."""
    buf = np.frombuffer(frame, np.uint8).copy() if len(frame) else np.zeros(1, np.uint8)
    w = np.zeros(n_params(arch), np.float64)
    kind, st, f64 = C.c_int(0), C.c_int(0), C.c_int(0)
    ver, cnt = C.c_uint64(0), C.c_uint64(0)
    rc = lib().gho_decode_frame(C.byref(arch), _p(buf, C.c_uint8), C.c_int64(len(frame)),
                                C.byref(kind), _p(w), C.byref(ver), C.byref(cnt), C.byref(f64),
                                C.byref(st))
    return rc, st.value, kind.value, w, ver.value, cnt.value, f64.value


def ref_encode(arch_text: str, kind: int, w, version=0, sample_count=1, wire_f64=0) -> bytes:
    """The reference's own encoder (oracle/_ref, proto.cpp encode)."""
    buf = np.zeros(1 << 26, np.uint8) if w is not None and len(w) > 1 << 20 else np.zeros(1 << 20, np.uint8)
    n = C.c_int64(0)
    wv = None if w is None else np.ascontiguousarray(w, np.float64)
    rc = ref().ghr_encode(kind, None if arch_text is None else arch_text.encode(), _p(wv),
                          version, sample_count, wire_f64, _p(buf, C.c_uint8), len(buf), C.byref(n))
    if rc != 0:
        raise RuntimeError(f"ghr_encode status {rc}")
    return bytes(buf[: n.value])


def finite_diff(arch: Arch, w, x, y, eps=1e-5):
    g = np.zeros(n_params(arch), np.float64)
    rc = lib().gho_finite_diff(C.byref(arch), _p(np.ascontiguousarray(w, np.float64)),
                               _p(np.ascontiguousarray(x, np.float64)),
                               _p(np.ascontiguousarray(y, np.int32), C.c_int32), len(y), eps, _p(g))
    if rc != OK:
        raise RuntimeError(f"gho_finite_diff status {rc}")
    return g


def sgd_step(w, v, g, lr, mu):
    w = np.array(w, np.float64); v = np.array(v, np.float64)
    rc = lib().gho_sgd_step(_p(w), _p(v), _p(np.ascontiguousarray(g, np.float64)), len(w), lr, mu)
    return rc, w, v


def data_spec(n_files, samples_per_file, seq_len=10, input_dim=5, n_classes=3, delta=5.0,
              seed=1234) -> DataSpec:
    return DataSpec(n_files, samples_per_file, seq_len, input_dim, n_classes, 0, delta, seed)


def generate(spec: DataSpec):
    n = spec.n_files * spec.samples_per_file
    x = np.zeros((n, spec.seq_len * spec.input_dim), np.float64)
    y = np.zeros(n, np.int32)
    lib().gho_generate(C.byref(spec), _p(x), _p(y, C.c_int32))
    return x, y


def epoch_indices(spec: DataSpec, W, k, epoch, shuffle_seed, shuffle=True):
    f0 = C.c_int32(); nf = C.c_int32()
    lib().gho_shard_files(spec.n_files, W, k, C.byref(f0), C.byref(nf))
    out = np.zeros(nf.value * spec.samples_per_file, np.int64)
    cnt = lib().gho_epoch_indices(C.byref(spec), W, k, epoch, shuffle_seed, int(shuffle),
                                  _p(out, C.c_int64))
    assert cnt == out.shape[0]
    return out


def train_cfg(**kw) -> TrainCfg:
    d = dict(algo=DOWNPOUR, n_workers=2, batch_size=100, epochs=1, lr=0.01, mu=0.9,
             alpha=0.5, tau=10, shuffle=1, weight_seed=7, shuffle_seed=99, wire_f64=0,
             max_updates=0, groups=0, flush_k=1, parent_lr=1.0, parent_mu=0.0)
    d.update(kw)
    c = TrainCfg()
    for k, v in d.items():
        setattr(c, k, v)
    return c


@dataclass
class RunOut:
    w: np.ndarray
    v: np.ndarray | None
    stats: RunStats
    loss: np.ndarray
    extra: dict


def run_sync(arch: Arch, spec: DataSpec, x, y, cfg: TrainCfg, max_trace=100000) -> RunOut:
    P = n_params(arch)
    w = np.zeros(P); v = np.zeros(P)
    trace = np.full(max(cfg.max_updates, 1) if cfg.max_updates else max_trace, np.nan)
    st = RunStats()
    rc = lib().gho_run_sync(C.byref(arch), C.byref(spec), _p(x), _p(y, C.c_int32),
                            C.byref(cfg), _p(w), _p(v), _p(trace), C.byref(st))
    if rc != OK:
        raise RuntimeError(f"gho_run_sync status {rc}")
    n = st.updates + st.rejected
    return RunOut(w, v, st, trace[:n], {})


def run_replay(arch: Arch, spec: DataSpec, x, y, cfg: TrainCfg, order,
               allow_error=False) -> RunOut:
    P = n_params(arch)
    order = np.ascontiguousarray(order, np.int32)
    w = np.zeros(P); v = np.zeros(P)
    ww = np.zeros((cfg.n_workers, P))
    stale = np.zeros(len(order), np.int64)
    trace = np.zeros(len(order))
    st = RunStats()
    rc = lib().gho_run_replay(C.byref(arch), C.byref(spec), _p(x), _p(y, C.c_int32),
                              C.byref(cfg), _p(order, C.c_int32), C.c_int64(len(order)),
                              _p(w), _p(v), _p(ww), _p(stale, C.c_int64), _p(trace),
                              C.byref(st))
    if rc != OK and not allow_error:
        raise RuntimeError(f"gho_run_replay status {rc}")
    return RunOut(w, v, st, trace, {"worker_w": ww, "staleness": stale, "rc": rc})


def run_hier(arch: Arch, spec: DataSpec, x, y, cfg: TrainCfg, max_trace=100000) -> RunOut:
    P = n_params(arch)
    w = np.zeros(P)
    gw = np.zeros((cfg.groups, P))
    trace = np.full(cfg.max_updates if cfg.max_updates else max_trace, np.nan)
    st = RunStats()
    rc = lib().gho_run_hier(C.byref(arch), C.byref(spec), _p(x), _p(y, C.c_int32),
                            C.byref(cfg), _p(w), _p(gw), _p(trace), C.byref(st))
    if rc != OK:
        raise RuntimeError(f"gho_run_hier status {rc}")
    return RunOut(w, None, st, trace, {"group_w": gw})


# ---- reference-library entry points (oracle/_ref) ----

def ref_forward_backward(arch_text: str, w, x, y):
    n = len(y)
    K = parse_arch(arch_text).b[parse_arch(arch_text).n_layers - 1]
    g = np.zeros(len(w)); probs = np.zeros((n, K)); lo = C.c_double()
    rc = ref().ghr_forward_backward(arch_text.encode(), _p(np.ascontiguousarray(w, np.float64)),
                                    _p(np.ascontiguousarray(x, np.float64)),
                                    _p(np.ascontiguousarray(y, np.int32), C.c_int32), n, _p(g),
                                    _p(probs), C.byref(lo))
    if rc != OK:
        raise RuntimeError(f"ghr_forward_backward {rc}: {ref().ghr_last_error().decode()}")
    return g, probs, lo.value


def ref_run_sync(arch_text: str, spec: DataSpec, x, y, cfg: TrainCfg) -> RunOut:
    P = n_params(parse_arch(arch_text))
    w = np.zeros(P); v = np.zeros(P)
    trace = np.full(cfg.max_updates if cfg.max_updates else 100000, np.nan)
    st = RunStats()
    rc = ref().ghr_run_sync(arch_text.encode(), C.byref(spec),
                            None if x is None else _p(x),
                            None if y is None else _p(y, C.c_int32),
                            C.byref(cfg), _p(w), _p(v), _p(trace), C.byref(st))
    if rc != OK:
        raise RuntimeError(f"ghr_run_sync {rc}: {ref().ghr_last_error().decode()}")
    n = st.updates + st.rejected
    return RunOut(w, v, st, trace[:n], {})


def ref_bench_sync(arch_text: str, spec: DataSpec, cfg: TrainCfg, warmup: int, timed: int):
    sec = C.c_double(); n = C.c_int64()
    rc = ref().ghr_bench_sync(arch_text.encode(), C.byref(spec), C.byref(cfg), warmup, timed,
                              C.byref(sec), C.byref(n))
    if rc != OK:
        raise RuntimeError(f"ghr_bench_sync {rc}: {ref().ghr_last_error().decode()}")
    return sec.value, n.value
