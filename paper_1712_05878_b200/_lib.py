"""ctypes binding of libghc.so (include/ghc.h).

Fails loudly: importing the product on a host where the in-tree library was
not built raises; every non-OK status raises the matching reference error
class (errors.hpp:10-45).  There is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GHC_LIB_PATH: load another in-tree build (A/B experiments, tools/ablate.sh)
LIB_PATH = os.environ.get("GHC_LIB_PATH") or os.path.join(HERE, "_build", "libghc.so")


class GradhubError(RuntimeError):
    """Base of the reference exception taxonomy."""


class ShapeError(GradhubError):            # errors.hpp:10-14
    pass


class NonFiniteGradientError(GradhubError):  # errors.hpp:16-21
    pass


class CacheMismatchError(GradhubError):    # errors.hpp:23-27
    pass


class ConfigError(GradhubError):           # errors.hpp:29-32
    pass


class TransportError(GradhubError):        # errors.hpp:34-38
    pass


class ProtocolError(GradhubError):         # errors.hpp:40-45
    pass


class CudaError(GradhubError):
    pass


class NcclError(GradhubError):
    pass


_STATUS = {1: ShapeError, 2: NonFiniteGradientError, 3: CacheMismatchError, 4: ConfigError,
           5: TransportError, 6: ProtocolError, 7: CudaError, 8: NcclError}

# Every symbol include/ghc.h declares: (name, restype, argtypes)
_vp, _i32, _i64, _u64, _f32, _sz, _cp = (C.c_void_p, C.c_int32, C.c_int64, C.c_uint64,
                                         C.c_float, C.c_size_t, C.c_char_p)
SIGNATURES = [
    ("ghc_version", _cp, []),
    ("ghc_last_error", _cp, []),
    ("ghc_status_name", _cp, [C.c_int]),
    ("ghc_device_count", C.c_int, [_vp]),
    ("ghc_ctx_create", C.c_int, [C.c_int, _vp]),
    ("ghc_ctx_destroy", None, [_vp]),
    ("ghc_ctx_sync", C.c_int, [_vp]),
    ("ghc_ctx_num_sms", C.c_int, [_vp]),
    ("ghc_ctx_launch_count", _u64, [_vp]),
    ("ghc_malloc", C.c_int, [_vp, _sz, _vp]),
    ("ghc_free", C.c_int, [_vp, _vp]),
    ("ghc_host_alloc", C.c_int, [_sz, _vp]),
    ("ghc_ipc_handle", C.c_int, [_vp, _vp, _vp]),
    ("ghc_ipc_open", C.c_int, [_vp, _vp, _vp]),
    ("ghc_ipc_close", C.c_int, [_vp, _vp]),
    ("ghc_host_free", C.c_int, [_vp]),
    ("ghc_memcpy_h2d", C.c_int, [_vp, _vp, _vp, _sz]),
    ("ghc_memcpy_d2h", C.c_int, [_vp, _vp, _vp, _sz]),
    ("ghc_memcpy_d2d", C.c_int, [_vp, _vp, _vp, _sz]),
    ("ghc_memset", C.c_int, [_vp, _vp, C.c_int, _sz]),
    ("ghc_memcpy_peer", C.c_int, [_vp, _vp, _i32, _vp, _i32, _sz]),
    ("ghc_weights_import_f64", C.c_int, [_vp, _vp, _vp, _i64, _vp]),
    ("ghc_nll_sum", C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    ("ghc_stream_hold", C.c_int, [_vp]),
    ("ghc_stream_release", C.c_int, [_vp]),
    ("ghc_timer_start", C.c_int, [_vp]),
    ("ghc_timer_stop", C.c_int, [_vp, _vp]),
    ("ghc_plan_create", C.c_int, [_vp, _cp, _vp]),
    ("ghc_plan_destroy", None, [_vp]),
    ("ghc_plan_n_params", _i64, [_vp]),
    ("ghc_plan_input_width", _i64, [_vp]),
    ("ghc_plan_n_classes", _i32, [_vp]),
    ("ghc_plan_tensors", C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp]),
    ("ghc_plan_kernel_name", _cp, [_vp]),
    ("ghc_plan_check_error", C.c_int, [_vp]),
    ("ghc_plan_set_probe", C.c_int, [_vp, _vp]),
    ("ghc_plan_max_clusters", _i32, [_vp]),
    ("ghc_plan_cluster_size", _i32, [_vp]),
    ("ghc_diag_barrier_bench", C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp]),
    ("ghc_diag_launch_bench", C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    ("ghc_arch_info", C.c_int, [_cp, _vp, _vp, _vp]),
    ("ghc_init_weights_text", C.c_int, [_cp, _u64, _vp]),
    ("ghc_init_weights", C.c_int, [_vp, _u64, _vp]),
    ("ghc_worker_grad", C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _f32, _vp, _vp]),
    ("ghc_worker_grads", C.c_int, [_vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    ("ghc_forward", C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    ("ghc_forward_cache", C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    ("ghc_gemm_nt", C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                              _i32, _vp, _vp, _i32, _f32]),
    ("ghc_transpose", C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32]),
    ("ghc_sgd_apply", C.c_int, [_vp, _vp, _vp, _vp, _i64, _f32, _f32, _vp, _vp]),
    ("ghc_elastic_pull", C.c_int, [_vp, _vp, _vp, _i64, _f32]),
    ("ghc_easgd_worker_step", C.c_int, [_vp, _vp, _vp, _vp, _i64, _f32, _f32, _u64, _u64, _vp]),
    ("ghc_sgd_step_out", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _f32, _f32, _vp, _vp]),
    ("ghc_easgd_worker_step_out", C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _f32, _f32, _u64, _u64, _vp]),
    ("ghc_easgd_center_step", C.c_int, [_vp, _vp, _vp, _i64, _f32, _vp]),
    ("ghc_weighted_mean", C.c_int, [_vp, _vp, _vp, _vp, _i32, _i64]),
    ("ghc_master_create", C.c_int, [_vp, _vp, _f32, _f32, _vp]),
    ("ghc_master_destroy", None, [_vp]),
    ("ghc_master_weights", C.c_int, [_vp, _vp, _vp]),
    ("ghc_master_read", C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    ("ghc_master_sync_rounds", C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _i32, _vp]),
    ("ghc_master_apply", C.c_int, [_vp, _vp]),
    ("ghc_packed_row_floats", _i32, [_i32]),
    ("ghc_dataset_pack", C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    ("ghc_resident_start", C.c_int, [_vp, _i64, C.c_double, _vp]),
    ("ghc_resident_submit", C.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    ("ghc_resident_wait", C.c_int, [_vp, _u64]),
    ("ghc_resident_submit_stream", C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    ("ghc_resident_check", C.c_int, [_vp]),
    ("ghc_resident_bench_calls", C.c_int, [_vp, _vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp]),
    ("ghc_resident_times", C.c_int, [_vp, _vp]),
    ("ghc_resident_stop", C.c_int, [_vp]),
    ("ghc_comm_unique_id", C.c_int, [_vp]),
    ("ghc_comm_init", C.c_int, [_vp, _vp, _i32, _i32, _vp]),
    ("ghc_comm_split", C.c_int, [_vp, _i32, _i32, _vp]),
    ("ghc_comm_destroy", None, [_vp]),
    ("ghc_comm_rank", _i32, [_vp]),
    ("ghc_comm_size", _i32, [_vp]),
    ("ghc_comm_reduce_sum", C.c_int, [_vp, _vp, _vp, _i64, _i32]),
    ("ghc_comm_broadcast", C.c_int, [_vp, _vp, _i64, _i32]),
    ("ghc_comm_allreduce_sum", C.c_int, [_vp, _vp, _vp, _i64]),
    ("ghc_dist_sync_rounds", C.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _i64, _vp, _i32, _vp]),
    ("ghc_p2p_create", C.c_int, [_vp, _i32, _i32, _vp]),
    ("ghc_p2p_create_virtual", C.c_int, [_vp, _i32, _vp]),
    ("ghc_p2p_export", C.c_int, [_vp, _vp]),
    ("ghc_p2p_import", C.c_int, [_vp, _vp]),
    ("ghc_p2p_destroy", None, [_vp]),
    ("ghc_p2p_diag_push", C.c_int, [_vp, _i32, C.c_uint32, _i32]),
    ("ghc_p2p_diag_check", C.c_int, [_vp, _i32, C.c_uint32, _i32, _vp]),
    ("ghc_p2p_row_elems", _i32, [_vp]),
    ("ghc_p2p_barrier", C.c_int, [_vp]),
    ("ghc_p2p_sync_rounds", C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp]),
    ("ghc_session_create", C.c_int, [_vp, _vp, _vp, _vp]),
    ("ghc_session_destroy", None, [_vp]),
    ("ghc_session_run", C.c_int, [_vp, _vp, _i64, _vp, _vp, _i64]),
    ("ghc_session_set_validation", C.c_int, [_vp, _vp, _vp, _i64, _i32]),
    ("ghc_session_load_data", C.c_int, [_vp, _vp, _vp, _i64]),
    ("ghc_session_validations", C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp]),
    ("ghc_validate", C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    ("ghc_frame_size", C.c_int, [_vp, _i32, _i32, _vp]),
    ("ghc_encode_frame", C.c_int, [_vp, _i32, _i32, _vp, _u64, _u64, _vp, _i64, _vp]),
    ("ghc_decode_frame", C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ghc_session_read", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    ("ghc_data_generate", C.c_int, [_vp, _i32, _i32, _vp, _vp]),
    ("ghc_data_shard", C.c_int, [_i32, _i32, _i32, _vp, _vp]),
    ("ghc_data_epoch_indices", C.c_int, [_vp, _i32, _i32, _i32, _u64, _i32, _vp, _vp]),
]

_lib = None

# Nsight Compute / Systems inject into the process and serialise kernels:
# cooperative cluster launches are not replayable there (plain cluster
# launches of the same grid are — it never exceeds the co-resident clusters),
# and kernels that wait on other kernels (the stream gate, the resident round
# service) cannot make progress.
PROFILER_ENV = ("NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "CUDA_INJECTION64_PATH")


def under_profiler() -> bool:
    return any(os.environ.get(k) for k in PROFILER_ENV)


def load():
    """Load the in-tree libghc.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1712_05878_b200.build` "
                              "(no CPU fallback exists)")
        if under_profiler():
            os.environ.setdefault("GHC_NO_COOP", "1")
        lib = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = load().ghc_last_error().decode(errors="replace")
        raise _STATUS.get(status, GradhubError)(f"{what}: {msg}" if what else msg)


class DataSpec(C.Structure):
    """ghc_data_spec (SPEC.md:421-423 DatasetSpec)."""
    _fields_ = [("n_files", C.c_int32), ("samples_per_file", C.c_int32),
                ("seq_len", C.c_int32), ("input_dim", C.c_int32), ("n_classes", C.c_int32),
                ("pad_", C.c_int32), ("delta", C.c_double), ("seed", C.c_uint64)]


class TrainConfig(C.Structure):
    """ghc_train_config (SPEC.md:547-550 TrainConfig)."""
    _fields_ = [("algo", C.c_int32), ("mode", C.c_int32), ("n_workers", C.c_int32),
                ("batch_size", C.c_int32), ("epochs", C.c_int32), ("tau", C.c_int32),
                ("lr", C.c_float), ("mu", C.c_float), ("alpha", C.c_float),
                ("shuffle", C.c_int32), ("weight_seed", C.c_uint64),
                ("shuffle_seed", C.c_uint64), ("groups", C.c_int32), ("flush_k", C.c_int32),
                ("parent_lr", C.c_float), ("parent_mu", C.c_float),
                ("max_updates", C.c_int32), ("pad_", C.c_int32)]
