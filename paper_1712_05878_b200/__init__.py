"""B200-native (sm_100a) Downpour/EASGD hot path of arXiv 1712.05878 (mpi_learn).

The compute lives in libghc.so (paper_1712_05878_b200/csrc, C ABI in
include/ghc.h); this package is the Python host mirror of the reference's
Model / Algo / Data interface used by the tests and the bench.
"""
from .gradhub import (Architecture, arch_info, CacheMismatchError, ConfigError, Context,  # noqa: F401
                      CudaError, DeviceArray, GradhubError, Master, NonFiniteGradientError,
                      OptimState, ProtocolError, ShapeError, TransportError, batches, data_spec,
                      easgd_center_step, easgd_worker_step, elastic_pull, epoch_indices, forward,
                      forward_backward, generate, init_weights, sgd_step, shard_files,
                      worker_grad_device, worker_grads_device, Session, train_config, DOWNPOUR,
                      EASGD, SYNC,
                      REPLAY, validate, HostArray, encode_frame, decode_frame,
                      FRAME_SHUTDOWN, FRAME_WEIGHTS, FRAME_GRADIENT, Resident, pack_rows,
                      pack_dataset)

BENCH_ARCH = "lstm(5,20,10),softmax(20,3)"
