/*
 * ghc.h — C ABI of the B200-native Downpour/EASGD hot path ("gradhub-cuda").
 *
 * The drop-in boundary for arXiv 1712.05878's reference (`gradhub`,
 * /root/reference/proj): the reference's C++ Model / Algo / Data interfaces
 * and master/worker loop stay the caller-facing API (see INTEGRATION.md for
 * the C++ shim a maintainer adds); underneath them every compute step runs
 * as a hand-written sm_100a kernel behind these extern "C" entry points.
 *
 *  - plain pointers and sizes only; no C++ or torch types cross the ABI;
 *  - device pointers are `d_*`, host pointers `h_*`; sizes in elements;
 *  - every call is stream-ordered on the context's CUDA stream and
 *    asynchronous unless it says otherwise; ghc_ctx_sync() is the explicit
 *    sync point;
 *  - errors never throw: each call returns a ghc_status that maps 1:1 onto
 *    the reference exception classes (errors.hpp:10-45); ghc_last_error()
 *    returns the thread's last message.  There is no CPU fallback: on a host
 *    without a usable sm_100 device ghc_ctx_create fails with GHC_ERR_CUDA.
 *
 * Reference interface each entry point replaces is cited per function.
 */
#ifndef GHC_H
#define GHC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ghc_status {
  GHC_OK = 0,
  GHC_ERR_SHAPE = 1,          /* ShapeError              errors.hpp:10-14 */
  GHC_ERR_NONFINITE = 2,      /* NonFiniteGradientError  errors.hpp:16-21 */
  GHC_ERR_CACHE_MISMATCH = 3, /* CacheMismatchError      errors.hpp:23-27 */
  GHC_ERR_CONFIG = 4,         /* ConfigError             errors.hpp:29-32 */
  GHC_ERR_TRANSPORT = 5,      /* TransportError          errors.hpp:34-38 */
  GHC_ERR_PROTOCOL = 6,       /* ProtocolError           errors.hpp:40-45 */
  GHC_ERR_CUDA = 7,           /* CUDA runtime / launch failure (new)       */
  GHC_ERR_NCCL = 8            /* NCCL failure (new)                         */
} ghc_status;

typedef struct ghc_ctx ghc_ctx;       /* one per (GPU, host thread): stream + scratch */
typedef struct ghc_plan ghc_plan;     /* Architecture compiled to a kernel plan      */
typedef struct ghc_master ghc_master; /* device-resident master state (w, v, version) */

const char* ghc_version(void);
const char* ghc_last_error(void);
const char* ghc_status_name(ghc_status s);

/* ------------------------------------------------------------------ */
/* Context, memory, timing                                            */
/* ------------------------------------------------------------------ */
ghc_status ghc_device_count(int* n);
ghc_status ghc_ctx_create(int device, ghc_ctx** out);
void ghc_ctx_destroy(ghc_ctx* ctx);
ghc_status ghc_ctx_sync(ghc_ctx* ctx);
int ghc_ctx_num_sms(const ghc_ctx* ctx);
/* Kernel launches this context issued so far (evidence for the bench). */
uint64_t ghc_ctx_launch_count(const ghc_ctx* ctx);
ghc_status ghc_malloc(ghc_ctx* ctx, size_t bytes, void** d_ptr);
ghc_status ghc_free(ghc_ctx* ctx, void* d_ptr);
ghc_status ghc_host_alloc(size_t bytes, void** h_ptr); /* pinned */
ghc_status ghc_host_free(void* h_ptr);
ghc_status ghc_memcpy_h2d(ghc_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
ghc_status ghc_memcpy_d2h(ghc_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);
ghc_status ghc_memcpy_d2d(ghc_ctx* ctx, void* d_dst, const void* d_src, size_t bytes);
/* CUDA IPC of a ghc_malloc'd buffer (base pointer) for the async / EASGD
 * mailboxes across processes (transport.hpp:22-44 "nvlink" backend, P2P
 * copies): handle = GHC_IPC_HANDLE_BYTES bytes; ghc_memcpy_d2d moves data
 * into / out of a mapped peer buffer over NVLink. */
#define GHC_IPC_HANDLE_BYTES 64
ghc_status ghc_ipc_handle(ghc_ctx* ctx, void* d_base, uint8_t* out_handle);
ghc_status ghc_ipc_open(ghc_ctx* ctx, const uint8_t* handle, void** d_ptr);
ghc_status ghc_ipc_close(ghc_ctx* ctx, void* d_ptr);
ghc_status ghc_memset(ghc_ctx* ctx, void* d_dst, int value, size_t bytes);
/* Peer copy between GPUs of one process (cudaMemcpyPeerAsync: NVLink on a
 * B200 box) on ctx's stream — the payload hop of the in-process "nvlink"
 * Endpoint (adapter/gradhub_cuda.cpp; replaces transport.cpp:25-177's
 * mailbox copy). */
ghc_status ghc_memcpy_peer(ghc_ctx* ctx, void* d_dst, int32_t dst_device, const void* d_src,
                           int32_t src_device, size_t bytes);
/* WeightSet upload for the drop-in adapter: d_w32[i] = (float)d_w64[i] (the
 * f32 wire, proto.cpp) and *d_hash = order-independent 64-bit hash of every
 * (index, f64 bits) — the device-side stale-cache token that replaces
 * weights_checksum (nn.cpp:66-81) in forward/backward's guard (nn.cpp:
 * 116-119, 253-260).  d_w32 and d_hash are nullable. */
ghc_status ghc_weights_import_f64(ghc_ctx* ctx, float* d_w32, const double* d_w64, int64_t p,
                                  uint64_t* d_hash);
/* loss (nn.cpp:234-248): *h_sum = Σ_s −log d_probs[s][d_y[s]] (f64, fixed
 * order); GHC_ERR_SHAPE if a label is outside [0,K).  Synchronising. */
ghc_status ghc_nll_sum(ghc_ctx* ctx, const double* d_probs, const int32_t* d_y, int64_t n,
                       int32_t k, double* h_sum);
/* Device timing without host launch overhead (nvbench's blocking kernel):
 * ghc_stream_hold queues a 1-thread kernel that spins on a pinned flag, the
 * caller queues timer_start + the timed work, then ghc_stream_release lets
 * it all run back to back; ghc_timer_stop as usual.  The gate times out
 * after 5 s. */
ghc_status ghc_stream_hold(ghc_ctx* ctx);
ghc_status ghc_stream_release(ghc_ctx* ctx);
/* CUDA-event timer on the context stream: start, then stop returns ms. */
ghc_status ghc_timer_start(ghc_ctx* ctx);
ghc_status ghc_timer_stop(ghc_ctx* ctx, float* ms);

/* ------------------------------------------------------------------ */
/* Model: Architecture (arch.hpp:36-57) → kernel plan                 */
/* ------------------------------------------------------------------ */
/* Grammar of parse_architecture (arch.hpp:54-57, arch.cpp:173-214):
 * "lstm(D,H,T),dense(i,o,act)*,softmax(i,K)"; validated as arch.cpp:26-73. */
ghc_status ghc_plan_create(ghc_ctx* ctx, const char* arch_text, ghc_plan** out);
void ghc_plan_destroy(ghc_plan* plan);
int64_t ghc_plan_n_params(const ghc_plan* plan);   /* Architecture::n_params  arch.cpp:114 */
int64_t ghc_plan_input_width(const ghc_plan* plan); /* Architecture::input_width arch.cpp:75 */
int32_t ghc_plan_n_classes(const ghc_plan* plan);   /* Architecture::n_classes arch.cpp:83 */
/* Parameter tensors in weight-set order (arch.cpp:95-112). */
ghc_status ghc_plan_tensors(const ghc_plan* plan, int64_t* offset, int64_t* dim0,
                            int64_t* dim1, int cap, int* n_tensors);
/* Diagnostics: when d_probe != NULL every fused launch records %globaltimer
 * at 7 phase boundaries per round and CTA into d_probe[(round*ctas+cta)*16+i]
 * (+ 5 points inside warp 0's first sample at i = 8..12)
 * (weights loaded, samples done, partial stored, barrier 1, reduce, barrier
 * 2).  NULL disables (the default). */
ghc_status ghc_plan_set_probe(ghc_plan* plan, uint64_t* d_probe);
/* Diagnostics: ns per grid-wide barrier for implementation `impl`
 * (0 atomic counter, 1 gather/broadcast flags, 2 all-poll-all flags,
 * 3 hardware cluster barrier of 8 CTAs) over `ctas` co-resident CTAs. */
ghc_status ghc_diag_barrier_bench(ghc_ctx* ctx, int32_t impl, int32_t ctas, int32_t threads,
                                  int32_t iters, double* ns_per);
/* Synchronise the context's stream and report (then clear) the plan's
 * device error bit: GHC_ERR_SHAPE "loss: label out of range [0,K)" if any
 * launch of this plan since the last check met a label outside [0,K)
 * (nn.cpp:241-244); GHC_OK otherwise. */
ghc_status ghc_plan_check_error(ghc_plan* plan);
/* Diagnostics: device-side cost of launching an empty kernel with the round
 * kernel's launch configuration piece by piece (variant bit 0 cooperative,
 * bit 1 clusters of 4, bit 2 `smem` bytes of dynamic shared memory): one
 * gated launch (median) and per launch over 200 back to back, in µs. */
ghc_status ghc_diag_launch_bench(ghc_ctx* ctx, int32_t variant, int32_t ctas, int32_t threads,
                                 int32_t smem, double* us_single, double* us_b2b);
/* Name of the fused kernel the plan dispatches to (diagnostics). */
const char* ghc_plan_kernel_name(const ghc_plan* plan);
/* Cluster variant geometry: co-resident clusters and cluster size (0 = flat). */
int32_t ghc_plan_max_clusters(const ghc_plan* plan);
int32_t ghc_plan_cluster_size(const ghc_plan* plan);

/* Host-only architecture check (no device needed): parse + validate and
 * report the sizes; GHC_ERR_CONFIG with the reference's message on error. */
ghc_status ghc_arch_info(const char* arch_text, int64_t* n_params, int64_t* input_width,
                         int32_t* n_classes);
/* init_weights from the architecture text (host only). */
ghc_status ghc_init_weights_text(const char* arch_text, uint64_t seed, double* h_w);

/* init_weights (nn.cpp:83-98), host-side and bit-identical to the reference
 * (mt19937_64 + Glorot-uniform bounds).  h_w: n_params doubles. */
ghc_status ghc_init_weights(const ghc_plan* plan, uint64_t seed, double* h_w);

/* ------------------------------------------------------------------ */
/* Worker minibatch step: forward (nn.cpp:100-232) + loss (nn.cpp:     */
/* 234-248) + backward (nn.cpp:250-399) fused in one launch.          */
/* ------------------------------------------------------------------ */
/* d_grad[P] = grad_scale * Σ_s ∂ℓ_s/∂w   (grad_scale = 1/n reproduces the
 *                                        reference's batch mean, nn.cpp:283-297)
 * d_loss_sum[0] = Σ_s ℓ_s                 (loss() = d_loss_sum / n)
 * Samples: rows d_x[s] / d_y[s] for s < n when d_idx == NULL, otherwise the
 * rows d_idx[s] of a device-resident dataset (d_x, d_y).  A label outside
 * [0,K) (nn.cpp:241-244 throws ShapeError) sets the plan's device error bit
 * without a host round trip; the launch itself stays asynchronous and the
 * bit is reported as GHC_ERR_SHAPE by the next synchronising call on the
 * plan — ghc_plan_check_error, ghc_master_read, ghc_validate,
 * ghc_session_run — which also clears it.
 * Deterministic: fixed reduction order, bit-identical across repeats. */
ghc_status ghc_worker_grad(ghc_plan* plan, const float* d_w, const float* d_x,
                           const int32_t* d_y, const int32_t* d_idx, int64_t n,
                           float grad_scale, float* d_grad, float* d_loss_sum);

/* n_workers (≤ 8) independent worker gradients in ONE launch: worker k at
 * weights d_w + k·w_stride over rows h_idx[k][0 .. h_n[k]) (h_idx: host
 * array of device pointers; an entry may be NULL → rows 0 .. h_n[k]-1),
 * scaled by 1/h_n[k], into d_grad + k·g_stride; its loss sum into
 * d_loss[k] (nullable).  The grid is split into n_workers virtual ranks of
 * the fused round kernel with no cross-rank sum (the session's sync EASGD
 * round, whose workers' gradients are independent within a round); shapes
 * without that kernel variant fall back to n_workers ghc_worker_grad calls.
 * Same semantics as ghc_worker_grad per worker (nn.cpp:250-399); the
 * reduction order differs (fewer clusters per worker), deterministic. */
ghc_status ghc_worker_grads(ghc_plan* plan, int32_t n_workers, const float* d_w, int64_t w_stride,
                            const float* d_x, const int32_t* d_y, const int32_t* const* h_idx,
                            const int32_t* h_n, float* d_grad, int64_t g_stride, float* d_loss);

/* Forward only: class probabilities d_probs[n×K] (nullable) and loss sum. */
ghc_status ghc_forward(ghc_plan* plan, const float* d_w, const float* d_x,
                       const int32_t* d_y, const int32_t* d_idx, int64_t n,
                       float* d_probs, float* d_loss_sum);

/* The LSTM layer's LayerCache (nn.hpp:15-23) for a batch: gates [n×T×4H]
 * (i,f,g,o after the nonlinearity), cell c_t, tanh(c_t), hidden h_t
 * [n×T×H], each nullable.  Computed by the generic GEMM-based LSTM
 * (generic.cu: per-timestep tcgen05 GEMMs + cell kernels) — the fused round
 * kernels never materialise them.  The first layer must be an LSTM. */
ghc_status ghc_forward_cache(ghc_plan* plan, const float* d_w, const float* d_x, int64_t n,
                             float* d_gates, float* d_cell, float* d_tanh, float* d_hidden);

/* ------------------------------------------------------------------ */
/* Dense layers (nn.cpp:129-145, 312-334) on tcgen05 tensor cores       */
/* ------------------------------------------------------------------ */
enum { GHC_EPI_STORE = 0, GHC_EPI_BIAS_ACT = 1, GHC_EPI_DACT = 2 };
/* C[M×N] = A[M×K] · B[N×K]ᵀ (both K-major, row-major fp32 in HBM), 3×TF32
 * on tcgen05 with fp32 TMEM accumulation; fused epilogue:
 *   GHC_EPI_STORE    C = alpha·acc
 *   GHC_EPI_BIAS_ACT C = act(acc + bias[n])                 (act: 0 tanh, 1 relu, 2 identity)
 *   GHC_EPI_DACT     C = acc · act'(Y[m][n]) (act' from the activation output Y) */
ghc_status ghc_gemm_nt(ghc_ctx* ctx, const float* d_a, const float* d_b, float* d_c, int32_t m,
                       int32_t n, int32_t k, int32_t lda, int32_t ldb, int32_t ldc, int32_t epi,
                       int32_t act, const float* d_bias, const float* d_y, int32_t ldy,
                       float alpha);
/* out[c][r] = in[r][c]. */
ghc_status ghc_transpose(ghc_ctx* ctx, float* d_out, const float* d_in, int32_t rows,
                         int32_t cols, int32_t ldin, int32_t ldout);

/* ------------------------------------------------------------------ */
/* Algo (optim.cpp) on device buffers                                  */
/* ------------------------------------------------------------------ */
/* sgd_step (optim.cpp:39-65): v = mu*v - lr*g; w += v, in place.  If any
 * g is non-finite the WHOLE update is rejected (optim.cpp:49-51): w, v stay
 * untouched, *d_status = GHC_ERR_NONFINITE (else GHC_OK) and *d_version is
 * not incremented.  Hyper-parameters validated as optim.cpp:20-29.  One
 * launch, no host sync (the status lands in device memory). */
ghc_status ghc_sgd_apply(ghc_ctx* ctx, float* d_w, float* d_v, const float* d_g,
                         int64_t p, float lr, float mu, int32_t* d_status,
                         uint64_t* d_version);
/* sgd_step with the reference's value semantics (optim.cpp:39-65 returns a
 * new WeightSet / OptimState): reads w, v, g and writes the updated weights
 * and velocity to w_out, v_out in ONE pass (20 B/param; the in-place
 * ghc_sgd_apply must see all of g before its first write: two passes).
 * Non-finite g → *d_status = GHC_ERR_NONFINITE and w_out / v_out hold no
 * update (the caller keeps w, v — never written); else GHC_OK and
 * *d_version += 1.  Outputs must not overlap the inputs (GHC_ERR_CONFIG). */
ghc_status ghc_sgd_step_out(ghc_ctx* ctx, const float* d_w, const float* d_v, const float* d_g,
                            float* d_w_out, float* d_v_out, int64_t p, float lr, float mu,
                            int32_t* d_status, uint64_t* d_version);
/* easgd_worker_step (optim.cpp:82-105) with value semantics, one pass:
 * w_out = w - lr*g, pulled toward c when batch_index % tau == 0.
 * Non-finite g → *d_status = GHC_ERR_NONFINITE (w untouched, w_out no update). */
ghc_status ghc_easgd_worker_step_out(ghc_ctx* ctx, const float* d_w, const float* d_c,
                                     const float* d_g, float* d_w_out, int64_t p, float lr,
                                     float alpha, uint64_t tau, uint64_t batch_index,
                                     int32_t* d_status);
/* elastic_pull (optim.cpp:67-80): w -= alpha*(w - c). */
ghc_status ghc_elastic_pull(ghc_ctx* ctx, float* d_w, const float* d_c, int64_t p,
                            float alpha);
/* easgd_worker_step (optim.cpp:82-105): w -= lr*g; pull toward c when
 * batch_index % tau == 0.  Non-finite g → *d_status = GHC_ERR_NONFINITE and
 * w untouched. */
ghc_status ghc_easgd_worker_step(ghc_ctx* ctx, float* d_w, const float* d_c,
                                 const float* d_g, int64_t p, float lr, float alpha,
                                 uint64_t tau, uint64_t batch_index, int32_t* d_status);
/* easgd_center_step (optim.cpp:107-123): c += alpha*(w - c); version += 1.
 * alpha validated in (0,1) (optim.cpp:31-37). */
ghc_status ghc_easgd_center_step(ghc_ctx* ctx, float* d_c, const float* d_w, int64_t p,
                                 float alpha, uint64_t* d_version);
/* Sync-round combine: out = Σ_i c_i * slot_i / Σ_i c_i in
 * slot (rank) order; slots are contiguous [W][P]. */
ghc_status ghc_weighted_mean(ghc_ctx* ctx, float* d_out, const float* d_slots,
                             const double* h_counts, int32_t n_slots, int64_t p);

/* ------------------------------------------------------------------ */
/* Master: device-resident Downpour master state + fused sync rounds   */
/* ------------------------------------------------------------------ */
/* Holds w and v double-buffered in HBM, the version counter and the
 * commit/reject flag; the update of round r is committed on device only if
 * its combined gradient is finite, with no host sync. */
ghc_status ghc_master_create(ghc_plan* plan, const double* h_w0, float lr, float mu,
                             ghc_master** out);
void ghc_master_destroy(ghc_master* m);
/* Current weights / velocity (device pointers valid until the next round). */
ghc_status ghc_master_weights(ghc_master* m, float** d_w, float** d_v);
ghc_status ghc_master_read(ghc_master* m, float* h_w, float* h_v, uint64_t* version,
                           uint64_t* rejected);
/* n_rounds synchronous Downpour rounds of ONE worker colocated with the
 * master (1 master + 1 worker per GPU) in ONE persistent
 * launch: per round gather the batch d_idx[r*stride ..] from the resident
 * dataset (d_idx == NULL: round r uses rows r*stride .. r*stride+n-1),
 * forward+loss+backward, deterministic cross-CTA gradient reduce, finite
 * check, sgd_step, commit.  d_counts[r] = samples in round r (nullable → n
 * each).  d_loss_out[r] = loss sum of round r (nullable).
 * d_x, d_y and d_loss_out only need to be device-ACCESSIBLE: pinned host
 * memory (ghc_host_alloc) streams the batches straight from the host — each
 * CTA prefetches its next-round rows over PCIe during the current round and
 * the round's loss is stored to host memory (zero-copy end-to-end path). */
ghc_status ghc_master_sync_rounds(ghc_master* m, const float* d_x, const int32_t* d_y,
                                  const int32_t* d_idx, int64_t stride,
                                  const int32_t* d_counts, int64_t n, int32_t n_rounds,
                                  float* d_loss_out);
/* Apply a combined gradient produced elsewhere (NCCL reduce, virtual workers):
 * d_g[P] is the already-combined gradient.  sgd_step (optim.cpp:39-65) in one
 * stream-ordered pass from the current w/v buffer into the other; the device
 * flips the current buffer and bumps the version, or — any non-finite g —
 * leaves it untouched and counts a rejection (optim.cpp:49-51; read back with
 * ghc_master_read).  No host synchronisation. */
ghc_status ghc_master_apply(ghc_master* m, const float* d_g);

/* Packed dataset rows for the fused sync rounds: row r = x[r][0..width) |
 * label r (int32 bits) | zero pad, stride ghc_packed_row_floats(width) =
 * the next multiple of 32 floats (128 B: the DRAM fetch granularity the
 * random gather sees, measured — 224-B rows still cost 311 B per sample).
 * A gathered sample is then whole 128-B lines with its label inside.  Pass the packed array
 * as d_x with d_y == NULL to ghc_master_sync_rounds / ghc_p2p_sync_rounds /
 * the resident service (SIMT cluster round kernel). */
int32_t ghc_packed_row_floats(int32_t width);
ghc_status ghc_dataset_pack(ghc_ctx* ctx, const float* d_x, const int32_t* d_y, int64_t rows,
                            int32_t width, float* d_out);
/* Resident round service: the persistent sync-round kernel launched ONCE
 * for master m (fused SIMT cluster kernel, n samples per round, n within one
 * sample per warp slot) and fed commands — a segment of `rounds` sync rounds
 * on batches x/y (idx/stride as ghc_master_sync_rounds), losses to loss_out
 * — through doorbells instead of a cooperative cluster launch per call
 * (≈ 13 µs of device-side launch + prologue + teardown, measured).
 *   ghc_resident_submit        host path: pinned ring + doorbell (returns seq);
 *   ghc_resident_wait          spins on the pinned completion word;
 *   ghc_resident_submit_stream stream path: a submit + a wait kernel on ctx's
 *                              stream (CUDA events around them time the rounds);
 *   ghc_resident_check         reads the service's error flags (synchronising);
 *   ghc_resident_stop          STOP, kernel exit, master state published; frees r.
 * With no command for idle_seconds (default 2) the kernel stops itself and
 * later calls report GHC_ERR_CUDA.  The master must not be used by other
 * calls while the service runs.  One submission path at a time. */
typedef struct ghc_resident ghc_resident;
ghc_status ghc_resident_start(ghc_master* m, int64_t n, double idle_seconds, ghc_resident** out);
ghc_status ghc_resident_submit(ghc_resident* r, const float* x, const int32_t* y, const int32_t* idx,
                               int64_t stride, int32_t rounds, float* loss_out, uint64_t* seq);
ghc_status ghc_resident_wait(ghc_resident* r, uint64_t seq);
ghc_status ghc_resident_submit_stream(ghc_resident* r, ghc_ctx* ctx, const float* x, const int32_t* y,
                                      const int32_t* idx, int64_t stride, int32_t rounds, float* loss_out,
                                      uint64_t* seq);
ghc_status ghc_resident_check(ghc_resident* r);
/* A C++ caller's per-batch loop (benchmark of the per-call API without an
 * interpreter): batch k at x + k·x_batch_stride (y likewise, NULL = packed
 * rows), one round per ghc_resident_submit, up to `depth` batches in
 * flight (1 = submit + wait per batch); *us_per_call = host wall time per
 * call. */
ghc_status ghc_resident_bench_calls(ghc_resident* r, const float* x, int64_t x_batch_stride,
                                    const int32_t* y, int64_t y_batch_stride, int32_t n_calls,
                                    int32_t depth, float* loss_out, double* us_per_call);
/* Diagnostics (%globaltimer ns), t[133]: [0..4] the last stream-submitted
 * command: submit, first / last CTA past the doorbell, completion published,
 * wait kernel saw it; then per command seq % 64: (last CTA past the
 * doorbell, completion published).  Synchronising. */
ghc_status ghc_resident_times(ghc_resident* r, uint64_t* t);
ghc_status ghc_resident_stop(ghc_resident* r);


/* ------------------------------------------------------------------ */
/* Exchange across GPUs (one process per GPU) over NCCL / NVLink 5:     */
/* replaces Endpoint send/recv (transport.hpp:22-44) + establish()      */
/* (transport.cpp:533-586, new backend "nvlink").                       */
/* ------------------------------------------------------------------ */
typedef struct ghc_comm ghc_comm;
#define GHC_UNIQUE_ID_BYTES 128
enum { GHC_EXCHANGE_REDUCE_BCAST = 0, GHC_EXCHANGE_ALLREDUCE = 1 };

/* Rank 0 creates the id; the caller moves the bytes to every rank. */
ghc_status ghc_comm_unique_id(uint8_t* out_id);
ghc_status ghc_comm_init(ghc_ctx* ctx, const uint8_t* id, int32_t rank, int32_t nranks,
                         ghc_comm** out);
/* Topology::hierarchical groups (transport.cpp:520-531): ranks with equal
 * color form a sub-communicator ordered by key; *out = NULL for color < 0. */
ghc_status ghc_comm_split(ghc_comm* parent, int32_t color, int32_t key, ghc_comm** out);
void ghc_comm_destroy(ghc_comm* comm);
int32_t ghc_comm_rank(const ghc_comm* comm);
int32_t ghc_comm_size(const ghc_comm* comm);
ghc_status ghc_comm_reduce_sum(ghc_comm* comm, const float* d_send, float* d_recv, int64_t count,
                               int32_t root);
ghc_status ghc_comm_broadcast(ghc_comm* comm, float* d_buf, int64_t count, int32_t root);
ghc_status ghc_comm_allreduce_sum(ghc_comm* comm, const float* d_send, float* d_recv,
                                  int64_t count);

/* Synchronous Downpour rounds across the communicator:
 * rank k is worker k and gathers its batch d_idx[r*stride ..] from its
 * resident shard; h_counts[r*nranks + k] is worker k's sample count in round
 * r (0 once it has sent DONE; known on every rank from the deterministic
 * data layer).  exchange = REDUCE_BCAST: gradients reduced to the master on
 * rank 0, sgd_step there, weights broadcast (the reference protocol);
 * ALLREDUCE: every rank holds a bit-identical master replica.  The master
 * object on every rank must be created from the same initial weights. */
ghc_status ghc_dist_sync_rounds(ghc_master* m, ghc_comm* comm, int32_t exchange,
                                const float* d_x, const int32_t* d_y, const int32_t* d_idx,
                                int64_t stride, const int32_t* h_counts, int32_t n_rounds,
                                float* d_loss_out);

/* ------------------------------------------------------------------ */
/* Fused NVLink exchange (replaces, for the sync round, Endpoint         */
/* GRADIENT/WEIGHTS send/recv transport.hpp:22-44 + the master loop      */
/* SPEC.md:340-366, and the NCCL reduce/broadcast of ghc_dist_*): the    */
/* persistent round kernel of every rank pushes its rank-local gradient  */
/* sub-slices into every rank's receive buffer over peer memory, counts  */
/* arrivals per column, sums the ranks in rank order and applies         */
/* sgd_step — each rank holds a bit-identical master replica.            */
/* ------------------------------------------------------------------ */
typedef struct ghc_p2p ghc_p2p;
/* Rank `rank` of an nranks (2..8) exchange over plan's fused kernel (the
 * same architecture, GPU model and batch size on every rank). */
ghc_status ghc_p2p_create(ghc_plan* plan, int32_t rank, int32_t nranks, ghc_p2p** out);
/* All nranks ranks as virtual ranks sharing ONE grid on this GPU (same
 * kernel code, peer pointers into one allocation): single-GPU testing. */
ghc_status ghc_p2p_create_virtual(ghc_plan* plan, int32_t nranks, ghc_p2p** out);
/* This rank's cudaIpc handle (GHC_IPC_HANDLE_BYTES) for the bootstrap. */
ghc_status ghc_p2p_export(ghc_p2p* p, uint8_t* out_handle);
/* Map every other rank's buffers: handles = nranks handles in rank order. */
ghc_status ghc_p2p_import(ghc_p2p* p, const uint8_t* handles);
void ghc_p2p_destroy(ghc_p2p* p);
/* n_rounds sync Downpour rounds in ONE persistent launch per rank.  Rank k
 * (virtual rank k) trains in round r on rows d_idx[k*idx_vstride + r*stride
 * + s] (rows r*stride + s with d_idx == NULL) for s < d_counts[r*nranks + k]
 * (d_counts nullable → n_max each); the gradient is the sample-weighted mean
 * over all ranks.  d_loss_out[r] = loss sum over ranks. */
ghc_status ghc_p2p_sync_rounds(ghc_master* m, ghc_p2p* p, const float* d_x, const int32_t* d_y,
                               const int32_t* d_idx, int64_t stride, int64_t idx_vstride,
                               const int32_t* d_counts, int64_t n_max, int32_t n_rounds,
                               float* d_loss_out);
/* Diagnostics of the cross-process hop (no co-resident round kernels): push
 * n tagged elements into row `rank` of rank `dst`'s receive rows (system-
 * scope stores through the IPC mapping, then a stream sync), and check on the
 * owner that row `src` holds them with tag `tag` (*h_bad = mismatches). */
ghc_status ghc_p2p_diag_push(ghc_p2p* p, int32_t dst, uint32_t tag, int32_t n);
ghc_status ghc_p2p_diag_check(ghc_p2p* p, int32_t src, uint32_t tag, int32_t n, int32_t* h_bad);
/* Elements per receive row (the fused kernel's padded gradient row, EP). */
int32_t ghc_p2p_row_elems(const ghc_p2p* p);
/* Device-side barrier of the nranks ranks, queued on the context stream
 * (system-scope flag stores into every peer's mapped line, then a poll of
 * this rank's line): work queued after it starts on all ranks within about
 * one NVLink round trip.  Every rank must call it equally often.  Virtual
 * exchanges: no-op.  (No reference counterpart: measurement plumbing for
 * timing the fused exchange across processes without host skew.) */
ghc_status ghc_p2p_barrier(ghc_p2p* p);

/* ------------------------------------------------------------------ */
/* Data layer, host side, bit-identical to the oracle */
/* ------------------------------------------------------------------ */
typedef struct ghc_data_spec {
  int32_t n_files;
  int32_t samples_per_file;
  int32_t seq_len;
  int32_t input_dim;
  int32_t n_classes;
  int32_t pad_;
  double delta;
  uint64_t seed;
} ghc_data_spec;

/* generate_synthetic for files [f0, f0+nf): rows of seq_len*input_dim f32
 * (the on-disk/wire precision) + labels. */
ghc_status ghc_data_generate(const ghc_data_spec* spec, int32_t f0, int32_t nf,
                             float* h_x, int32_t* h_y);
/* shard_files. */
ghc_status ghc_data_shard(int32_t n_files, int32_t n_workers, int32_t worker,
                          int32_t* first_file, int32_t* n_files_out);
/* batches: the epoch permutation of worker's shard as
 * GLOBAL sample indices; returns the count in *count. */
ghc_status ghc_data_epoch_indices(const ghc_data_spec* spec, int32_t n_workers,
                                  int32_t worker, int32_t epoch, uint64_t shuffle_seed,
                                  int32_t shuffle, int64_t* h_out, int64_t* count);

/* Wire frames on the device (proto.cpp:214-386): the
 * reference's GHUB frame of a WEIGHTS (kind 1, version) / GRADIENT (kind 2,
 * basis_version, sample_count ≥ 1) message over the arch's tensors, f32
 * (wire_f64 = 0) or f64 values; kind 0 = SHUTDOWN.  Byte-identical to the
 * reference encoder.  d_out must be 16-byte aligned (cudaMalloc is). */
ghc_status ghc_frame_size(const ghc_plan* plan, int32_t kind, int32_t wire_f64, int64_t* bytes);
ghc_status ghc_encode_frame(ghc_plan* plan, int32_t kind, int32_t wire_f64, const float* d_w,
                            uint64_t version, uint64_t sample_count, uint8_t* d_out, int64_t cap,
                            int64_t* len);
/* Validates the frame (bad magic / unsupported version / truncated / length
 * overflow / unknown type / malformed payload → GHC_ERR_PROTOCOL with
 * *decode_status = the reference's DecodeStatus 1..6; tensors not matching
 * the arch → GHC_ERR_SHAPE) and unpacks the values into d_w[P] (f64 frames
 * rounded to f32).  *kind: 1 WEIGHTS, 2 GRADIENT, 0 SHUTDOWN, -type for the
 * other message types.  d_frame must be 4-byte aligned (16-byte aligned
 * frames take the vector path). */
ghc_status ghc_decode_frame(ghc_plan* plan, const uint8_t* d_frame, int64_t len, int32_t* kind,
                            float* d_w, uint64_t* version, uint64_t* sample_count,
                            int32_t* wire_f64, int32_t* decode_status);

/* validate: the master's serial held-out evaluation —
 * one fused forward over the n held-out samples, then *h_correct = samples
 * whose argmax_k p_k (lowest k on ties) equals the label and *h_loss_mean =
 * mean -ln p_y.  Synchronous.  n < 1 → GHC_ERR_CONFIG. */
ghc_status ghc_validate(ghc_plan* plan, const float* d_w, const float* d_x, const int32_t* d_y,
                        int64_t n, int64_t* h_correct, double* h_loss_mean);

/* ------------------------------------------------------------------ */
/* Roles: a training session of W workers on this     */
/* device ("virtual workers"), the C++ master/worker loops over the     */
/* kernels above.  Dataset generated by the data layer and resident.    */
/* ------------------------------------------------------------------ */
typedef struct ghc_session ghc_session;
enum { GHC_ALGO_DOWNPOUR = 0, GHC_ALGO_EASGD = 1 };
enum { GHC_MODE_SYNC = 0, GHC_MODE_REPLAY = 1 };

/* TrainConfig. */
typedef struct ghc_train_config {
  int32_t algo;         /* GHC_ALGO_*                                        */
  int32_t mode;         /* GHC_MODE_SYNC | GHC_MODE_REPLAY (async, replayed)  */
  int32_t n_workers;
  int32_t batch_size;
  int32_t epochs;
  int32_t tau;          /* EASGD exchange period                             */
  float lr;
  float mu;
  float alpha;          /* EASGD elastic force                               */
  int32_t shuffle;
  uint64_t weight_seed;
  uint64_t shuffle_seed;
  int32_t groups;       /* hierarchical sub-masters (0 = flat)               */
  int32_t flush_k;      /* hierarchical flush period K                       */
  float parent_lr;      /* top master (pass-through: 1, 0)                   */
  float parent_mu;
  int32_t max_updates;  /* sync / hierarchical rounds cap (0 = all epochs)   */
  int32_t pad_;
} ghc_train_config;

ghc_status ghc_session_create(ghc_plan* plan, const ghc_train_config* cfg,
                              const ghc_data_spec* spec, ghc_session** out);
void ghc_session_destroy(ghc_session* s);
/* Runs the session.  REPLAY (async Downpour / EASGD): h_order[k] = worker
 * whose next batch the master processes at step k (EASGD: whose next local
 * batch runs; it exchanges when its batch_index % tau == 0).  SYNC EASGD
 * without an order = round-robin.  h_loss (nullable): per-round / per-step
 * mean loss; h_staleness (nullable): per-step version - basis_version;
 * at most trace_cap entries of each are written. */
ghc_status ghc_session_run(ghc_session* s, const int32_t* h_order, int64_t n_order,
                           float* h_loss, int64_t* h_staleness, int64_t trace_cap);
/* Final master weights (Downpour / top master) or EASGD center, velocity,
 * every worker's local weights [W][P], sub-master weights [G][P];
 * stats = {version, rejected, samples absorbed, rounds/steps}. */
ghc_status ghc_session_read(ghc_session* s, float* h_w, float* h_v, float* h_worker_w,
                            float* h_group_w, uint64_t* stats);
/* Replace the session's dataset rows (generated from the spec at create)
 * with caller data of the same shape: h_x[rows][seq_len*input_dim],
 * h_y[rows], rows = n_files*samples_per_file (SPEC.md:421-448 files hold
 * f32).  Shards, index streams and batches are unchanged.  Used to feed the
 * reference's own data (or a poisoned row: non-finite parity tests). */
ghc_status ghc_session_load_data(ghc_session* s, const float* h_x, const int32_t* h_y,
                                 int64_t rows);
/* Held-out set of the master's serial validation:
 * validate every `every` master updates (0 = only at the end) and once at
 * the end of every ghc_session_run (no duplicate if the cadence already
 * validated that version).  Hierarchical sessions validate at the end. */
ghc_status ghc_session_set_validation(ghc_session* s, const float* h_x, const int32_t* h_y,
                                      int64_t n, int32_t every);
/* VALIDATE_RESULT records so far: *count = total; the first min(cap, total)
 * are written (version, accuracy = correct / n, mean loss). */
ghc_status ghc_session_validations(ghc_session* s, int64_t cap, uint64_t* versions,
                                   double* accuracy, double* loss, int64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* GHC_H */
