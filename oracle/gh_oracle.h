/*
 * gh_oracle.h — CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * Plain-C, double-precision restatement of the reference (arXiv 1712.05878
 * `gradhub`, /root/reference/proj) for the Downpour/EASGD hot path, plus the
 * SPEC-only roles/data layers the reference describes but does not ship.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the CPU baseline.
 * The product (paper_1712_05878_b200, libghc.so) never links or calls it.
 *
 * Every function cites the reference file:line (or SPEC.md line) it restates.
 */
#ifndef GH_ORACLE_H
#define GH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the exception taxonomy of errors.hpp:10-45. */
enum {
  GHO_OK = 0,
  GHO_SHAPE = 1,          /* ShapeError              errors.hpp:10-14 */
  GHO_NONFINITE = 2,      /* NonFiniteGradientError  errors.hpp:16-21 */
  GHO_CACHE_MISMATCH = 3, /* CacheMismatchError      errors.hpp:23-27 */
  GHO_CONFIG = 4,         /* ConfigError             errors.hpp:29-32 */
  GHO_TRANSPORT = 5,      /* TransportError          errors.hpp:34-38 */
  GHO_PROTOCOL = 6        /* ProtocolError           errors.hpp:40-45 */
};

/* Layer kinds (arch.hpp:12-33). */
enum { GHO_DENSE = 0, GHO_LSTM = 1, GHO_SOFTMAX = 2 };
/* Activations (arch.hpp:10). */
enum { GHO_TANH = 0, GHO_RELU = 1, GHO_IDENTITY = 2 };

#define GHO_MAX_LAYERS 16

typedef struct {
  int32_t n_layers;
  int32_t kind[GHO_MAX_LAYERS];
  /* dense: (in, out, act); lstm: (D, H, T); softmax: (in, K, unused) */
  int32_t a[GHO_MAX_LAYERS];
  int32_t b[GHO_MAX_LAYERS];
  int32_t c[GHO_MAX_LAYERS];
} gho_arch;

/* ---- rng.hpp:13-74 -------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int32_t mti;
  int32_t has_spare;
  double spare;
} gho_rng;

void gho_rng_seed(gho_rng* r, uint64_t seed);
uint64_t gho_rng_u64(gho_rng* r);
double gho_rng_uniform01(gho_rng* r);
double gho_rng_uniform(gho_rng* r, double lo, double hi);
double gho_rng_normal(gho_rng* r);
uint64_t gho_rng_below(gho_rng* r, uint64_t n);
void gho_rng_shuffle_i64(gho_rng* r, int64_t* v, int64_t n);
uint64_t gho_mix_seed(uint64_t a, uint64_t b);

/* ---- arch.cpp ------------------------------------------------------- */
int gho_arch_parse(const char* text, gho_arch* out);
int gho_arch_validate(const gho_arch* a);
int64_t gho_arch_n_params(const gho_arch* a);
int64_t gho_arch_input_width(const gho_arch* a);
int32_t gho_arch_n_classes(const gho_arch* a);
/* Parameter tensor table in weight-set order (arch.cpp:95-112).
 * Returns the tensor count; fills offsets/sizes/dim0/dim1 (dim1=0 for 1-D). */
int gho_arch_tensors(const gho_arch* a, int64_t* offset, int64_t* size,
                     int64_t* dim0, int64_t* dim1, int cap);

/* ---- nn.cpp --------------------------------------------------------- */
void gho_init_weights(const gho_arch* a, uint64_t seed, double* w);
/* forward (nn.cpp:100-232) + loss (nn.cpp:234-248) + backward (nn.cpp:250-399).
 * grad may be NULL (forward+loss only); probs may be NULL. */
int gho_forward_backward(const gho_arch* a, const double* w, const double* x,
                         const int32_t* y, int64_t n, double* grad,
                         double* probs, double* loss_out);
/* validate (SPEC-only): forward over a held-out set;
 * *correct = samples whose argmax_k p_k (lowest k on ties, the
 * std::max_element convention) equals the label, *loss_mean = mean -ln p_y.
 * n < 1 → GHO_CONFIG ("empty held-out set → configuration error"). */
int gho_validate(const gho_arch* a, const double* w, const double* x, const int32_t* y,
                 int64_t n, int64_t* correct, double* loss_mean);
/* finite_diff_gradient (nn.cpp:407-426). */
int gho_finite_diff(const gho_arch* a, const double* w, const double* x,
                    const int32_t* y, int64_t n, double eps, double* grad);
/* weights_checksum (nn.cpp:66-81). */
uint64_t gho_weights_checksum(const gho_arch* a, const double* w);

/* ---- optim.cpp ------------------------------------------------------ */
int gho_sgd_step(double* w, double* v, const double* g, int64_t p, double lr,
                 double mu);
void gho_elastic_pull(double* w, const double* center, int64_t p, double alpha);
int gho_easgd_worker_step(double* w, const double* center, const double* g,
                          int64_t p, double lr, double alpha, uint64_t tau,
                          uint64_t batch_index);
int gho_easgd_center_step(double* c, const double* worker, int64_t p,
                          double alpha);

/* ---- proto.cpp wire rounding (proto.cpp:79,125) ---------------------- */
void gho_wire_round(double* dst, const double* src, int64_t p, int wire_f64);
/* ---- proto.cpp frames (restated) -------------------------------------- */
/* kind: 0 SHUTDOWN, 1 WEIGHTS {version}, 2 GRADIENT {basis_version,
 * sample_count}; tensors = the arch's parameter tensors in weight-set order
 * (arch.cpp:95-112), values f32 (wire_f64 = 0) or f64 (type | 0x40).
 * Layout (proto.cpp:214-272): "GHUB" | u16 version 1 | u8 type | u64 payload
 * length | payload; tensor block = u32 count, per tensor u8 rank, u32 dims,
 * values; all little-endian. */
int64_t gho_frame_size(const gho_arch* a, int kind, int wire_f64);
int gho_encode_frame(const gho_arch* a, int kind, const double* w, uint64_t version,
                     uint64_t sample_count, int wire_f64, uint8_t* out, int64_t cap,
                     int64_t* len);
/* decode (proto.cpp:288-386) + the arch check the roles do when they build a
 * WeightSet: *status = DecodeStatus (0 ok, 1 bad_magic, 2 unsupported_version,
 * 3 truncated, 4 length_overflow, 5 unknown_type, 6 malformed_payload);
 * returns GHO_PROTOCOL on a decode failure, GHO_SHAPE when the tensors do not
 * match the arch; w receives the values widened to f64. */
int gho_decode_frame(const gho_arch* a, const uint8_t* in, int64_t len, int* kind, double* w,
                     uint64_t* version, uint64_t* sample_count, int* wire_f64, int* status);

/* ---- data (decisions in DESIGN.md "Data layer") ---- */
typedef struct {
  int32_t n_files;
  int32_t samples_per_file;
  int32_t seq_len;
  int32_t input_dim;
  int32_t n_classes;
  int32_t pad_;
  double delta;
  uint64_t seed;
} gho_data_spec;

/* x: n_files*samples_per_file rows of seq_len*input_dim (f32-representable
 * doubles, the on-disk wire precision); y: labels. */
void gho_generate(const gho_data_spec* s, double* x, int32_t* y);
/* Only the rows of files [f0, f0+nf) (same values as gho_generate). */
void gho_generate_files(const gho_data_spec* s, int32_t f0, int32_t nf,
                        double* x, int32_t* y);
int gho_shard_files(int32_t n_files, int32_t n_workers, int32_t worker,
                    int32_t* first_file, int32_t* n_files_out);
/* Global sample indices of `worker`'s shard for `epoch`, shuffled when
 * `shuffle` != 0. Returns the count. */
int64_t gho_epoch_indices(const gho_data_spec* s, int32_t n_workers,
                          int32_t worker, int32_t epoch, uint64_t shuffle_seed,
                          int32_t shuffle, int64_t* out);

/* ---- roles ---------------------------------------- */
enum { GHO_DOWNPOUR = 0, GHO_EASGD = 1 };

typedef struct {
  int32_t algo;
  int32_t n_workers;
  int32_t batch_size;
  int32_t epochs;
  double lr;
  double mu;
  double alpha;
  int32_t tau;
  int32_t shuffle;
  uint64_t weight_seed;
  uint64_t shuffle_seed;
  int32_t wire_f64;
  int32_t max_updates; /* master updates (sync rounds / async steps); 0 = all */
  int32_t groups;      /* hierarchical: number of sub-masters (0 = flat) */
  int32_t flush_k;     /* hierarchical: flush period K */
  double parent_lr;
  double parent_mu;
} gho_train_cfg;

typedef struct {
  int64_t updates;       /* accepted master updates */
  int64_t rejected;      /* non-finite updates rejected */
  int64_t samples;       /* Σ sample_count over accepted gradients */
  uint64_t version;      /* final master version */
} gho_run_stats;

/* Synchronous Downpour: rank-ordered sample-weighted mean.
 * x,y: the FULL dataset (gho_generate). w_out/v_out: final master state.
 * loss_trace (nullable, max_updates entries): sample-weighted batch loss. */
int gho_run_sync(const gho_arch* a, const gho_data_spec* s, const double* x,
                 const int32_t* y, const gho_train_cfg* cfg, double* w_out,
                 double* v_out, double* loss_trace, gho_run_stats* st);

/* Replayed order (SPEC.md:349-357 async Downpour; SPEC.md:149-166,343 EASGD).
 * order[k] = worker index whose next batch is processed at step k.
 * Downpour: each step is one GRADIENT → sgd_step → reply to that worker.
 * EASGD:    each step is one local worker batch; on batch_index % tau == 0
 *           the worker exchanges with the center (updated-center ordering).
 * staleness (nullable, n_order): Downpour staleness per step.
 * worker_w (nullable, n_workers*P): final local weights of every worker. */
int gho_run_replay(const gho_arch* a, const gho_data_spec* s, const double* x,
                   const int32_t* y, const gho_train_cfg* cfg,
                   const int32_t* order, int64_t n_order, double* w_out,
                   double* v_out, double* worker_w, int64_t* staleness,
                   double* loss_trace, gho_run_stats* st);

/* Hierarchical masters: `groups` sub-masters, each a sync
 * Downpour master over n_workers/groups workers; every flush_k accepted group
 * updates each sub-master uplinks (snapshot - current) with the absorbed
 * sample count; the top master combines the groups synchronously (sample
 * weighted, group order) and applies sgd_step(parent_lr, parent_mu). */
int gho_run_hier(const gho_arch* a, const gho_data_spec* s, const double* x,
                 const int32_t* y, const gho_train_cfg* cfg, double* w_out,
                 double* group_w_out, double* loss_trace, gho_run_stats* st);

#ifdef __cplusplus
}
#endif

#endif /* GH_ORACLE_H */
