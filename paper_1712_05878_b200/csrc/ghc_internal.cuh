// ghc_internal.cuh — definitions shared by the libghc translation units
// (ghc.cu: model/algo/master; dist.cu: NCCL exchange).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ghc.h"
#include "host_model.hpp"
#include "lstm_round.cuh"
#include "lstm_step.cuh"
#include "lstm_tc.cuh"
#include "update_kernels.cuh"

using namespace ghc;

ghc_status ghc_fail(ghc_status s, const std::string& msg);
#define fail ghc_fail

#define CU(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(GHC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
  } while (0)

// ---- fused LSTM→softmax kernel table (one instantiation per shape) ----
struct LstmEntry {
  int D, H, T, K;
  void (*fn)(StepArgs);        // flat variant (grid barriers)      lstm_step.cuh
  // cluster variants, index ci → clusters of kClusterSizes[ci] = 4 / 8 / 2
  void (*fn_round[3])(StepArgs);   // SIMT round kernel (lstm_round.cuh)
  void (*fn_res[3])(StepArgs);     // its resident-service variant (null for trunks)
  void (*fn_tc[3])(StepArgs);      // tensor-core cluster variant (lstm_tc.cuh); null: n/a
  void (*fn_multi[3])(StepArgs);   // per-worker gradients in one launch (MULTI; null: n/a)
  int P, ppad, ep[3];
  size_t (*smem)(int);
  size_t (*smem_round[3])(int);
  size_t (*smem_tc[3])(int);
  const char* name;
};

constexpr int kClusterSizes[3] = {4, 8, 2};

// The instantiated fused-kernel shapes (defined in ghc.cu only).
const std::vector<LstmEntry>& lstm_table();
// LSTM trunk shapes for layered archs (K unused; defined in ghc.cu).
const std::vector<LstmEntry>& trunk_table();

struct ghc_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::atomic<uint64_t> launches{0};
  float* splitk_ws = nullptr;  // split-K GEMM partials (dense.cu), grown on demand
  size_t splitk_bytes = 0;
  MasterDev* scratch_ms = nullptr;  // barrier state of the context-level cooperative kernels
  unsigned char* hdr_scratch = nullptr;  // decode: gathered frame-header bytes (codec.cu), kHdrScratch
  int* gate_h = nullptr;            // ghc_stream_hold: pinned flag (host view)
  int* gate_d = nullptr;            //                  (device view)
};

struct LayeredWorkspace;
struct GenericLstmWorkspace;

namespace ghc {
// ghc_gemm_nt with an optional transposed copy of C (CT[n][m], stride ldct)
// written by the GEMM epilogue (dense.cu).
ghc_status gemm_nt_ct(ghc_ctx* c, const float* d_a, const float* d_b, float* d_c, int32_t M,
                      int32_t N, int32_t K, int32_t lda, int32_t ldb, int32_t ldc, int32_t epi,
                      int32_t act, const float* d_bias, const float* d_y, int32_t ldy, float alpha,
                      float* d_ct, int32_t ldct);
// C[M×N] = A·Bᵀ with K split over ≈ one wave (ordered partials; long-K
// weight gradients of the generic LSTM path, dense.cu).
ghc_status gemm_nt_splitk(ghc_ctx* c, const float* d_a, const float* d_b, float* d_c, int32_t M,
                          int32_t N, int32_t K, int32_t lda, int32_t ldb, int32_t ldc);
}  // namespace ghc

struct ghc_plan {
  ghc_ctx* ctx = nullptr;
  bool layered = false;                 // dense layers: layered.cu path
  const LstmEntry* trunk = nullptr;     // LSTM trunk kernel of a layered arch
  LayeredWorkspace* ws = nullptr;
  bool generic_lstm = false;            // LSTM layer outside the kernel tables: generic.cu
  GenericLstmWorkspace* gws = nullptr;
  int max_warps = 8;      // warps/CTA that fit the fused kernel's smem
  unsigned long long* probe = nullptr;  // phase-timing probe (diagnostics)
  unsigned* bar = nullptr;  // flag barrier: (2 + max_ctas) 128-B lines
  int max_clusters = 0;      // co-resident clusters of the chosen cluster size
  int cluster_size = 8;      // 4 or 8 (chosen at plan creation from occupancy)
  int cs_index = 1;          // 0: clusters of 4, 1: clusters of 8
  int round_warps = 8;       // warps/CTA that fit the cluster variant's smem
  bool use_cluster = true;   // GHC_STEP=flat selects the flat variant
  bool use_tc = false;       // cluster variant runs lstm_round_tc_kernel (8 samples/CTA pass)
  Model model;
  const LstmEntry* lstm = nullptr;
  int max_ctas = 0;       // co-resident CTAs of the fused kernel
  float* part = nullptr;  // [max_ctas][ppad]
  unsigned long long* tpart = nullptr;  // tagged rows of the single-GPU exchange
  unsigned long long* tw = nullptr;
  MasterDev* ms = nullptr;  // scratch barrier state for grad/fwd launches
  int* err = nullptr;
  std::string kname;
};

struct ghc_master {
  ghc_plan* plan = nullptr;
  float* g_scratch = nullptr;  // layered archs: the round's combined gradient
  float** bufs = nullptr;      // device copy of {w[0], w[1], v[0], v[1]} (sgd_db_kernel)
  float* w[2] = {nullptr, nullptr};
  float* v[2] = {nullptr, nullptr};
  MasterDev* ms = nullptr;
  MasterDev* ms_apply = nullptr;  // barrier state for the in-place sgd_apply_kernel
  MasterDev* ms_db = nullptr;     // bad flag + arrival counter of sgd_db_kernel
  float lr = 0.01f, mu = 0.0f;
  int64_t P = 0;
  // host copy of ms->cur: valid until a launch that may flip the buffers
  // (the fused rounds, ghc_master_apply) — saves a blocking D2H per call
  int host_cur = 0;
  bool host_cur_known = true;
};

// Current buffer index of the master (cached; one D2H read when unknown).
extern "C" ghc_status ghc_master_current(ghc_master* m, int* cur);
// Force-load the stream gate kernel (before a resident kernel starts).
extern "C" ghc_status ghc_preload_gate();
// sgd_step on the master's double buffers in ONE pass (sgd_db_kernel, det
// mode + db_fixup_kernel): the buffers flip on every call, so the host keeps
// knowing the current index; lr / mu as given (the top master of a
// hierarchy uses its parent settings).
extern "C" ghc_status master_apply_det(ghc_master* m, const float* d_g, float lr, float mu);

namespace {

// Launch geometry of the fused step: ≈ one CTA per SM, one warp per sample.
inline void step_geometry(const ghc_plan* p, int64_t n, int& ctas, int& warps) {
  const int sms = p->ctx->num_sms;
  warps = static_cast<int>((n + sms - 1) / sms);
  if (warps < 1) warps = 1;
  if (warps > p->max_warps) warps = p->max_warps;
  int64_t c = (n + warps - 1) / warps;
  if (c < 1) c = 1;
  if (c > p->max_ctas) c = p->max_ctas;
  ctas = static_cast<int>(c);
}

// vr > 1: vr virtual ranks share the grid (cross-rank exchange, SIMT kernel),
// each with max_clusters / vr clusters and n_max samples per round.
inline ghc_status launch_step(ghc_plan* p, StepArgs& a, int64_t n_max, int vr = 1,
                              cudaStream_t stream = nullptr, bool multi = false) {
  if (!p->lstm) return fail(GHC_ERR_CONFIG, "plan has no fused worker kernel");
  if (a.res && !(p->use_cluster && p->max_clusters > 0 && !p->use_tc))
    return fail(GHC_ERR_CONFIG, "resident rounds need the SIMT cluster round kernel");
  a.err = p->err;
  a.probe = p->probe;
  a.bar = p->bar;
  if (p->use_cluster && p->max_clusters > 0) {
    // ≈ one CTA per SM; SIMT variant: one warp per sample, TC variant: the
    // CTA's 8 warps step 8 samples together (kTcSamples per pass)
    const int cs = p->cluster_size;
    const bool tc = p->use_tc && a.GX <= 1;
    const int maxc = p->max_clusters / vr;
    if (maxc < 1) return fail(GHC_ERR_CONFIG, "too many virtual ranks for the co-resident clusters");
    int warps;
    int64_t per_cta;  // samples per CTA in one pass
    if (tc) {
      warps = 8;
      per_cta = kTcSamples;
    } else {
      const int spw = kSamplesPerWarp;
      const int64_t slots = static_cast<int64_t>(maxc) * cs * spw;
      warps = static_cast<int>((n_max + slots - 1) / slots);
      warps = warps < 1 ? 1 : (warps > p->round_warps ? p->round_warps : warps);
      per_cta = static_cast<int64_t>(warps) * spw;
    }
    int64_t ctas = (n_max + per_cta - 1) / per_cta;
    int64_t nc = (ctas + cs - 1) / cs;
    if (nc < 1) nc = 1;
    if (nc > maxc) nc = maxc;
    a.VR = vr;
    a.part = p->part;
    a.tpart = p->tpart;
    a.tw = p->tw;
    a.pstride = p->lstm->ep[p->cs_index];
    a.pipelined = n_max <= nc * cs * per_cta;
    if (a.res && !a.pipelined)
      return fail(GHC_ERR_CONFIG, "resident rounds: the batch must fit one sample per warp slot");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nc * cs * vr));
    cfg.blockDim = dim3(static_cast<unsigned>(warps * 32));
    cfg.dynamicSmemBytes = tc ? p->lstm->smem_tc[p->cs_index](warps)
                              : p->lstm->smem_round[p->cs_index](warps);
    cfg.stream = stream ? stream : p->ctx->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    // GHC_NO_COOP=1: plain cluster launch (ncu cannot replay cooperative
    // cluster launches); the grid never exceeds the co-resident clusters
    // reported by cudaOccupancyMaxActiveClusters, so the spin barriers hold.
    static const bool no_coop = [] {
      const char* e = std::getenv("GHC_NO_COOP");
      return e && e[0] == '1';
    }();
    cfg.numAttrs = no_coop ? 1 : 2;
    void (*fn)(StepArgs) = multi ? p->lstm->fn_multi[p->cs_index]
                           : tc  ? p->lstm->fn_tc[p->cs_index]
                                 : (a.res ? p->lstm->fn_res[p->cs_index] : p->lstm->fn_round[p->cs_index]);
    if (!fn) return fail(GHC_ERR_CONFIG, "no kernel variant for this launch");
    if (a.res || multi) {  // same shared-memory opt-in as the ordinary variant
      CU(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(cfg.dynamicSmemBytes)));
    }
    CU(cudaLaunchKernelEx(&cfg, fn, a));
    p->ctx->launches++;
    return GHC_OK;
  }
  int ctas, warps;
  step_geometry(p, n_max, ctas, warps);
  a.part = p->part;
  a.pstride = p->lstm->ppad;
  a.pipelined = n_max <= static_cast<int64_t>(ctas) * warps;
  const size_t smem = p->lstm->smem(warps);
  void* args[] = {&a};
  CU(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(p->lstm->fn), dim3(ctas),
                                 dim3(warps * 32), args, smem, p->ctx->stream));
  p->ctx->launches++;
  return GHC_OK;
}

inline int occupancy_grid(ghc_ctx* c, const void* fn, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  if (per_sm < 1) per_sm = 1;
  return per_sm * c->num_sms;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace


// layered.cu — worker step for archs with dense layers; g_out == nullptr ⇒
// forward only (probs nullable, loss_out nullable).
ghc_status layered_step(ghc_plan* p, const float* w, const float* x, const int32_t* y,
                        const int32_t* idx, int64_t n, float scale, float* g_out,
                        float* loss_out, float* probs);
void layered_free(LayeredWorkspace* ws);

// generic.cu — LSTM layer of any shape as per-timestep tcgen05 GEMMs + cell kernels.
ghc_status generic_lstm_fwd(ghc_plan* p, const float* w, const float* X, int n, float* hT_out);
ghc_status generic_lstm_bwd(ghc_plan* p, const float* w, const float* X, int n, const float* dhT,
                            float* g_out);
ghc_status generic_lstm_cache(ghc_plan* p, int n, float* d_gates, float* d_cell, float* d_tanh,
                              float* d_hidden);
void generic_lstm_free(GenericLstmWorkspace* ws);

// LSTM trunk (flat kernel of p->trunk, modes MODE_TRUNK_*), cooperative.
inline ghc_status launch_trunk(ghc_plan* p, StepArgs& a, int64_t n) {
  const LstmEntry* e = p->trunk;
  const int sms = p->ctx->num_sms;
  int warps = static_cast<int>((n + sms - 1) / sms);
  warps = warps < 1 ? 1 : (warps > 8 ? 8 : warps);
  int64_t ctas = (n + warps - 1) / warps;
  if (ctas > p->max_ctas) ctas = p->max_ctas;
  a.part = p->part;
  a.pstride = e->ppad;
  a.err = p->err;
  a.bar = p->bar;
  a.pipelined = 0;
  void* args[] = {&a};
  CU(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(e->fn), dim3(static_cast<unsigned>(ctas)),
                                 dim3(warps * 32), args, e->smem(warps), p->ctx->stream));
  p->ctx->launches++;
  return GHC_OK;
}
