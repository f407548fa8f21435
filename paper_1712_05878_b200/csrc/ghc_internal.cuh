// ghc_internal.cuh — definitions shared by the libghc translation units
// (ghc.cu: model/algo/master; dist.cu: NCCL exchange).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ghc.h"
#include "host_model.hpp"
#include "lstm_step.cuh"
#include "update_kernels.cuh"

using namespace ghc;

ghc_status ghc_fail(ghc_status s, const std::string& msg);
#define fail ghc_fail

namespace {

#define CU(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(GHC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
  } while (0)

// ---- fused LSTM→softmax kernel table (one instantiation per shape) ----
struct LstmEntry {
  int D, H, T, K;
  void (*fn)(StepArgs);
  int P, ppad;
  size_t (*smem)(int);
  const char* name;
};

template <int D, int H, int T, int K>
LstmEntry make_entry(const char* name) {
  using N = LstmNet<D, H, T, K>;
  return LstmEntry{D, H, T, K, &lstm_softmax_step_kernel<D, H, T, K>, N::P, N::PPAD,
                   &N::smem_bytes, name};
}

const std::vector<LstmEntry>& lstm_table() {
  static const std::vector<LstmEntry> t = {
      make_entry<5, 20, 10, 3>("lstm_softmax_step<D5,H20,T10,K3>"),  // SPEC.md:109 bench net
      make_entry<5, 8, 10, 3>("lstm_softmax_step<D5,H8,T10,K3>"),
      make_entry<3, 4, 5, 3>("lstm_softmax_step<D3,H4,T5,K3>"),
      make_entry<2, 16, 3, 4>("lstm_softmax_step<D2,H16,T3,K4>"),
      make_entry<5, 32, 10, 3>("lstm_softmax_step<D5,H32,T10,K3>"),
      make_entry<4, 12, 6, 5>("lstm_softmax_step<D4,H12,T6,K5>"),
  };
  return t;
}

}  // namespace

struct ghc_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::atomic<uint64_t> launches{0};
};

struct ghc_plan {
  ghc_ctx* ctx = nullptr;
  int max_warps = 8;      // warps/CTA that fit the fused kernel's smem
  unsigned long long* probe = nullptr;  // phase-timing probe (diagnostics)
  Model model;
  const LstmEntry* lstm = nullptr;
  int max_ctas = 0;       // co-resident CTAs of the fused kernel
  float* part = nullptr;  // [max_ctas][ppad]
  MasterDev* ms = nullptr;  // scratch barrier state for grad/fwd launches
  int* err = nullptr;
  std::string kname;
};

struct ghc_master {
  ghc_plan* plan = nullptr;
  float* w[2] = {nullptr, nullptr};
  float* v[2] = {nullptr, nullptr};
  MasterDev* ms = nullptr;
  MasterDev* ms_apply = nullptr;  // barrier state for ghc_master_apply
  float lr = 0.01f, mu = 0.0f;
  int64_t P = 0;
};

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

inline ghc_status launch_step(ghc_plan* p, StepArgs& a, int64_t n_max) {
  if (!p->lstm) return fail(GHC_ERR_CONFIG, "plan has no fused worker kernel");
  int ctas, warps;
  step_geometry(p, n_max, ctas, warps);
  a.part = p->part;
  a.pstride = p->lstm->ppad;
  a.err = p->err;
  a.probe = p->probe;
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

