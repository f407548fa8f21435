// dense.cu — C ABI for the dense-layer GEMM (tcgen05, 3×TF32) and transpose.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dense_gemm.cuh"
#include "ghc_internal.cuh"

using namespace ghc;

namespace {
template <int BN>
ghc_status launch_gemm(ghc_ctx* c, const GemmArgs& g) {
  constexpr int stage = 2 * gemm_detail::BM * gemm_detail::BK * 4 + 2 * BN * gemm_detail::BK * 4;
  const size_t smem = 2 * stage;
  static bool attr_set = false;
  if (!attr_set) {
    CU(cudaFuncSetAttribute(tcgen05_gemm_nt_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    attr_set = true;
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + gemm_detail::BM - 1) / gemm_detail::BM);
  tcgen05_gemm_nt_kernel<BN><<<grid, 128, smem, c->stream>>>(g);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// fp32 [rows][ld] K-major operand, box = one 16-byte K-chunk × box_rows rows.
bool make_map(CUtensorMap* tm, const float* base, int rows, int K, int ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15u) || (ld % 4)) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
  const cuuint32_t box[2] = {4, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// GHC_GEMM=legacy forces the register-staged kernel (A/B comparisons).
bool tma_allowed() {
  static const bool ok = [] {
    const char* e = std::getenv("GHC_GEMM");
    return !(e && std::string(e) == "legacy");
  }();
  return ok;
}

template <int BN>
ghc_status launch_gemm_tma(ghc_ctx* c, const GemmArgs& g, const CUtensorMap& ta,
                           const CUtensorMap& tb) {
  constexpr int stage = 2 * gemm_detail::BM * gemm_detail::BK * 4 + 2 * BN * gemm_detail::BK * 4;
  const size_t smem = gemm_detail::kTmaStages * stage;
  static bool attr_set = false;
  if (!attr_set) {
    CU(cudaFuncSetAttribute(tcgen05_gemm_tma_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    attr_set = true;
  }
  const int nz = g.kchunk > 0 ? (g.K + g.kchunk - 1) / g.kchunk : 1;
  dim3 grid((g.N + BN - 1) / BN, (g.M + gemm_detail::BM - 1) / gemm_detail::BM, nz);
  tcgen05_gemm_tma_kernel<BN><<<grid, 192, smem, c->stream>>>(ta, tb, g);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

// CTA-pair kernel (tcgen05 cta_group::2, 256 × 2·NH tiles): large M and N.
// GHC_GEMM=single keeps the single-CTA kernel (A/B comparisons).
bool pair_allowed() {
  static const bool ok = [] {
    const char* e = std::getenv("GHC_GEMM");
    return !(e && (std::string(e) == "single" || std::string(e) == "legacy"));
  }();
  return ok;
}

#ifndef GHC_PAIR_BK
#define GHC_PAIR_BK 16
#endif
constexpr int kPairBK = GHC_PAIR_BK;                  // K elements per stage
constexpr int kPairStages = 96 / kPairBK;             // 6 × 32 KB (BK 16) or 3 × 64 KB (BK 32)
template <int NH>
ghc_status launch_gemm_pair(ghc_ctx* c, const GemmArgs& g, const CUtensorMap& ta,
                            const CUtensorMap& tb) {
  constexpr int BKP = kPairBK, SP = kPairStages;
  constexpr int stage = 2 * gemm_detail::BM * BKP * 4 + 2 * NH * BKP * 4;
  const size_t smem = SP * stage;
  static bool attr_set = false;
  if (!attr_set) {
    CU(cudaFuncSetAttribute(tcgen05_gemm_pair_kernel<NH, BKP, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    attr_set = true;
  }
  dim3 grid(2 * ((g.N + 2 * NH - 1) / (2 * NH)), (g.M + 2 * gemm_detail::BM - 1) / (2 * gemm_detail::BM));
  tcgen05_gemm_pair_kernel<NH, BKP, SP><<<grid, 320, smem, c->stream>>>(ta, tb, g);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

// Narrow outputs with a long K (dX of the N = 20 input layer, K = 4096: only
// ⌈M/128⌉ = 8 tiles for 148 SMs): split K over ≈ one wave of CTAs into
// per-split partials, then one deterministic combine + epilogue pass.
ghc_status launch_gemm_splitk(ghc_ctx* c, const GemmArgs& g, const CUtensorMap& ta,
                              const CUtensorMap& tb, int nsplit) {
  int kchunk = (g.K + nsplit - 1) / nsplit;
  kchunk = (kchunk + gemm_detail::BK - 1) / gemm_detail::BK * gemm_detail::BK;
  const int nz = (g.K + kchunk - 1) / kchunk;
  const size_t need = sizeof(float) * static_cast<size_t>(nz) * g.M * g.N;
  if (need > c->splitk_bytes) {
    cudaFree(c->splitk_ws);  // synchronising: no launch still uses the old buffer
    c->splitk_ws = nullptr;
    c->splitk_bytes = 0;
    CU(cudaMalloc(&c->splitk_ws, need));
    c->splitk_bytes = need;
  }
  GemmArgs p = g;  // partials: raw sums, [nz][M][N]
  p.C = c->splitk_ws;
  p.CT = nullptr;
  p.ldc = g.N;
  p.epi = EPI_STORE;
  p.alpha = 1.0f;
  p.kchunk = kchunk;
  if (ghc_status st = launch_gemm_tma<32>(c, p, ta, tb)) return st;
  const long long n = static_cast<long long>(g.M) * g.N;
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 4LL * c->num_sms));
  splitk_reduce_kernel<<<blocks, 256, 0, c->stream>>>(c->splitk_ws, nz, g);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}
}  // namespace

namespace ghc {
ghc_status gemm_nt_ct(ghc_ctx* c, const float* d_a, const float* d_b, float* d_c, int32_t M,
                      int32_t N, int32_t K, int32_t lda, int32_t ldb, int32_t ldc, int32_t epi,
                      int32_t act, const float* d_bias, const float* d_y, int32_t ldy, float alpha,
                      float* d_ct, int32_t ldct) {
  if (M < 1 || N < 1 || K < 1) return ghc_fail(GHC_ERR_SHAPE, "gemm: empty operand");
  GemmArgs g{d_a, d_b, d_c, d_bias, d_y, M, N, K, lda, ldb, ldc, ldy, act, alpha, epi};
  g.CT = d_ct;
  g.ldct = ldct;
  // N tile: one 128×BN tile per CTA, one CTA per SM (≈190 KB of stages), so a
  // launch takes ⌈tiles / SMs⌉ waves of time ∝ BN.  Pick the BN with the
  // least waves × BN (ties → the larger tile): M = 1000, N = 4096 → BN = 112,
  // 296 tiles = exactly 2 waves on 148 SMs instead of 256 tiles in 2 waves of
  // 128-wide tiles.
  int bn = 32;
  if (N > 32) {
    const long long mt = (M + gemm_detail::BM - 1) / gemm_detail::BM;
    long long best = -1;
    for (int cand : {128, 112, 96, 64}) {
      const long long tiles = mt * ((N + cand - 1) / cand);
      const long long cost = (tiles + c->num_sms - 1) / c->num_sms * cand;
      if (best < 0 || cost < best) {
        best = cost;
        bn = cand;
      }
    }
  }
  CUtensorMap ta, tb;
  if (pair_allowed() && M >= 256 && N >= 256 && K >= 4 * gemm_detail::BK &&
      make_map(&ta, d_a, M, K, lda, gemm_detail::BM) && make_map(&tb, d_b, N, K, ldb, 128))
    return launch_gemm_pair<128>(c, g, ta, tb);
  if (tma_allowed() && make_map(&ta, d_a, M, K, lda, gemm_detail::BM) &&
      make_map(&tb, d_b, N, K, ldb, bn)) {
    const long long tiles = static_cast<long long>((M + gemm_detail::BM - 1) / gemm_detail::BM) *
                            ((N + bn - 1) / bn);
    if (bn == 32 && tiles * 4 <= c->num_sms && K >= 8 * gemm_detail::BK) {
      const int nsplit = static_cast<int>(std::min<long long>(c->num_sms / tiles, K / (4 * gemm_detail::BK)));
      if (nsplit >= 2) return launch_gemm_splitk(c, g, ta, tb, nsplit);
    }
    switch (bn) {
      case 32: return launch_gemm_tma<32>(c, g, ta, tb);
      case 64: return launch_gemm_tma<64>(c, g, ta, tb);
      case 96: return launch_gemm_tma<96>(c, g, ta, tb);
      case 112: return launch_gemm_tma<112>(c, g, ta, tb);
      default: return launch_gemm_tma<128>(c, g, ta, tb);
    }
  }
  // register-staged fallback (GHC_GEMM=legacy / unaligned operands): no CT
  // epilogue there, so transpose the result afterwards
  if (ghc_status st = N <= 32 ? launch_gemm<32>(c, g) : launch_gemm<128>(c, g)) return st;
  if (d_ct) return ghc_transpose(c, d_ct, d_c, M, N, ldc, ldct);
  return GHC_OK;
}
// Long-K weight-gradient GEMMs (K = n·T of the generic LSTM path): always
// split K over ≈ one wave into ordered partials — each partial accumulates a
// short K range in TMEM (3×TF32 error grows with the accumulated K), and the
// combine adds them in split order (deterministic).
ghc_status gemm_nt_splitk(ghc_ctx* c, const float* d_a, const float* d_b, float* d_c, int32_t M,
                          int32_t N, int32_t K, int32_t lda, int32_t ldb, int32_t ldc) {
  if (M < 1 || N < 1 || K < 1) return ghc_fail(GHC_ERR_SHAPE, "gemm: empty operand");
  GemmArgs g{d_a, d_b, d_c, nullptr, nullptr, M, N, K, lda, ldb, ldc, 0, 2, 1.0f, GHC_EPI_STORE};
  g.CT = nullptr;
  g.ldct = 0;
  CUtensorMap ta, tb;
  if (tma_allowed() && N <= 32 && make_map(&ta, d_a, M, K, lda, gemm_detail::BM) &&
      make_map(&tb, d_b, N, K, ldb, 32)) {
    const long long tiles = (M + gemm_detail::BM - 1) / gemm_detail::BM;
    const int nsplit = static_cast<int>(
        std::max<long long>(1, std::min<long long>(c->num_sms / tiles, K / (4 * gemm_detail::BK))));
    if (nsplit >= 2) return launch_gemm_splitk(c, g, ta, tb, nsplit);
  }
  if (N > 32) {  // column blocks of 32: each block takes the split-K path
    for (int n0 = 0; n0 < N; n0 += 32) {
      const int nb = std::min(32, N - n0);
      if (ghc_status st = gemm_nt_splitk(c, d_a, d_b + static_cast<long long>(n0) * ldb, d_c + n0, M, nb, K,
                                         lda, ldb, ldc))
        return st;
    }
    return GHC_OK;
  }
  return gemm_nt_ct(c, d_a, d_b, d_c, M, N, K, lda, ldb, ldc, GHC_EPI_STORE, 2, nullptr, nullptr, 0,
                    1.0f, nullptr, 0);
}
}  // namespace ghc

extern "C" {

ghc_status ghc_gemm_nt(ghc_ctx* c, const float* d_a, const float* d_b, float* d_c, int32_t M,
                       int32_t N, int32_t K, int32_t lda, int32_t ldb, int32_t ldc, int32_t epi,
                       int32_t act, const float* d_bias, const float* d_y, int32_t ldy,
                       float alpha) {
  return gemm_nt_ct(c, d_a, d_b, d_c, M, N, K, lda, ldb, ldc, epi, act, d_bias, d_y, ldy, alpha,
                    nullptr, 0);
}

ghc_status ghc_transpose(ghc_ctx* c, float* d_out, const float* d_in, int32_t rows, int32_t cols,
                         int32_t ldin, int32_t ldout) {
  if (ldin % 4 == 0 && ldout % 4 == 0 && aligned16(d_in) && aligned16(d_out) &&
      static_cast<long long>(rows) * cols >= (1 << 16)) {
    dim3 g4((cols + 63) / 64, (rows + 63) / 64);
    transpose4_kernel<<<g4, 256, 0, c->stream>>>(d_out, d_in, rows, cols, ldin, ldout);
    CU(cudaGetLastError());
    c->launches++;
    return GHC_OK;
  }
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(d_out, d_in, rows, cols, ldin, ldout);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

}  // extern "C"
