// dense.cu — C ABI for the dense-layer GEMM (tcgen05, 3×TF32) and transpose.
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
}  // namespace

extern "C" {

ghc_status ghc_gemm_nt(ghc_ctx* c, const float* d_a, const float* d_b, float* d_c, int32_t M,
                       int32_t N, int32_t K, int32_t lda, int32_t ldb, int32_t ldc, int32_t epi,
                       int32_t act, const float* d_bias, const float* d_y, int32_t ldy,
                       float alpha) {
  if (M < 1 || N < 1 || K < 1) return ghc_fail(GHC_ERR_SHAPE, "gemm: empty operand");
  GemmArgs g{d_a, d_b, d_c, d_bias, d_y, M, N, K, lda, ldb, ldc, ldy, act, alpha, epi};
  if (N <= 32) return launch_gemm<32>(c, g);
  return launch_gemm<128>(c, g);
}

ghc_status ghc_transpose(ghc_ctx* c, float* d_out, const float* d_in, int32_t rows, int32_t cols,
                         int32_t ldin, int32_t ldout) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(d_out, d_in, rows, cols, ldin, ldout);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

}  // extern "C"
