// dense_gemm.cuh — tcgen05 (5th-gen tensor core) GEMM for the dense layers of
// the wide-layer variant (nn.cpp:129-145 forward, nn.cpp:312-334 backward).
//
//   C[M×N] = A[M×K] · B[N×K]ᵀ      (both operands K-major, fp32 in HBM)
//
// * 3×TF32: every fp32 operand x is split in smem into hi = tf32(x) and
//   lo = tf32(x − hi); D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi with fp32
//   accumulation in TMEM — fp32-level accuracy (the reference is f64; a plain
//   TF32 product would be ~1e-3 relative and fail parity).
// * Tile 128 × BN (BN = 128 or 32) × 32 per stage, 2-stage smem pipeline:
//   all threads load+split the next K-block while the tensor core runs the
//   current one; one elected thread issues the 12 tcgen05.mma (4 K-steps × 3)
//   and commits to the stage's mbarrier.
// * Operands in the canonical K-major SWIZZLE_NONE layout (core matrix = 8
//   rows × 16 B; LBO = stride between the two 16-B K-chunks of one MMA,
//   SBO = stride between 8-row groups — CUTLASS mma_sm100_desc.hpp).
// * Epilogue: tcgen05.ld 32x32b.x32 → registers → fused bias / activation /
//   activation-derivative / scale → st.global (the (epi, act) switch once per
//   chunk: each variant a branch-free unrolled loop).
// * Large M and N: tcgen05_gemm_pair_kernel (below) — a CTA pair
//   (cta_group::2) per 256 × 256 tile, half the shared-memory operand bytes
//   per output, accumulator segments drained to registers for accuracy.
#pragma once

#include <type_traits>

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ghc_device.cuh"  // GHC_CHECK

namespace ghc {

enum GemmEpi : int {
  EPI_STORE = 0,     // C = acc * alpha
  EPI_BIAS_ACT = 1,  // C = act(acc + bias[n])            (forward, act in {tanh, relu, id})
  EPI_DACT = 2,      // C = acc * act'(Y[m][n])            (backward dX, act' from the layer output)
};

struct GemmArgs {
  const float* A;  // [M][lda]
  const float* B;  // [N][ldb]
  float* C;        // [M][ldc]
  const float* bias;  // EPI_BIAS_ACT
  const float* Y;     // EPI_DACT: [M][ldy]
  int M, N, K;
  int lda, ldb, ldc, ldy;
  int act;      // 0 tanh, 1 relu, 2 identity (arch.hpp:10)
  float alpha;
  int epi;
  int kchunk = 0;  // split-K: CTA z covers K range [z·kchunk, (z+1)·kchunk) (multiple of BK)
  float* CT = nullptr;  // optional transposed copy: CT[n][m] (row stride ldct) — the
  int ldct = 0;         // K-major operand of the next weight-gradient GEMM, written
                        // coalesced by the epilogue instead of a separate transpose
};

namespace gemm_detail {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per stage along K (= 8 chunks of 16 B)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, SWIZZLE_NONE smem descriptor (sm_100 "version 1").
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  // base_offset 0, lbo_mode 0, layout_type SWIZZLE_NONE (0)
  return d;
}

// kind::tf32, D f32, A/B TF32, both K-major, M = 128.
__host__ __device__ constexpr uint32_t make_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// Bounded wait: a descriptor / commit bug traps (kernel error) instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  for (long long spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase));
    if (done) return;
    if (spin > (1ll << 26)) __trap();
  }
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ float act_f(float z, int act) {
  if (act == 1) return z > 0.f ? z : 0.f;
  if (act == 0) return tanhf(z);
  return z;
}
// derivative from the activation OUTPUT y (nn.cpp:26-36 rewritten in y):
// tanh' = 1 − y², relu' = [y > 0] (≡ [z > 0]), identity' = 1
__device__ __forceinline__ float dact_from_y(float y, int act) {
  if (act == 1) return y > 0.f ? 1.f : 0.f;
  if (act == 0) return 1.f - y * y;
  return 1.f;
}

}  // namespace gemm_detail

// Block: 128 threads (4 warps).  Warp w owns TMEM lanes 32w..32w+31 = tile
// rows; one thread of warp 0 issues the MMAs.
template <int BN>
__global__ void __launch_bounds__(128, 1) tcgen05_gemm_nt_kernel(GemmArgs g) {
  using namespace gemm_detail;
  static_assert(BN == 32 || BN == 64 || BN == 128 || BN == 256, "N tile");
  constexpr int A_BYTES = BM * BK * 4;                 // one operand copy per stage
  constexpr int B_BYTES = BN * BK * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;     // hi + lo of A and B
  extern __shared__ __align__(1024) uint8_t gsm[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

  // NACC accumulators in TMEM, K-blocks rotate over them: the tensor core's
  // fp32 accumulation truncates, so fewer adds into each (smaller) partial
  // sum + round-to-nearest FADDs of the partials in the epilogue cut the
  // K-proportional bias (measured: DESIGN.md §4, dense layers).
  constexpr int NACC = 4;
  constexpr int TCOLS = NACC * BN < 32 ? 32 : NACC * BN;
  static_assert(TCOLS <= 512, "TMEM columns");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  // Canonical K-major layout inside one operand copy:
  //   [chunk c = 0..7 (16 B of K)][row group = rows/8][row % 8][16 B]
  //   LBO = rows*16 (next chunk), SBO = 128 (next 8-row group)
  auto store_tile = [&](uint8_t* base_hi, uint8_t* base_lo, const float* src, int ld, int rows,
                        int row0, int row_lim, int k0) {
    // lane = chunk_local*8 + r8 ; a warp covers 8 rows × 4 chunks per pass
    for (int it = warp; it < (rows / 8) * 2; it += 4) {
      const int rg = it >> 1;               // 8-row group
      const int ch = (it & 1) * 4 + (lane >> 3);
      const int r = rg * 8 + (lane & 7);
      const int grow = row0 + r;
      const int gk = k0 + ch * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (grow < row_lim) {
        const float* p = src + (long long)grow * ld + gk;
        if (gk + 3 < g.K && (((uintptr_t)p) & 15u) == 0) {
          v = __ldg(reinterpret_cast<const float4*>(p));
        } else {
          if (gk < g.K) v.x = __ldg(p);
          if (gk + 1 < g.K) v.y = __ldg(p + 1);
          if (gk + 2 < g.K) v.z = __ldg(p + 2);
          if (gk + 3 < g.K) v.w = __ldg(p + 3);
        }
      }
      float4 h, l;
      h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - h.x);
      h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - h.y);
      h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - h.z);
      h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - h.w);
      const int off = ch * rows * 16 + rg * 128 + (lane & 7) * 16;
      *reinterpret_cast<float4*>(base_hi + off) = h;
      *reinterpret_cast<float4*>(base_lo + off) = l;
    }
  };

  const int nkb = (g.K + BK - 1) / BK;
  const uint32_t idesc = make_idesc(BN);
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb & 1;
    uint8_t* st = gsm + s * STAGE;
    if (kb >= 2) mbar_wait(&mbar[s], ((kb - 2) >> 1) & 1);  // MMAs that read this stage are done
    store_tile(st, st + A_BYTES, g.A, g.lda, BM, m0, g.M, kb * BK);
    store_tile(st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES, g.B, g.ldb, BN, n0, g.N, kb * BK);
    asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy stores → tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = smem_u32(st), a_lo = a_hi + A_BYTES;
      const uint32_t b_hi = smem_u32(st + 2 * A_BYTES), b_lo = b_hi + B_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {  // K = 8 tf32 = 2 chunks per MMA
        const uint32_t ao = ks * 2 * BM * 16, bo = ks * 2 * BN * 16;
        const uint64_t dah = make_desc(a_hi + ao, BM * 16, 128);
        const uint64_t dal = make_desc(a_lo + ao, BM * 16, 128);
        const uint64_t dbh = make_desc(b_hi + bo, BN * 16, 128);
        const uint64_t dbl = make_desc(b_lo + bo, BN * 16, 128);
        const uint32_t acc0 = (kb >= NACC || ks > 0) ? 1u : 0u;  // first use zero-inits
        const uint32_t d = tmem + static_cast<uint32_t>((kb % NACC) * BN);
        umma_tf32(d, dah, dbh, idesc, acc0);  // hi·hi
        umma_tf32(d, dah, dbl, idesc, 1u);    // hi·lo
        umma_tf32(d, dal, dbh, idesc, 1u);    // lo·hi
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar[s])));
    }
  }
  // last K-block's MMAs complete ⇒ all complete (issue order)
  const int last = nkb - 1;
  mbar_wait(&mbar[last & 1], (last >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // ---- epilogue: TMEM → registers → fused op → HBM ----
  const int row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    for (int a = 0; a < NACC && a < nkb; ++a) {
      uint32_t v[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + a * BN + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] += __uint_as_float(v[i]);
    }
    if (row < g.M) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int col = n0 + c0 + i;
        if (col >= g.N) continue;
        float o = acc[i];
        if (g.epi == EPI_BIAS_ACT) {
          o = act_f(o + g.bias[col], g.act);
        } else if (g.epi == EPI_DACT) {
          o *= dact_from_y(g.Y[(long long)row * g.ldy + col], g.act);
        } else {
          o *= g.alpha;
        }
        g.C[(long long)row * g.ldc + col] = o;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TCOLS));
}

// ---------------------------------------------------------------------------
// TMA-fed, warp-specialised variant (the default when strides allow TMA).
//
//   warp 0      : TMA producer — per stage 8 boxes of A (16 B of K × 128 rows)
//                 and 8 of B; a box of one 16-byte K-chunk lands as rows × 16 B
//                 contiguous = one column of core matrices of the canonical
//                 K-major SWIZZLE_NONE layout (LBO = rows·16, SBO = 128).  TMA
//                 zero-fills the M/N/K edges.
//   warp 1      : TMEM allocation, one elected thread issues the 12 MMAs of a
//                 stage (4 K-steps × 3×TF32) and commits to the stage's
//                 "empty" barrier.
//   warps 2..5  : split — the raw fp32 tile IS the "hi" operand (the tensor
//                 core ignores the low 13 mantissa bits); they write only
//                 lo = x − trunc_tf32(x) (exact), then the epilogue (TMEM lane
//                 quarter = warp % 4).
// Stages: STAGES × (A_hi, A_lo, B_hi, B_lo) in smem; barriers full (TMA bytes),
// split (128 arrivals), empty (MMA commit), done (last commit).
namespace gemm_detail {

constexpr int kTmaStages = 3;

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace gemm_detail

// tcgen05.ld of W ∈ {16, 32} consecutive 32-bit TMEM columns (32 lanes × W)
template <int W>
__device__ __forceinline__ void tmem_ld(uint32_t (&v)[W], uint32_t taddr) {
  static_assert(W == 16 || W == 32, "chunk");
  if constexpr (W == 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;");
}

// The epilogue op on W consecutive columns of one row: the (epi, act) switch
// is taken once per chunk, so each variant is a branch-free unrolled loop
// (a per-element switch serialised the epilogue: ≈ 10 µs per 128 × 112 tile).
// Columns ≥ N compute throw-away values (never stored).
template <int W>
__device__ __forceinline__ void epilogue_ops(float (&acc)[W], const GemmArgs& g, int row, int col0) {
  using namespace gemm_detail;
  if (g.epi == EPI_BIAS_ACT) {
    float b[W];
#pragma unroll
    for (int i = 0; i < W; ++i) b[i] = col0 + i < g.N ? __ldg(g.bias + col0 + i) : 0.f;
    if (g.act == 1) {
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = fmaxf(acc[i] + b[i], 0.f);
    } else if (g.act == 2) {
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] += b[i];
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = tanhf(acc[i] + b[i]);
    }
  } else if (g.epi == EPI_DACT) {
    float y[W];
    const float* yr = g.Y + (long long)row * g.ldy;
#pragma unroll
    for (int i = 0; i < W; ++i) y[i] = col0 + i < g.N ? __ldg(yr + col0 + i) : 0.f;
    if (g.act == 1) {
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = y[i] > 0.f ? acc[i] : 0.f * acc[i];
    } else if (g.act == 0) {
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] *= 1.f - y[i] * y[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) acc[i] *= g.alpha;
  }
}

template <int BN>
__global__ void __launch_bounds__(192, 1)
    tcgen05_gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                            const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
  using namespace gemm_detail;
  // BN: any multiple of 16 up to 128 (kind::tf32, M = 128 needs N % 16 == 0);
  // the host picks it so the tile count fills whole waves of the SMs.
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 128, "N tile");
  constexpr int S = kTmaStages;
  constexpr int A_BYTES = BM * BK * 4;
  constexpr int B_BYTES = BN * BK * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // A_hi | A_lo | B_hi | B_lo
  constexpr int NACC = 4;                           // rotating accumulators (accuracy)
  constexpr int TCOLS = NACC * BN <= 32 ? 32 : NACC * BN <= 64 ? 64 : NACC * BN <= 128 ? 128
                       : NACC * BN <= 256 ? 256 : 512;  // power of two
  static_assert(NACC * BN <= 512, "TMEM columns");
  extern __shared__ __align__(1024) uint8_t gsm[];
  __shared__ uint64_t full[S], split[S], empty[S], done;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  // split-K (g.kchunk > 0): this CTA's K range and its own partial-C slice
  const int kbase = g.kchunk > 0 ? static_cast<int>(blockIdx.z) * g.kchunk : 0;
  const int klen = g.kchunk > 0 ? min(g.kchunk, g.K - kbase) : g.K;
  const int nkb = (klen + BK - 1) / BK;
  if (g.kchunk > 0) g.C += static_cast<long long>(blockIdx.z) * g.M * g.ldc;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        uint8_t* st = gsm + s * STAGE;
        mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
#pragma unroll
        for (int c = 0; c < BK / 4; ++c) {
          tma_load_2d(st + c * BM * 16, &tmA, kbase + kb * BK + 4 * c, m0, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + c * BN * 16, &tmB, kbase + kb * BK + 4 * c, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = make_idesc(BN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        mbar_wait(&split[s], (kb / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_hi = smem_u32(gsm + s * STAGE), a_lo = a_hi + A_BYTES;
        const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
        const uint32_t d = tmem + static_cast<uint32_t>((kb % NACC) * BN);
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t ao = ks * 2 * BM * 16, bo = ks * 2 * BN * 16;
          const uint64_t dah = make_desc(a_hi + ao, BM * 16, 128);
          const uint64_t dal = make_desc(a_lo + ao, BM * 16, 128);
          const uint64_t dbh = make_desc(b_hi + bo, BN * 16, 128);
          const uint64_t dbl = make_desc(b_lo + bo, BN * 16, 128);
          const uint32_t acc0 = (kb >= NACC || ks > 0) ? 1u : 0u;
          umma_tf32(d, dal, dbh, idesc, acc0);  // lo·hi (small terms first)
          umma_tf32(d, dah, dbl, idesc, 1u);    // hi·lo
          umma_tf32(d, dah, dbh, idesc, 1u);    // hi·hi
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&empty[s])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&done)));
    }
  } else {
    // ---------------- split: lo = x - trunc_tf32(x) ----------------
    const int t = tid - 64;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      uint8_t* st = gsm + s * STAGE;
      auto split_tile = [&](const uint8_t* hi, uint8_t* lo, int bytes) {
        for (int i = t; i < bytes / 16; i += 128) {
          const uint4 x = reinterpret_cast<const uint4*>(hi)[i];
          float4 l;
          l.x = __uint_as_float(x.x) - __uint_as_float(x.x & 0xFFFFE000u);
          l.y = __uint_as_float(x.y) - __uint_as_float(x.y & 0xFFFFE000u);
          l.z = __uint_as_float(x.z) - __uint_as_float(x.z & 0xFFFFE000u);
          l.w = __uint_as_float(x.w) - __uint_as_float(x.w & 0xFFFFE000u);
          reinterpret_cast<float4*>(lo)[i] = l;
        }
      };
      split_tile(st, st + A_BYTES, A_BYTES);
      split_tile(st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES, B_BYTES);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores → tensor core
      mbar_arrive(&split[s]);
    }
    // ---------------- epilogue: TMEM lane quarter = warp % 4 ----------------
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    const bool vec = (g.N % 4 == 0) && (g.ldc % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(g.C) & 15u) == 0);
    // 32-column chunks (+ one 16-column tail when BN % 32 == 16)
    auto chunk = [&](auto width, int c0) {
      constexpr int W = decltype(width)::value;
      float acc[W];
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = 0.f;
      for (int a = 0; a < NACC && a < nkb; ++a) {
        uint32_t v[W];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + a * BN + c0;
        tmem_ld<W>(v, taddr);
#pragma unroll
        for (int i = 0; i < W; ++i) acc[i] += __uint_as_float(v[i]);
      }
      if (row < g.M) {
        epilogue_ops<W>(acc, g, row, n0 + c0);
        float* crow = g.C + (long long)row * g.ldc + n0 + c0;
        if (vec && n0 + c0 + W <= g.N) {
#pragma unroll
          for (int i = 0; i < W; i += 4)
            reinterpret_cast<float4*>(crow)[i / 4] = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < W; ++i)
            if (n0 + c0 + i < g.N) crow[i] = acc[i];
        }
        if (g.CT) {  // lanes = consecutive rows → each store is one coalesced 128-B line
#pragma unroll
          for (int i = 0; i < W; ++i)
            if (n0 + c0 + i < g.N) g.CT[(long long)(n0 + c0 + i) * g.ldct + row] = acc[i];
        }
      }
    };
#pragma unroll 1
    for (int c0 = 0; c0 + 32 <= BN; c0 += 32) chunk(std::integral_constant<int, 32>{}, c0);
    if constexpr (BN % 32 == 16) chunk(std::integral_constant<int, 16>{}, BN - 16);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of 2 CTAs on the two SMs
// of a TPC computes one 256 × NP tile.  CTA r holds A rows m0 + 128r.. and B
// rows (= C columns) n0 + r·NH.. (NH = NP/2) in its own shared memory; the
// leader (r = 0) issues `tcgen05.mma.cta_group::2` with M = 256, N = NP, which
// reads each CTA's halves from its own SM — per SM, one MMA covers 128 × NP
// outputs for the operand bytes of 128 × NH: half the shared-memory reads per
// output of the single-CTA kernel (whose 3×TF32 stage is bound by the smem
// port).  Accumulators: CTA r's TMEM holds its 128 rows × NP.
// Barriers: each CTA's TMA completes its own `full`; every worker warp of
// both CTAs arrives on the leader's `split` (count 16, mapa'd address); the
// leader's commits arrive on `empty` / accumulator barriers of both CTAs
// (multicast).
namespace gemm_detail {
__host__ __device__ constexpr uint32_t make_idesc_m(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {  // → the same barrier in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {  // arrive on CTA 0's copy
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
}  // namespace gemm_detail

// Accuracy: the tensor core's fp32 accumulation truncates (error ∝ adds per
// accumulator).  Two 256-column TMEM accumulators alternate
// over segments of DS K-blocks; the 8 worker warps drain a finished segment
// into fp32 registers (round-to-nearest FADD; 128 columns × 1 row per
// thread) S K-blocks after it ends, while the tensor core fills the other.
// Warps: 0 TMA producer, 1 MMA issuer (leader CTA), 2..9 split + drain +
// epilogue (TMEM lane quarter = warp % 4, column half = (warp − 2) / 4).
template <int NH, int BKP, int SP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    tcgen05_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
  using namespace gemm_detail;
  constexpr int NP = 2 * NH;  // the pair's N (MMA N ≤ 256, multiple of 16)
  static_assert(NP == 256, "pair N tile: two 256-column accumulators fill TMEM");
  constexpr int S = SP;
  constexpr int DS = 512 / BKP;  // K-blocks per accumulator segment (K = 512: ≤ 192 adds per accumulator)
  static_assert(DS > S, "a segment is drained S K-blocks after it ends, before its accumulator is reused");
  constexpr int A_BYTES = BM * BKP * 4;
  constexpr int B_BYTES = NH * BKP * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // A_hi | A_lo | B_hi | B_lo (this CTA's halves)
  constexpr int TCOLS = 512;
  constexpr int NW = 256;  // worker threads
  extern __shared__ __align__(1024) uint8_t gsm[];
  __shared__ uint64_t full[S], split[S], empty[S], accfull[2], accempty[2];
  __shared__ uint32_t tmem_base_s;

  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * 2 * BM + static_cast<int>(rank) * BM;  // this CTA's A / C rows
  const int n0 = (blockIdx.x >> 1) * NP;                             // the pair's C columns
  const int nb0 = n0 + static_cast<int>(rank) * NH;                  // this CTA's B rows
  const int nkb = (g.K + BKP - 1) / BKP;
  const int nseg = (nkb + DS - 1) / DS;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 16);  // one arrival per worker warp of both CTAs
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], 16);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer (each CTA: its own halves) ----------------
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        uint8_t* st = gsm + s * STAGE;
        mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
#pragma unroll
        for (int c = 0; c < BKP / 4; ++c) {
          tma_load_2d(st + c * BM * 16, &tmA, kb * BKP + 4 * c, m0, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + c * NH * 16, &tmB, kb * BKP + 4 * c, nb0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = make_idesc_m(2 * BM, NP);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        const int seg = kb / DS, acc = seg & 1;
        const bool first = kb % DS == 0, last = kb % DS == DS - 1 || kb == nkb - 1;
        if (first && seg >= 2) mbar_wait(&accempty[acc], ((seg >> 1) - 1) & 1);  // drained
        mbar_wait(&split[s], (kb / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_hi = smem_u32(gsm + s * STAGE), a_lo = a_hi + A_BYTES;
        const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
        const uint32_t d = tmem + static_cast<uint32_t>(acc * NP);
#pragma unroll
        for (int ks = 0; ks < BKP / 8; ++ks) {
          const uint32_t ao = ks * 2 * BM * 16, bo = ks * 2 * NH * 16;
          const uint64_t dah = make_desc(a_hi + ao, BM * 16, 128);
          const uint64_t dal = make_desc(a_lo + ao, BM * 16, 128);
          const uint64_t dbh = make_desc(b_hi + bo, NH * 16, 128);
          const uint64_t dbl = make_desc(b_lo + bo, NH * 16, 128);
          const uint32_t acc0 = (first && ks == 0) ? 0u : 1u;
          umma_tf32_pair(d, dal, dbh, idesc, acc0);  // lo·hi (small terms first)
          umma_tf32_pair(d, dah, dbl, idesc, 1u);    // hi·lo
          umma_tf32_pair(d, dah, dbh, idesc, 1u);    // hi·hi
        }
        commit_pair(&empty[s]);
        if (last) commit_pair(&accfull[acc]);
      }
    }
  } else {
    // ---------------- workers: split, drain, epilogue ----------------
    const int t = tid - 64;
    const int q = warp & 3, h = (warp - 2) >> 2;
    float sum[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) sum[i] = 0.f;
    auto drain = [&](int seg) {
      const int acc = seg & 1;
      mbar_wait(&accfull[acc], (seg >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t v[16];
        tmem_ld<16>(v, tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * NP + h * 128 + c * 16);
#pragma unroll
        for (int i = 0; i < 16; ++i) sum[c * 16 + i] += __uint_as_float(v[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) arrive_leader(&accempty[acc]);
    };
    int drained = 0;
    for (int kb = 0;; ++kb) {
      if (kb < nkb) {
        const int s = kb % S;
        mbar_wait(&full[s], (kb / S) & 1);
        uint8_t* st = gsm + s * STAGE;
        auto split_tile = [&](const uint8_t* hi, uint8_t* lo, int bytes) {
#pragma unroll 2
          for (int i = t; i < bytes / 16; i += NW) {
            const uint4 x = reinterpret_cast<const uint4*>(hi)[i];
            float4 l;
            l.x = __uint_as_float(x.x) - __uint_as_float(x.x & 0xFFFFE000u);
            l.y = __uint_as_float(x.y) - __uint_as_float(x.y & 0xFFFFE000u);
            l.z = __uint_as_float(x.z) - __uint_as_float(x.z & 0xFFFFE000u);
            l.w = __uint_as_float(x.w) - __uint_as_float(x.w & 0xFFFFE000u);
            reinterpret_cast<float4*>(lo)[i] = l;
          }
        };
        split_tile(st, st + A_BYTES, A_BYTES);
        split_tile(st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES, B_BYTES);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores → tensor core
        __syncwarp();
        if (lane == 0) arrive_leader(&split[s]);
      } else if (drained >= nseg) {
        break;
      }
      // a segment is drained S K-blocks after its last one was split (one
      // call site: the 128 running sums stay in registers)
      if (drained < nseg && (kb >= nkb || min(nkb, (drained + 1) * DS) - 1 + S <= kb)) drain(drained++);
    }
    // ---------------- epilogue through shared memory ----------------
    // (the stages are idle: every TMA load was consumed and the last
    // accumulator commit tracked every MMA).  Sums → smem [128][257], then
    // warps sweep rows with lanes along columns: coalesced C / Y / bias
    // accesses and one loop body (instead of 128 unrolled epilogues).
    constexpr int LD = NP + 1;
    float* tile = reinterpret_cast<float*>(gsm);
#ifdef GHC_CHECKED
    {
      unsigned dyn;
      asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
      GHC_CHECK(BM * LD * 4 <= dyn && S * STAGE <= dyn);
    }
#endif
    {
      const int r = q * 32 + lane;
#pragma unroll
      for (int i = 0; i < 128; ++i) tile[r * LD + h * 128 + i] = sum[i];
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int wk = t >> 5;  // worker warp 0..7
    const bool vec = (g.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(g.C) & 15u) == 0);
#pragma unroll 1
    for (int r = wk; r < BM; r += 8) {
      const int row = m0 + r;
      if (row >= g.M) break;
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 128) {  // lane: 4 consecutive columns
        const int c = c0 + 4 * lane;
        float o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = tile[r * LD + c + i];
        epilogue_ops<4>(o, g, row, n0 + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) tile[r * LD + c + i] = o[i];
        float* crow = g.C + (long long)row * g.ldc + n0 + c;
        if (vec && n0 + c + 4 <= g.N) {
          *reinterpret_cast<float4*>(crow) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (n0 + c + i < g.N) crow[i] = o[i];
        }
      }
    }
    if (g.CT) {  // transposed copy: lanes along rows → coalesced CT rows
      asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll 1
      for (int c = wk; c < NP; c += 8) {
        const int col = n0 + c;
        if (col >= g.N) break;
#pragma unroll
        for (int r = lane; r < BM; r += 32) {
          const int row = m0 + r;
          if (row < g.M) g.CT[(long long)col * g.ldct + row] = tile[r * LD + c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // no CTA frees TMEM / leaves while its peer's MMAs or arrivals are in flight
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

// Split-K combine: C = epilogue(Σ_z part[z]) in z order (deterministic),
// with the same epilogues as the GEMM kernels.
static __global__ void splitk_reduce_kernel(const float* __restrict__ part, int nz, GemmArgs g) {
  using namespace gemm_detail;
  const long long n = static_cast<long long>(g.M) * g.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(i / g.N), col = static_cast<int>(i % g.N);
    float o = 0.f;
    for (int z = 0; z < nz; ++z) o += part[(static_cast<long long>(z) * g.M + row) * g.N + col];
    if (g.epi == EPI_BIAS_ACT) o = act_f(o + __ldg(g.bias + col), g.act);
    else if (g.epi == EPI_DACT) o *= dact_from_y(__ldg(g.Y + (long long)row * g.ldy + col), g.act);
    else o *= g.alpha;
    g.C[(long long)row * g.ldc + col] = o;
    if (g.CT) g.CT[(long long)col * g.ldct + row] = o;
  }
}

// Out-of-place transpose: out[c][r] = in[r][c] (32×32 smem tiles).
static __global__ void transpose_kernel(float* __restrict__ out, const float* __restrict__ in, int rows,
                                 int cols, int ldin, int ldout) {
  __shared__ float t[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = blockIdx.y * 32 + i;
    t[i][threadIdx.x] = (r < rows && c < cols) ? in[(long long)r * ldin + c] : 0.f;
  }
  __syncthreads();
  const int r2 = blockIdx.y * 32 + threadIdx.x;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c2 = blockIdx.x * 32 + i;
    if (c2 < cols && r2 < rows) out[(long long)c2 * ldout + r2] = t[threadIdx.x][i];
  }
}

// Vectorised out-of-place transpose (64×64 tiles, float4 loads and stores):
// the per-round Wᵀ of the 4096-wide layer; needs 16-B aligned rows.
static __global__ void __launch_bounds__(256) transpose4_kernel(float* __restrict__ out,
                                                                const float* __restrict__ in, int rows,
                                                                int cols, int ldin, int ldout) {
  __shared__ float t[64][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  for (int i = ty; i < 64; i += 16) {
    const int r = r0 + i, c = c0 + 4 * tx;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < rows) {
      const float* p = in + (long long)r * ldin + c;
      if (c + 3 < cols) {
        v = __ldg(reinterpret_cast<const float4*>(p));
      } else {
        if (c < cols) v.x = p[0];
        if (c + 1 < cols) v.y = p[1];
        if (c + 2 < cols) v.z = p[2];
      }
    }
    t[i][4 * tx] = v.x;
    t[i][4 * tx + 1] = v.y;
    t[i][4 * tx + 2] = v.z;
    t[i][4 * tx + 3] = v.w;
  }
  __syncthreads();
  for (int i = ty; i < 64; i += 16) {
    const int c = c0 + i, r = r0 + 4 * tx;
    if (c >= cols) continue;
    const float4 v = make_float4(t[4 * tx][i], t[4 * tx + 1][i], t[4 * tx + 2][i], t[4 * tx + 3][i]);
    float* p = out + (long long)c * ldout + r;
    if (r + 3 < rows) {
      *reinterpret_cast<float4*>(p) = v;
    } else {
      if (r < rows) p[0] = v.x;
      if (r + 1 < rows) p[1] = v.y;
      if (r + 2 < rows) p[2] = v.z;
    }
  }
}

}  // namespace ghc
