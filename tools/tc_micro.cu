// tc_micro.cu — isolates the loops of lstm_tc.cuh on one CTA (8 warps) and
// times each warp with clock64: the weight-gradient tile rows (with and
// without their shared-memory operand loads) and the forward recurrence step
// (with/without the named barrier).  Ground truth for DESIGN.md §4.
#include <cstdio>
#include <cstdint>

#include "../paper_1712_05878_b200/csrc/lstm_tc.cuh"

using namespace ghc;
using L = TcLayout<5, 20, 10, 3, 4>;
constexpr int T = 10, S = 8, H = 20, KS = L::KS, RSA = L::RSA, RSD = L::RSD;

template <int MODE>
__global__ void wgrad_bench(float* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) float sm[];
  float* AF = sm;
  float* DZ = sm + (T + 1) * S * RSA;
  for (int i = threadIdx.x; i < (T + 1) * S * RSA + T * S * RSD; i += blockDim.x)
    sm[i] = __uint_as_float(tf32_rna(1.0f + 1e-3f * (i % 97)));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  float res = 0.f;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    const int nt_count = warp < 4 ? 4 : 1;
    const int mt2 = warp < 4 ? warp : 4;
    const int nt0 = warp < 4 ? 0 : warp - 4;
    float acc[4][4];
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) acc[j][i] = 0.f;
    const int o0 = L::frag_off(16 * mt2 + g), o1 = L::frag_off(16 * mt2 + g + 8);
    if (MODE == 0) {  // as in the kernel: loads inside the t loop
#pragma unroll 2
      for (int t = 0; t < T; ++t) {
        const float* d0 = DZ + (t * S + c) * RSD;
        const float* d1 = d0 + 4 * RSD;
        const uint32_t ah2[4] = {__float_as_uint(d0[o0]), __float_as_uint(d0[o1]), __float_as_uint(d1[o0]),
                                 __float_as_uint(d1[o1])};
        const uint32_t al2[4] = {__float_as_uint(d0[o0 + 2]), __float_as_uint(d0[o1 + 2]),
                                 __float_as_uint(d1[o0 + 2]), __float_as_uint(d1[o1 + 2])};
        const float* b0 = AF + (t * S + c) * RSA;
        const float* b1 = b0 + 4 * RSA;
        if (nt_count == 4) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ob = L::frag_off(8 * j + g);
            mma3(acc[j], ah2, al2, make_float4(b0[ob], b1[ob], b0[ob + 2], b1[ob + 2]));
          }
        } else {
          const int ob = L::frag_off(8 * nt0 + g);
          mma3(acc[0], ah2, al2, make_float4(b0[ob], b1[ob], b0[ob + 2], b1[ob + 2]));
        }
      }
    } else {  // MODE 1: same HMMA sequence, operands from registers only
      uint32_t ah2[4] = {(uint32_t)lane, 1u, 2u, 3u}, al2[4] = {4u, 5u, 6u, (uint32_t)rep};
      float4 bb = make_float4(1.f, 2.f, 3.f, 4.f);
#pragma unroll 2
      for (int t = 0; t < T; ++t) {
        if (nt_count == 4) {
#pragma unroll
          for (int j = 0; j < 4; ++j) mma3(acc[j], ah2, al2, bb);
        } else {
          mma3(acc[0], ah2, al2, bb);
        }
      }
    }
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) res += acc[j][i];
  }
  long long t1 = clock64();
  out[threadIdx.x] = res;
  if (lane == 0) cyc[warp] = (t1 - t0) / reps;
}

// forward recurrence of lstm_round_tc_kernel (5 warps), optional named barrier
template <bool BAR>
__global__ void fwd_bench(float* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) float sm[];
  float* AF = sm;
  float* cache = sm + (T + 1) * S * RSA;
  for (int i = threadIdx.x; i < (T + 1) * S * RSA; i += blockDim.x) sm[i] = 0.01f * (i % 7);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  if (warp >= L::MTF) return;
  uint32_t ah[KS][4], al[KS][4];
  for (int ks = 0; ks < KS; ++ks)
    for (int i = 0; i < 4; ++i) {
      ah[ks][i] = tf32_rna(0.1f * (i + ks));
      al[ks][i] = tf32_rna(1e-4f * lane);
    }
  const int q = g & 3;
  const int uu = 4 * warp + (g >> 2) + 2 * (q >> 1);
  const int ss = 2 * c + (q & 1);
  long long t0 = clock64();
  float cst = 0.f;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      float acc[KS][4];
      const float4* brow = reinterpret_cast<const float4*>(AF + (t * S + g) * RSA) + c;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[ks][i] = 0.0f;
        mma3(acc[ks], ah[ks], al[ks], brow[4 * ks]);
      }
      float e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        e[i] = acc[0][i];
#pragma unroll
        for (int ks = 1; ks < KS; ++ks) e[i] += acc[ks][i];
      }
      transpose4(e, q);
      const float ig = sigmoid_f(e[0]), fg = sigmoid_f(e[1]), gg = tanh_f(e[2]), og = sigmoid_f(e[3]);
      cst = fmaf(fg, cst, ig * gg);
      const float tc = tanh_f(cst);
      float* ct = cache + ((t * H + uu) * S + ss) * 8;
      reinterpret_cast<float4*>(ct)[0] = make_float4(ig, fg, gg, og);
      reinterpret_cast<float2*>(ct)[2] = make_float2(cst, tc);
      put_split(AF + ((t + 1) * S + ss) * RSA, L::frag_off(uu), og * tc);
      if (BAR) named_bar(1, 32 * L::MTF);
      else __syncwarp();
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = cst;
  if (lane == 0) cyc[warp] = (t1 - t0) / (reps * T);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8 * sizeof(long long));
  long long h[8];
  const int smem = 200 * 1024;
  auto run = [&](const char* name, void (*k)(float*, long long*, int), int threads) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(cyc, 0, 8 * sizeof(long long));
    k<<<1, threads, smem>>>(out, cyc, 50);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    std::printf("%-34s", name);
    for (int w = 0; w < 8; ++w) std::printf(" %6lld", h[w]);
    std::printf("   (cycles per warp)\n");
  };
  run("wgrad rows, smem operands", wgrad_bench<0>, 256);
  run("wgrad rows, register operands", wgrad_bench<1>, 256);
  run("forward step, named barrier", fwd_bench<true>, 256);
  run("forward step, no barrier", fwd_bench<false>, 256);
  cudaError_t e = cudaGetLastError();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
