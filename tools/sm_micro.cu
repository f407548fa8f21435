// sm_micro.cu — per-SM pipe throughput probes for the fused round kernel's
// inner loops (one CTA on one SM, `warps` warps, clock64 around a loop):
//   lds128_bcast  LDS.128, every lane the same address (the dz / h broadcast)
//   lds128_dist   LDS.128, lane-distinct conflict-free addresses
//   lds32_bcast   LDS.32 broadcast
//   shfl          SHFL.IDX
//   ffma2         independent FFMA2 chains
//   ffma          independent FFMA chains
//   mufu_ex2      MUFU.EX2
// Prints cycles per warp-instruction per SM (i.e. the SM-wide cost).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_micro tools/sm_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;

template <int MODE>
__global__ void probe(float* out, long long* cyc) {
  __shared__ __align__(16) float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i < 8 ? __int_as_float((i * 5 + 3) & 7) : 1.0f + 1e-7f * i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float4(lane, 1, 2, 3);
  float2 a2[8];
  for (int i = 0; i < 8; ++i) a2[i] = make_float2(lane, i);
  const float4* p4 = reinterpret_cast<const float4*>(sm);
  int off = (threadIdx.x >> 5) * 8;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
    if constexpr (MODE == 0) {  // LDS.128 broadcast: 8 loads / iter
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 u = p4[(off + i + it) & 1023];
        acc[i].x += u.x;
        acc[i].y += u.y;
        acc[i].z += u.z;
        acc[i].w += u.w;
      }
    } else if constexpr (MODE == 1) {  // LDS.128 lane-distinct
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 u = p4[(lane + 32 * i + it) & 1023];
        acc[i].x += u.x;
        acc[i].y += u.y;
        acc[i].z += u.z;
        acc[i].w += u.w;
      }
    } else if constexpr (MODE == 2) {  // LDS.32 broadcast
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i].x += sm[(off + i + it) & 4095];
    } else if constexpr (MODE == 3) {  // SHFL
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i].x += __shfl_sync(0xffffffffu, acc[(i + 1) & 7].y, (it + i) & 31);
    } else if constexpr (MODE == 4) {  // FFMA2
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) a2[i] = __ffma2_rn(a2[i], make_float2(1.0000001f, 0.9999999f), make_float2(1e-9f, 2e-9f));
    } else if constexpr (MODE == 5) {  // FFMA
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i].x = fmaf(acc[i].x, 1.0000001f, 1e-9f);
    } else if constexpr (MODE == 6) {  // MUFU.EX2
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(acc[i].x));
        acc[i].x = y * 0.5f;
      }
    } else if constexpr (MODE == 7) {  // latency: dependent FFMA
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[0].x = fmaf(acc[0].x, 1.0000001f, 1e-9f);
    } else if constexpr (MODE == 8) {  // latency: dependent FFMA2
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[0] = __ffma2_rn(a2[0], make_float2(1.0000001f, 0.9999999f), make_float2(1e-9f, 2e-9f));
    } else if constexpr (MODE == 9) {  // latency: dependent MUFU.EX2
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(acc[0].x));
    } else if constexpr (MODE == 10) {  // latency: dependent MUFU.RCP
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(acc[0].x));
    } else if constexpr (MODE == 11) {  // latency: dependent SHFL
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[0].x = __shfl_xor_sync(0xffffffffu, acc[0].x, 1 + (i & 3));
    } else if constexpr (MODE == 12) {  // latency: dependent LDS (pointer chase)
#pragma unroll
      for (int i = 0; i < 8; ++i) off = __float_as_int(sm[off & 4095]) & 7;
    } else {  // latency: STS -> __syncwarp -> LDS of another lane's value
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        sm[2048 + lane] = acc[0].x;
        __syncwarp();
        acc[0].x = sm[2048 + ((lane + 1) & 31)] + 1.0f;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = (float)off;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y + acc[i].z + acc[i].w + a2[i].x + a2[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int per_iter) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  for (int w : {1, 2, 4, 8}) {
    probe<MODE><<<1, 32 * w>>>(out, cyc);
    probe<MODE><<<1, 32 * w>>>(out, cyc);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double per = (double)c / ((double)kIters * per_iter * w);
    printf("%-14s warps=%d  SM cycles per warp-instr %.2f  (per warp %.2f)\n", name, w, per, per * w);
  }
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("lds128_bcast", 8);
  run<1>("lds128_dist", 8);
  run<2>("lds32_bcast", 8);
  run<3>("shfl", 8);
  run<4>("ffma2", 32);
  run<5>("ffma", 32);
  run<6>("mufu_ex2", 8);
  run<7>("lat_ffma", 8);
  run<8>("lat_ffma2", 8);
  run<9>("lat_ex2", 8);
  run<10>("lat_rcp", 8);
  run<11>("lat_shfl", 8);
  run<12>("lat_lds", 8);
  run<13>("lat_sts_lds", 8);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
