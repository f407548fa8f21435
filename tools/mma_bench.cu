// mma_bench.cu — micro-benchmark of the legacy warp-level tensor path on
// sm_100a (mma.sync m16n8k8 tf32 / m16n8k16 bf16): dependent-chain latency
// and per-SM-sub-partition issue throughput.  Used to size the CTA-cooperative
// LSTM recurrence.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CHAINS, bool BF16>
__global__ void bench(int iters, float* out, long long* cyc) {
  float d[CHAINS][4];
  for (int c = 0; c < CHAINS; ++c)
    for (int i = 0; i < 4; ++i) d[c][i] = 0.f;
  const uint32_t a = __float_as_uint(1.0f + threadIdx.x * 1e-7f), b = __float_as_uint(0.5f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (BF16) mma_bf16(d[c], a, a, a, a, b, b);
      else mma_tf32(d[c], a, a, a, a, b, b);
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma_bench(int iters, float* out, long long* cyc) {
  float d[8];
  for (int i = 0; i < 8; ++i) d[i] = threadIdx.x;
  const float x = 1.0001f, y = 0.9999f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = fmaf(d[i], x, y);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char* name, F kern, int warps, int iters, int per_iter, float* out, long long* cyc) {
  kern<<<1, 32 * warps>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per = (double)c / ((double)iters * per_iter);
  std::printf("%-28s warps=%2d  cycles/instr/warp=%7.2f  => SM-wide instr/clk=%.3f\n", name, warps,
              per, warps / per);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 12);
  const int it = 4096;
  for (int w : {1, 4, 8, 16}) {
    run("tf32 m16n8k8 chain=1", bench<1, false>, w, it, 1, out, cyc);
    run("tf32 m16n8k8 chain=4", bench<4, false>, w, it, 4, out, cyc);
    run("tf32 m16n8k8 chain=8", bench<8, false>, w, it, 8, out, cyc);
    run("bf16 m16n8k16 chain=1", bench<1, true>, w, it, 1, out, cyc);
    run("bf16 m16n8k16 chain=8", bench<8, true>, w, it, 8, out, cyc);
    run("ffma chain=8", ffma_bench, w, it, 8, out, cyc);
  }
  cudaError_t e = cudaGetLastError();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
