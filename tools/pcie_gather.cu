// pcie_gather.cu — zero-copy gather of shuffled 256-B dataset rows from
// pinned host memory, the e2e bench's access pattern (lstm_round.cuh
// fetch_rows): 128 CTAs x 8 warps, one row per warp per round, the next
// round's row requested one round ahead, a busy loop of `work_ns` standing
// in for the round's compute.  Variants of the copy:
//   0: 4-B cp.async per lane (the kernel's: 50 x + 1 label element, + the
//      4-B index of the round after next)
//   1: 16-B cp.async.cg, 16 lanes per 256-B row (+ the 4-B index)
//   2: variant 1 with the indices of all rounds in device memory
// Prints µs per round for each (variant, work_ns).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_gather tools/pcie_gather.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void cp4(void* d, const void* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void cp16(void* d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256, 1) gather(const float* rows, const int* idx, int rounds, int B, int variant,
                                                 long long work_ns, float* sink) {
  __shared__ __align__(16) float buf[8][2][64];
  __shared__ int sidx[8][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * 8 + warp;
  if (s >= B) return;
  auto fetch_row = [&](int row, int b) {
    const float* src = rows + (long long)row * 64;
    if (variant == 0) {
      cp4(&buf[warp][b][lane], src + lane);
      if (lane < 18) cp4(&buf[warp][b][32 + lane], src + 32 + lane);
      if (lane == 0) cp4(&buf[warp][b][50], src + 50);
    } else {
      if (lane < 16) cp16(&buf[warp][b][4 * lane], src + 4 * lane);
    }
  };
  // prologue: round 0's row, round 1's index
  fetch_row(__ldg(idx + s), 0);
  if (lane == 0) cp4(&sidx[warp][1], idx + (long long)B + s);
  commit();
  float acc = 0.f;
  for (int r = 0; r < rounds; ++r) {
    wait_all();
    __syncwarp();
    if (r + 1 < rounds) {
      const int row = sidx[warp][1];  // fetched a round earlier
      __syncwarp();
      fetch_row(row, (r + 1) & 1);
      if (lane == 0 && r + 2 < rounds) cp4(&sidx[warp][1], idx + (long long)(r + 2) * B + s);
      commit();
    }
    acc += buf[warp][r & 1][lane] + buf[warp][r & 1][50];
    const unsigned long long t0 = gt();
    while ((long long)(gt() - t0) < work_ns) {
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int B = 1000, rounds = 400;
  const long long nrows = 182000000ll / 256;  // the e2e dataset: 182 MB of packed rows
  float* hrows;
  int* hidx;
  CK(cudaHostAlloc(&hrows, nrows * 256, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hidx, (size_t)rounds * B * 4, cudaHostAllocMapped));
  for (long long i = 0; i < nrows * 64; ++i) hrows[i] = (float)(i & 1023);
  srand(1);
  for (long long i = 0; i < (long long)rounds * B; ++i) hidx[i] = (int)(((long long)rand() * 7919 + rand()) % nrows);
  int* didx;
  CK(cudaMalloc(&didx, (size_t)rounds * B * 4));
  CK(cudaMemcpy(didx, hidx, (size_t)rounds * B * 4, cudaMemcpyHostToDevice));
  float *drows, *sink;
  CK(cudaHostGetDevicePointer(&drows, hrows, 0));
  int* hidx_d;
  CK(cudaHostGetDevicePointer(&hidx_d, hidx, 0));
  CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"rows\": %d, \"row_bytes\": 256, \"results\": [", B);
  bool first = true;
  for (int variant = 0; variant < 3; ++variant)
    for (long long w : {0ll, 4000ll, 8000ll, 10000ll, 11000ll, 12000ll}) {
      const int* ip = variant == 2 ? didx : hidx_d;
      gather<<<125, 256>>>(drows, ip, 20, B, variant, w, sink);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      gather<<<125, 256>>>(drows, ip, rounds, B, variant, w, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s{\"variant\": %d, \"work_ns\": %lld, \"us_per_round\": %.3f, \"GBps\": %.1f}", first ? "" : ", ",
             variant, w, 1e3 * ms / rounds, (double)B * 260 * rounds / (ms * 1e-3) / 1e9);
      first = false;
    }
  printf("]}\n");
}
