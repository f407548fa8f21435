// pcie_latency.cu — latency of zero-copy loads from pinned host memory as the
// round kernel's prologue sees them: one warp per sample (125 CTAs x 8
// warps), each reading its 4-B gather index and then its 256-B row, on pages
// the GPU has not touched since the allocation / since the last launch.
// %globaltimer per warp: index load, then row load (dependent).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_latency tools/pcie_latency.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe(const float* rows, const int* idx, int B, int nwarps_active, unsigned long long* out, float* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * 8 + warp;
  if (s >= nwarps_active) return;
  const unsigned long long t0 = gt();
  int r;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(idx + s) : "memory");
  const unsigned long long t1 = gt() + (r & 0) ;
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(rows + (long long)r * 64 + lane) : "memory");
  const unsigned long long t2 = gt() + (__float_as_uint(v) & 0);
  if (lane == 0) {
    out[3 * s] = t0;
    out[3 * s + 1] = t1;
    out[3 * s + 2] = t2;
  }
  if (v == 12345.f) sink[0] = v;
}

int main() {
  const int B = 1000;
  const long long nrows = 182000000ll / 256;
  float* hrows;
  int* hidx;
  CK(cudaHostAlloc(&hrows, nrows * 256, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hidx, 64 * B * 4, cudaHostAllocMapped));
  for (long long i = 0; i < nrows * 64; i += 1024) hrows[i] = 1.f;
  srand(3);
  for (int i = 0; i < 64 * B; ++i) hidx[i] = (int)(((long long)rand() * 7919 + rand()) % nrows);
  float *drows, *sink;
  int* didx;
  CK(cudaHostGetDevicePointer(&drows, hrows, 0));
  CK(cudaHostGetDevicePointer(&didx, hidx, 0));
  unsigned long long *dout, *hout;
  CK(cudaMalloc(&dout, 3 * B * 8));
  CK(cudaMalloc(&sink, 4));
  hout = (unsigned long long*)malloc(3 * B * 8);
  printf("[");
  int k = 0;
  for (int active : {1, 1000})
    for (int rep = 0; rep < 4; ++rep) {
      // rep 0: indices / rows never touched; rep 1: same indices again;
      // rep 2, 3: fresh index block (other rows) in a new launch
      const int blk = rep == 1 ? 2 * k : 2 * k + rep;
      probe<<<125, 256>>>(drows, didx + (blk % 64) * B, B, active, dout, sink);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hout, dout, 3 * B * 8, cudaMemcpyDeviceToHost));
      std::vector<double> a, b, c;
      unsigned long long tmin = ~0ull;
      for (int s = 0; s < active; ++s) tmin = std::min(tmin, hout[3 * s]);
      for (int s = 0; s < active; ++s) {
        a.push_back((hout[3 * s + 1] - hout[3 * s]) / 1e3);
        b.push_back((hout[3 * s + 2] - hout[3 * s + 1]) / 1e3);
        c.push_back((hout[3 * s + 2] - tmin) / 1e3);
      }
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      std::sort(c.begin(), c.end());
      printf("%s{\"warps\": %d, \"rep\": %d, \"idx_us_med\": %.2f, \"idx_us_max\": %.2f, \"row_us_med\": %.2f, "
             "\"row_us_max\": %.2f, \"all_done_us\": %.2f}\n",
             k ? ", " : "", active, rep, a[a.size() / 2], a.back(), b[b.size() / 2], b.back(), c.back());
      ++k;
    }
  printf("]\n");
}
