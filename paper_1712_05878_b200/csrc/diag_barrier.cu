// diag_barrier.cu — micro-benchmark of grid-wide barrier implementations for
// the persistent round loop (diagnostics only; informs DESIGN.md §Sync).
//   impl 0: atomic counter + generation word (grid_barrier, ghc_device.cuh)
//   impl 1: gather/broadcast flags (flag_barrier, lstm_step.cuh)
//   impl 2: all-poll-all: every CTA polls every CTA's padded flag (relaxed)
//   impl 3: cluster barrier only (barrier.cluster; cluster of 8) — lower bound
#include "ghc_internal.cuh"

using namespace ghc;

namespace {

__device__ __forceinline__ void barrier_allpoll(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * kFlagStride, epoch);
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    while ((int)(ld_relaxed_gpu(flags + b * kFlagStride) - epoch) < 0) {
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncthreads();
}

// impl 4: all-poll, no fences (relaxed signalling floor; NOT a valid barrier)
__device__ __forceinline__ void barrier_nofence(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * kFlagStride), "r"(epoch) : "memory");
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    while ((int)(ld_relaxed_gpu(flags + b * kFlagStride) - epoch) < 0) {
    }
  __syncthreads();
}
// impl 5: column barrier: only the CTAs with equal blockIdx % 8 (16-18 CTAs)
__device__ __forceinline__ void barrier_column(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * kFlagStride, epoch);
  const int col = blockIdx.x & 7, ncol = (gridDim.x - col + 7) / 8;
  if (threadIdx.x < ncol) {
    const int b = col + 8 * threadIdx.x;
    while ((int)(ld_relaxed_gpu(flags + b * kFlagStride) - epoch) < 0) {
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// impl 6: all-poll with acquire loads (no trailing fence)
__device__ __forceinline__ void barrier_acqpoll(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * kFlagStride, epoch);
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + b * kFlagStride) : "memory");
    } while ((int)(v - epoch) < 0);
  }
  __syncthreads();
}

__global__ void barrier_bench_kernel(int impl, int iters, MasterDev* ms, unsigned* bar,
                                     unsigned long long* out) {
  unsigned epoch = bar[0];
  __syncthreads();
  const unsigned long long t0 = globaltimer();
  for (int i = 0; i < iters; ++i) {
    if (impl == 0) grid_barrier(ms);
    else if (impl == 1) flag_barrier(bar, ++epoch, 0);
    else if (impl == 2) barrier_allpoll(bar + 2 * kFlagStride, ++epoch);
    else if (impl == 4) barrier_nofence(bar + 2 * kFlagStride, ++epoch);
    else if (impl == 5) barrier_column(bar + 2 * kFlagStride, ++epoch);
    else if (impl == 6) barrier_acqpoll(bar + 2 * kFlagStride, ++epoch);
    else asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  const unsigned long long t1 = globaltimer();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (blockIdx.x == 0 && threadIdx.x == 0) bar[0] = epoch;
}

}  // namespace

extern "C" ghc_status ghc_diag_barrier_bench(ghc_ctx* c, int32_t impl, int32_t ctas,
                                             int32_t threads, int32_t iters, double* ns_per) {
  MasterDev* ms = nullptr;
  unsigned* bar = nullptr;
  unsigned long long* out = nullptr;
  CU(cudaSetDevice(c->device));
  CU(cudaMalloc(&ms, sizeof(MasterDev)));
  CU(cudaMemset(ms, 0, sizeof(MasterDev)));
  const size_t bar_bytes = sizeof(unsigned) * 32 * (2 + static_cast<size_t>(ctas));
  CU(cudaMalloc(&bar, bar_bytes));
  CU(cudaMemset(bar, 0, bar_bytes));
  CU(cudaMalloc(&out, sizeof(unsigned long long) * ctas));
  CU(cudaDeviceSynchronize());  // memsets (legacy stream) before the launch on ctx->stream
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeCooperative;
  attr[na].val.cooperative = 1;
  ++na;
  if (impl == 3) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 8;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  for (int rep = 0; rep < 2; ++rep)  // warm-up, then measured
    CU(cudaLaunchKernelEx(&cfg, barrier_bench_kernel, (int)impl, (int)iters, ms, bar, out));
  CU(cudaStreamSynchronize(c->stream));
  std::vector<unsigned long long> h(static_cast<size_t>(ctas));
  CU(cudaMemcpy(h.data(), out, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost));
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  *ns_per = static_cast<double>(mx) / iters;
  cudaFree(ms);
  cudaFree(bar);
  cudaFree(out);
  return GHC_OK;
}
