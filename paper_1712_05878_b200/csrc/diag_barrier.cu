// diag_barrier.cu — micro-benchmark of grid-wide barrier implementations for
// the persistent round loop (diagnostics only; informs DESIGN.md §Sync).
//   impl 0: atomic counter + generation word (grid_barrier, ghc_device.cuh)
//   impl 1: gather/broadcast flags (flag_barrier, lstm_step.cuh)
//   impl 2: all-poll-all: every CTA polls every CTA's padded flag (relaxed)
//   impl 3: cluster barrier only (barrier.cluster; cluster of 8) — lower bound
#include <algorithm>

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

// ---------------------------------------------------------------------------
// Launch cost of the round kernel's launch configuration, piece by piece
// (diagnostics for the fixed per-call cost): an empty kernel
// of `ctas` × `threads` with the flags of `variant` — bit 0: cooperative,
// bit 1: clusters of 4, bit 2: `smem` bytes of dynamic shared memory.
// us_single: median CUDA-event time of one launch queued behind a gate
// (device-side launch + teardown only); us_b2b: per launch over 200
// back-to-back launches.
namespace {
__global__ void empty_kernel(int* sink) {
  if (sink && threadIdx.x == 0 && blockIdx.x == 0) *sink = 1;
}
}  // namespace

extern "C" ghc_status ghc_diag_launch_bench(ghc_ctx* c, int32_t variant, int32_t ctas, int32_t threads,
                                            int32_t smem, double* us_single, double* us_b2b) {
  CU(cudaSetDevice(c->device));
  if (variant & 4)
    CU(cudaFuncSetAttribute(reinterpret_cast<const void*>(empty_kernel),
                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = (variant & 4) ? smem : 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (variant & 1) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (variant & 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 4;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  int* sink = nullptr;
  CU(cudaLaunchKernelEx(&cfg, empty_kernel, sink));  // warm-up
  CU(cudaStreamSynchronize(c->stream));
  std::vector<float> t;
  for (int i = 0; i < 21; ++i) {
    if (ghc_status s = ghc_stream_hold(c)) return s;
    CU(cudaEventRecord(c->ev0, c->stream));
    CU(cudaLaunchKernelEx(&cfg, empty_kernel, sink));
    CU(cudaEventRecord(c->ev1, c->stream));
    if (ghc_status s = ghc_stream_release(c)) return s;
    CU(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  *us_single = 1e3 * t[t.size() / 2];
  if (ghc_status s = ghc_stream_hold(c)) return s;
  CU(cudaEventRecord(c->ev0, c->stream));
  for (int i = 0; i < 200; ++i) CU(cudaLaunchKernelEx(&cfg, empty_kernel, sink));
  CU(cudaEventRecord(c->ev1, c->stream));
  if (ghc_status s = ghc_stream_release(c)) return s;
  CU(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  *us_b2b = 1e3 * ms / 200;
  return GHC_OK;
}
