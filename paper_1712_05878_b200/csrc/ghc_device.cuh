// ghc_device.cuh — device-side building blocks shared by the sm_100a kernels:
// device-resident master state, a grid barrier for persistent (cooperatively
// launched) kernels, fast activations and warp reductions.
#pragma once

#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

// Checked build (build.py --checked → _build_checked/libghc.so, -DGHC_CHECKED):
// the index arithmetic of every shared-memory region and tagged L2 row is
// asserted at its use — an access past its own region (into a neighbouring
// buffer of the same CTA, which the hardware cannot flag) traps with the
// source line instead of corrupting state.  The sanitizer stand-in on a pool
// where compute-sanitizer is closed; the product build
// compiles the checks away.
#ifdef GHC_CHECKED
#define GHC_CHECK(c)                                                                             \
  do {                                                                                           \
    if (!(c)) {                                                                                  \
      printf("GHC_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c,       \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define GHC_CHECK(c) \
  do {               \
  } while (0)
#endif
// [p, p + n) lies inside [base, base + size)   (element pointers of one type)
#define GHC_CHECK_RANGE(p, n, base, size) \
  GHC_CHECK((p) >= (base) && (p) + (n) <= (base) + (size))

namespace ghc {

// Device-resident master state (one per ghc_master / per fused launch).
// Lives in HBM so that commit/reject decisions never need a host sync.
struct MasterDev {
  unsigned bar_count;          // grid-barrier arrivals
  unsigned bar_gen;            // grid-barrier generation
  int cur;                     // which of the double-buffered w/v is current
  int status;                  // last round: 0 = accepted, GHC_ERR_NONFINITE = rejected
  unsigned long long version;  // accepted master updates (optim.cpp:63)
  unsigned long long rejected; // rejected (non-finite) updates
  unsigned long long round;    // rounds run so far (flag parity)
  int flag[2];                 // per-round non-finite flags (parity round & 1)
  unsigned arrive;             // last-CTA-done counter (single-barrier kernels)
  int pad_;
  unsigned long long samples;  // samples of the accepted rounds (run stats)
};

// Sense-free generation barrier across all CTAs of a cooperative launch.
// Thread 0 of each CTA arrives on a device-scope counter (release), the last
// arriver bumps the generation, the others spin (acquire).  Loads of data
// written by other CTAs after the barrier use ld.global.cg (__ldcg) so no
// stale L1 line can be observed.
__device__ __forceinline__ void grid_barrier(MasterDev* ms) {
  __syncthreads();
  if (threadIdx.x == 0) {
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> gen(ms->bar_gen);
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(ms->bar_count);
    const unsigned g = gen.load(cuda::memory_order_relaxed);
    __threadfence();
    const unsigned arrived = cnt.fetch_add(1u, cuda::memory_order_acq_rel);
    if (arrived == gridDim.x - 1) {
      cnt.store(0u, cuda::memory_order_relaxed);
      gen.store(g + 1u, cuda::memory_order_release);
    } else {
      while (gen.load(cuda::memory_order_acquire) == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// sigmoid / tanh as branch-free MUFU sequences: ex2.approx.ftz + rcp.approx.ftz
// (each ≤ 2 ulp).  The IEEE __frcp_rn path compiles to a branch + CALL per
// reciprocal (BSSY/BSYNC), which serialises the four gate activations; these
// are 4-5 instructions with no control flow, abs error ≲ 3e-7 — well inside
// the fp32 parity budget (the reference uses libm exp/tanh, nn.cpp:15-19).
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigmoid_f(float x) {
  return rcp_approx(1.0f + ex2_approx(-1.4426950408889634f * x));
}
__device__ __forceinline__ float tanh_f(float x) {
  return 1.0f - 2.0f * rcp_approx(ex2_approx(2.8853900817779268f * x) + 1.0f);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// cp.async (LDGSTS): 4-byte global → shared copies that complete
// asynchronously; the issuing thread waits with cp_async_wait<N>() (at most N
// newest groups still pending) and a __syncwarp publishes them to the warp.
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool is_finite_f(float v) { return isfinite(v); }

}  // namespace ghc
