// update_kernels.cuh — the master update path (optim.cpp) as HBM-bound sm_100a
// kernels: float4-vectorised, grid-stride, one CTA wave sized to the SM count.
//
//   sgd_apply       optim.cpp:39-65 + all_finite tensor.cpp:29-36
//                   (20 B/param: read w, v, g; write w, v)
//   easgd_worker    optim.cpp:82-105 (12 B/param, +12 on pull batches)
//   easgd_center    optim.cpp:107-123 (12 B/param)
//   elastic_pull    optim.cpp:67-80   (12 B/param)
//   weighted_mean   SPEC.md:358-366 sync combine ((W+1)·4 B/param)
//
// Whole-update rejection without a host sync: the kernels that must reject a
// non-finite gradient run as cooperative launches — phase A checks g
// (warp-shuffle/`__syncthreads_or` reduce → one device flag), a grid barrier,
// phase B applies the update only if the flag is clear; g is re-read in phase
// B through L2 (evict-last hint in phase A), so DRAM traffic stays ≈20 B/param.
#pragma once

#include "ghc_device.cuh"

namespace ghc {

// Load that asks L2 to keep the line (evict_last policy): g is re-read in
// phase B of the rejecting kernels.
__device__ __forceinline__ float4 ld_g4_keep(const float4* p) {
  float4 r;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ bool finite4(float4 v) {
  return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
}

// Phase A of the rejecting kernels: any non-finite g → ms->flag[0].
__device__ __forceinline__ int check_finite_all(const float* g, long long P, int vec,
                                                MasterDev* ms) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long n4 = vec ? (P >> 2) : 0;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  int bad = 0;
  for (long long i = tid; i < n4; i += nth) bad |= !finite4(ld_g4_keep(g4 + i));
  for (long long i = (n4 << 2) + tid; i < P; i += nth) bad |= !isfinite(g[i]);
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(&ms->flag[0], 1);
  grid_barrier(ms);
  return __ldcg(&ms->flag[0]);
}

// Last CTA out resets the flag and publishes status / version.
__device__ __forceinline__ void finish_rejecting(MasterDev* ms, int rej, int* status,
                                                 unsigned long long* version,
                                                 unsigned long long* rejected) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&ms->arrive, 1u);
    if (prev == gridDim.x - 1) {
      ms->arrive = 0;
      ms->flag[0] = 0;
      if (status) *status = rej ? 2 /*GHC_ERR_NONFINITE*/ : 0;
      if (version && !rej) *version += 1ull;
      if (rejected && rej) *rejected += 1ull;
      __threadfence();
    }
  }
}

static __global__ void __launch_bounds__(256) sgd_apply_kernel(float* __restrict__ w, float* __restrict__ v,
                                                        const float* __restrict__ g, long long P, int vec,
                                                        float lr, float mu, MasterDev* ms,
                                                        int* status, unsigned long long* version,
                                                        unsigned long long* rejected) {
  const int rej = check_finite_all(g, P, vec, ms);
  if (!rej) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long n4 = vec ? (P >> 2) : 0;
    float4* w4 = reinterpret_cast<float4*>(w);
    float4* v4 = reinterpret_cast<float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (long long i = tid; i < n4; i += nth) {
      const float4 gv = __ldcg(g4 + i);
      float4 vv = __ldcs(v4 + i);
      float4 wv = __ldcs(w4 + i);
      vv.x = fmaf(mu, vv.x, -lr * gv.x);
      vv.y = fmaf(mu, vv.y, -lr * gv.y);
      vv.z = fmaf(mu, vv.z, -lr * gv.z);
      vv.w = fmaf(mu, vv.w, -lr * gv.w);
      wv.x += vv.x;
      wv.y += vv.y;
      wv.z += vv.z;
      wv.w += vv.w;
      __stcs(v4 + i, vv);
      __stcs(w4 + i, wv);
    }
    for (long long i = (n4 << 2) + tid; i < P; i += nth) {
      const float vn = fmaf(mu, v[i], -lr * __ldcg(g + i));
      v[i] = vn;
      w[i] += vn;
    }
  }
  finish_rejecting(ms, rej, status, version, rejected);
}

// One streaming pass of sgd_step (optim.cpp:59-60) from (w, v, g) into
// (w2, v2): 20 B/param; returns this thread's "saw a non-finite g" bit.
__device__ __forceinline__ int sgd_pass(const float* __restrict__ w, const float* __restrict__ v,
                                        const float* __restrict__ g, float* __restrict__ w2,
                                        float* __restrict__ v2, long long P, int vec, float lr,
                                        float mu) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long n4 = vec ? (P >> 2) : 0;
  int bad = 0;
  for (long long i = tid; i < n4; i += nth) {
    const float4 gv = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 vv = __ldcs(reinterpret_cast<const float4*>(v) + i);
    float4 wv = __ldcs(reinterpret_cast<const float4*>(w) + i);
    bad |= !finite4(gv);
    vv.x = fmaf(mu, vv.x, -lr * gv.x);
    vv.y = fmaf(mu, vv.y, -lr * gv.y);
    vv.z = fmaf(mu, vv.z, -lr * gv.z);
    vv.w = fmaf(mu, vv.w, -lr * gv.w);
    wv.x += vv.x;
    wv.y += vv.y;
    wv.z += vv.z;
    wv.w += vv.w;
    __stcs(reinterpret_cast<float4*>(v2) + i, vv);
    __stcs(reinterpret_cast<float4*>(w2) + i, wv);
  }
  for (long long i = (n4 << 2) + tid; i < P; i += nth) {
    const float gi = g[i];
    bad |= !isfinite(gi);
    const float vn = fmaf(mu, v[i], -lr * gi);
    v2[i] = vn;
    w2[i] = w[i] + vn;
  }
  return bad;
}

// The grid's OR of the per-thread bad bits, seen by the last CTA to arrive
// (flags->flag[0] / arrive reset for the next launch); returns -1 in every
// other CTA, else the OR (0 / 1).  No grid barrier.
__device__ __forceinline__ int last_cta_or(int bad, MasterDev* flags) {
  bad = __syncthreads_or(bad);
  int res = -1;
  if (threadIdx.x == 0) {
    if (bad) atomicOr(&flags->flag[0], 1);
    __threadfence();
    const unsigned prev = atomicAdd(&flags->arrive, 1u);
    if (prev == gridDim.x - 1) {  // last CTA: every write and flag of the grid is visible
      __threadfence();
      res = atomicAdd(&flags->flag[0], 0) ? 1 : 0;
      flags->flag[0] = 0;
      flags->arrive = 0;
    }
  }
  return res;
}

// sgd_step with value semantics (the drop-in's `sgd_step(w, g, s)` returns
// new weights / state): (w, v, g) → (w2, v2) in one pass, 20 B/param — the
// in-place form has to see all of g before its first write (two passes).  A
// non-finite g sets *status = GHC_ERR_NONFINITE (w2, v2 then hold no update;
// the inputs were never written), else 0 and *version += 1.
static __global__ void __launch_bounds__(256) sgd_out_kernel(const float* __restrict__ w,
                                                      const float* __restrict__ v,
                                                      const float* __restrict__ g,
                                                      float* __restrict__ w2, float* __restrict__ v2,
                                                      long long P, int vec, float lr, float mu,
                                                      MasterDev* flags, int* status,
                                                      unsigned long long* version) {
  const int rej = last_cta_or(sgd_pass(w, v, g, w2, v2, P, vec, lr, mu), flags);
  if (rej >= 0) {
    if (status) *status = rej ? 2 /*GHC_ERR_NONFINITE*/ : 0;
    if (version && !rej) *version += 1ull;
    __threadfence();
  }
}

// easgd_worker_step with value semantics: w2 = w − lr·g, pulled toward c on
// pull rounds (optim.cpp:82-105), one pass (16 B/param on pull rounds).
static __global__ void __launch_bounds__(256) easgd_worker_out_kernel(
    const float* __restrict__ w, const float* __restrict__ c, const float* __restrict__ g,
    float* __restrict__ w2, long long P, int vec, float lr, float alpha, int pull, MasterDev* flags,
    int* status) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long n4 = vec ? (P >> 2) : 0;
  int bad = 0;
  for (long long i = tid; i < n4; i += nth) {
    const float4 gv = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 wv = __ldcs(reinterpret_cast<const float4*>(w) + i);
    bad |= !finite4(gv);
    wv.x -= lr * gv.x;  // optim.cpp:97-98
    wv.y -= lr * gv.y;
    wv.z -= lr * gv.z;
    wv.w -= lr * gv.w;
    if (pull) {  // optim.cpp:76
      const float4 cv = __ldcs(reinterpret_cast<const float4*>(c) + i);
      wv.x -= alpha * (wv.x - cv.x);
      wv.y -= alpha * (wv.y - cv.y);
      wv.z -= alpha * (wv.z - cv.z);
      wv.w -= alpha * (wv.w - cv.w);
    }
    __stcs(reinterpret_cast<float4*>(w2) + i, wv);
  }
  for (long long i = (n4 << 2) + tid; i < P; i += nth) {
    const float gi = g[i];
    bad |= !isfinite(gi);
    float wv = w[i] - lr * gi;
    if (pull) wv -= alpha * (wv - c[i]);
    w2[i] = wv;
  }
  const int rej = last_cta_or(bad, flags);
  if (rej >= 0 && status) {
    *status = rej ? 2 : 0;
    __threadfence();
  }
}

// sgd_step for the double-buffered master (optim.cpp:39-65) in ONE pass:
// read w, v, g of the current buffer, write the new w, v into the other one
// (20 B/param, the algorithmic minimum); the last CTA out commits by flipping
// ms->cur (version + 1) or rejects a non-finite gradient whole (optim.cpp:
// 49-51 — the current buffer was never written).  No grid barrier, no
// separate finite-check pass.  `flags` holds the cross-CTA bad flag and the
// arrival counter.
//
// det = 1 (the master paths that track the buffer index on the host): the
// buffers flip on EVERY call; a rejected update leaves flags->flag[1] = 1
// and db_fixup_kernel (launched right after) copies the old w, v into the new
// buffers — the rare path pays the copy, the common path stays one pass.
static __global__ void __launch_bounds__(256) sgd_db_kernel(float* const* __restrict__ wb,
                                                     float* const* __restrict__ vb,
                                                     const float* __restrict__ g, long long P,
                                                     int vec, float lr, float mu, MasterDev* ms,
                                                     MasterDev* flags, int det = 0) {
  const int cur = __ldcg(&ms->cur);
  int bad = sgd_pass(wb[cur], vb[cur], g, wb[cur ^ 1], vb[cur ^ 1], P, vec, lr, mu);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    if (bad) atomicOr(&flags->flag[0], 1);
    __threadfence();
    const unsigned prev = atomicAdd(&flags->arrive, 1u);
    if (prev == gridDim.x - 1) {  // last CTA: every write and flag of the grid is visible
      __threadfence();
      const int rej = atomicAdd(&flags->flag[0], 0);
      if (rej) {
        ms->rejected += 1ull;
        ms->status = 2;  // GHC_ERR_NONFINITE
        if (det) ms->cur = cur ^ 1;
      } else {
        ms->cur = cur ^ 1;
        ms->version += 1ull;
        ms->status = 0;
      }
      flags->flag[1] = det && rej;
      flags->flag[0] = 0;
      flags->arrive = 0;
      __threadfence();
    }
  }
}

// After a rejected det-mode sgd_db: the new current buffers get the old
// state (the update is rejected whole, optim.cpp:49-51).  Every CTA reads the
// same stream-ordered flag; the common (accepted) case returns at once.
static __global__ void __launch_bounds__(256) db_fixup_kernel(float* const* __restrict__ wb,
                                                       float* const* __restrict__ vb, long long P,
                                                       const MasterDev* ms, const MasterDev* flags) {
  if (!__ldcg(&flags->flag[1])) return;
  const int cur = __ldcg(&ms->cur);
  const float* w = wb[cur ^ 1];
  const float* v = vb[cur ^ 1];
  float* w2 = wb[cur];
  float* v2 = vb[cur];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x) {
    w2[i] = w[i];
    v2[i] = v[i];
  }
}

static __global__ void __launch_bounds__(256) easgd_worker_kernel(float* __restrict__ w,
                                                           const float* __restrict__ c,
                                                           const float* __restrict__ g,
                                                           long long P, int vec, float lr,
                                                           float alpha, int pull, MasterDev* ms,
                                                           int* status) {
  const int rej = check_finite_all(g, P, vec, ms);
  if (!rej) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long n4 = vec ? (P >> 2) : 0;
    float4* w4 = reinterpret_cast<float4*>(w);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const float4* c4 = reinterpret_cast<const float4*>(c);
    for (long long i = tid; i < n4; i += nth) {
      const float4 gv = __ldcg(g4 + i);
      float4 wv = __ldcs(w4 + i);
      wv.x -= lr * gv.x;  // optim.cpp:97-98
      wv.y -= lr * gv.y;
      wv.z -= lr * gv.z;
      wv.w -= lr * gv.w;
      if (pull) {  // optim.cpp:76
        const float4 cv = __ldcs(c4 + i);
        wv.x -= alpha * (wv.x - cv.x);
        wv.y -= alpha * (wv.y - cv.y);
        wv.z -= alpha * (wv.z - cv.z);
        wv.w -= alpha * (wv.w - cv.w);
      }
      __stcs(w4 + i, wv);
    }
    for (long long i = (n4 << 2) + tid; i < P; i += nth) {
      float wv = w[i] - lr * __ldcg(g + i);
      if (pull) wv -= alpha * (wv - c[i]);
      w[i] = wv;
    }
  }
  finish_rejecting(ms, rej, status, nullptr, nullptr);
}

// c += alpha*(w - c)  (optim.cpp:118) — also used for elastic_pull with the
// roles swapped: w -= alpha*(w - c)  ≡  w += alpha*(c - w).
static __global__ void __launch_bounds__(256) elastic_kernel(float* __restrict__ dst,
                                                      const float* __restrict__ src,
                                                      long long P, int vec, float alpha,
                                                      int pull, unsigned long long* version) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long n4 = vec ? (P >> 2) : 0;
  float4* d4 = reinterpret_cast<float4*>(dst);
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (long long i = tid; i < n4; i += nth) {
    float4 d = __ldcs(d4 + i);
    const float4 s = __ldcs(s4 + i);
    if (pull) {
      d.x -= alpha * (d.x - s.x);
      d.y -= alpha * (d.y - s.y);
      d.z -= alpha * (d.z - s.z);
      d.w -= alpha * (d.w - s.w);
    } else {
      d.x += alpha * (s.x - d.x);
      d.y += alpha * (s.y - d.y);
      d.z += alpha * (s.z - d.z);
      d.w += alpha * (s.w - d.w);
    }
    __stcs(d4 + i, d);
  }
  for (long long i = (n4 << 2) + tid; i < P; i += nth) {
    if (pull) dst[i] -= alpha * (dst[i] - src[i]);
    else dst[i] += alpha * (src[i] - dst[i]);
  }
  if (version && blockIdx.x == 0 && threadIdx.x == 0) *version += 1ull;
}

constexpr int kMaxSlots = 64;
struct SlotWeights {
  float c[kMaxSlots];
};

// out = Σ_i c_i * slot_i / Σ c_i, slot order fixed (deterministic).
static __global__ void __launch_bounds__(256) weighted_mean_kernel(float* __restrict__ out,
                                                            const float* __restrict__ slots,
                                                            int W, long long P, long long sstride,
                                                            int vec, SlotWeights cw,
                                                            float inv_total) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long n4 = vec ? (P >> 2) : 0;
  for (long long i = tid; i < n4; i += nth) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < W; ++k) {
      const float4 s = __ldcs(reinterpret_cast<const float4*>(slots + (long long)k * sstride) + i);
      acc.x = fmaf(cw.c[k], s.x, acc.x);
      acc.y = fmaf(cw.c[k], s.y, acc.y);
      acc.z = fmaf(cw.c[k], s.z, acc.z);
      acc.w = fmaf(cw.c[k], s.w, acc.w);
    }
    acc.x *= inv_total;
    acc.y *= inv_total;
    acc.z *= inv_total;
    acc.w *= inv_total;
    __stcs(reinterpret_cast<float4*>(out) + i, acc);
  }
  for (long long i = (n4 << 2) + tid; i < P; i += nth) {
    float acc = 0.f;
    for (int k = 0; k < W; ++k) acc = fmaf(cw.c[k], slots[(long long)k * sstride + i], acc);
    out[i] = acc * inv_total;
  }
}

}  // namespace ghc
