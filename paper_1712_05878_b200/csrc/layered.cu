// layered.cu — worker step for architectures with dense layers
// (arch.hpp:54-57: lstm(D,H,T)? dense(i,o,act)* softmax(i,K)), e.g. the
// wide-layer variant of config c5: lstm(5,20,10),dense(20,4096,relu),
// dense(4096,4096,relu),softmax(4096,3) — P = 16,881,699.
//
//   forward  nn.cpp:100-232  LSTM trunk kernel (h_T) → per dense layer one
//            tcgen05 GEMM with fused bias+activation (dense_gemm.cuh) →
//            softmax-CE head kernel (probs, ℓ, dlogits·scale, dZ_L fused)
//   backward nn.cpp:276-399  per dense layer: db = colsum(dZ), dW = dZᵀ·A and
//            dA = dZ·W on tcgen05 (act' of the previous layer fused into the
//            dA epilogue), then the LSTM trunk kernel from dh_T
// Every reduction over samples has a fixed order (bit-deterministic).
#include "dense_gemm.cuh"
#include "ghc_internal.cuh"

using namespace ghc;

namespace {

__global__ void gather_rows_kernel(float* __restrict__ out, int32_t* __restrict__ yout,
                                   const float* __restrict__ x, const int32_t* __restrict__ y,
                                   const int32_t* __restrict__ idx, int n, int width) {
  const int s = blockIdx.x;
  if (s >= n) return;
  const int row = idx[s];
  for (int i = threadIdx.x; i < width; i += blockDim.x)
    out[(long long)s * width + i] = x[(long long)row * width + i];
  if (threadIdx.x == 0) yout[s] = y[row];
}

// Softmax-CE head (nn.cpp:202-248 forward, 276-311 backward), one warp per
// sample: z = Ws·a + bs, p = softmax(z), ℓ = −log p_y, dz = (p − onehot)·scale;
// dA = Wsᵀ·dz, times act'(a) when `a` is a dense layer's output.
template <int KMAX>
__global__ void head_kernel(const float* __restrict__ A, int in, const float* __restrict__ Ws,
                            const float* __restrict__ bs, int K, const int32_t* __restrict__ y,
                            int n, float scale, float* __restrict__ dlogits,
                            float* __restrict__ loss_vec, float* __restrict__ dA, int dact,
                            float* __restrict__ probs, int* err) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const float* a = A + (long long)warp * in;
  float z[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) z[k] = 0.f;
  for (int i = lane; i < in; i += 32) {
    const float av = a[i];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) z[k] = fmaf(Ws[(long long)k * in + i], av, z[k]);
  }
  float zmax = -3.0e38f;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < K) {
      z[k] = warp_sum(z[k]) + bs[k];
      zmax = fmaxf(zmax, z[k]);
    }
  }
  int label = y[warp];
  if (label < 0 || label >= K) {
    if (lane == 0) atomicOr(err, 1);
    label = 0;
  }
  float den = 0.f, zy = 0.f;
  float e[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    e[k] = k < K ? expf(z[k] - zmax) : 0.f;
    den += e[k];
    zy = k == label ? z[k] : zy;
  }
  const float inv = 1.0f / den;
  float dz[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) dz[k] = k < K ? (e[k] * inv - (k == label ? 1.f : 0.f)) * scale : 0.f;
  if (lane == 0) loss_vec[warp] = logf(den) - (zy - zmax);
  if (lane < K) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k == lane) {
        if (dlogits) dlogits[(long long)warp * K + k] = dz[k];
        if (probs) probs[(long long)warp * K + k] = e[k] * inv;
      }
  }
  if (dA) {
    for (int i = lane; i < in; i += 32) {
      float d = 0.f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) d = fmaf(Ws[(long long)k * in + i], dz[k], d);
      if (dact >= 0) d *= gemm_detail::dact_from_y(a[i], dact);
      dA[(long long)warp * in + i] = d;
    }
  }
}

// The same head with one 256-thread block per sample and float4 rows (the
// wide variant's 4096-wide layer: a warp per sample left the row loop
// latency-bound at ~10 % of HBM).  Fixed reduction order: per-thread partial
// over its float4 chunks, butterfly within the warp, then the warps in order
// (every thread forms the same sums from shared memory).
template <int KMAX>
__global__ void __launch_bounds__(256) head_block_kernel(
    const float* __restrict__ A, int in, const float* __restrict__ Ws, const float* __restrict__ bs, int K,
    const int32_t* __restrict__ y, int n, float scale, float* __restrict__ dlogits, float* __restrict__ loss_vec,
    float* __restrict__ dA, int dact, float* __restrict__ probs, int* err) {
  __shared__ float red[KMAX][8];
  const int s = blockIdx.x;
  if (s >= n) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int in4 = in >> 2;
  const float4* a4 = reinterpret_cast<const float4*>(A + (long long)s * in);
  float z[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) z[k] = 0.f;
#pragma unroll 4
  for (int i = threadIdx.x; i < in4; i += blockDim.x) {
    const float4 av = a4[i];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(Ws + (long long)k * in) + i);
        z[k] = fmaf(w.x, av.x, z[k]);
        z[k] = fmaf(w.y, av.y, z[k]);
        z[k] = fmaf(w.z, av.z, z[k]);
        z[k] = fmaf(w.w, av.w, z[k]);
      }
  }
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const float v = warp_sum(z[k]);
    if (lane == 0 && k < K) red[k][warp] = v;
  }
  __syncthreads();
  float zmax = -3.0e38f;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < K) {
      float t = 0.f;
      for (int w = 0; w < nw; ++w) t += red[k][w];
      z[k] = t + bs[k];
      zmax = fmaxf(zmax, z[k]);
    }
  }
  int label = y[s];
  if (label < 0 || label >= K) {
    if (threadIdx.x == 0) atomicOr(err, 1);
    label = 0;
  }
  float den = 0.f, zy = 0.f, e[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    e[k] = k < K ? expf(z[k] - zmax) : 0.f;
    den += e[k];
    zy = k == label ? z[k] : zy;
  }
  const float inv = 1.0f / den;
  float dz[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) dz[k] = k < K ? (e[k] * inv - (k == label ? 1.f : 0.f)) * scale : 0.f;
  if (threadIdx.x == 0) {
    loss_vec[s] = logf(den) - (zy - zmax);
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) {
        if (dlogits) dlogits[(long long)s * K + k] = dz[k];
        if (probs) probs[(long long)s * K + k] = e[k] * inv;
      }
  }
  if (dA) {
    float4* d4 = reinterpret_cast<float4*>(dA + (long long)s * in);
#pragma unroll 4
    for (int i = threadIdx.x; i < in4; i += blockDim.x) {
      float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) {
          const float4 w = __ldg(reinterpret_cast<const float4*>(Ws + (long long)k * in) + i);
          d.x = fmaf(w.x, dz[k], d.x);
          d.y = fmaf(w.y, dz[k], d.y);
          d.z = fmaf(w.z, dz[k], d.z);
          d.w = fmaf(w.w, dz[k], d.w);
        }
      if (dact >= 0) {
        const float4 av = a4[i];
        d.x *= gemm_detail::dact_from_y(av.x, dact);
        d.y *= gemm_detail::dact_from_y(av.y, dact);
        d.z *= gemm_detail::dact_from_y(av.z, dact);
        d.w *= gemm_detail::dact_from_y(av.w, dact);
      }
      d4[i] = d;
    }
  }
}

// One-launch column reduction for wide rows (cols % 4 == 0, 16-B rows):
// block = 4 column quads (16 columns) × 64 row lanes; row lane ry sums rows
// ry, ry + 64, … (eight float4 loads in flight per thread; up to 4
// coefficient columns k0..k0+3 from one read of X), then the 64 row-lane
// sums per column are added by a fixed pairwise tree in shared memory —
// deterministic; one launch instead of the two-stage partial + final pair (two launches of
// ≈ 8 µs each per call in the wide round).
__global__ void __launch_bounds__(256) colsum4_kernel(float* __restrict__ out, int ldo,
                                                      const float* __restrict__ X, int ldx,
                                                      const float* __restrict__ coef, int kc, int n,
                                                      int cols) {
  constexpr int QX = 4, RY = 64, U = 8;
  __shared__ float4 red[4][RY][QX + 1];
  const int qx = threadIdx.x & (QX - 1), ry = threadIdx.x / QX;
  const int q = blockIdx.x * QX + qx;  // column quad
  const int k0 = 4 * blockIdx.y;
  const int nk = coef ? min(4, kc - k0) : 1;
  float4 acc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (4 * q < cols) {
    for (int s0 = ry; s0 < n; s0 += RY * U) {
      float4 v[U];
      float cf[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + RY * u;
        v[u] = s < n ? __ldg(reinterpret_cast<const float4*>(X + (long long)s * ldx) + q)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          cf[u][k] = coef ? (s < n && k < nk ? __ldg(coef + (long long)s * kc + k0 + k) : 0.f) : 1.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k >= nk) break;
          acc[k].x = fmaf(cf[u][k], v[u].x, acc[k].x);
          acc[k].y = fmaf(cf[u][k], v[u].y, acc[k].y);
          acc[k].z = fmaf(cf[u][k], v[u].z, acc[k].z);
          acc[k].w = fmaf(cf[u][k], v[u].w, acc[k].w);
        }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nk) red[k][ry][qx] = acc[k];
#pragma unroll
  for (int h = RY / 2; h > 0; h >>= 1) {  // fixed pairwise tree over the row lanes
    __syncthreads();
    if (ry < h) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= nk) break;
        const float4 a = red[k][ry][qx], b = red[k][ry + h][qx];
        red[k][ry][qx] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < QX * nk) {
    const int k = threadIdx.x / QX, qq = threadIdx.x % QX;
    const int c = 4 * (blockIdx.x * QX + qq);
    if (c < cols) {
      const float4 o = red[k][0][qq];
      float* dst = out + (long long)(k0 + k) * ldo + c;
      dst[0] = o.x;
      dst[1] = o.y;
      dst[2] = o.z;
      dst[3] = o.w;
    }
  }
}

// Stage 1 of a deterministic column reduction over samples:
// part[chunk][k][c] = Σ_{s ∈ chunk} coef[s][k] · X[s][c]   (coef == nullptr → 1)
__global__ void colsum_partial_kernel(float* __restrict__ part, const float* __restrict__ X,
                                      int ldx, const float* __restrict__ coef, int kc, int n,
                                      int cols, int chunk) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.y;
  const int k0 = 4 * blockIdx.z;  // coefficient columns k0..k0+3 (kc up to the head's K)
  if (c >= cols) return;
  const int s0 = ch * chunk, s1 = min(n, s0 + chunk);
  const int nk = min(4, kc - k0);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int s = s0; s < s1; ++s) {
    const float xv = X[(long long)s * ldx + c];
    if (coef) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nk) acc[k] = fmaf(coef[(long long)s * kc + k0 + k], xv, acc[k]);
    } else {
      acc[0] += xv;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nk) part[((long long)ch * kc + k0 + k) * cols + c] = acc[k];
}

// Stage 2: out[k*ldo + c] = Σ_chunk part[chunk][k][c] (chunk order).
__global__ void colsum_final_kernel(float* __restrict__ out, int ldo, const float* __restrict__ part,
                                    int kc, int cols, int nchunks) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (c >= cols) return;
  float t = 0.f;
#pragma unroll 8
  for (int ch = 0; ch < nchunks; ++ch) t += part[((long long)ch * kc + k) * cols + c];
  out[(long long)k * ldo + c] = t;
}

__global__ void sum_kernel(float* out, const float* v, int n) {
  __shared__ float red[256];
  float t = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += v[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

struct Buf {
  float* p = nullptr;
  size_t cap = 0;
  ghc_status ensure(size_t n) {
    if (n <= cap) return GHC_OK;
    cudaFree(p);
    p = nullptr;
    cap = 0;
    CU(cudaMalloc(&p, sizeof(float) * (n ? n : 1)));
    cap = n;
    return GHC_OK;
  }
};

}  // namespace

struct LayeredWorkspace {
  Buf xg, yg, h, dh, logits, loss, part, zT, aT, wT;
  std::vector<Buf> act;   // Y_l per dense layer
  std::vector<Buf> actT;  // Y_lᵀ [width][n] (written by the forward GEMM's epilogue)
  Buf dz[2];
  Buf dzT[2];             // dZᵀ written by the dA GEMM's epilogue
};

namespace {

ghc_status colsum(ghc_ctx* c, LayeredWorkspace& ws, float* out, int ldo, const float* X, int ldx,
                  const float* coef, int kc, int n, int cols) {
  if (cols >= 256 && cols % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15u) == 0) {
    const int kcc = coef ? kc : 1;
    colsum4_kernel<<<dim3((cols / 4 + 3) / 4, (kcc + 3) / 4), 256, 0, c->stream>>>(out, ldo, X, ldx, coef,
                                                                                  kcc, n, cols);
    c->launches++;
    CU(cudaGetLastError());
    return GHC_OK;
  }
  const int nch = n < 32 ? n : 32;
  const int chunk = (n + nch - 1) / nch;
  if (ghc_status s = ws.part.ensure(static_cast<size_t>(nch) * kc * cols)) return s;
  colsum_partial_kernel<<<dim3((cols + 127) / 128, nch, (kc + 3) / 4), 128, 0, c->stream>>>(
      ws.part.p, X, ldx, coef, kc, n, cols, chunk);
  colsum_final_kernel<<<dim3((cols + 127) / 128, kc), 128, 0, c->stream>>>(out, ldo, ws.part.p,
                                                                          kc, cols, nch);
  c->launches += 2;
  CU(cudaGetLastError());
  return GHC_OK;
}

ghc_status transpose(ghc_ctx* c, float* out, const float* in, int rows, int cols) {
  return ghc_transpose(c, out, in, rows, cols, cols, rows);
}

}  // namespace

// Layered worker step (declared in ghc_internal.cuh).  probs != nullptr →
// forward only (probs + loss).
ghc_status layered_step(ghc_plan* p, const float* w, const float* x, const int32_t* y,
                        const int32_t* idx, int64_t n64, float scale, float* g_out,
                        float* loss_out, float* probs) {
  ghc_ctx* c = p->ctx;
  const Model& m = p->model;
  const int n = static_cast<int>(n64);
  if (!p->ws) p->ws = new LayeredWorkspace();
  LayeredWorkspace& ws = *p->ws;
  const int width = static_cast<int>(m.input_width);
  // 1. gather the batch
  const float* X = x;
  const int32_t* Y = y;
  if (idx) {
    if (ghc_status s = ws.xg.ensure(static_cast<size_t>(n) * width)) return s;
    if (ghc_status s = ws.yg.ensure(static_cast<size_t>(n))) return s;
    gather_rows_kernel<<<n, 64, 0, c->stream>>>(ws.xg.p, reinterpret_cast<int32_t*>(ws.yg.p), x,
                                                y, idx, n, width);
    c->launches++;
    X = ws.xg.p;
    Y = reinterpret_cast<const int32_t*>(ws.yg.p);
  }
  const auto& L = m.layers;
  const bool has_lstm = L.front().kind == LayerKind::lstm;
  const int nd = static_cast<int>(L.size()) - 1 - (has_lstm ? 1 : 0);  // dense layers
  ws.act.resize(static_cast<size_t>(nd));
  ws.actT.resize(static_cast<size_t>(nd));
  const bool want_grad = g_out != nullptr;
  // 2. LSTM trunk forward → h_T [n × H]
  const float* a = X;
  int a_w = width;
  int ti = 0;
  if (has_lstm) {
    const int H = L[0].b;
    if (ghc_status s = ws.h.ensure(static_cast<size_t>(n) * H)) return s;
    if (p->generic_lstm) {
      if (ghc_status s = generic_lstm_fwd(p, w, X, n, ws.h.p)) return s;
    } else {
      StepArgs sa{};
      sa.x = X;
      sa.y = Y;
      sa.n = n;
      sa.rounds = 1;
      sa.grad_scale = 1.0f;
      sa.w_in = w;
      sa.ms = p->ms;
      sa.hio = ws.h.p;
      sa.mode = MODE_TRUNK_FWD;
      if (ghc_status s = launch_trunk(p, sa, n)) return s;
    }
    a = ws.h.p;
    a_w = H;
    ti = 3;
  }
  // 3. dense layers forward
  std::vector<const float*> A_in(static_cast<size_t>(nd));
  std::vector<int> in_w(static_cast<size_t>(nd)), ti_l(static_cast<size_t>(nd));
  for (int l = 0; l < nd; ++l) {
    const Layer& d = L[static_cast<size_t>(l + (has_lstm ? 1 : 0))];
    if (ghc_status s = ws.act[static_cast<size_t>(l)].ensure(static_cast<size_t>(n) * d.b)) return s;
    A_in[static_cast<size_t>(l)] = a;
    in_w[static_cast<size_t>(l)] = a_w;
    ti_l[static_cast<size_t>(l)] = ti;
    const float* W = w + m.tensors[static_cast<size_t>(ti)].offset;
    const float* b = w + m.tensors[static_cast<size_t>(ti + 1)].offset;
    // Y_l feeds layer l+1's weight gradient as the K-major Y_lᵀ: the epilogue
    // writes it (coalesced) instead of a separate transpose pass
    float* yT = nullptr;
    if (want_grad && l + 1 < nd) {
      if (ghc_status s = ws.actT[static_cast<size_t>(l)].ensure(static_cast<size_t>(n) * d.b)) return s;
      yT = ws.actT[static_cast<size_t>(l)].p;
    }
    if (ghc_status s = gemm_nt_ct(c, a, W, ws.act[static_cast<size_t>(l)].p, n, d.b, d.a, a_w, d.a,
                                  d.b, GHC_EPI_BIAS_ACT, static_cast<int>(d.act), b, nullptr, 0, 1.0f,
                                  yT, n))
      return s;
    a = ws.act[static_cast<size_t>(l)].p;
    a_w = d.b;
    ti += 2;
  }
  // 4. head
  const Layer& sm = L.back();
  const int K = sm.b;
  if (K > 32) return fail(GHC_ERR_CONFIG, "softmax head: at most 32 classes");
  const float* Ws = w + m.tensors[static_cast<size_t>(ti)].offset;
  const float* bs = w + m.tensors[static_cast<size_t>(ti + 1)].offset;
  const bool fwd_only = g_out == nullptr;
  if (ghc_status s = ws.logits.ensure(static_cast<size_t>(n) * K)) return s;
  if (ghc_status s = ws.loss.ensure(static_cast<size_t>(n))) return s;
  if (ghc_status s = ws.dz[0].ensure(static_cast<size_t>(n) * a_w)) return s;
  const bool need_dA = !fwd_only && (nd > 0 || has_lstm);
  const int dact = nd > 0 ? static_cast<int>(L[L.size() - 2].act) : -1;
  {
    const int warps_per_block = 8;
    const dim3 grid((n + warps_per_block - 1) / warps_per_block);
    const bool vec = (a_w % 4) == 0 && a_w >= 512 && (reinterpret_cast<uintptr_t>(a) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(Ws) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(ws.dz[0].p) & 15u) == 0;
    if (vec && K <= 4)
      head_block_kernel<4><<<n, 256, 0, c->stream>>>(
          a, a_w, Ws, bs, K, Y, n, scale, ws.logits.p, ws.loss.p, need_dA ? ws.dz[0].p : nullptr,
          dact, probs, p->err);
    else if (vec)
      head_block_kernel<32><<<n, 256, 0, c->stream>>>(
          a, a_w, Ws, bs, K, Y, n, scale, ws.logits.p, ws.loss.p, need_dA ? ws.dz[0].p : nullptr,
          dact, probs, p->err);
    else if (K <= 4)
      head_kernel<4><<<grid, 32 * warps_per_block, 0, c->stream>>>(
          a, a_w, Ws, bs, K, Y, n, scale, ws.logits.p, ws.loss.p, need_dA ? ws.dz[0].p : nullptr,
          dact, probs, p->err);
    else
      head_kernel<32><<<grid, 32 * warps_per_block, 0, c->stream>>>(
          a, a_w, Ws, bs, K, Y, n, scale, ws.logits.p, ws.loss.p, need_dA ? ws.dz[0].p : nullptr,
          dact, probs, p->err);
    c->launches++;
    CU(cudaGetLastError());
  }
  if (loss_out) {
    sum_kernel<<<1, 256, 0, c->stream>>>(loss_out, ws.loss.p, n);
    c->launches++;
  }
  if (fwd_only) return GHC_OK;
  // 5. head gradients: gWs[k][i] = Σ_s dz[s][k]·a[s][i]; gbs[k] = Σ_s dz[s][k]
  if (ghc_status s = colsum(c, ws, g_out + m.tensors[static_cast<size_t>(ti)].offset, a_w, a, a_w,
                            ws.logits.p, K, n, a_w))
    return s;
  if (ghc_status s = colsum(c, ws, g_out + m.tensors[static_cast<size_t>(ti + 1)].offset, 1,
                            ws.logits.p, K, nullptr, 1, n, K))
    return s;
  // 6. dense layers backward (dz[cur] holds dZ_l = dA_l ⊙ act'_l)
  int cur = 0;
  for (int l = nd - 1; l >= 0; --l) {
    const Layer& d = L[static_cast<size_t>(l + (has_lstm ? 1 : 0))];
    const int in = in_w[static_cast<size_t>(l)], out = d.b;
    const int tw = ti_l[static_cast<size_t>(l)];
    float* dZ = ws.dz[cur].p;
    // db_l (nn.cpp:325)
    if (ghc_status s = colsum(c, ws, g_out + m.tensors[static_cast<size_t>(tw + 1)].offset, out, dZ,
                              out, nullptr, 1, n, out))
      return s;
    // dW_l = dZᵀ·A (nn.cpp:327-329): C[out×in] = dZᵀ[out×n] · (Aᵀ[in×n])ᵀ
    // K-major operands: dZᵀ from the previous dA GEMM's epilogue (the head's dZ
    // is transposed here), Aᵀ from the forward epilogue (the trunk's h here)
    const float* zT = ws.dzT[cur].p;
    if (l == nd - 1) {
      if (ghc_status s = ws.zT.ensure(static_cast<size_t>(out) * n)) return s;
      if (ghc_status s = transpose(c, ws.zT.p, dZ, n, out)) return s;
      zT = ws.zT.p;
    }
    const float* aT = l > 0 ? ws.actT[static_cast<size_t>(l - 1)].p : nullptr;
    if (l == 0) {
      if (ghc_status s = ws.aT.ensure(static_cast<size_t>(in) * n)) return s;
      if (ghc_status s = transpose(c, ws.aT.p, A_in[static_cast<size_t>(l)], n, in)) return s;
      aT = ws.aT.p;
    }
    if (ghc_status s = ghc_gemm_nt(c, zT, aT, g_out + m.tensors[static_cast<size_t>(tw)].offset,
                                   out, in, n, n, n, in, GHC_EPI_STORE, 2, nullptr, nullptr, 0, 1.0f))
      return s;
    // dA_{l-1} = dZ·W (nn.cpp:330) [n×in] = dZ[n×out] · (Wᵀ[in×out])ᵀ, act' fused
    if (l > 0 || has_lstm) {
      if (ghc_status s = ws.wT.ensure(static_cast<size_t>(in) * out)) return s;
      if (ghc_status s = transpose(c, ws.wT.p, w + m.tensors[static_cast<size_t>(tw)].offset, out, in))
        return s;
      float* dst;
      float* dstT = nullptr;
      int epi, act_prev;
      const float* Yprev = nullptr;
      if (l > 0) {
        if (ghc_status s = ws.dz[cur ^ 1].ensure(static_cast<size_t>(n) * in)) return s;
        if (ghc_status s = ws.dzT[cur ^ 1].ensure(static_cast<size_t>(n) * in)) return s;
        dst = ws.dz[cur ^ 1].p;
        dstT = ws.dzT[cur ^ 1].p;
        epi = GHC_EPI_DACT;
        act_prev = static_cast<int>(L[static_cast<size_t>(l - 1 + (has_lstm ? 1 : 0))].act);
        Yprev = ws.act[static_cast<size_t>(l - 1)].p;
      } else {
        if (ghc_status s = ws.dh.ensure(static_cast<size_t>(n) * in)) return s;
        dst = ws.dh.p;
        epi = GHC_EPI_STORE;
        act_prev = 2;
      }
      if (ghc_status s = gemm_nt_ct(c, dZ, ws.wT.p, dst, n, in, out, out, out, in, epi, act_prev,
                                    nullptr, Yprev, in, 1.0f, dstT, n))
        return s;
      cur ^= 1;
    }
  }
  // 7. LSTM trunk backward from dh_T (nn.cpp:335-396)
  if (has_lstm && p->generic_lstm) {
    const float* dH = nd > 0 ? ws.dh.p : ws.dz[0].p;
    return generic_lstm_bwd(p, w, X, n, dH, g_out);
  }
  if (has_lstm) {
    const float* dH = nd > 0 ? ws.dh.p : ws.dz[0].p;
    StepArgs sa{};
    sa.x = X;
    sa.y = Y;
    sa.n = n;
    sa.rounds = 1;
    sa.grad_scale = 1.0f;
    sa.w_in = w;
    sa.ms = p->ms;
    sa.hio = const_cast<float*>(dH);
    sa.g_out = g_out;
    sa.mode = MODE_TRUNK_GRAD;
    if (ghc_status s = launch_trunk(p, sa, n)) return s;
  }
  return GHC_OK;
}

void layered_free(LayeredWorkspace* ws) {
  if (!ws) return;
  Buf* all[] = {&ws->xg, &ws->yg, &ws->h, &ws->dh, &ws->logits, &ws->loss, &ws->part,
                &ws->zT, &ws->aT, &ws->wT, &ws->dz[0], &ws->dz[1], &ws->dzT[0], &ws->dzT[1]};
  for (Buf* b : all) cudaFree(b->p);
  for (Buf& b : ws->act) cudaFree(b.p);
  for (Buf& b : ws->actT) cudaFree(b.p);
  delete ws;
}
