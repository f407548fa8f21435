// lstm_step.cuh — the fused worker step for `lstm(D,H,T) → softmax(H,K)`
// (the SPEC benchmark net) on sm_100a.
//
// One launch runs, for every sample of a round, the reference's
//   forward   nn.cpp:146-201 (LSTM, gate order i,f,g,o, arch.hpp:20-22)
//             nn.cpp:202-229 (softmax) + loss nn.cpp:234-248
//   backward  nn.cpp:276-311 (softmax, dz = (p-onehot)*scale, nn.cpp:283-297)
//             nn.cpp:335-396 (BPTT, dc carried through f, dh = Whᵀ dz)
// then a deterministic cross-CTA reduction of the per-CTA partial gradients
// and — in MODE_SGD — the master's sgd_step (optim.cpp:39-65) with the
// whole-update non-finite rejection (optim.cpp:49-51) committed on device.
//
// Mapping (B200, 148 SMs): one warp per sample, lane j owns hidden unit j
// (H ≤ 32) and the four gate rows {j, H+j, 2H+j, 3H+j}; its rows of Wx/Wh
// live in registers for the forward recurrence, its column of Wh for
// dh = Whᵀdz in the backward; h_t and the gate cache live in shared memory.
// Samples of a round are spread over ≈ one CTA per SM so the 1000
// transcendentals/sample run on every SM's MUFU pipe.  The recurrence is a
// K=25 contraction per timestep — far below a tcgen05 tile — so the kernel is
// FFMA/latency-bound by design.
#pragma once

#include "ghc_device.cuh"

namespace ghc {

enum StepMode : int { MODE_GRAD = 0, MODE_SGD = 1, MODE_FWD = 2 };

struct StepArgs {
  const float* x;         // dataset (or batch) rows, T*D floats each
  const int32_t* y;       // labels
  const int32_t* idx;     // gather indices into x/y (nullable: row s)
  long long stride;       // idx offset per round
  const int32_t* counts;  // samples per round (nullable: n)
  int n;
  int rounds;
  float grad_scale;       // MODE_GRAD: grad = scale * Σ_s ∇ℓ_s
  const float* w_in;      // MODE_GRAD / MODE_FWD weights
  float* w0;              // MODE_SGD double buffers
  float* w1;
  float* v0;
  float* v1;
  float lr;
  float mu;
  MasterDev* ms;
  float* part;            // [gridDim.x][pstride] partial sums (+ loss slot)
  int pstride;
  float* g_out;           // MODE_GRAD: reduced gradient [P]
  float* loss_out;        // per-round loss sum (nullable)
  float* probs_out;       // MODE_FWD: n×K (nullable)
  int* err;               // bit 0: label out of range (nn.cpp:241-244)
  unsigned long long* probe;  // nullable: [rounds][gridDim][8] %globaltimer per phase
  int mode;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int D, int H, int T, int K>
struct LstmNet {
  static_assert(H >= 1 && H <= 32, "one lane per hidden unit");
  static_assert(K >= 1 && K <= 32, "classes");
  static constexpr int G4 = 4 * H;
  static constexpr int OFF_WX = 0;                 // Wx[4H×D]  arch.cpp:103
  static constexpr int OFF_WH = G4 * D;            // Wh[4H×H]  arch.cpp:104
  static constexpr int OFF_B = OFF_WH + G4 * H;    // b[4H]     arch.cpp:105
  static constexpr int OFF_WS = OFF_B + G4;        // Ws[K×H]   arch.cpp:108
  static constexpr int OFF_BS = OFF_WS + K * H;    // bs[K]     arch.cpp:109
  static constexpr int P = OFF_BS + K;
  static constexpr int PPAD = (P + 1 + 3) & ~3;    // + loss slot, 16-B rows
  static constexpr int XW = T * D;
  static constexpr int S_X = 0;                          // x_t rows
  static constexpr int S_H = (XW + 3) & ~3;              // h[T][H]
  static constexpr int S_C = S_H + ((T * H + 3) & ~3);   // cache[T][6][H]
  static constexpr int S_DZ = S_C + T * 6 * H;           // dz[T][4H]
  static constexpr int WARP_FLOATS = (S_DZ + T * G4 + 3) & ~3;
  static size_t smem_bytes(int nw) {
    return sizeof(float) * (size_t)(PPAD + nw * WARP_FLOATS + nw * PPAD + 32);
  }
};

// Forward + softmax/loss (+ backward when BWD) of one sample; the sample's
// gradient is ADDED into the warp's partial `wp` (lane j touches only the
// entries of its own gate rows, lane 0 the output bias) — no atomics.
template <int D, int H, int T, int K, bool BWD>
__device__ __forceinline__ float lstm_sample(const float* __restrict__ wsm, float* __restrict__ ws,
                                             float* __restrict__ wp,
                                             const float* __restrict__ xrow, int label, float scale,
                                             int lane, float* probs_row) {
  using N = LstmNet<D, H, T, K>;
  const bool act = lane < H;
  const int j = act ? lane : 0;
  float* xs = ws + N::S_X;
  float* hs = ws + N::S_H;
  float* cs = ws + N::S_C;
  float* dzs = ws + N::S_DZ;  // dz[t][4H], t = 0..T-1

  for (int i = lane; i < N::XW; i += 32) xs[i] = __ldg(xrow + i);
  __syncwarp();

  // ---------------- forward recurrence (nn.cpp:160-200) ----------------
  {
    float wx[4][D], wh[4][H], bb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bb[q] = wsm[N::OFF_B + q * H + j];
#pragma unroll
      for (int d = 0; d < D; ++d) wx[q][d] = wsm[N::OFF_WX + (q * H + j) * D + d];
#pragma unroll
      for (int k = 0; k < H; ++k) wh[q][k] = wsm[N::OFF_WH + (q * H + j) * H + k];
    }
    float c = 0.0f;
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      float a0[4], a1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a0[q] = bb[q];
        a1[q] = 0.0f;
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const float xv = xs[t * D + d];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (d & 1) a1[q] = fmaf(wx[q][d], xv, a1[q]);
          else a0[q] = fmaf(wx[q][d], xv, a0[q]);
        }
      }
      if (t > 0) {
        const float* hp = hs + (t - 1) * H;
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const float hv = hp[k];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (k & 1) a1[q] = fmaf(wh[q][k], hv, a1[q]);
            else a0[q] = fmaf(wh[q][k], hv, a0[q]);
          }
        }
      }
      const float ig = sigmoid_f(a0[0] + a1[0]);
      const float fg = sigmoid_f(a0[1] + a1[1]);
      const float gg = tanh_f(a0[2] + a1[2]);
      const float og = sigmoid_f(a0[3] + a1[3]);
      c = fmaf(fg, c, ig * gg);
      const float tc = tanh_f(c);
      if (act) {
        float* ct = cs + t * 6 * H + j;
        ct[0 * H] = ig;
        ct[1 * H] = fg;
        ct[2 * H] = gg;
        ct[3 * H] = og;
        ct[4 * H] = c;
        ct[5 * H] = tc;
        hs[t * H + j] = og * tc;
      }
      __syncwarp();
    }
  }

  // ---------------- softmax + loss (nn.cpp:202-248) ----------------
  const float hT = act ? hs[(T - 1) * H + j] : 0.0f;
  float z[K];
  float zmax = -3.0e38f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    z[k] = warp_sum(act ? wsm[N::OFF_WS + k * H + j] * hT : 0.0f) + wsm[N::OFF_BS + k];
    zmax = fmaxf(zmax, z[k]);
  }
  float e[K];
  float den = 0.0f, zy = 0.0f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    e[k] = expf(z[k] - zmax);
    den += e[k];
    if (k == label) zy = z[k];
  }
  const float inv_den = 1.0f / den;
  const float lossv = logf(den) - (zy - zmax);
  if (probs_row != nullptr) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane == k) probs_row[k] = e[k] * inv_den;
  }
  if constexpr (!BWD) return lossv;

  // ---------------- backward: softmax (nn.cpp:276-311) ----------------
  float dh = 0.0f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float dzk = (e[k] * inv_den - (k == label ? 1.0f : 0.0f)) * scale;
    if (act) wp[N::OFF_WS + k * H + j] += dzk * hT;
    if (lane == 0) wp[N::OFF_BS + k] += dzk;
    dh = fmaf(act ? wsm[N::OFF_WS + k * H + j] : 0.0f, dzk, dh);
  }

  // ------- backward pass 1: the BPTT chain (nn.cpp:351-392), dz → smem -------
  {
    float wt[4 * H];  // column j of Wh: Wh[r][j]
#pragma unroll
    for (int r = 0; r < 4 * H; ++r) wt[r] = wsm[N::OFF_WH + r * H + j];
    float dc = 0.0f;
#pragma unroll 1
    for (int t = T - 1; t >= 0; --t) {
      const float* ct = cs + t * 6 * H + j;
      const float ig = ct[0 * H], fg = ct[1 * H], gg = ct[2 * H], og = ct[3 * H];
      const float tc = ct[5 * H];
      const float cp = t > 0 ? cs[(t - 1) * 6 * H + 4 * H + j] : 0.0f;
      const float dout = dh * tc;
      dc = fmaf(dh * og, 1.0f - tc * tc, dc);
      const float di = dc * gg, dg = dc * ig, df = dc * cp;
      float* dzt = dzs + t * 4 * H;
      if (act) {
        dzt[0 * H + j] = di * ig * (1.0f - ig);
        dzt[1 * H + j] = df * fg * (1.0f - fg);
        dzt[2 * H + j] = dg * (1.0f - gg * gg);
        dzt[3 * H + j] = dout * og * (1.0f - og);
      }
      __syncwarp();
      if (t > 0) {  // dh_{t-1} = Whᵀ dz_t (the reference also does this at t=0, unused)
        float p[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int r = 0; r < 4 * H; ++r) p[r & 3] = fmaf(wt[r], dzt[r], p[r & 3]);
        dh = (p[0] + p[1]) + (p[2] + p[3]);
        dc *= fg;
      }
    }
  }

  // ------- backward pass 2: dWx, dWh, db = Σ_t dz_t ⊗ [x_t, h_{t-1}] -------
  if (act) {
    float dz[T][4];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < 4; ++q) dz[t][q] = dzs[t * 4 * H + q * H + j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float s = 0.0f;
#pragma unroll
      for (int t = 0; t < T; ++t) s += dz[t][q];
      wp[N::OFF_B + q * H + j] += s;
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float xv = xs[t * D + d];
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fmaf(dz[t][q], xv, s[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) wp[N::OFF_WX + (q * H + j) * D + d] += s[q];
    }
#pragma unroll 2
    for (int k = 0; k < H; ++k) {
      float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int t = 1; t < T; ++t) {
        const float hv = hs[(t - 1) * H + k];
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = fmaf(dz[t][q], hv, s[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) wp[N::OFF_WH + (q * H + j) * H + k] += s[q];
    }
  }
  __syncwarp();
  return lossv;
}

template <int D, int H, int T, int K>
__global__ void __launch_bounds__(256, 1) lstm_softmax_step_kernel(StepArgs a) {
  using N = LstmNet<D, H, T, K>;
  extern __shared__ __align__(16) float smem[];
  const int NW = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* wsm = smem;
  float* ws = smem + N::PPAD + warp * N::WARP_FLOATS;
  float* wpart = smem + N::PPAD + NW * N::WARP_FLOATS;  // [NW][PPAD]; reused as `red`
  float* lossw = wpart + NW * N::PPAD;                   // [32]
  const int G = gridDim.x;
  const int E = N::P + 1;  // gradient + loss slot

  int cur = 0;
  unsigned long long round0 = 0;
  unsigned long long accepted = 0, rejected = 0;
  int last_status = 0;
  if (a.mode == MODE_SGD) {
    cur = __ldcg(&a.ms->cur);
    round0 = __ldcg(&a.ms->round);
  }

  for (int r = 0; r < a.rounds; ++r) {
    const float* w = a.mode == MODE_SGD ? (cur ? a.w1 : a.w0) : a.w_in;
    const int n = a.counts ? __ldg(a.counts + r) : a.n;
    const int32_t* idx = a.idx ? a.idx + (long long)r * a.stride : nullptr;
    const float scale = a.mode == MODE_SGD ? 1.0f / (float)n : a.grad_scale;
    const int parity = (int)((round0 + (unsigned long long)r) & 1ull);

    unsigned long long* pr =
        a.probe ? a.probe + ((long long)r * gridDim.x + blockIdx.x) * 8 : nullptr;
    if (pr && threadIdx.x == 0) pr[0] = globaltimer();
    for (int p = threadIdx.x; p < N::P; p += blockDim.x) wsm[p] = __ldcg(w + p);
    __syncthreads();
    if (pr && threadIdx.x == 0) pr[1] = globaltimer();

    // ---- per-warp samples of this CTA's contiguous chunk ----
    float* wp = wpart + warp * N::PPAD;
    if (a.mode != MODE_FWD) {
      for (int p = lane; p < N::PPAD; p += 32) wp[p] = 0.0f;
      __syncwarp();
    }
    float lsum = 0.0f;
    const int spc = (n + G - 1) / G;
    const int s0 = blockIdx.x * spc;
    const int s1 = min(n, s0 + spc);
    for (int s = s0 + warp; s < s1; s += NW) {
      const int row = idx ? __ldg(idx + s) : s;
      int label = __ldg(a.y + row);
      if (label < 0 || label >= K) {
        if (lane == 0) atomicOr(a.err, 1);
        label = 0;
      }
      const float* xrow = a.x + (long long)row * N::XW;
      if (a.mode == MODE_FWD) {
        lsum += lstm_sample<D, H, T, K, false>(
            wsm, ws, wp, xrow, label, scale, lane,
            a.probs_out ? a.probs_out + (long long)s * K : nullptr);
      } else {
        lsum += lstm_sample<D, H, T, K, true>(wsm, ws, wp, xrow, label, scale, lane, nullptr);
      }
    }
    if (lane == 0) lossw[warp] = lsum;
    __syncthreads();
    if (pr && threadIdx.x == 0) pr[2] = globaltimer();

    // ---- CTA partial (fixed warp order) → global ----
    float* prow = a.part + (long long)blockIdx.x * a.pstride;
    if (a.mode != MODE_FWD) {
      for (int p = threadIdx.x; p < N::P; p += blockDim.x) {
        float t = 0.0f;
        for (int w2 = 0; w2 < NW; ++w2) t += wpart[w2 * N::PPAD + p];
        __stcg(prow + p, t);
      }
    }
    if (threadIdx.x == 0) {
      float t = 0.0f;
      for (int w2 = 0; w2 < NW; ++w2) t += lossw[w2];
      __stcg(prow + N::P, t);
    }
    if (pr && threadIdx.x == 0) pr[3] = globaltimer();
    grid_barrier(a.ms);
    if (pr && threadIdx.x == 0) pr[4] = globaltimer();
    if (a.mode == MODE_SGD && blockIdx.x == 0 && threadIdx.x == 0) a.ms->flag[parity ^ 1] = 0;

    // ---- distributed deterministic reduction of slice [p0,p1) over CTAs ----
    const int slice = (E + G - 1) / G;
    const int p0 = a.mode == MODE_FWD ? (blockIdx.x == 0 ? N::P : E) : blockIdx.x * slice;
    const int p1 = a.mode == MODE_FWD ? E : min(E, p0 + slice);
    const float* wcur = w;
    float* wnext = cur ? a.w0 : a.w1;
    const float* vcur = cur ? a.v1 : a.v0;
    float* vnext = cur ? a.v0 : a.v1;
    int bad = 0;
    float* red = wpart;
    const int cols = min(max(p1 - p0, 1), (int)blockDim.x);
    const int groups = blockDim.x / cols;
    for (int base = p0; base < p1; base += cols) {
      const int nc = min(cols, p1 - base);
      const int c = threadIdx.x % cols, gidx = threadIdx.x / cols;
      float sum = 0.0f;
      if (c < nc && gidx < groups)
        for (int b = gidx; b < G; b += groups) sum += __ldcg(a.part + (long long)b * a.pstride + base + c);
      if (gidx < groups) red[gidx * cols + c] = sum;
      __syncthreads();
      if (threadIdx.x < nc) {
        float tot = 0.0f;
        for (int g2 = 0; g2 < groups; ++g2) tot += red[g2 * cols + threadIdx.x];
        const int p = base + threadIdx.x;
        if (p == N::P) {
          if (a.loss_out) a.loss_out[r] = tot;
        } else if (a.mode == MODE_GRAD) {
          a.g_out[p] = tot;
        } else if (a.mode == MODE_SGD) {
          if (!is_finite_f(tot)) bad = 1;
          // sgd_step (optim.cpp:59-60): v = mu*v - lr*g; w += v
          const float vn = fmaf(a.mu, __ldcg(vcur + p), -a.lr * tot);
          __stcg(vnext + p, vn);
          __stcg(wnext + p, __ldcg(wcur + p) + vn);
        }
      }
      __syncthreads();
    }
    if (a.mode == MODE_SGD) {
      bad = __syncthreads_or(bad);
      if (bad && threadIdx.x == 0) atomicOr(&a.ms->flag[parity], 1);
      if (pr && threadIdx.x == 0) pr[5] = globaltimer();
      grid_barrier(a.ms);
      if (pr && threadIdx.x == 0) pr[6] = globaltimer();
      const int rej = __ldcg(&a.ms->flag[parity]);
      if (rej) {
        ++rejected;
        last_status = 2;  // GHC_ERR_NONFINITE: keep w/v (optim.cpp:49-51)
      } else {
        cur ^= 1;
        ++accepted;
        last_status = 0;
      }
    }
  }
  if (a.mode == MODE_SGD && blockIdx.x == 0 && threadIdx.x == 0) {
    a.ms->cur = cur;
    a.ms->version += accepted;
    a.ms->rejected += rejected;
    a.ms->round = round0 + (unsigned long long)a.rounds;
    a.ms->status = last_status;
  }
}

}  // namespace ghc
