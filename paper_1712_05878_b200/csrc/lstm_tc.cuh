// lstm_tc.cuh — tensor-core variant of the cluster-resident sync round.
//
// Same math and the same round plumbing (ClusterXchg, lstm_round.cuh) as
// lstm_round_kernel, different sample phase.  Instead of one warp per sample
// with one lane per hidden unit (FFMA chains, 20 of 32 lanes busy), the 8
// samples of a CTA step through time TOGETHER and every contraction runs on
// the warp-level tensor path (mma.sync m16n8k8, 3×TF32 split so products keep
// fp32 accuracy: a·b ≈ a_hi·b_hi + a_hi·b_lo + a_lo·b_hi):
//
//   forward  (nn.cpp:160-200)  Z_t[4H × 8] = [Wh | Wx | b] · [h_{t-1}; x_t; 1]
//            M = gate rows, N = the CTA's 8 samples, K = H+D+1 padded to 8.
//            Rows are permuted so an m-tile holds the 4 gates of 4 units; a
//            4×4 butterfly transpose (4 shuffles) then gives every lane the
//            four gates of ONE (unit, sample) pair — all 32 lanes run the cell.
//   backward (nn.cpp:351-392)  dh_{t-1}[H × 8] = Whᵀ · dz_t, K = 4H split over
//            the CTA's warps, partials summed in fixed order.
//   weights  (nn.cpp:394-420)  dW[4H × (H+D+1)] = Σ_{t,s} dz_t,s ⊗ [h_{t-1}; x_t; 1]
//            one GEMM over K = (t, s) writing the CTA partial directly (no
//            per-warp partials to reduce).
//
// Measured on B200 (tools/mma_bench.cu): m16n8k8 tf32 = 21-cycle latency,
// one issue per 8 cycles per SM sub-partition — the per-timestep chains here
// are 12 MMAs deep at most.  Requires H % 4 == 0 (4 units per m-tile).
#pragma once

#include <type_traits>

#include "lstm_round.cuh"

namespace ghc {

constexpr int kTcSamples = 8;  // samples per CTA pass = MMA N

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// x = hi + lo, both TF32 (hi + lo reconstructs x exactly for the head).
__device__ __forceinline__ float2 split_tf32(float x) {
  const uint32_t h = tf32_rna(x);
  return make_float2(__uint_as_float(h), __uint_as_float(tf32_rna(x - __uint_as_float(h))));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// d += A·B in 3×TF32 (small terms first).  b = {b0_hi, b1_hi, b0_lo, b1_lo}
// (one LDS.128 from a fragment-ordered plane, see TcLayout::frag_off).
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     float4 b) {
  const uint32_t bh0 = __float_as_uint(b.x), bh1 = __float_as_uint(b.y);
  mma_tf32(d, al[0], al[1], al[2], al[3], bh0, bh1);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], __float_as_uint(b.z), __float_as_uint(b.w));
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
}
__device__ __forceinline__ void split_frag(const float (&v)[4], uint32_t (&h)[4], uint32_t (&l)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 s = split_tf32(v[i]);
    h[i] = __float_as_uint(s.x);
    l[i] = __float_as_uint(s.y);
  }
}
// 4×4 transpose across the lanes (lane ^ 4, lane ^ 8) that share c and g>>2:
// on entry lane q = g&3 holds element i of row q, on exit element i of column q.
__device__ __forceinline__ void transpose4(float (&e)[4], int q) {
  const bool b0 = q & 1;
  float x0 = b0 ? e[0] : e[1], x1 = b0 ? e[2] : e[3];
  x0 = __shfl_xor_sync(0xffffffffu, x0, 4);
  x1 = __shfl_xor_sync(0xffffffffu, x1, 4);
  if (b0) {
    e[0] = x0;
    e[2] = x1;
  } else {
    e[1] = x0;
    e[3] = x1;
  }
  const bool b1 = q & 2;
  float y0 = b1 ? e[0] : e[2], y1 = b1 ? e[1] : e[3];
  y0 = __shfl_xor_sync(0xffffffffu, y0, 8);
  y1 = __shfl_xor_sync(0xffffffffu, y1, 8);
  if (b1) {
    e[0] = y0;
    e[1] = y1;
  } else {
    e[2] = y0;
    e[3] = y1;
  }
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int D, int H, int T, int K, int CS>
struct TcLayout {
  using N = LstmNet<D, H, T, K>;
  static_assert(H % 4 == 0, "4 units per forward m-tile");
  static constexpr int S = kTcSamples;                 // samples per CTA pass (MMA N)
  static constexpr int NW = 8;                         // warps per CTA
  static constexpr int G4 = 4 * H;
  static constexpr int KC = (H + D + 1 + 7) & ~7;      // [h_{t-1} | x_t | 1 | 0…]
  static constexpr int KS = KC / 8;                    // forward k-steps
  // AF / DZ rows are stored in B-fragment order: for k-step ks and c = 0..3
  // the 4 floats {hi(k), hi(k+4), lo(k), lo(k+4)}, k = 8ks + c, so one
  // LDS.128 yields a lane's whole 3×TF32 B fragment.  Row strides ≡ 16 mod 32
  // floats keep the 8 lanes of an LDS.128 phase on distinct banks.
  static constexpr int row_stride(int ks) { return 16 * ks + ((ks & 1) ? 0 : 16); }
  static constexpr int RSA = row_stride(KS);           // AF row (one (t, s))
  static constexpr int MTF = G4 / 16;                  // forward m-tiles (warps)
  static_assert(MTF <= NW, "H ≤ 32");
  static constexpr int MTH = (H + 15) / 16;            // dh m-tiles (units)
  static constexpr int HP = MTH * 16;
  static constexpr int KSH = G4 / 8;                   // dh k-steps (gate rows)
  static constexpr int KP = NW / MTH;                  // dh k-split over warps
  static constexpr int KSHW = (KSH + KP - 1) / KP;     // k-steps per dh warp (max)
  static constexpr int RSD = row_stride(KSH);          // DZ row (one (t, s))
  static constexpr int NTW = KS;                       // weight-grad n-tiles
  static constexpr int MTW = G4 / 16;                  // weight-grad m-tiles
  static constexpr int XWP = (T * D + 3) & ~3;
  static constexpr int E = N::P + 1;
  static constexpr int SL = (((E + CS - 1) / CS) + 3) & ~3;
  static constexpr int EP = SL * CS;
  // shared memory map (floats, 16-B aligned sections)
  static constexpr int r4(int v) { return (v + 3) & ~3; }
  static constexpr int O_W0 = 0;
  static constexpr int O_W1 = O_W0 + N::PPAD;
  static constexpr int O_PART = O_W1 + N::PPAD;                      // CTA partial [P+1]
  static constexpr int O_VSL = O_PART + N::PPAD;                     // vsl[SL] vtmp[SL] badv[CS]
  static constexpr int O_AF = O_VSL + 2 * SL + r4(CS);               // [T+1][S][RSA]
  static constexpr int O_CACHE = O_AF + (T + 1) * S * RSA;           // [T][H][S][8]
  static constexpr int O_DZ = O_CACHE + T * H * S * 8;               // [T][S][RSD]
  static constexpr int O_DHP = O_DZ + T * S * RSD;                   // [KP][HP][S]
  static constexpr int O_XST = O_DHP + KP * HP * S;                  // [2][S][XWP]
  static constexpr int O_LAB = O_XST + 2 * S * XWP;                  // ints: lab[2][S], next[S]
  static constexpr int O_DZK = O_LAB + r4(3 * S);                    // [S][K]
  static constexpr int O_LOSS = O_DZK + r4(S * K);                   // [S]
  static constexpr int TOTAL = O_LOSS + S;
  static size_t smem_bytes(int) { return sizeof(float) * (size_t)TOTAL; }
  // offset of hi(k) inside a fragment-ordered row; lo(k) is at +2
  __device__ static int frag_off(int k) { return (k >> 3) * 16 + (k & 3) * 4 + ((k >> 2) & 1); }
};

__device__ __forceinline__ void put_split(float* row, int off, float v) {
  const float2 p = split_tf32(v);
  row[off] = p.x;
  row[off + 2] = p.y;
}

template <int D, int H, int T, int K, int CS>
__global__ void __launch_bounds__(256, 1) lstm_round_tc_kernel(StepArgs a) {
  using N = LstmNet<D, H, T, K>;
  using L = TcLayout<D, H, T, K, CS>;
  constexpr int S = L::S, KS = L::KS, RSA = L::RSA, RSD = L::RSD, HP = L::HP, KP = L::KP;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = gridDim.x;
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  float* cpart = smem + L::O_PART;
  float* AF = smem + L::O_AF;
  float* cache = smem + L::O_CACHE;
  float* DZ = smem + L::O_DZ;
  float* dhp = smem + L::O_DHP;
  float* xst = smem + L::O_XST;
  int* lab = reinterpret_cast<int*>(smem + L::O_LAB);
  float* dzk = smem + L::O_DZK;
  float* lss = smem + L::O_LOSS;

  ClusterXchg<N::P, L::SL, L::EP, CS> xc;
  xc.init(a, cluster, smem + L::O_VSL, smem + L::O_VSL + L::SL,
          reinterpret_cast<int*>(smem + L::O_VSL + 2 * L::SL));
  unsigned long long round0 = 0;
  int cur = 0;
  const bool sgd = xc.sgd;
  const bool bwd = a.mode != MODE_FWD;
  if (sgd) {
    cur = __ldcg(&a.ms->cur);
    round0 = __ldcg(&a.ms->round);
  }
  float* gw = sgd ? (cur ? a.w1 : a.w0) : nullptr;
  float* gv = sgd ? (cur ? a.v1 : a.v0) : nullptr;
  xc.load_state(a, sgd ? gw : a.w_in, gv, smem + L::O_W0);
  float* wa = smem + L::O_W0;
  float* wb = smem + L::O_W1;

  // AF rows: h_{-1} = 0, bias column = 1, K padding = 0 (x columns per pass).
  for (int i = threadIdx.x; i < (T + 1) * S * RSA; i += blockDim.x) AF[i] = 0.0f;
  __syncthreads();
  for (int i = threadIdx.x; i < (T + 1) * S; i += blockDim.x) AF[i * RSA + L::frag_off(H + D)] = 1.0f;

  auto first_sample = [&](int r, int& s0, int& s1) {
    const int n = a.counts ? __ldg(a.counts + r) : a.n;
    const int spc = (n + G - 1) / G;
    s0 = blockIdx.x * spc;
    s1 = min(n, s0 + spc);
  };
  auto row_of = [&](int r, int s) {
    // no gather table: round r reads rows r*stride + s (stride 0: rows s)
    return a.idx ? __ldg(a.idx + (long long)r * a.stride + s) : (int)((long long)r * a.stride + s);
  };
  // warp w stages sample slot w of a pass: x row (cp.async) + label
  auto fetch_nocommit = [&](int row, int b) {
    const float* xrow = a.x + (long long)row * (T * D);
    float* dst = xst + (b * S + warp) * L::XWP;
    for (int i = lane; i < T * D; i += 32) cp_async4(dst + i, xrow + i);
    if (lane == 0) cp_async4(lab + b * S + warp, a.y + row);
  };
  auto fetch_idx_nocommit = [&](int r) {  // slot w's gather index of round r → lab[2S+w]
    if (!a.idx || lane != 0 || r >= a.rounds) return;
    int sx, sx1;
    first_sample(r, sx, sx1);
    if (sx + warp < sx1) cp_async4(lab + 2 * S + warp, a.idx + (long long)r * a.stride + sx + warp);
  };
  if (a.pipelined) {
    int s0, s1;
    first_sample(0, s0, s1);
    if (s0 + warp < s1) fetch_nocommit(row_of(0, s0 + warp), 0);
    fetch_idx_nocommit(1);
    cp_async_commit();
  }
  __syncthreads();

  for (int r = 0; r < a.rounds; ++r) {
    const int n = a.counts ? __ldg(a.counts + r) : a.n;
    const float scale = sgd ? 1.0f / (float)n : a.grad_scale;
    unsigned long long* pr =
        a.probe ? a.probe + ((long long)r * gridDim.x + blockIdx.x) * 16 : nullptr;
    if (pr && threadIdx.x == 0) pr[0] = globaltimer();
    for (int p = threadIdx.x; p < N::PPAD; p += blockDim.x) cpart[p] = 0.0f;

    int s0, s1;
    first_sample(r, s0, s1);
    if (a.pipelined) {
      // rows of round r / indices of round r+1 were requested a round ago;
      // request round r+1's rows and round r+2's indices before computing
      cp_async_wait<0>();
      __syncwarp();
      if (r + 1 < a.rounds) {
        int sn0, sn1;
        first_sample(r + 1, sn0, sn1);
        const int row = a.idx ? lab[2 * S + warp] : (int)((long long)(r + 1) * a.stride + sn0 + warp);
        __syncwarp();
        if (sn0 + warp < sn1) fetch_nocommit(row, (r + 1) & 1);
        fetch_idx_nocommit(r + 2);
        cp_async_commit();
      }
    }

    // ---------------- one pass per 8 samples ----------------
    for (int sb = s0; sb < s1; sb += S) {
      const int cnt = min(S, s1 - sb);
      const int buf = a.pipelined ? (r & 1) : 0;
      if (!a.pipelined) {  // synchronous staging (batches > 8 samples per CTA)
        if (warp < cnt) {
          const int row = row_of(r, sb + warp);
          float* dst = xst + warp * L::XWP;
          for (int i = lane; i < T * D; i += 32) dst[i] = __ldg(a.x + (long long)row * (T * D) + i);
          if (lane == 0) lab[warp] = __ldg(a.y + row);
        }
      }
      __syncthreads();  // staged rows visible; previous pass done with AF/cache
      for (int i = threadIdx.x; i < S * T * D; i += blockDim.x) {
        const int s = i / (T * D), rem = i % (T * D);
        const int t = rem / D, d = rem % D;
        const float v = s < cnt ? xst[(buf * S + s) * L::XWP + rem] : 0.0f;
        put_split(AF + (t * S + s) * RSA, L::frag_off(H + d), v);
      }
      __syncthreads();
      if (pr && threadIdx.x == 0) pr[8] = globaltimer();

      // ---- forward recurrence: warp m owns units 4m..4m+3 (all 4 gates) ----
      if (warp < L::MTF) {
        uint32_t ah[KS][4], al[KS][4];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          float v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rho = g + 8 * (i & 1);              // a0:(g,c) a1:(g+8,c) a2:(g,c+4) a3:(g+8,c+4)
            const int k = 8 * ks + c + 4 * (i >> 1);
            const int row = (rho & 3) * H + 4 * warp + (rho >> 2);  // gate q = rho&3, unit
            v[i] = k < H ? wa[N::OFF_WH + row * H + k]
                         : (k < H + D ? wa[N::OFF_WX + row * D + (k - H)]
                                      : (k == H + D ? wa[N::OFF_B + row] : 0.0f));
          }
          split_frag(v, ah[ks], al[ks]);
        }
        const int q = g & 3;
        const int uu = 4 * warp + (g >> 2) + 2 * (q >> 1);
        const int ss = 2 * c + (q & 1);
        float cst = 0.0f;
#pragma unroll 1
        for (int t = 0; t < T; ++t) {
          float acc[KS][4];
          const float4* brow = reinterpret_cast<const float4*>(AF + (t * S + g) * RSA) + c;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[ks][i] = 0.0f;
            mma3(acc[ks], ah[ks], al[ks], brow[4 * ks]);
          }
          float e[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            e[i] = acc[0][i];
#pragma unroll
            for (int ks = 1; ks < KS; ++ks) e[i] += acc[ks][i];
          }
          transpose4(e, q);  // e = pre-activations i, f, g, o of (uu, ss)
          const float ig = sigmoid_f(e[0]);
          const float fg = sigmoid_f(e[1]);
          const float gg = tanh_f(e[2]);
          const float og = sigmoid_f(e[3]);
          cst = fmaf(fg, cst, ig * gg);
          const float tc = tanh_f(cst);
          float* ct = cache + ((t * H + uu) * S + ss) * 8;
          reinterpret_cast<float4*>(ct)[0] = make_float4(ig, fg, gg, og);
          reinterpret_cast<float2*>(ct)[2] = make_float2(cst, tc);
          put_split(AF + ((t + 1) * S + ss) * RSA, L::frag_off(uu), og * tc);
          named_bar(1, 32 * L::MTF);
        }
      }
      __syncthreads();
      if (pr && threadIdx.x == 0) pr[9] = globaltimer();

      // ---- softmax + loss (nn.cpp:202-248), warp w = sample slot w ----
      {
        const int s = warp;
        const bool valid = s < cnt;
        const bool act = lane < H;
        const int j = act ? lane : 0;
        const float* hrow = AF + (T * S + s) * RSA + L::frag_off(j);
        const float hT = act ? hrow[0] + hrow[2] : 0.0f;
        int label = valid ? lab[(a.pipelined ? (r & 1) : 0) * S + s] : 0;
        if (label < 0 || label >= K) {
          if (lane == 0 && valid) atomicOr(a.err, 1);
          label = 0;
        }
        const float scl = valid ? scale : 0.0f;
        float z[K], ek[K];
        float zmax = -3.0e38f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          z[k] = warp_sum(act ? wa[N::OFF_WS + k * H + j] * hT : 0.0f) + wa[N::OFF_BS + k];
          zmax = fmaxf(zmax, z[k]);
        }
        float den = 0.0f, zy = 0.0f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          ek[k] = expf(z[k] - zmax);
          den += ek[k];
          if (k == label) zy = z[k];
        }
        const float inv = 1.0f / den;
        if (lane == 0) lss[s] = valid ? logf(den) - (zy - zmax) : 0.0f;
        if (valid && a.probs_out && lane < K) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (lane == k) a.probs_out[(long long)(sb + s) * K + k] = ek[k] * inv;
        }
        if (bwd) {  // nn.cpp:276-311: dz = (p - onehot)·scale, dh_T = Wsᵀ dz
          float dh = 0.0f;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float d = (ek[k] * inv - (k == label ? 1.0f : 0.0f)) * scl;
            if (lane == 0) dzk[s * K + k] = d;
            dh = fmaf(act ? wa[N::OFF_WS + k * H + j] : 0.0f, d, dh);
          }
          if (act) dhp[j * S + s] = dh;
        }
      }
      __syncthreads();
      // head gradients and loss: fixed-order sums over the pass's samples
      for (int i = threadIdx.x; i < K * H + K + 1; i += blockDim.x) {
        if (i < K * H) {
          if (!bwd) continue;
          const int k = i / H, j = i % H;
          float acc = 0.0f;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const float* hrow = AF + (T * S + s) * RSA + L::frag_off(j);
            acc = fmaf(dzk[s * K + k], hrow[0] + hrow[2], acc);
          }
          cpart[N::OFF_WS + i] += acc;
        } else if (i < K * H + K) {
          if (!bwd) continue;
          const int k = i - K * H;
          float acc = 0.0f;
#pragma unroll
          for (int s = 0; s < S; ++s) acc += dzk[s * K + k];
          cpart[N::OFF_BS + k] += acc;
        } else {
          float acc = 0.0f;
#pragma unroll
          for (int s = 0; s < S; ++s) acc += lss[s];
          cpart[N::P] += acc;
        }
      }
      if (pr && threadIdx.x == 0) pr[10] = globaltimer();

      if (bwd) {
        // ---- BPTT chain (nn.cpp:351-392): thread (u, s) elementwise, dh on MMA ----
        const bool ew = threadIdx.x < H * S;
        const int u = threadIdx.x / S, s = threadIdx.x % S;
        const int mt = warp % L::MTH, kp = warp / L::MTH;
        const bool mw = warp < L::MTH * KP;
        uint32_t bh[L::KSHW][4], bl[L::KSHW][4];
        if (mw) {
#pragma unroll
          for (int jj = 0; jj < L::KSHW; ++jj) {
            const int ks = kp + KP * jj;
            float v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int uu = 16 * mt + g + 8 * (i & 1);
              const int rr = 8 * ks + c + 4 * (i >> 1);
              v[i] = (ks < L::KSH && uu < H) ? wa[N::OFF_WH + rr * H + uu] : 0.0f;
            }
            split_frag(v, bh[jj], bl[jj]);
          }
        }
        float dc = 0.0f;
#pragma unroll 1
        for (int t = T - 1; t >= 0; --t) {
          if (ew) {
            float dh = dhp[u * S + s];
            if (t < T - 1)
#pragma unroll
              for (int k2 = 1; k2 < KP; ++k2) dh += dhp[(k2 * HP + u) * S + s];
            const float* ct = cache + ((t * H + u) * S + s) * 8;
            const float4 g4 = reinterpret_cast<const float4*>(ct)[0];
            const float ig = g4.x, fg = g4.y, gg = g4.z, og = g4.w;
            const float tc = ct[5];
            const float cp = t > 0 ? cache[(((t - 1) * H + u) * S + s) * 8 + 4] : 0.0f;
            const float dout = dh * tc;
            dc = fmaf(dh * og, 1.0f - tc * tc, dc);
            const float di = dc * gg, dg = dc * ig, df = dc * cp;
            float* dzt = DZ + (t * S + s) * RSD;
            put_split(dzt, L::frag_off(0 * H + u), di * ig * (1.0f - ig));
            put_split(dzt, L::frag_off(1 * H + u), df * fg * (1.0f - fg));
            put_split(dzt, L::frag_off(2 * H + u), dg * (1.0f - gg * gg));
            put_split(dzt, L::frag_off(3 * H + u), dout * og * (1.0f - og));
            dc *= fg;
          }
          __syncthreads();
          if (t == 0) break;
          if (mw) {  // dh_{t-1}[u][s] partial over this warp's gate rows
            float acc[L::KSHW][4];
            const float4* brow = reinterpret_cast<const float4*>(DZ + (t * S + g) * RSD) + c;
#pragma unroll
            for (int jj = 0; jj < L::KSHW; ++jj) {
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[jj][i] = 0.0f;
              const int ks = min(kp + KP * jj, L::KSH - 1);  // past the end: A = 0
              mma3(acc[jj], bh[jj], bl[jj], brow[4 * ks]);
            }
            float e[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              e[i] = acc[0][i];
#pragma unroll
              for (int jj = 1; jj < L::KSHW; ++jj) e[i] += acc[jj][i];
            }
            float* o = dhp + (kp * HP + 16 * mt + g) * S + 2 * c;
            reinterpret_cast<float2*>(o)[0] = make_float2(e[0], e[1]);
            reinterpret_cast<float2*>(o + 8 * S)[0] = make_float2(e[2], e[3]);
          }
          __syncthreads();
        }
        if (pr && threadIdx.x == 0) pr[11] = globaltimer();

        // ---- weight gradients: dW[r][k] = Σ_{t,s} dz[t][s][r] · AF[t][s][k] ----
        // M = gate rows (MTW m-tiles), N = [h|x|1] columns (NTW n-tiles),
        // K = (t, s).  Warps 0..MF-1 own whole rows of output tiles (each A
        // fragment loaded once per t); the MTW-MF leftover m-tiles are split
        // per n-tile over the warps starting at 4, so the 4 SM sub-partitions
        // issue equal HMMA counts for the bench shape (MTW = 5).
        auto wgrad_tiles = [&](auto nt_count, int mt2, int nt0) {
          constexpr int NT = decltype(nt_count)::value;
          float acc[NT][4];
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][i] = 0.0f;
          const int o0 = L::frag_off(16 * mt2 + g), o1 = L::frag_off(16 * mt2 + g + 8);
#pragma unroll 2
          for (int t = 0; t < T; ++t) {
            // A = dzᵀ: rows r = 16mt+g (+8), cols s = c (+4);  B = AF: rows s, col k
            const float* d0 = DZ + (t * S + c) * RSD;
            const float* d1 = d0 + 4 * RSD;
            const uint32_t ah2[4] = {__float_as_uint(d0[o0]), __float_as_uint(d0[o1]),
                                     __float_as_uint(d1[o0]), __float_as_uint(d1[o1])};
            const uint32_t al2[4] = {__float_as_uint(d0[o0 + 2]), __float_as_uint(d0[o1 + 2]),
                                     __float_as_uint(d1[o0 + 2]), __float_as_uint(d1[o1 + 2])};
            const float* b0 = AF + (t * S + c) * RSA;
            const float* b1 = b0 + 4 * RSA;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const int ob = L::frag_off(8 * (nt0 + j) + g);
              mma3(acc[j], ah2, al2, make_float4(b0[ob], b1[ob], b0[ob + 2], b1[ob + 2]));
            }
          }
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int rr = 16 * mt2 + g + 8 * (i >> 1);
              const int k = 8 * (nt0 + j) + 2 * c + (i & 1);
              int idx = -1;
              if (k < H) idx = N::OFF_WH + rr * H + k;
              else if (k < H + D) idx = N::OFF_WX + rr * D + (k - H);
              else if (k == H + D) idx = N::OFF_B + rr;
              if (idx >= 0) cpart[idx] += acc[j][i];
            }
        };
        constexpr int MF = (L::MTW / 4) * 4;
        for (int mt2 = warp; mt2 < MF; mt2 += L::NW)
          wgrad_tiles(std::integral_constant<int, L::NTW>{}, mt2, 0);
        for (int i = (warp + L::NW - 4) % L::NW; i < (L::MTW - MF) * L::NTW; i += L::NW)
          wgrad_tiles(std::integral_constant<int, 1>{}, MF + i / L::NTW, i % L::NTW);
        if (pr && threadIdx.x == 0) pr[12] = globaltimer();
      }
    }
    __syncthreads();
    if (pr && threadIdx.x == 0) pr[2] = pr[3] = globaltimer();
    cluster.sync();  // CTA partials of the whole cluster complete
    if (pr && threadIdx.x == 0) pr[4] = globaltimer();
    xc.exchange(a, cluster, r, cpart, wa, wb, pr, n);
  }
  xc.publish(a, gw, gv, wa, round0);
}

}  // namespace ghc
