// lstm_round.cuh — cluster-resident variant of the fused sync-round kernel.
//
// Same per-sample math as lstm_step.cuh (lstm_sample), different round
// plumbing, designed from the measured B200 sync costs (DESIGN.md §Sync:
// grid-wide flag barrier ≈ 1.4-2.5 µs, hardware cluster barrier ≈ 0.28 µs):
//
//   1. each CTA reduces its warps' gradients into a CTA partial in smem;
//   2. cluster barrier; CTA j of each cluster (CS = 4 or 8 CTAs, chosen per
//      plan from occupancy) reduces slice j of the
//      gradient over its cluster through DSMEM (fixed peer order) and stores
//      that cluster partial to HBM/L2;
//   3. ONE column barrier per round: the NC CTAs holding slice j (one per
//      cluster) wait only for each other;
//   4. CTA j sums slice j over the NC cluster partials (fixed order — the
//      result is bit-identical in every cluster), applies sgd_step
//      (optim.cpp:39-65) with its velocity slice kept in smem across rounds,
//      and stores the new weights of slice j straight into the weight buffer
//      of every CTA of its cluster (DSMEM stores);
//   5. cluster barrier; the non-finite flag is OR-ed over the cluster (whose CS
//      slices cover the whole gradient → a global decision) and the update is
//      committed or rejected (optim.cpp:49-51) by a buffer swap — weights
//      never round-trip through global memory between rounds.
#pragma once

#include <cooperative_groups.h>

#include "lstm_step.cuh"

namespace ghc {

namespace cg = cooperative_groups;

// Samples interleaved per warp (static ILP, lstm_samples<..., SPW>).
#ifndef GHC_SPW
#define GHC_SPW 1
#endif
constexpr int kSamplesPerWarp = GHC_SPW;

// ---------------------------------------------------------------------------
// Single-GPU exchange, reduce-scatter / all-gather over epoch-tagged L2 rows
// (the default of the SIMT round kernel).  Per round:
//   a. every CTA pushes slice q of its CTA partial to cluster peer q
//      (st.async + the peer's mbarrier complete_tx — no cluster barrier);
//   b. CTA j sums its CS received rows (rank order) = the cluster partial of
//      slice j and stores it to L2 as 64-bit (value, tag) elements;
//   c. CTA (cluster c, rank j) polls the NC cluster rows of SUB-slice c of
//      slice j until every tag is this round's, sums them in cluster order,
//      applies sgd_step to the sub-slice (its velocity lives here) and stores
//      the new weights tagged (tag = 2·epoch + non-finite bit);
//   d. CTA j polls the NC sub-slices of slice j, ORs their non-finite bits and
//      pushes the slice (+ its flag) to every CTA of its cluster (st.async);
//   e. every CTA waits for its CS slices; reject (optim.cpp:49-51) if any flag.
// A 64-bit element store is single-copy atomic, so a reader that sees the
// tag sees the value: no fences, no flag barriers.  Rows are double-buffered
// by epoch parity; a cluster reaches round r+2's stores only after every
// cluster consumed round r (its round r+1 rows depend on them).
template <int P, int SL, int EP, int CS, bool MULTI = false>
struct ClusterRS {
  static constexpr int E = P + 1;
  static constexpr int kRowBatch = 32;  // tagged cluster rows polled per batch (all of them for ≤ 32 clusters)
  float* recv;           // [2][CS][SL]
  float* vsub;           // [SL] velocity of this CTA's sub-slice
  float* vnew;           // [SL]
  float* wnew;           // [SL] spare (the new weights go straight to the tagged row)
  int* badr;             // [2][CS][4] non-finite flags pushed by the slice owners
  uint64_t* mbp;         // [2] partial rows arrived
  uint64_t* mbw;         // [2] new weights arrived
  int crank, cid, NC, e0, SS, s0, s1;
  int GX, NCr, vrank, rank, cl;  // ranks; clusters per rank; this CTA's (virtual) rank, cluster in rank
  unsigned epoch;   // this plan's round counter: tags of the rank-local rows
  unsigned xepoch;  // the cross-rank exchange's counter (kept with its buffers, equal on all ranks)
  unsigned long long accepted, rejected, acc_samples;
  int last_status;
  bool sgd;

  __device__ static uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
  __device__ static uint32_t mapa(const void* p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sa(p)), "r"(rank));
    return r;
  }
  __device__ static void st_async(uint32_t addr, float4 v, uint32_t mbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mbar)
        : "memory");
  }
  __device__ static void wait(uint64_t* bar, unsigned parity) {
    for (long long spin = 0;; ++spin) {
      uint32_t done;
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(sa(bar)), "r"(parity)
          : "memory");
      if (done) return;
      if (spin > (1ll << 28)) __trap();  // never hang the GPU on a protocol bug
    }
  }
  __device__ static void st_tag(unsigned long long* p, float v, unsigned tag) {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
  }
  __device__ static unsigned long long ld_tag(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
  }
  // four consecutive tagged elements (32-B aligned): two 16-B loads
  __device__ static void ld_tag4(const unsigned long long* p, unsigned long long (&w)[4]) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w[0]), "=l"(w[1]) : "l"(p) : "memory");
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w[2]), "=l"(w[3]) : "l"(p + 2) : "memory");
  }

  // smem: recv (2·CS·SL floats), vsub / vnew / wnew (SL each), badr (8·CS ints), 4 mbarriers
  static constexpr int smem_floats() { return 2 * CS * SL + 3 * SL + 8 * CS + 8; }

  __device__ void init(const StepArgs& a, cg::cluster_group& cluster, float* base) {
    recv = base;
    vsub = recv + 2 * CS * SL;
    vnew = vsub + SL;
    wnew = vnew + SL;
    badr = reinterpret_cast<int*>(wnew + SL);
    mbp = reinterpret_cast<uint64_t*>(badr + 8 * CS);  // 8-byte aligned: offsets are multiples of 4 floats
    mbw = mbp + 2;
    crank = (int)cluster.block_rank();
    cid = blockIdx.x / CS;
    NC = gridDim.x / CS;
    e0 = crank * SL;
    GX = max(1, a.GX);
    NCr = NC / max(1, a.VR);
    vrank = cid / NCr;
    cl = cid % NCr;
    rank = a.rank0 + vrank;
    SS = (((SL + NCr - 1) / NCr) + 3) & ~3;
    s0 = e0 + cl * SS;
    s1 = min(min(e0 + SL, E), s0 + SS);
    GHC_CHECK(crank < CS && cid < NC && vrank < max(1, a.VR) && cl < NCr && SL % 4 == 0);
    GHC_CHECK(s1 <= s0 || (s0 >= e0 && s1 <= e0 + SL && s1 - s0 <= SL && s1 <= EP));
    GHC_CHECK(a.GX <= 1 || rank < GX);
    epoch = __ldcg(a.bar);
    xepoch = GX > 1 ? __ldcg(a.gcnt[rank] + CS * kFlagStride) : 0u;
    accepted = rejected = acc_samples = 0;
    last_status = 0;
    sgd = a.mode == MODE_SGD;
    if (threadIdx.x == 0) {
      for (int i = 0; i < 2; ++i) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(mbp + i)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(mbw + i)));
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }

  // Prologue: the current weights into shared memory (all loads of a
  // thread in flight before its stores — the loop with interleaved smem
  // stores serialised one L2 round trip per element) and the velocity of
  // this CTA's sub-slice.
  __device__ void load_state(const float* gw, const float* gv, float* wbuf) {
    const float vs = (sgd && s0 + (int)threadIdx.x < s1 && s0 + (int)threadIdx.x < P) ? __ldcg(gv + s0 + threadIdx.x) : 0.f;
    if ((reinterpret_cast<uintptr_t>(gw) & 15u) == 0) {
      constexpr int P4 = P / 4;
      const float4* g4 = reinterpret_cast<const float4*>(gw);
      for (int base = threadIdx.x; base < P4; base += 4 * blockDim.x) {
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = base + i * blockDim.x;
          v[i] = q < P4 ? __ldcg(g4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = base + i * blockDim.x;
          if (q < P4) reinterpret_cast<float4*>(wbuf)[q] = v[i];
        }
      }
      for (int p = 4 * P4 + threadIdx.x; p < P; p += blockDim.x) wbuf[p] = __ldcg(gw + p);
    } else {
      for (int p = threadIdx.x; p < P; p += blockDim.x) wbuf[p] = __ldcg(gw + p);
    }
    if (sgd) {
      if (s0 + (int)threadIdx.x < s1) vsub[threadIdx.x] = vs;
      for (int e = s0 + blockDim.x + threadIdx.x; e < s1; e += blockDim.x) vsub[e - s0] = e < P ? __ldcg(gv + e) : 0.f;
    }
  }

  // Push this rank's sum of element e into row `rank` of every rank's receive
  // rows (uint64 [2][GX][EP], P2P-mapped; system scope — the ranks are other
  // GPUs), then poll this rank's copy of the GX rows and sum in rank order.
  __device__ float cross_rank_sum(const StepArgs& a, int par, int e, float mine, unsigned tag) const {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(mine);
    GHC_CHECK(GX <= kMaxRanks && rank < GX && e < EP);
    for (int q = 0; q < GX; ++q) {
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.gpart[q]) +
                                ((long long)par * GX + rank) * EP + e;
      asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(dst), "l"(w) : "memory");
    }
    const unsigned long long* src =
        reinterpret_cast<const unsigned long long*>(a.gpart[rank]) + (long long)par * GX * EP + e;
    unsigned long long v[kMaxRanks];
    bool ok;
    long long spin = 0;
    do {
      if (++spin > (1ll << 26)) __trap();
      ok = true;
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q) {
        if (q >= GX) break;
        asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v[q]) : "l"(src + (long long)q * EP) : "memory");
        ok &= (unsigned)(v[q] >> 32) == tag;
      }
    } while (!ok);
    float t = 0.0f;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) {
      if (q >= GX) break;
      t += __uint_as_float((unsigned)v[q]);
    }
    return t;
  }

  // wparts: nw warp partials [nw][pstride] (P gradient entries + loss slot);
  // their sum (warp order) is the CTA partial, formed while pushing.
  // r: round index within the segment (loss slot); rb: rounds run by this
  // launch so far (mbarrier phases — a resident launch serves many segments).
  __device__ void exchange(const StepArgs& a, int r, unsigned long long rb, float* loss_out,
                           const float* wparts, int nw, int pstride, float*& wa, float*& wb,
                           unsigned long long* pr, int ntot) {
    ++epoch;
    ++xepoch;
    const int par = epoch & 1;                 // L2 rows: epoch parity (survives launches)
    const int mb = (int)(rb & 1);              // mbarriers: re-initialised per launch
    const unsigned ph = (unsigned)(rb >> 1) & 1;
    const unsigned tag = epoch << 1;
    if (threadIdx.x == 0) {  // arm: bytes the peers will push this round
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(mbp + mb)),
                   "r"(CS * SL * 4)
                   : "memory");
      if (sgd)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(mbw + mb)),
                     "r"(CS * (SL * 4 + 16))
                     : "memory");
    }
    // (a) slice q of the CTA partial (Σ warp partials, warp order) → peer q
    for (int i = threadIdx.x; i < CS * (SL / 4); i += blockDim.x) {
      const int q = i / (SL / 4), k = 4 * (i % (SL / 4));
      const int e = q * SL + k;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < E) {
        GHC_CHECK_RANGE(wparts + (long long)(nw - 1) * pstride + e, 4, wparts, (long long)nw * pstride);
        v = reinterpret_cast<const float4*>(wparts + e)[0];
        for (int w = 1; w < nw; ++w) {
          const float4 u = reinterpret_cast<const float4*>(wparts + (long long)w * pstride + e)[0];
          v.x += u.x;
          v.y += u.y;
          v.z += u.z;
          v.w += u.w;
        }
      }
      GHC_CHECK_RANGE(recv + (mb * CS + crank) * SL + k, 4, recv, 2 * CS * SL);
      st_async(mapa(recv + (mb * CS + crank) * SL + k, q), v, mapa(mbp + mb, q));
    }
    wait(mbp + mb, ph);
    if (pr && threadIdx.x == 0) pr[4] = globaltimer();
    // (b) cluster partial of slice j → tagged L2 row
    unsigned long long* rows = a.tpart + (long long)par * NC * EP;
    for (int k = threadIdx.x; k < SL; k += blockDim.x) {
      float t = 0.0f;
#pragma unroll
      for (int q = 0; q < CS; ++q) t += recv[(mb * CS + q) * SL + k];
      GHC_CHECK(e0 + k < EP && cid < NC);
      st_tag(rows + (long long)cid * EP + e0 + k, t, tag);
    }
    if (pr && threadIdx.x == 0) pr[5] = globaltimer();
    // (c) sub-slice [s0, s1) over this rank's NCr clusters (cluster order);
    //     GX ranks: + one hop over NVLink — push the rank sum, tagged, into
    //     row `rank` of every rank's receive rows, then sum the GX rows in rank
    //     order (bit-identical on every rank) → sgd_step
    unsigned long long* tw = a.tw + ((long long)vrank * 2 + par) * EP;
    const unsigned long long* myrows = rows + (long long)vrank * NCr * EP;
    for (int e = s0 + threadIdx.x; e < s1; e += blockDim.x) {
      GHC_CHECK(e < EP && e - s0 < SL && vrank * NCr + NCr <= NC);
      float t = 0.0f;
      for (int c0 = 0; c0 < NCr; c0 += kRowBatch) {
        unsigned long long v[kRowBatch];
        bool ok;
        long long spin = 0;
        do {
          if (++spin > (1ll << 26)) __trap();  // never hang the GPU on a protocol bug
          ok = true;
#pragma unroll
          for (int i = 0; i < kRowBatch; ++i) {
            v[i] = c0 + i < NCr ? ld_tag(myrows + (long long)(c0 + i) * EP + e) : ((unsigned long long)tag << 32);
            ok &= (unsigned)(v[i] >> 32) == tag;
          }
        } while (!ok);
#pragma unroll
        for (int i = 0; i < kRowBatch; ++i)
          if (c0 + i < NCr) t += __uint_as_float((unsigned)v[i]);
      }
      if (GX > 1) t = cross_rank_sum(a, xepoch & 1, e, t, xepoch);
      if (e == P) {
        if constexpr (MULTI) {
          if (loss_out) loss_out[vrank] = t;  // worker vrank's loss sum
        } else {
          if (loss_out) loss_out[r] = t;
        }
      } else if (a.mode == MODE_GRAD) {
        if constexpr (MULTI) a.g_out[vrank * a.g_vstride + e] = t;  // worker vrank's gradient
        else a.g_out[e] = t;
      } else if (sgd) {
        // sgd_step (optim.cpp:59-60): v = mu*v - lr*g; w += v.  Each element
        // carries its own non-finite bit in its tag (2·epoch + bit); step (d)
        // ORs the bits of a slice and (e) the slices' flags, so one
        // non-finite entry anywhere rejects the whole update (optim.cpp:49-51)
        // without a CTA barrier here.
        const unsigned bad_e = is_finite_f(t) ? 0u : 1u;
        const float vn = fmaf(a.mu, vsub[e - s0], -a.lr * t);
        vnew[e - s0] = vn;
        st_tag(tw + e, wa[e] + vn, tag | bad_e);
      }
    }
    if (!sgd) {
      __syncthreads();
      return;
    }
    // weights-row elements that no sub-slice owns (e ≥ E, e == P) get a plain tag
    if (cl == 0)
      for (int e = max(E - 1, e0) + threadIdx.x; e < e0 + SL; e += blockDim.x)
        if (e >= E || e == P) st_tag(tw + e, 0.0f, tag);
    if (pr && threadIdx.x == 0) pr[6] = globaltimer();
    // (d) gather slice j of the new weights, OR the flags, push to the cluster
    int sbad = 0;
    for (int k = 4 * threadIdx.x; k < SL; k += 4 * blockDim.x) {
      GHC_CHECK(e0 + k + 4 <= EP);
      // two polls in flight (the second issued before the first is checked):
      // a value that lands is seen ≈ half an L2 round trip sooner
      unsigned long long v[4], u[4];
      auto ready = [&](const unsigned long long (&x)[4]) {
        bool ok = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) ok &= ((unsigned)(x[i] >> 32) | 1u) == (tag | 1u);
        return ok;
      };
      ld_tag4(tw + e0 + k, v);
      for (long long spin = 0;; ++spin) {
        if (spin > (1ll << 26)) __trap();
        ld_tag4(tw + e0 + k, u);
        if (ready(v)) break;
        ld_tag4(tw + e0 + k, v);
        if (ready(u)) {
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = u[i];
          break;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) sbad |= (int)((v[i] >> 32) & 1u);
      const float4 w4 = make_float4(__uint_as_float((unsigned)v[0]), __uint_as_float((unsigned)v[1]),
                                    __uint_as_float((unsigned)v[2]), __uint_as_float((unsigned)v[3]));
#pragma unroll
      for (int q = 0; q < CS; ++q) st_async(mapa(wb + e0 + k, q), w4, mapa(mbw + mb, q));
    }
    sbad = __syncthreads_or(sbad);
    if (threadIdx.x < CS)
      st_async(mapa(badr + (mb * CS + crank) * 4, threadIdx.x), make_float4(__int_as_float(sbad), 0.f, 0.f, 0.f),
               mapa(mbw + mb, threadIdx.x));
    if (pr && threadIdx.x == 0) pr[7] = globaltimer();
    // (e) all CS slices + flags landed → commit or reject
    wait(mbw + mb, ph);
    if (pr && threadIdx.x == 0) pr[13] = globaltimer();
    int rej = 0;
#pragma unroll
    for (int q = 0; q < CS; ++q) rej |= badr[(mb * CS + q) * 4];
    if (rej) {
      ++rejected;
      last_status = 2;  // GHC_ERR_NONFINITE: keep w/v (optim.cpp:49-51)
    } else {
      for (int e = s0 + threadIdx.x; e < s1; e += blockDim.x) vsub[e - s0] = vnew[e - s0];
      float* t = wa;
      wa = wb;
      wb = t;
      ++accepted;
      acc_samples += (unsigned long long)ntot;
      last_status = 0;
    }
    // No CTA barrier here: every thread waited on the mbarrier itself (the
    // new weights are visible to it), vsub/vnew entries are owned by one
    // thread, and the next writes into the other weight buffer come from
    // peers' step (d) of the next round, which needs this CTA's step (b) —
    // after the barrier that closes the next round's samples.
  }

  __device__ void publish(const StepArgs& a, float* gw, float* gv, const float* wa,
                          unsigned long long round0, unsigned long long rounds) {
    if (sgd) {
      if (cid == 0)
        for (int e = threadIdx.x; e < P; e += blockDim.x) gw[e] = wa[e];
      for (int e = s0 + threadIdx.x; e < s1 && e < P; e += blockDim.x) gv[e] = vsub[e - s0];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.bar[0] = epoch;
      if (GX > 1)
        for (int v = 0; v < max(1, a.VR); ++v) a.gcnt[a.rank0 + v][CS * kFlagStride] = xepoch;
      if (sgd) {
        a.ms->version += accepted;
        a.ms->rejected += rejected;
        a.ms->samples += acc_samples;
        a.ms->round = round0 + rounds;
        a.ms->status = last_status;
      }
    }
  }
};

template <int D, int H, int T, int K, int CS>
struct RoundLayout {
  using N = LstmNet<D, H, T, K>;
  static constexpr int SPW = kSamplesPerWarp;
  static constexpr int E = N::P + 1;                          // grad + loss
  static constexpr int SL = (((E + CS - 1) / CS) + 3) & ~3;   // slice per cluster rank
  static constexpr int EP = SL * CS;                          // padded row
  // weight buffers receive whole slices (st.async) → at least EP floats
  static constexpr int WBP = N::PPAD > EP ? N::PPAD : EP;
  static constexpr int RSF = ClusterRS<N::P, SL, EP, CS>::smem_floats();
  __host__ __device__ static size_t smem_bytes(int nw) {
    return sizeof(float) * (size_t)(2 * WBP + nw * SPW * N::WARP_FLOATS + nw * N::PPAD + 2 * SL +
                                    ((CS + 3) & ~3) + RSF);
  }
};

// Steps 2–5 of the round (file header) and the final publish, shared by the
// SIMT kernel below and the tensor-core kernel of lstm_tc.cuh.  The caller
// holds the complete CTA partial (P gradient entries + loss in slot P) in its
// own shared memory at `cpart`, and every CTA of the cluster has passed a
// cluster.sync() since its partial was completed.
#ifndef GHC_XCHG_BATCH
#define GHC_XCHG_BATCH 32
#endif
constexpr int kXchgBatch = GHC_XCHG_BATCH;  // cluster-partial rows loaded per batch (step 4)

template <int P, int SL, int EP, int CS>
struct ClusterXchg {
  static constexpr int E = P + 1;
  float* vsl;   // [SL] velocity slice (SGD), kept in smem across rounds
  float* vtmp;  // [SL]
  int* badv;    // [CS] non-finite flags, written by peers
  int crank, cid, NC, e0, e1;
  int NCr, vrank, rank, cl;  // clusters per rank, this CTA's virtual/global rank, cluster in rank
  unsigned epoch, xepoch;
  unsigned long long accepted, rejected, acc_samples;
  int last_status;
  bool sgd;

  __device__ void init(const StepArgs& a, cg::cluster_group& cluster, float* vs, float* vt, int* bv) {
    vsl = vs;
    vtmp = vt;
    badv = bv;
    crank = (int)cluster.block_rank();
    cid = blockIdx.x / CS;
    NC = gridDim.x / CS;
    e0 = crank * SL;
    e1 = min(E, e0 + SL);
    NCr = NC / max(1, a.VR);
    vrank = cid / NCr;
    cl = cid % NCr;
    rank = a.rank0 + vrank;
    epoch = __ldcg(a.bar);
    // cross-rank exchange epoch: kept next to this rank's arrival counters
    xepoch = a.GX > 1 ? __ldcg(a.gcnt[rank] + CS * kFlagStride) : 0u;
    accepted = rejected = acc_samples = 0;
    last_status = 0;
    sgd = a.mode == MODE_SGD;
  }

  // Master weights/velocity of the current buffer → wbuf (all P) and vsl.
  __device__ void load_state(const StepArgs& a, const float* gw, const float* gv, float* wbuf) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) wbuf[p] = __ldcg(gw + p);
    if (sgd)
      for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) vsl[e - e0] = e < P ? __ldcg(gv + e) : 0.f;
  }

  // Σ_{i<nrow} rows[i][e..e+3] in row order, kXchgBatch L2 loads in flight.
  __device__ static float4 sum_rows(const float* rows, int nrow, long long stride, int e) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < nrow; c0 += kXchgBatch) {
      float4 v[kXchgBatch];
#pragma unroll
      for (int i = 0; i < kXchgBatch; ++i)
        v[i] = c0 + i < nrow ? __ldcg(reinterpret_cast<const float4*>(rows + (c0 + i) * stride + e))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < kXchgBatch; ++i) {
        t.x += v[i].x;
        t.y += v[i].y;
        t.z += v[i].z;
        t.w += v[i].w;
      }
    }
    return t;
  }

  // (4x) Cross-rank exchange of slice j over NVLink peer memory, "LL" style
  // (as NCCL's low-latency protocol): every value travels with the exchange
  // epoch in ONE 8-byte store, so a reader that sees the epoch sees the
  // value — no fences, no counters (a system-scope fence costs ~8 µs/round,
  // measured).  Receive buffer per rank: uint2 [2 parity][GX][EP].
  //   push: cluster cl of this rank sums sub-slice cl of slice j over the
  //         rank's NCr cluster partials (fixed order) and stores it, tagged,
  //         into row `rank` of EVERY rank's receive buffer;
  //   sum:  every CTA of column j polls the GX rows of slice j in its own
  //         receive buffer until all tags equal this epoch and adds them in
  //         rank order — bit-identical on every rank.
  // Parity double buffer: a rank pushes round r+2 only after every rank's
  // column-j CTAs pushed round r+1, i.e. after they finished reading round r.
  // (value, tag) as ONE 64-bit element: single-copy atomic in the PTX model
  // (a v2.b32 vector access is only atomic per 32-bit element)
  __device__ static void st_tagged(uint2* p, float v, unsigned tag) {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
  }
  __device__ static uint2 ld_tagged(const uint2* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return make_uint2((unsigned)w, (unsigned)(w >> 32));
  }
  __device__ void xchg_push(const StepArgs& a, int par, const float* gcol) {
    ++xepoch;
    const int SS = (((SL + NCr - 1) / NCr) + 3) & ~3;
    const int lo = e0 + cl * SS, hi = min(e1, lo + SS);
    for (int e = lo + 4 * threadIdx.x; e < hi; e += 4 * blockDim.x) {
      const float4 t = sum_rows(gcol, NCr, EP, e);
      for (int q = 0; q < a.GX; ++q) {
        uint2* dst = reinterpret_cast<uint2*>(a.gpart[q]) + ((long long)par * a.GX + rank) * EP + e;
        st_tagged(dst + 0, t.x, xepoch);
        st_tagged(dst + 1, t.y, xepoch);
        st_tagged(dst + 2, t.z, xepoch);
        st_tagged(dst + 3, t.w, xepoch);
      }
    }
  }
  // Σ_q row q of this rank's receive buffer at columns e..e+3, rank order.
  __device__ float4 xchg_sum(const StepArgs& a, int par, int e) const {
    const uint2* base = reinterpret_cast<const uint2*>(a.gpart[rank]) + (long long)par * a.GX * EP + e;
    uint2 v[kMaxRanks][4];
    bool ready;
    do {
      ready = true;
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q) {
        if (q >= a.GX) break;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          v[q][i] = ld_tagged(base + (long long)q * EP + i);
          ready &= v[q][i].y == xepoch;
        }
      }
    } while (!ready);
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) {
      if (q >= a.GX) break;
      t.x += __uint_as_float(v[q][0].x);
      t.y += __uint_as_float(v[q][1].x);
      t.z += __uint_as_float(v[q][2].x);
      t.w += __uint_as_float(v[q][3].x);
    }
    return t;
  }

  __device__ void exchange(const StepArgs& a, cg::cluster_group& cluster, int r, float* cpart,
                           float*& wa, float*& wb, unsigned long long* pr, int ntot) {
    const int par = r & 1;
    // ---- (2) slice j over the cluster via DSMEM → cluster partial in HBM ----
    float* grow = a.part + ((long long)par * NC + cid) * EP;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      float t = 0.0f;
#pragma unroll
      for (int q = 0; q < CS; ++q) t += cluster.map_shared_rank(cpart, q)[e];
      __stcg(grow + e, t);
    }
    if (pr && threadIdx.x == 0) pr[5] = globaltimer();

    // ---- (3) column barrier: the NC CTAs that own slice j ----
    ++epoch;
    __syncthreads();
    unsigned* flags = a.bar + 2 * kFlagStride;
    if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * kFlagStride, epoch);
    for (int c = vrank * NCr + threadIdx.x; c < (vrank + 1) * NCr; c += blockDim.x) {
      const unsigned* f = flags + (c * CS + crank) * kFlagStride;
      while ((int)(ld_relaxed_gpu(f) - epoch) < 0) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    if (pr && threadIdx.x == 0) pr[6] = globaltimer();

    // ---- (4) slice j over all clusters (fixed order) → update → broadcast ----
    // float4 columns: SL and EP are multiples of 4, e0 too.
    // One rank: sum the NC cluster partials of slice j (every cluster does
    // this redundantly — one barrier instead of two).  GX ranks: cross-rank
    // two-level reduce (4x below), then sum the GX rank partials of slice j.
    int bad = 0;
    const float* gcol = a.part + ((long long)par * NC + vrank * NCr) * EP;
    if (a.GX > 1) {
      xchg_push(a, par, gcol);
      if (pr && threadIdx.x == 0) pr[14] = pr[15] = globaltimer();
    }
    for (int e = e0 + 4 * threadIdx.x; e < e1; e += 4 * blockDim.x) {
      const float4 t = a.GX > 1 ? xchg_sum(a, par, e) : sum_rows(gcol, NCr, EP, e);
      const float tv[4] = {t.x, t.y, t.z, t.w};
      float wn[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ee = e + i;
        wn[i] = 0.0f;
        if (ee >= e1) continue;
        if (ee == P) {
          if (cid == 0 && a.loss_out) a.loss_out[r] = tv[i];
        } else if (a.mode == MODE_GRAD) {
          if (cid == 0) a.g_out[ee] = tv[i];
        } else if (sgd) {
          if (!is_finite_f(tv[i])) bad = 1;
          // sgd_step (optim.cpp:59-60): v = mu*v - lr*g; w += v
          const float vn = fmaf(a.mu, vsl[ee - e0], -a.lr * tv[i]);
          vtmp[ee - e0] = vn;
          wn[i] = wa[ee] + vn;
        }
      }
      if (sgd) {  // new weights → every CTA of the cluster (DSMEM, float4)
        const float4 w4 = make_float4(wn[0], wn[1], wn[2], wn[3]);
#pragma unroll
        for (int q = 0; q < CS; ++q)
          reinterpret_cast<float4*>(cluster.map_shared_rank(wb, q) + e)[0] = w4;
      }
    }
    if (sgd) {
      bad = __syncthreads_or(bad);
      if (threadIdx.x < CS) cluster.map_shared_rank(badv, (int)threadIdx.x)[crank] = bad;
    }
    if (pr && threadIdx.x == 0) pr[7] = globaltimer();
    cluster.sync();  // new weights + flags landed in every CTA of the cluster
    if (pr && threadIdx.x == 0) pr[13] = globaltimer();
    if (sgd) {
      int rej = 0;
#pragma unroll
      for (int q = 0; q < CS; ++q) rej |= badv[q];
      if (rej) {
        ++rejected;
        last_status = 2;  // GHC_ERR_NONFINITE: keep w/v (optim.cpp:49-51)
      } else {
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) vsl[e - e0] = vtmp[e - e0];
        float* t = wa;
        wa = wb;
        wb = t;
        ++accepted;
        acc_samples += (unsigned long long)ntot;
        last_status = 0;
      }
      __syncthreads();
    }
  }

  // Master state back to HBM (cluster 0 holds the same bits as every cluster).
  __device__ void publish(const StepArgs& a, float* gw, float* gv, const float* wa,
                          unsigned long long round0) {
    if (sgd && cid == 0) {
      for (int e = e0 + threadIdx.x; e < e1 && e < P; e += blockDim.x) {
        gw[e] = wa[e];
        gv[e] = vsl[e - e0];
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.bar[0] = epoch;
      if (a.GX > 1)
        for (int v = 0; v < max(1, a.VR); ++v) a.gcnt[a.rank0 + v][CS * kFlagStride] = xepoch;
      if (sgd) {
        a.ms->version += accepted;
        a.ms->rejected += rejected;
        a.ms->samples += acc_samples;
        a.ms->round = round0 + (unsigned long long)a.rounds;
        a.ms->status = last_status;
      }
    }
  }
};

// RES: the resident round service variant (commands from a.res); a separate
// instantiation so the ordinary launch carries none of its state (registers).
template <int D, int H, int T, int K, int CS, bool RES = false, bool MULTI = false>
__global__ void __launch_bounds__(256, 1) lstm_round_kernel(StepArgs a) {
  using N = LstmNet<D, H, T, K>;
  using RL = RoundLayout<D, H, T, K, CS>;
  constexpr int SL = RL::SL;
  constexpr int SPW = RL::SPW;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = gridDim.x;
  const unsigned long long t_entry = a.probe ? globaltimer() : 0ull;

  extern __shared__ __align__(16) float smem[];
  const int NW = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* wbuf0 = smem;
  float* wbuf1 = smem + RL::WBP;
  float* ws = smem + 2 * RL::WBP + warp * SPW * N::WARP_FLOATS;  // SPW sample slots
  float* wpart = smem + 2 * RL::WBP + NW * SPW * N::WARP_FLOATS;  // [NW][PPAD]; [0] = CTA partial
  float* vsl = wpart + NW * N::PPAD;                           // [SL] velocity slice
  ClusterRS<N::P, SL, RL::EP, CS, MULTI> rs;  // the round's exchange (one GPU or GX ranks)
#ifdef GHC_CHECKED
  {  // the host sized the launch's shared memory with the same layout
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    GHC_CHECK(RL::smem_bytes(NW) <= dyn);
  }
#endif
  rs.init(a, cluster, vsl + 2 * SL + ((CS + 3) & ~3));

  unsigned long long round0 = 0;
  int cur = 0;
  const bool sgd = rs.sgd;
  if (sgd) {
    cur = __ldcg(&a.ms->cur);
    round0 = __ldcg(&a.ms->round);
  }
  float* gw = sgd ? (cur ? a.w1 : a.w0) : nullptr;  // master weights in HBM
  float* gv = sgd ? (cur ? a.v1 : a.v0) : nullptr;
  if constexpr (MULTI) rs.load_state(a.w_in + rs.vrank * a.w_vstride, gv, wbuf0);  // worker vrank's weights
  else rs.load_state(sgd ? gw : a.w_in, gv, wbuf0);
  cluster.sync();  // peers' mbarriers initialised before any st.async
  float* wa = wbuf0;  // weights the samples use
  float* wb = wbuf1;  // peers deposit the next weights here

  // ---- sample assignment + cp.async prefetch ----
  // CTA b owns samples [b*spc, min(n,(b+1)*spc)); warp w, slot sp handles
  // s0 + w + sp*NW.  Pipelined launches (n ≤ slots) prefetch every slot's
  // next-round row during the current round: the index one round ahead, the
  // row after this round's compute (cp.async into the slot's other buffer).
  // Virtual rank v of the grid owns CTAs [v*Gr, (v+1)*Gr) and its own batch.
  const int Gr = G / max(1, a.VR);
  const int lb = blockIdx.x % Gr;
  const int GX = max(1, a.GX);
  auto n_of = [&](int r, int q) {
    if constexpr (MULTI) return a.n_v[q];  // worker q's batch (one round)
    return a.counts ? __ldg(a.counts + (long long)r * GX + q) : a.n;
  };
  // Without per-round counts every round has the same sample range and scale:
  // computed once (the integer division by the CTA count is a serial chain).
  const bool fixed_n = !MULTI && a.counts == nullptr;
  const int fs_spc = (a.n + Gr - 1) / Gr;
  const int fs_s0 = lb * fs_spc, fs_s1 = min(a.n, fs_s0 + fs_spc);
  auto first_sample = [&](int r, int& s, int& s1) {
    if (fixed_n) {
      s1 = fs_s1;
      s = fs_s0 + warp;
      return;
    }
    const int n = n_of(r, rs.rank);
    const int spc = (n + Gr - 1) / Gr;
    const int s0 = lb * spc;
    s1 = min(n, s0 + spc);
    s = s0 + warp;
  };
  // One segment of rounds per launch — or, resident (a.res), one segment per
  // command of the ResidentCtl queue: the data pointers, round count and
  // loss slots come from the command; weights, velocity, epochs and the
  // mbarrier phases carry over.
  const float* sx = a.x;
  const int32_t* sy = a.y;
  const int32_t* sidx = a.idx;
  long long sstride = a.stride;
  int srounds = a.rounds;
  float* sloss = a.loss_out;
  unsigned long long rg = 0;   // rounds run by this launch
  unsigned long long seq = 0;  // resident: command sequence number
  const int32_t* idxv = nullptr;
  auto slot_x = [&](int sp, int b) { return ws + sp * N::WARP_FLOATS + N::S_X + b * N::XWP; };
  auto slot_l = [&](int sp) { return reinterpret_cast<int*>(ws + sp * N::WARP_FLOATS + N::S_L); };
  // y == nullptr: packed dataset rows (ghc_dataset_pack) — x padded to a
  // 32-byte multiple with the label inside the padding: one row = whole
  // sectors, no separate label sector (DRAM traffic ≈ the algorithmic bytes)
  // this lane's row elements (lane, lane + 32) and their padded smem offsets:
  // round-invariant, so the per-row copy is two cp.async with no index math
  const int xo0 = lane < N::XW ? N::xoff(lane) : 0;
  const int xo1 = lane + 32 < N::XW ? N::xoff(lane + 32) : 0;
  auto fetch_rows = [&](int sp, int row, int b, const float* X, const int32_t* Y) {
    const float* xrow = X + (long long)row * (Y ? N::XW : N::XWPK);
    float* dst = slot_x(sp, b);
    if (lane < N::XW) cp_async4(dst + xo0, xrow + lane);
    if (lane + 32 < N::XW) cp_async4(dst + xo1, xrow + lane + 32);
    for (int i = lane + 64; i < N::XW; i += 32) cp_async4(dst + N::xoff(i), xrow + i);  // rows > 64 floats
    if (lane == 0) cp_async4(slot_l(sp) + b, Y ? static_cast<const void*>(Y + row) : xrow + N::XW);
  };
  auto fetch_nocommit = [&](int sp, int row, int b) { fetch_rows(sp, row, b, sx, sy); };
  // resident: the next command, peeked during this command's last round
  __shared__ ResidentCmd s_next;
  __shared__ int s_has_next, s_early;
  if (threadIdx.x == 0) s_has_next = s_early = 0;
  bool prefetched = false;  // this segment's round-0 rows are already in flight
  unsigned long long pk2[8];     // thread 0: slot of the command after next (loaded a segment early)
  unsigned long long pk2_seq = 0;
  // the next command's round-0 rows (fixed n: the same sample slots)
  auto fetch_next_segment = [&]() {
    const ResidentCmd nc = s_next;
    int sn, sn1;
    first_sample(0, sn, sn1);
    const int32_t* nidx = nc.idx ? nc.idx + (long long)rs.vrank * a.idx_vstride : nullptr;
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp)
      if (sn + sp * NW < sn1)
        fetch_rows(sp, nidx ? __ldg(nidx + sn + sp * NW) : sn + sp * NW, (int)((rg + 1) & 1), nc.x, nc.y);
    if (nidx && lane == 0 && nc.rounds > 1) {  // round 1's indices (slot_l[2])
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp)
        if (sn + sp * NW < sn1) cp_async4(slot_l(sp) + 2, nidx + nc.stride + sn + sp * NW);
    }
    cp_async_commit();
  };
  auto row_of = [&](int r, int s) {
    // no gather table: round r reads rows r*stride + s (stride 0: rows s)
    return idxv ? __ldg(idxv + (long long)r * sstride + s) : (int)((long long)r * sstride + s);
  };
  // gather indices of round r (pipelined path): one cp.async per slot into
  // slot_l[2], fetched a round before the rows they select
  auto fetch_idx_nocommit = [&](int r) {
    if (!idxv || lane != 0 || r >= srounds) return;
    int sx0, sx1;
    first_sample(r, sx0, sx1);
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp)
      if (sx0 + sp * NW < sx1) cp_async4(slot_l(sp) + 2, idxv + (long long)r * sstride + sx0 + sp * NW);
  };

  if (RES && blockIdx.x == 0 && threadIdx.x == 0) a.res->ctas = gridDim.x;
  if constexpr (RES) __syncthreads();  // s_has_next initialised before any thread reads it
  unsigned long long pk[8];  // thread 0: the next command's slot, loaded during the last round
  unsigned long long* prl = nullptr;  // probe row of the last round run (resident: segment-boundary probes)
  for (;;) {  // segments
  if constexpr (RES) {
    ResidentCmd cmd;
    const bool have = s_has_next != 0;
    if (!resident_next(a.res, ++seq, cmd, have, s_next)) break;
    if (prl && threadIdx.x == 0) prl[15] = globaltimer();  // next command in hand
    sx = cmd.x;
    sy = cmd.y;
    sidx = cmd.idx;
    sstride = cmd.stride;
    srounds = cmd.rounds;
    sloss = cmd.loss_out;
  }
  if constexpr (MULTI) idxv = a.idx_v[rs.vrank];
  else idxv = sidx ? sidx + (long long)rs.vrank * a.idx_vstride : nullptr;
  if (a.pipelined && srounds > 0 && !prefetched) {
    int s, s1;
    first_sample(0, s, s1);
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp)
      if (s + sp * NW < s1) fetch_nocommit(sp, row_of(0, s + sp * NW), (int)(rg & 1));
    fetch_idx_nocommit(1);
    cp_async_commit();
  }
  prefetched = false;
  // reset after the barrier: every thread has read `have` (s_has_next) for
  // this segment — the peeked-command fast path has no barrier of its own
  __syncthreads();
  if (threadIdx.x == 0) s_has_next = s_early = 0;

  for (int r = 0; r < srounds; ++r, ++rg) {
    int ntot = GX * a.n;  // samples of round r over all ranks (SPEC.md:358-366 weighted mean)
    if (!fixed_n) {
      ntot = 0;
      for (int q = 0; q < GX; ++q) ntot += n_of(r, q);
    }
    float scale = sgd ? 1.0f / (float)ntot : a.grad_scale;
    if constexpr (MULTI) scale = 1.0f / (float)n_of(r, rs.rank);  // worker mean
    unsigned long long* pr =
        a.probe ? a.probe + ((long long)(RES ? (long long)rg : r) * gridDim.x + blockIdx.x) * 16 : nullptr;
    if (pr && threadIdx.x == 0) {
      pr[0] = globaltimer();
      unsigned sm;
      asm("mov.u32 %0, %%smid;" : "=r"(sm));
      pr[1] = sm;  // which SM ran this CTA (diagnostics: per-SM skew)
    }

    // ---- samples ----
    float lsum = 0.0f;
    int s, s1;
    first_sample(r, s, s1);
    // One sample per warp (pipelined, SPW = 1): lstm_samples STORES every
    // gradient entry of the warp partial; otherwise zero it and accumulate.
    constexpr bool kStore = SPW == 1;
    float* wp = wpart + warp * N::PPAD;
    if (!(a.pipelined && kStore) || s >= s1) {
      for (int p = lane; p < N::PPAD / 4; p += 32)
        reinterpret_cast<float4*>(wp)[p] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
    }
    if (a.pipelined) {
      // Rows of round r and indices of round r+1 were requested at the start
      // of round r-1 (prologue for r = 0): a whole round of compute and
      // exchange hides their latency — PCIe included when x/y are pinned
      // host memory.  Now request round r+1's rows (into the buffer round
      // r-1 used) and round r+2's indices, then compute round r.
      cp_async_wait<0>();
      __syncwarp();
      if (r + 1 < srounds) {
        int sn, sn1;
        first_sample(r + 1, sn, sn1);
        int rows[SPW];
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp)
          rows[sp] = idxv ? slot_l(sp)[2] : (int)((long long)(r + 1) * sstride + sn + sp * NW);
        __syncwarp();
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp)
          if (sn + sp * NW < sn1) fetch_nocommit(sp, rows[sp], (int)((rg + 1) & 1));
        fetch_idx_nocommit(r + 2);
        cp_async_commit();
      } else if (RES) {
        // last round of a resident command.  The next command's slot was
        // loaded at the end of the previous command (pk2, no wait): if it is
        // valid now its first batch is fetched right away, a whole round
        // ahead (host-memory batches need it).  Otherwise load the slot now
        // and check it after the samples (then the fetch overlaps the
        // exchange only).
        if (threadIdx.x == 0) {
          ResidentCmd nc;
          s_early = (pk2_seq == seq + 1 && slot_valid(pk2, seq + 1, nc) && nc.op == 0 && nc.rounds > 0) ? 1 : 0;
          if (s_early) s_next = nc;
          else issue_slot_loads(a.res, seq + 1, pk);
        }
        __syncthreads();
        if (s_early && fixed_n) {
          fetch_next_segment();
          prefetched = true;
        }
      }
      if (s < s1) {
        const float* xsp[SPW];
        int lab[SPW];
        float scl[SPW];
        float* prb[SPW];
        float lo[SPW];
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp) {
          const bool valid = s + sp * NW < s1;
          const int use = valid ? sp : 0;  // empty slot: recompute slot 0 with weight 0
          xsp[sp] = slot_x(use, (int)(rg & 1));
          int l = slot_l(use)[rg & 1];
          if (l < 0 || l >= K) {
            if (lane == 0 && valid) atomicOr(a.err, 1);
            l = 0;
          }
          lab[sp] = l;
          scl[sp] = valid ? scale : 0.0f;
          prb[sp] = (valid && a.probs_out) ? a.probs_out + (long long)(s + sp * NW) * K : nullptr;
        }
        unsigned long long* ps = (pr && warp == 0) ? pr : nullptr;
        float* tio[SPW];
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp) tio[sp] = nullptr;
        if (a.mode == MODE_FWD)
          lstm_samples<D, H, T, K, false, SPW, true, !kStore>(wa, ws, wp, xsp, lab, scl, lane, prb,
                                                              lo, ps, tio);
        else
          lstm_samples<D, H, T, K, true, SPW, true, !kStore>(wa, ws, wp, xsp, lab, scl, lane, prb, lo,
                                                             ps, tio);
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp)
          if (s + sp * NW < s1) lsum += lo[sp];
      }
    } else {
      for (; s < s1; s += NW) {
        const int row = row_of(r, s);
        float* xs = slot_x(0, 0);
        const float* xrow = sx + (long long)row * (sy ? N::XW : N::XWPK);
        for (int i = lane; i < N::XW; i += 32) xs[N::xoff(i)] = __ldg(xrow + i);
        int label = sy ? __ldg(sy + row) : __float_as_int(__ldg(xrow + N::XW));
        __syncwarp();
        if (label < 0 || label >= K) {
          if (lane == 0) atomicOr(a.err, 1);
          label = 0;
        }
        if (a.mode == MODE_FWD)
          lsum += lstm_sample<D, H, T, K, false>(
              wa, ws, wp, xs, label, scale, lane,
              a.probs_out ? a.probs_out + (long long)s * K : nullptr, nullptr);
        else
          lsum += lstm_sample<D, H, T, K, true>(wa, ws, wp, xs, label, scale, lane, nullptr,
                                                nullptr);
        __syncwarp();
      }
    }
    if (lane == 0) wp[N::P] = lsum;  // loss rides in slot P
    const bool last_res = RES && a.pipelined && r + 1 == srounds;
    if (last_res && threadIdx.x == 0) {
      if (s_early) {
        s_has_next = 1;
      } else {
        ResidentCmd nc;
        s_has_next = (slot_valid(pk, seq + 1, nc) && nc.op == 0 && nc.rounds > 0) ? 1 : 0;
        if (s_has_next) s_next = nc;
      }
    }
    __syncthreads();
    if (last_res && s_has_next && !s_early && fixed_n) {  // late: overlaps the exchange
      fetch_next_segment();
      prefetched = true;
    }
    if (pr && threadIdx.x == 0) pr[2] = globaltimer();

    // (the CTA partial — Σ warp partials, warp order — is formed by ClusterRS (a))
    if (pr && threadIdx.x == 0) pr[3] = globaltimer();
    rs.exchange(a, r, rg, sloss, wpart, NW, N::PPAD, wa, wb, pr, ntot);
    prl = pr;
  }
  if constexpr (!RES) {
    break;
  } else {
    resident_done(a.res, sloss != nullptr && rs.s0 <= N::P && N::P < rs.s1);
    if (prl && threadIdx.x == 0) prl[14] = globaltimer();  // completion arrival issued
    // the slot after next, loaded as late as possible (a host queueing a few
    // commands ahead has filled it by now; after the arrival, whose release
    // would otherwise wait for these loads) and checked at the start of the
    // next command's last round
    if (threadIdx.x == 0) {
      issue_slot_loads(a.res, seq + 2, pk2);
      pk2_seq = seq + 2;
    }
  }
  }  // segments

  rs.publish(a, gw, gv, wa, round0, rg);
  if (a.probe && !RES && threadIdx.x == 0 && a.rounds > 0) {  // kernel entry / exit (launch anatomy)
    a.probe[(long long)blockIdx.x * 16 + 14] = t_entry;
    a.probe[((long long)(a.rounds - 1) * G + blockIdx.x) * 16 + 15] = globaltimer();
  }
  cluster.sync();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace ghc
