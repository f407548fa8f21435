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
// (H ≤ 32).  Forward: the 4H gate rows are spread over all 32 lanes (rows ℓ,
// ℓ+32, ℓ+64 with their Wx/Wh/b in registers), activated where computed and
// gathered per unit with one SHFL per gate (H ≤ 24, H % 4 == 0; otherwise
// lane j computes the rows {j, H+j, 2H+j, 3H+j} itself).  Backward: lane j
// holds column j of Wh for dh = Whᵀdz; h_t, the gate cache and dz live in
// shared memory.
// Samples of a round are spread over ≈ one CTA per SM so the 1000
// transcendentals/sample run on every SM's MUFU pipe.  The recurrence is a
// K=25 contraction per timestep — far below a tcgen05 tile — so the kernel is
// FFMA/latency-bound by design.
#pragma once

#include "ghc_device.cuh"

namespace ghc {

enum StepMode : int {
  MODE_GRAD = 0,       // fused lstm→softmax: gradient + loss
  MODE_SGD = 1,        // fused sync rounds with sgd_step
  MODE_FWD = 2,        // fused forward: probs + loss
  MODE_TRUNK_FWD = 3,  // LSTM trunk of a deeper net: write h_T rows (hio[s][H])
  MODE_TRUNK_GRAD = 4  // LSTM trunk backward from dh_T rows (hio[s][H]): Wx, Wh, b grads
};

constexpr int kMaxRanks = 8;  // GPUs of one NVLink domain in the fused exchange

// ---------------------------------------------------------------------------
// Resident round service (resident.cu): the persistent round kernel stays
// launched and serves a queue of commands — each one segment of sync rounds
// on its own batch pointers — so a call costs a doorbell, not a cooperative
// cluster launch (≈ 13 µs of launch + prologue + teardown, measured).
//   host submit:   pinned ring slot + pinned doorbell; CTA 0 relays it into
//                  the device ring and publishes the device bell;
//   stream submit: a 1-thread kernel on the caller's stream writes the slot
//                  and the bell; a 1-thread wait kernel on the same stream
//                  spins until the command completed (CUDA events around
//                  the pair time exactly the served rounds).
// Completion: every CTA arrives on a counter after the segment's last round;
// the last one publishes `done` (device) and the pinned host word.  With no
// command for idle_ns the kernel publishes a STOP itself (never strands the
// GPU) and marks the service expired.
struct ResidentCmd {
  const float* x;
  const int32_t* y;
  const int32_t* idx;
  long long stride;
  float* loss_out;
  int rounds;
  int op;  // 0 run, 1 stop
  unsigned long long seq;
  unsigned long long pad_;  // 64 B: four 16-byte loads from the host ring
};
constexpr int kResRing = 8;
struct ResidentCtl {
  ResidentCmd cmd[kResRing];
  unsigned long long claim;    // highest claimed command slot (submitter / relay / expiry)
  unsigned long long bell;     // highest published command (device)
  unsigned long long arrive;   // CTA completions, all commands
  unsigned long long done;     // highest completed command (device)
  int expired;                 // idle STOP published by the kernel itself
  int submit_failed;           // a stream submit found the service expired
  ResidentCmd* host_cmd;       // pinned ring (device-mapped pointer)
  unsigned long long* host_bell;  // pinned doorbell
  unsigned long long* host_done;  // pinned: [0] completed command, [1] expired
  unsigned long long idle_ns;
  unsigned long long t[8];     // diagnostics (%globaltimer): [0] submit, [1] first CTA past the
                               // bell, [2] last CTA past the bell, [3] done published, [4] wait saw it
  unsigned long long tlog[64][2];  // per command (seq % 64): last CTA past the bell, done published
  unsigned long long ctas;     // round-kernel CTAs (completion = arrive reaches seq · ctas)
};

__device__ __forceinline__ unsigned long long res_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long res_ld_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long res_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A command from the pinned host ring: four independent 16-byte system-
// scope loads (all in flight at once — field-by-field volatile loads paid a
// PCIe round trip each, measured).
static_assert(sizeof(ResidentCmd) == 64, "ResidentCmd: four 16-byte words");
__device__ __forceinline__ ResidentCmd load_host_cmd(const ResidentCmd* h) {
  unsigned long long v[8];
  const unsigned long long* p = reinterpret_cast<const unsigned long long*>(h);
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p) : "memory");
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[2]), "=l"(v[3]) : "l"(p + 2) : "memory");
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[4]), "=l"(v[5]) : "l"(p + 4) : "memory");
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[6]), "=l"(v[7]) : "l"(p + 6) : "memory");
  ResidentCmd c;
  memcpy(&c, v, sizeof(c));
  return c;
}

// Device ring slots are self-validating: the last word is a hash of the
// other seven, so one round of four relaxed 16-byte loads either yields the
// whole published command or fails the check (a slot is rewritten only for
// seq + kResRing) — a reader needs no doorbell load in front of it.
__device__ __forceinline__ unsigned long long cmd_check(const unsigned long long (&v)[8]) {
  unsigned long long h = 0x9e3779b97f4a7c15ull;
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    h ^= v[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xbf58476d1ce4e5b9ull;
  }
  return h | 1ull;  // never 0 (a zeroed slot never validates)
}
__device__ __forceinline__ void write_cmd(ResidentCtl* c, ResidentCmd cmd) {
  unsigned long long v[8];
  memcpy(v, &cmd, sizeof(cmd));
  v[7] = cmd_check(v);
  unsigned long long* p = reinterpret_cast<unsigned long long*>(&c->cmd[cmd.seq % kResRing]);
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = v[i];
}
// Issue the loads of slot `seq` (results land in v; consume later).
__device__ __forceinline__ void issue_slot_loads(const ResidentCtl* c, unsigned long long seq,
                                                 unsigned long long (&v)[8]) {
  const unsigned long long* p = reinterpret_cast<const unsigned long long*>(&c->cmd[seq % kResRing]);
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p) : "memory");
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[2]), "=l"(v[3]) : "l"(p + 2) : "memory");
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[4]), "=l"(v[5]) : "l"(p + 4) : "memory");
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[6]), "=l"(v[7]) : "l"(p + 6) : "memory");
}
__device__ __forceinline__ bool slot_valid(const unsigned long long (&v)[8], unsigned long long seq,
                                           ResidentCmd& out) {
  memcpy(&out, v, sizeof(out));
  return out.seq == seq && v[7] == cmd_check(v);
}

// Next command for this CTA (all threads return the same command; false on
// STOP).  `have`: this CTA already holds it (peeked during the last round).
static __device__ __noinline__ bool resident_wait_cmd(ResidentCtl* c, unsigned long long seq,
                                                      ResidentCmd& out) {
  __shared__ ResidentCmd s_cmd;
  if (threadIdx.x == 0) {
    {
      const unsigned long long t0 = res_now();
      for (unsigned it = 0;; ++it) {
        unsigned long long v[8];
        issue_slot_loads(c, seq, v);
        ResidentCmd cmd;
        if (slot_valid(v, seq, cmd)) {
          s_cmd = cmd;
          break;
        }
        // fallback relay of the host ring on CTA 0 (the relay kernel normally
        // does it) and the idle expiry
        if (blockIdx.x == 0) {
          const bool host_ready = res_ld_sys(c->host_bell) >= seq;
          const bool idle = !host_ready && res_now() - t0 > c->idle_ns;
          if ((host_ready || idle) && atomicCAS(&c->claim, seq - 1, seq) == seq - 1) {
            ResidentCmd w{};
            if (host_ready) {
              w = load_host_cmd(c->host_cmd + (seq % kResRing));
            } else {
              w.op = 1;  // idle: STOP
              w.seq = seq;
              c->expired = 1;
              volatile unsigned long long* hd = c->host_done;
              hd[1] = 1ull;
            }
            write_cmd(c, w);
            __threadfence_system();
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&c->bell), "l"(seq) : "memory");
          }
        } else if ((it & 1023u) == 0 && res_now() - t0 > c->idle_ns + 10000000000ull) {
          __trap();  // relay gone: never hang
        }
      }
    }
    const unsigned long long tb = res_now();
    atomicMin(&c->t[1], tb);
    atomicMax(&c->t[2], tb);
    atomicMax(&c->tlog[seq % 64][0], tb);
  }
  __syncthreads();
  out = s_cmd;
  __syncthreads();
  return out.op == 0;
}
// Fast path inline: the command was peeked during the last round (shared
// memory, behind a CTA barrier) — no barrier and no call (a call would make
// thread 0 wait for its in-flight slot loads to save their registers).
static __device__ __forceinline__ bool resident_next(ResidentCtl* c, unsigned long long seq, ResidentCmd& out,
                                                     bool have, const ResidentCmd& peeked) {
  if (have) {
    out = peeked;
    if (threadIdx.x == 0) atomicMax(&c->tlog[seq % 64][0], res_now());
    return out.op == 0;
  }
  return resident_wait_cmd(c, seq, out);
}

// The segment of command `seq` is complete on this CTA (its last exchange
// committed): one fire-and-forget arrival; the relay kernel (on a spare SM)
// publishes the completion once every CTA arrived — no round trip here.
static __device__ __forceinline__ void resident_done(ResidentCtl* c, bool wrote_loss) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // the CTA that stored this segment's losses (possibly to host memory)
    // makes them visible system-wide first; the others only release at gpu
    // scope (the relay's system fence before the host word is cumulative)
    if (wrote_loss) __threadfence_system();
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&c->arrive) : "memory");
  }
}

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
  unsigned long long* probe;  // nullable: [rounds][gridDim][16] %globaltimer per phase
  float* hio;             // TRUNK modes: h_T out / dh_T in, [n][H]
  unsigned* bar;          // flag barrier: epoch, go, then one 128-B line per CTA
  int pipelined;          // every round has ≤ 1 sample per warp (cp.async prefetch path)
  int mode;
  // ---- cross-rank exchange (lstm_round.cuh ClusterXchg, GX > 1) ----
  // GX ranks (one per GPU, or virtual ranks sharing one grid) each train on
  // their own batch and hold a bit-identical replica of the master.  counts
  // is then [rounds][GX]; idx of virtual rank v starts at idx + v*idx_vstride.
  int GX;                 // ranks in the exchange (1: single-GPU round)
  int VR;                 // virtual ranks in this grid (1 with one process per GPU)
  int rank0;              // global rank of this grid's first virtual rank
  long long idx_vstride;
  float* gpart[kMaxRanks];     // per rank: tagged receive rows uint2[2][GX][EP] (peer-mapped)
  unsigned long long* tpart;   // single-GPU exchange: tagged cluster rows [2][clusters][EP]
  unsigned long long* tw;      // single-GPU exchange: tagged new weights [2][EP]
  unsigned* gcnt[kMaxRanks];   // per rank: line [CS*kFlagStride] keeps the exchange epoch
  ResidentCtl* res;            // non-null: resident round service (commands in res)
  // ---- independent per-worker gradients in one launch (MULTI kernels) ----
  // virtual rank v computes worker v's gradient at weights w_in + v·w_vstride
  // over its own batch (rows idx_v[v][0 .. n_v[v])), scaled by 1/n_v[v], into
  // g_out + v·g_vstride, its loss sum into loss_out[v]; no cross-rank sum.
  const int32_t* idx_v[kMaxRanks];
  int n_v[kMaxRanks];
  long long w_vstride;
  long long g_vstride;
};

// Grid barrier for the persistent round loop (gather → broadcast):
// CTA b publishes `epoch | bad<<31` in its own 128-B line (release store);
// CTA 0 polls all G lines, one thread per line, with relaxed loads (no L1
// invalidate per poll), ORs the `bad` bits and publishes `go = epoch|bad`;
// every CTA polls `go` with one thread, then one acquire fence.  Two L2 hops,
// no serialised atomics, no hot line shared by all pollers.  Returns the OR of
// all CTAs' `bad` bits (a non-finite update is rejected grid-wide).
constexpr int kFlagStride = 32;  // uints: one 128-byte line per CTA flag
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_barrier(unsigned* bar, unsigned epoch, int bad) {
  __shared__ int s_bad;
  __syncthreads();
  unsigned* go = bar + kFlagStride;  // bar[0] epoch store, bar[32] go, flags from bar[64]
  unsigned* flags = bar + 2 * kFlagStride;
  if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * kFlagStride, epoch | (bad ? 0x80000000u : 0u));
  if (blockIdx.x == 0) {
    int any = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
      unsigned v;
      do {
        v = ld_relaxed_gpu(flags + b * kFlagStride);
      } while ((int)((v & 0x7fffffffu) - epoch) < 0);
      any |= (int)(v >> 31);
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      st_release_gpu(go, epoch | (any ? 0x80000000u : 0u));
    }
  }
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      v = ld_relaxed_gpu(go);
    } while ((int)((v & 0x7fffffffu) - epoch) < 0);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s_bad = (int)(v >> 31);
  }
  __syncthreads();
  return s_bad;
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
  static constexpr int XW = T * D;                       // global row width
  static constexpr int XWPK = (XW + 1 + 31) & ~31;       // packed row: x, label, pad to 128 B
  static constexpr int DP = (D + 3) & ~3;                // x_t padded to float4s in smem
  static constexpr int XWP = T * DP;
  static constexpr bool HV = (H % 4) == 0;               // h rows loadable as float4
  static constexpr int S_X = 0;                          // x rows [2][T][DP] (double buffer)
  static constexpr int S_L = 2 * XWP;                    // label[2], next idx (ints)
  static constexpr int S_H = S_L + 4;                    // h[T][H]
  static constexpr int S_C = S_H + ((T * H + 3) & ~3);   // cache[T][H][8]: i f g o | c tanh(c)
  static constexpr int S_DZ = S_C + T * H * 8;           // dz[T][4H]
  static constexpr int WARP_FLOATS = (S_DZ + T * G4 + 3) & ~3;
  // global row element i → smem offset (t*DP + d)
  __device__ static int xoff(int i) { return (i / D) * DP + (i % D); }
  static size_t smem_bytes(int nw) {
    return sizeof(float) * (size_t)(PPAD + nw * WARP_FLOATS + nw * PPAD + 32);
  }
};

// Forward + softmax/loss (+ backward when BWD) of SPW samples interleaved in
// one warp's instruction stream (static ILP: the samples share the weight
// registers and fill each other's dependency stalls).  Slot sp uses the
// per-sample scratch at ws + sp*WARP_FLOATS; its input row xs[sp] is already
// in shared memory (cp.async-prefetched by the caller).  Each sample's
// gradient (scaled by scale[sp]; 0 masks an empty slot) is ADDED into the
// warp partial `wp` — lane j touches only the entries of its own gate rows,
// lane 0 the output bias — no atomics.  loss[sp] receives ℓ of slot sp.
// HEAD = false: the LSTM is the trunk of a deeper net (arch.cpp: lstm first,
// dense layers after); the forward writes h_T to trunk_io[sp] and the
// backward starts from dh_T read from trunk_io[sp] (already scaled).
// ACC = false: the gradient entries are STORED into wp (one sample per warp
// and round: no zeroing of the 8.6 KB partial needed); true: added.
template <int D, int H, int T, int K, bool BWD, int SPW, bool HEAD = true, bool ACC = true>
__device__ __forceinline__ void lstm_samples(const float* __restrict__ wsm, float* __restrict__ ws,
                                             float* __restrict__ wp,
                                             const float* const (&xs)[SPW],
                                             const int (&label)[SPW], const float (&scale)[SPW],
                                             int lane, float* const (&probs_row)[SPW],
                                             float (&loss)[SPW], unsigned long long* pr,
                                             float* const (&trunk_io)[SPW]) {
  using N = LstmNet<D, H, T, K>;
  constexpr int DP = N::DP;
  const bool act = lane < H;
  // Lanes ≥ H shadow unit lane mod H: they compute the same values as that
  // unit's lane, so their shared-memory stores (same address, same value)
  // need no divergent branch in the recurrences.  Reductions and the weight
  // gradients still mask them with `act`.
  const int j = lane % H;
  auto put = [](float& dst, float v) {
    if constexpr (ACC) dst += v;
    else dst = v;
  };
  float* hs[SPW];
  float* cs[SPW];
  float* dzs[SPW];
#pragma unroll
  for (int sp = 0; sp < SPW; ++sp) {
    hs[sp] = ws + sp * N::WARP_FLOATS + N::S_H;
    cs[sp] = ws + sp * N::WARP_FLOATS + N::S_C;
    dzs[sp] = ws + sp * N::WARP_FLOATS + N::S_DZ;  // dz[t][4H]
    // the slot's last region ends inside the slot; x rows come from a slot's
    // double buffer (or the caller's staging row)
    GHC_CHECK(N::S_DZ + T * 4 * H <= N::WARP_FLOATS && N::S_C + T * H * 8 <= N::S_DZ &&
              N::S_H + T * H <= N::S_C && 2 * N::XWP <= N::S_L);
    GHC_CHECK(xs[sp] != nullptr && (reinterpret_cast<uintptr_t>(xs[sp]) & 15u) == 0);
  }
  // x_t (DP floats, float4 loads) and h_t (H floats, float4 when H%4==0)
  auto load_x = [&](int sp, int t, float (&v)[DP]) {
#pragma unroll
    for (int c = 0; c < DP / 4; ++c) {
      const float4 u = reinterpret_cast<const float4*>(xs[sp] + t * DP)[c];
      v[4 * c] = u.x;
      v[4 * c + 1] = u.y;
      v[4 * c + 2] = u.z;
      v[4 * c + 3] = u.w;
    }
  };
  auto load_h = [&](int sp, int t, float (&v)[H]) {
    if constexpr (N::HV) {
#pragma unroll
      for (int c = 0; c < H / 4; ++c) {
        const float4 u = reinterpret_cast<const float4*>(hs[sp] + t * H)[c];
        v[4 * c] = u.x;
        v[4 * c + 1] = u.y;
        v[4 * c + 2] = u.z;
        v[4 * c + 3] = u.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < H; ++k) v[k] = hs[sp][t * H + k];
    }
  };
  if (pr && lane == 0) pr[8] = globaltimer();

  // ---------------- forward recurrence (nn.cpp:160-200) ----------------
  // Packed FP32x2 FMAs (FFMA2, sm_100): each gate keeps two partial sums
  // (even / odd input index) — one FFMA2 advances both with the same rounding
  // as two FFMAs, so results are bit-identical to the scalar loop at half the
  // issue slots (3-register FFMA issues once per 2 cycles per SM sub-partition).
  //
  // Gate rows spread over all 32 lanes (H ≤ 24, H % 4 == 0): lane ℓ computes
  // rows ℓ, ℓ+32, ℓ+64 (< 4H) — NR = ⌈4H/32⌉ rows instead of 4 — activates
  // them (σ or tanh by the row's gate, branch-free), and lane u collects the
  // four gates of unit u with one SHFL per gate.  The recurrent product is
  // bound by FFMA2 issue (≈ 6.3 warp-cycles per FFMA2 with two
  // warps per sub-partition), so 3 rows × 10 instead of 4 × 10 FFMA2 per step
  // at H = 20.  Same operations in the same order per row: bit-identical to
  // the unit-per-lane loop below.
  constexpr int NR = (4 * H + 31) / 32;
  if constexpr (N::HV && NR < 4) {
    constexpr int DH = D / 2, HH = H / 2;
    float2 wxr[NR][DH > 0 ? DH : 1], whr[NR][HH];
    float wxt[NR], br[NR], al[NR], be[NR], ga[NR];
#pragma unroll
    for (int sl = 0; sl < NR; ++sl) {
      const int r = lane + 32 * sl;
      const bool ok = r < 4 * H;
      const int rr = ok ? r : 0;
      const float* rx = wsm + N::OFF_WX + rr * D;
      const float4* rh4 = reinterpret_cast<const float4*>(wsm + N::OFF_WH + rr * H);
#pragma unroll
      for (int m = 0; m < DH; ++m) wxr[sl][m] = ok ? make_float2(rx[2 * m], rx[2 * m + 1]) : make_float2(0.f, 0.f);
#pragma unroll
      for (int m = 0; m < H / 4; ++m) {
        const float4 u = ok ? rh4[m] : make_float4(0.f, 0.f, 0.f, 0.f);
        whr[sl][2 * m] = make_float2(u.x, u.y);
        whr[sl][2 * m + 1] = make_float2(u.z, u.w);
      }
      wxt[sl] = (ok && (D & 1)) ? rx[D - 1] : 0.0f;
      br[sl] = ok ? wsm[N::OFF_B + rr] : 0.0f;
      // σ(z) = rcp(1 + 2^(−z·log2e));  tanh(z) = 1 − 2·rcp(2^(2z·log2e) + 1)
      const bool tnh = (rr / H) == 2;
      al[sl] = tnh ? 2.8853900817779268f : -1.4426950408889634f;
      be[sl] = tnh ? -2.0f : 1.0f;
      ga[sl] = tnh ? 1.0f : 0.0f;
    }
    // gate q of unit u lives in lane (qH+u) mod 32, row slot (qH+u) / 32;
    // pick[q] = the slot this lane presents for gate q
    // (as bit masks: a select by a runtime slot index would compile to a
    // local-memory array access)
    unsigned pick[4][NR];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int sl = 0; sl < NR; ++sl) {
        const int r = lane + 32 * sl;
        pick[q][sl] = (r < 4 * H && r / H == q) ? 0xffffffffu : 0u;
      }
    int src[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) src[q] = (q * H + j) & 31;
    float c[SPW];
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp) c[sp] = 0.0f;
    // b + Wx·x_t of one sample (the first terms of each row's sum)
    auto xpart = [&](int sp, int t, float2 (&a)[NR]) {
      float xv[DP];
      load_x(sp, t, xv);
#pragma unroll
      for (int sl = 0; sl < NR; ++sl) {
        a[sl] = make_float2(br[sl], 0.0f);
#pragma unroll
        for (int m = 0; m < DH; ++m) a[sl] = __ffma2_rn(wxr[sl][m], make_float2(xv[2 * m], xv[2 * m + 1]), a[sl]);
        if (D & 1) a[sl].x = fmaf(wxt[sl], xv[D - 1], a[sl].x);
      }
    };
    // activations, gate gather, cell update, cache + h_t stores
    auto gates = [&](int sp, int t, const float2 (&a)[NR]) {
      float y[NR];
#pragma unroll
      for (int sl = 0; sl < NR; ++sl)
        y[sl] = fmaf(be[sl], rcp_approx(1.0f + ex2_approx(al[sl] * (a[sl].x + a[sl].y))), ga[sl]);
      float gq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        unsigned pv = 0u;
#pragma unroll
        for (int sl = 0; sl < NR; ++sl) pv |= __float_as_uint(y[sl]) & pick[q][sl];
        gq[q] = __shfl_sync(0xffffffffu, __uint_as_float(pv), src[q]);
      }
      const float ig = gq[0], fg = gq[1], gg = gq[2], og = gq[3];
      c[sp] = fmaf(fg, c[sp], ig * gg);
      const float tc = tanh_f(c[sp]);
      float* ct = cs[sp] + (t * H + j) * 8;
      reinterpret_cast<float4*>(ct)[0] = make_float4(ig, fg, gg, og);
      reinterpret_cast<float2*>(ct)[2] = make_float2(c[sp], tc);
      hs[sp][t * H + j] = og * tc;
    };
    // Software-pipelined over t: step t's chain is LDS h_{t-1} → Wh·h → σ/tanh
    // → h_t; the input projection of step t+1 (independent of h) is computed
    // inside step t, off that chain.  Same operations in the same order per
    // row as the straight loop: bit-identical.
    float2 accn[SPW][NR];
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp) xpart(sp, 0, accn[sp]);
    {
      float2 acc[SPW][NR];
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp)
#pragma unroll
        for (int sl = 0; sl < NR; ++sl) acc[sp][sl] = accn[sp][sl];
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) xpart(sp, T > 1 ? 1 : 0, accn[sp]);
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) gates(sp, 0, acc[sp]);
      __syncwarp();
    }
#pragma unroll 1
    for (int t = 1; t < T; ++t) {
      float2 acc[SPW][NR];
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) {
        float hv[H];
        load_h(sp, t - 1, hv);
#pragma unroll
        for (int sl = 0; sl < NR; ++sl) acc[sp][sl] = accn[sp][sl];
#pragma unroll
        for (int m = 0; m < HH; ++m)
#pragma unroll
          for (int sl = 0; sl < NR; ++sl)
            acc[sp][sl] = __ffma2_rn(whr[sl][m], make_float2(hv[2 * m], hv[2 * m + 1]), acc[sp][sl]);
      }
      const int tn = t + 1 < T ? t + 1 : t;  // last step: a harmless reload
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) xpart(sp, tn, accn[sp]);
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) gates(sp, t, acc[sp]);
      __syncwarp();
    }
  } else {
    constexpr int DH = D / 2, HH = H / 2;
    float2 wxp[4][DH > 0 ? DH : 1], whp[4][HH > 0 ? HH : 1];
    float wxt[4], wht[4], bb[4];  // odd-length tails (into the even partial sum)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float* rx = wsm + N::OFF_WX + (q * H + j) * D;
      const float* rh = wsm + N::OFF_WH + (q * H + j) * H;
      bb[q] = wsm[N::OFF_B + q * H + j];
#pragma unroll
      for (int m = 0; m < DH; ++m) wxp[q][m] = make_float2(rx[2 * m], rx[2 * m + 1]);
      if constexpr (N::HV) {  // row of Wh: 16-B aligned, lane stride 4H floats → conflict-free LDS.128
#pragma unroll
        for (int m = 0; m < H / 4; ++m) {
          const float4 u = reinterpret_cast<const float4*>(rh)[m];
          whp[q][2 * m] = make_float2(u.x, u.y);
          whp[q][2 * m + 1] = make_float2(u.z, u.w);
        }
      } else {
#pragma unroll
        for (int m = 0; m < HH; ++m) whp[q][m] = make_float2(rh[2 * m], rh[2 * m + 1]);
      }
      wxt[q] = (D & 1) ? rx[D - 1] : 0.0f;
      wht[q] = (H & 1) ? rh[H - 1] : 0.0f;
    }
    float c[SPW];
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp) c[sp] = 0.0f;
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      float2 acc[SPW][4];  // (Σ even-index terms + bias, Σ odd-index terms)
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) {
        float xv[DP];
        load_x(sp, t, xv);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[sp][q] = make_float2(bb[q], 0.0f);
#pragma unroll
          for (int m = 0; m < DH; ++m)
            acc[sp][q] = __ffma2_rn(wxp[q][m], make_float2(xv[2 * m], xv[2 * m + 1]), acc[sp][q]);
          if (D & 1) acc[sp][q].x = fmaf(wxt[q], xv[D - 1], acc[sp][q].x);
        }
      }
      if (t > 0) {
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp) {
          float hv[H];
          load_h(sp, t - 1, hv);
#pragma unroll
          for (int m = 0; m < HH; ++m)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              acc[sp][q] = __ffma2_rn(whp[q][m], make_float2(hv[2 * m], hv[2 * m + 1]), acc[sp][q]);
          if (H & 1)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[sp][q].x = fmaf(wht[q], hv[H - 1], acc[sp][q].x);
        }
      }
      float a0[SPW][4], a1[SPW][4];
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a0[sp][q] = acc[sp][q].x;
          a1[sp][q] = acc[sp][q].y;
        }
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) {
        const float ig = sigmoid_f(a0[sp][0] + a1[sp][0]);
        const float fg = sigmoid_f(a0[sp][1] + a1[sp][1]);
        const float gg = tanh_f(a0[sp][2] + a1[sp][2]);
        const float og = sigmoid_f(a0[sp][3] + a1[sp][3]);
        c[sp] = fmaf(fg, c[sp], ig * gg);
        const float tc = tanh_f(c[sp]);
        float* ct = cs[sp] + (t * H + j) * 8;
        reinterpret_cast<float4*>(ct)[0] = make_float4(ig, fg, gg, og);
        reinterpret_cast<float2*>(ct)[2] = make_float2(c[sp], tc);
        hs[sp][t * H + j] = og * tc;
      }
      __syncwarp();
    }
  }
  if (pr && lane == 0) pr[9] = globaltimer();

  float dh[SPW];
  if constexpr (!HEAD) {
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp) {
      loss[sp] = 0.0f;
      if (!BWD) {
        if (act && trunk_io[sp]) trunk_io[sp][j] = hs[sp][(T - 1) * H + j];
        dh[sp] = 0.0f;
      } else {
        dh[sp] = trunk_io[sp][j] * (scale[sp] != 0.0f ? 1.0f : 0.0f);
      }
    }
    if constexpr (!BWD) return;
  } else {
  // ---------------- softmax + loss (nn.cpp:202-248) ----------------
  float hT[SPW], e[SPW][K], inv_den[SPW];
#pragma unroll
  for (int sp = 0; sp < SPW; ++sp) {
    hT[sp] = act ? hs[sp][(T - 1) * H + j] : 0.0f;
    float z[K];
    float zmax = -3.0e38f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      z[k] = warp_sum(act ? wsm[N::OFF_WS + k * H + j] * hT[sp] : 0.0f) + wsm[N::OFF_BS + k];
      zmax = fmaxf(zmax, z[k]);
    }
    float den = 0.0f, zy = 0.0f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      e[sp][k] = ex2_approx((z[k] - zmax) * 1.4426950408889634f);  // MUFU: ≤ 2 ulp, z − zmax ≤ 0
      den += e[sp][k];
      // z[label] as a branch-free select: `if (k == label) zy = z[k]` lets the
      // compiler fold the unrolled loop into z[label] — a dynamically
      // indexed array in local memory (STL/LDL in the round kernel)
      zy = __uint_as_float((__float_as_uint(z[k]) & (k == label[sp] ? 0xffffffffu : 0u)) |
                           __float_as_uint(zy));
    }
    inv_den[sp] = 1.0f / den;
    loss[sp] = lg2_approx(den) * 0.6931471805599453f - (zy - zmax);  // den ∈ [1, K]
    if (probs_row[sp] != nullptr) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (lane == k) probs_row[sp][k] = e[sp][k] * inv_den[sp];
    }
  }
  if constexpr (!BWD) return;

  // ---------------- backward: softmax (nn.cpp:276-311) ----------------
#pragma unroll
  for (int sp = 0; sp < SPW; ++sp) dh[sp] = 0.0f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float gws = 0.0f, gbs = 0.0f;
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp) {
      const float dzk = (e[sp][k] * inv_den[sp] - (k == label[sp] ? 1.0f : 0.0f)) * scale[sp];
      gws = fmaf(dzk, hT[sp], gws);
      gbs += dzk;
      dh[sp] = fmaf(wsm[N::OFF_WS + k * H + j], dzk, dh[sp]);  // shadow lanes: = lane j's
    }
    if (act) put(wp[N::OFF_WS + k * H + j], gws);
    if (lane == 0) put(wp[N::OFF_BS + k], gbs);
  }
  }  // HEAD
  if (pr && lane == 0) pr[10] = globaltimer();

  // ------- backward pass 1: the BPTT chain (nn.cpp:351-392), dz → smem -------
  {
    float wt[4 * H];  // column j of Wh: Wh[r][j]
#pragma unroll
    for (int r = 0; r < 4 * H; ++r) wt[r] = wsm[N::OFF_WH + r * H + j];
    float dc[SPW];
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp) dc[sp] = 0.0f;
#pragma unroll 1
    for (int t = T - 1; t >= 0; --t) {
      float fgs[SPW];
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp) {
        const float* ct = cs[sp] + (t * H + j) * 8;
        const float4 g4 = reinterpret_cast<const float4*>(ct)[0];
        const float ig = g4.x, fg = g4.y, gg = g4.z, og = g4.w;
        const float tc = ct[5];
        const float cp = t > 0 ? cs[sp][((t - 1) * H + j) * 8 + 4] : 0.0f;
        fgs[sp] = fg;
        const float dout = dh[sp] * tc;
        dc[sp] = fmaf(dh[sp] * og, 1.0f - tc * tc, dc[sp]);
        const float di = dc[sp] * gg, dg = dc[sp] * ig, df = dc[sp] * cp;
        float* dzt = dzs[sp] + t * 4 * H;
        dzt[0 * H + j] = di * ig * (1.0f - ig);
        dzt[1 * H + j] = df * fg * (1.0f - fg);
        dzt[2 * H + j] = dg * (1.0f - gg * gg);
        dzt[3 * H + j] = dout * og * (1.0f - og);
      }
      __syncwarp();
      if (t > 0) {  // dh_{t-1} = Whᵀ dz_t (the reference also does this at t=0, unused)
#pragma unroll
        for (int sp = 0; sp < SPW; ++sp) {
          const float4* dz4 = reinterpret_cast<const float4*>(dzs[sp] + t * 4 * H);
          float2 p01 = make_float2(0.0f, 0.0f), p23 = make_float2(0.0f, 0.0f);  // FFMA2 pairs
#pragma unroll
          for (int r4 = 0; r4 < H; ++r4) {
            const float4 u = dz4[r4];
            p01 = __ffma2_rn(make_float2(wt[4 * r4], wt[4 * r4 + 1]), make_float2(u.x, u.y), p01);
            p23 = __ffma2_rn(make_float2(wt[4 * r4 + 2], wt[4 * r4 + 3]), make_float2(u.z, u.w), p23);
          }
          dh[sp] = (p01.x + p01.y) + (p23.x + p23.y);
          dc[sp] *= fgs[sp];
        }
      }
    }
  }
  if (pr && lane == 0) pr[11] = globaltimer();

  // ------- backward pass 2: dWx, dWh, db = Σ_{s,t} dz ⊗ [x_t, h_{t-1}] -------
  if (act) {
    float dz[SPW][T][4];
#pragma unroll
    for (int sp = 0; sp < SPW; ++sp)
#pragma unroll
      for (int t = 0; t < T; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) dz[sp][t][q] = dzs[sp][t * 4 * H + q * H + j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float acc = 0.0f;
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp)
#pragma unroll
        for (int t = 0; t < T; ++t) acc += dz[sp][t][q];
      put(wp[N::OFF_B + q * H + j], acc);
    }
    {
      float acc[4][D];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int d = 0; d < D; ++d) acc[q][d] = 0.0f;
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp)
#pragma unroll
        for (int t = 0; t < T; ++t) {
          float xv[DP];
          load_x(sp, t, xv);
#pragma unroll
          for (int d = 0; d < D; ++d)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][d] = fmaf(dz[sp][t][q], xv[d], acc[q][d]);
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int d = 0; d < D; ++d) put(wp[N::OFF_WX + (q * H + j) * D + d], acc[q][d]);
    }
    // dWh in column blocks of 4: 16 accumulators, h_{t-1} read as float4
    constexpr int KB = N::HV ? 4 : 1;
#pragma unroll 1
    for (int k0 = 0; k0 < H; k0 += KB) {
      float acc[KB][4];
#pragma unroll
      for (int kk = 0; kk < KB; ++kk)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[kk][q] = 0.0f;
#pragma unroll
      for (int sp = 0; sp < SPW; ++sp)
#pragma unroll
        for (int t = 1; t < T; ++t) {
          float hv[KB];
          if constexpr (KB == 4) {
            const float4 u = reinterpret_cast<const float4*>(hs[sp] + (t - 1) * H + k0)[0];
            hv[0] = u.x;
            hv[1] = u.y;
            hv[2] = u.z;
            hv[3] = u.w;
          } else {
            hv[0] = hs[sp][(t - 1) * H + k0];
          }
#pragma unroll
          for (int kk = 0; kk < KB; ++kk)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[kk][q] = fmaf(dz[sp][t][q], hv[kk], acc[kk][q]);
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) put(wp[N::OFF_WH + (q * H + j) * H + k0 + kk], acc[kk][q]);
    }
  }
  __syncwarp();
  if (pr && lane == 0) pr[12] = globaltimer();
}

// Single-sample convenience wrapper (flat kernel, non-pipelined paths).
template <int D, int H, int T, int K, bool BWD, bool HEAD = true>
__device__ __forceinline__ float lstm_sample(const float* __restrict__ wsm, float* __restrict__ ws,
                                             float* __restrict__ wp,
                                             const float* __restrict__ xs, int label,
                                             float scale, int lane, float* probs_row,
                                             unsigned long long* pr, float* trunk = nullptr) {
  const float* xa[1] = {xs};
  const int la[1] = {label};
  const float sa[1] = {scale};
  float* pa[1] = {probs_row};
  float* ta[1] = {trunk};
  float lo[1];
  lstm_samples<D, H, T, K, BWD, 1, HEAD>(wsm, ws, wp, xa, la, sa, lane, pa, lo, pr, ta);
  return lo[0];
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
  const int G = gridDim.x;
  const int E = N::P + 1;  // gradient + loss slot

  int cur = 0;
  unsigned long long round0 = 0;
  unsigned long long accepted = 0, rejected = 0, acc_samples = 0;
  int last_status = 0;
  if (a.mode == MODE_SGD) {
    cur = __ldcg(&a.ms->cur);
    round0 = __ldcg(&a.ms->round);
  }
  unsigned epoch = __ldcg(a.bar);
  const bool trunk = a.mode == MODE_TRUNK_FWD || a.mode == MODE_TRUNK_GRAD;

  // Sample s of round r handled by this warp: CTA b owns [b*spc, (b+1)*spc).
  auto first_sample = [&](int r, int& s, int& s1) {
    const int n = a.counts ? __ldg(a.counts + r) : a.n;
    const int spc = (n + G - 1) / G;
    const int s0 = blockIdx.x * spc;
    s1 = min(n, s0 + spc);
    s = s0 + warp;
  };
  float* xbuf = ws + N::S_X;  // [2][XWP]
  int* lbuf = reinterpret_cast<int*>(ws + N::S_L);
  // Asynchronous copy of sample row `row` (x + label) into buffer `b`.
  auto fetch_async = [&](int row, int b) {
    const float* xrow = a.x + (long long)row * N::XW;
    float* dst = xbuf + b * N::XWP;
    for (int i = lane; i < N::XW; i += 32) cp_async4(dst + N::xoff(i), xrow + i);
    if (lane == 0) cp_async4(lbuf + b, a.y + row);
    cp_async_commit();
  };
  auto row_of = [&](int r, int s) {
    // no gather table: round r reads rows r*stride + s (stride 0: rows s)
    return a.idx ? __ldg(a.idx + (long long)r * a.stride + s) : (int)((long long)r * a.stride + s);
  };
  if (a.pipelined) {
    int s, s1;
    first_sample(0, s, s1);
    if (s < s1) fetch_async(row_of(0, s), 0);
  }

  for (int r = 0; r < a.rounds; ++r) {
    const float* w = a.mode == MODE_SGD ? (cur ? a.w1 : a.w0) : a.w_in;
    const int n = a.counts ? __ldg(a.counts + r) : a.n;
    const float scale = a.mode == MODE_SGD ? 1.0f / (float)n : a.grad_scale;

    unsigned long long* pr =
        a.probe ? a.probe + ((long long)r * gridDim.x + blockIdx.x) * 16 : nullptr;
    if (pr && threadIdx.x == 0) pr[0] = globaltimer();
    if ((reinterpret_cast<uintptr_t>(w) & 15u) == 0) {
      for (int p = threadIdx.x; p < N::P / 4; p += blockDim.x)
        reinterpret_cast<float4*>(wsm)[p] = __ldcg(reinterpret_cast<const float4*>(w) + p);
      for (int p = (N::P & ~3) + threadIdx.x; p < N::P; p += blockDim.x) wsm[p] = __ldcg(w + p);
    } else {
      for (int p = threadIdx.x; p < N::P; p += blockDim.x) wsm[p] = __ldcg(w + p);
    }
    float* wp = wpart + warp * N::PPAD;
    if (a.mode != MODE_FWD) {
      for (int p = lane; p < N::PPAD / 4; p += 32)
        reinterpret_cast<float4*>(wp)[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    if (pr && threadIdx.x == 0) pr[1] = globaltimer();

    // ---- per-warp samples of this CTA's contiguous chunk ----
    float lsum = 0.0f;
    int s, s1;
    first_sample(r, s, s1);
    if (a.pipelined) {
      // ≤ 1 sample per warp per round; its row is already in flight (or landed)
      // in buffer r&1.  Ask for next round's index now, the row after compute.
      int sn = 0, sn1 = 0;
      const bool next = r + 1 < a.rounds;
      if (next) {
        first_sample(r + 1, sn, sn1);
        if (sn < sn1 && a.idx && lane == 0)
          cp_async4(lbuf + 2, a.idx + (long long)(r + 1) * a.stride + sn);
        cp_async_commit();
      }
      if (s < s1) {
        if (next) cp_async_wait<1>();  // this round's row (older group) has landed
        else cp_async_wait<0>();       // no newer group on the last round
        __syncwarp();
        int label = lbuf[r & 1];
        // the trunk of a deeper net has no labels here (the head kernel checks them)
        if (!trunk && (label < 0 || label >= K)) {
          if (lane == 0) atomicOr(a.err, 1);
          label = 0;
        }
        unsigned long long* ps = (pr && warp == 0) ? pr : nullptr;
        const float* xs = xbuf + (r & 1) * N::XWP;
        if (a.mode == MODE_FWD) {
          lsum = lstm_sample<D, H, T, K, false>(
              wsm, ws, wp, xs, label, scale, lane,
              a.probs_out ? a.probs_out + (long long)s * K : nullptr, ps);
        } else if (a.mode == MODE_TRUNK_FWD) {
          lstm_sample<D, H, T, K, false, false>(wsm, ws, wp, xs, label, scale, lane, nullptr, ps,
                                                a.hio + (long long)s * H);
        } else if (a.mode == MODE_TRUNK_GRAD) {
          lstm_sample<D, H, T, K, true, false>(wsm, ws, wp, xs, label, scale, lane, nullptr, ps,
                                               a.hio + (long long)s * H);
        } else {
          lsum = lstm_sample<D, H, T, K, true>(wsm, ws, wp, xs, label, scale, lane, nullptr, ps);
        }
      }
      if (next && sn < sn1) {
        cp_async_wait<0>();
        __syncwarp();
        const int row = a.idx ? lbuf[2] : (int)((long long)(r + 1) * a.stride + sn);
        __syncwarp();
        fetch_async(row, (r + 1) & 1);
      }
    } else {
      for (; s < s1; s += NW) {
        const int row = row_of(r, s);
        float* xs = xbuf;
        for (int i = lane; i < N::XW; i += 32) xs[N::xoff(i)] = __ldg(a.x + (long long)row * N::XW + i);
        int label = __ldg(a.y + row);
        __syncwarp();
        if (!trunk && (label < 0 || label >= K)) {
          if (lane == 0) atomicOr(a.err, 1);
          label = 0;
        }
        if (trunk) label = 0;
        if (a.mode == MODE_FWD) {
          lsum += lstm_sample<D, H, T, K, false>(
              wsm, ws, wp, xs, label, scale, lane,
              a.probs_out ? a.probs_out + (long long)s * K : nullptr, nullptr);
        } else if (a.mode == MODE_TRUNK_FWD) {
          lstm_sample<D, H, T, K, false, false>(wsm, ws, wp, xs, label, scale, lane, nullptr,
                                                nullptr, a.hio + (long long)s * H);
        } else if (a.mode == MODE_TRUNK_GRAD) {
          lstm_sample<D, H, T, K, true, false>(wsm, ws, wp, xs, label, scale, lane, nullptr,
                                               nullptr, a.hio + (long long)s * H);
        } else {
          lsum += lstm_sample<D, H, T, K, true>(wsm, ws, wp, xs, label, scale, lane, nullptr,
                                                nullptr);
        }
        __syncwarp();
      }
    }
    if (lane == 0) wp[N::P] = lsum;  // the loss rides in the padded slot P
    __syncthreads();
    if (pr && threadIdx.x == 0) pr[2] = globaltimer();

    // ---- CTA partial (fixed warp order) → global, float4 ----
    float4* prow = reinterpret_cast<float4*>(a.part + (long long)blockIdx.x * a.pstride);
    for (int p = threadIdx.x; p < N::PPAD / 4; p += blockDim.x) {
      float4 t = reinterpret_cast<const float4*>(wpart)[p];
      for (int w2 = 1; w2 < NW; ++w2) {
        const float4 u = reinterpret_cast<const float4*>(wpart + w2 * N::PPAD)[p];
        t.x += u.x;
        t.y += u.y;
        t.z += u.z;
        t.w += u.w;
      }
      __stcg(prow + p, t);
    }
    if (pr && threadIdx.x == 0) pr[3] = globaltimer();
    flag_barrier(a.bar, ++epoch, 0);
    if (pr && threadIdx.x == 0) pr[4] = globaltimer();

    // ---- distributed deterministic reduction of slice [p0,p1) over CTAs ----
    const int slice = (E + G - 1) / G;
    const bool fwd_only = a.mode == MODE_FWD || a.mode == MODE_TRUNK_FWD;
    const int p0 = fwd_only ? (blockIdx.x == 0 ? N::P : E) : blockIdx.x * slice;
    const int p1 = fwd_only ? E : min(E, p0 + slice);
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
      const int p = base + c;
      // master state for this parameter, loaded while the partials fly
      float wv = 0.f, vv = 0.f;
      if (a.mode == MODE_SGD && threadIdx.x < nc && base + threadIdx.x < N::P) {
        wv = __ldcg(wcur + base + threadIdx.x);
        vv = __ldcg(vcur + base + threadIdx.x);
      }
      float sum = 0.0f;
      if (c < nc && gidx < groups) {
        for (int b0 = gidx; b0 < G; b0 += 16 * groups) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int b = b0 + i * groups;
            v[i] = b < G ? __ldcg(a.part + (long long)b * a.pstride + p) : 0.0f;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) sum += v[i];
        }
      }
      if (gidx < groups) red[gidx * cols + c] = sum;
      __syncthreads();
      if (threadIdx.x < nc) {
        float tot = 0.0f;
        for (int g2 = 0; g2 < groups; ++g2) tot += red[g2 * cols + threadIdx.x];
        const int pp = base + threadIdx.x;
        if (pp == N::P) {
          if (a.loss_out) a.loss_out[r] = tot;
        } else if (a.mode == MODE_GRAD) {
          a.g_out[pp] = tot;
        } else if (a.mode == MODE_TRUNK_GRAD) {
          if (pp < N::OFF_WS) a.g_out[pp] = tot;  // trunk: Wx, Wh, b only
        } else if (a.mode == MODE_SGD) {
          if (!is_finite_f(tot)) bad = 1;
          // sgd_step (optim.cpp:59-60): v = mu*v - lr*g; w += v
          const float vn = fmaf(a.mu, vv, -a.lr * tot);
          __stcg(vnext + pp, vn);
          __stcg(wnext + pp, wv + vn);
        }
      }
      __syncthreads();
    }
    if (a.mode == MODE_SGD) {
      if (pr && threadIdx.x == 0) pr[5] = globaltimer();
      const int rej = flag_barrier(a.bar, ++epoch, bad);
      if (pr && threadIdx.x == 0) pr[6] = globaltimer();
      if (rej) {
        ++rejected;
        last_status = 2;  // GHC_ERR_NONFINITE: keep w/v (optim.cpp:49-51)
      } else {
        cur ^= 1;
        ++accepted;
        acc_samples += (unsigned long long)n;
        last_status = 0;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.bar[0] = epoch;
    if (a.mode == MODE_SGD) {
      a.ms->cur = cur;
      a.ms->version += accepted;
      a.ms->rejected += rejected;
      a.ms->samples += acc_samples;
      a.ms->round = round0 + (unsigned long long)a.rounds;
      a.ms->status = last_status;
    }
  }
}

}  // namespace ghc
