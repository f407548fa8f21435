// resident.cu — the resident round service (ghc_resident_*, include/ghc.h):
// the persistent sync-round kernel (lstm_round.cuh) launched once, serving
// commands (one segment of rounds each) through doorbells instead of a
// cooperative cluster launch per call.  Measured on B200 (tools/
// launch_anatomy.py): a launch of the round kernel costs ≈ 13 µs of launch,
// prologue and teardown on the device before/after its rounds; a served
// command costs a doorbell hop.  Protocol and completion: lstm_step.cuh
// (ResidentCtl).  One submission path at a time (host ring or stream), in
// order.
#include <chrono>
#include <thread>
#include <vector>

#include "ghc_internal.cuh"

struct ghc_resident {
  ghc_master* m = nullptr;
  ghc_plan* p = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t relay_stream = nullptr;       // the host-ring relay kernel
  ResidentCtl* ctl = nullptr;                // device
  ResidentCmd* h_cmd = nullptr;              // pinned, mapped
  unsigned long long* h_bell = nullptr;      // pinned, mapped
  unsigned long long* h_done = nullptr;      // pinned, mapped [2]
  uint64_t next = 1;
  int64_t n = 0;
  bool stopped = false;
};

namespace {

// The relay on a spare SM (the round kernel leaves 20 of 148 free):
//  * publishes each host-ring command into the device ring as soon as it
//    lands (the round CTAs only ever read L2, and a queued next command is
//    visible when a command's last round starts — its first batch is then
//    fetched during that round's exchange);
//  * publishes completions: command s is done once every round CTA arrived
//    for it (arrive ≥ s · ctas; the CTAs only fire a reduction) — device word
//    for the stream waiter, pinned word for the host.
// CTA 0 of the round kernel keeps a fallback relay; the claim word makes
// either one write a slot once.
// Two warps: warp 0 publishes completions (L2 polling only — a completion
// is seen within one L2 round trip), warp 1 relays host commands (its
// doorbell polls cross PCIe, ≈ 1–2 µs each, and must not delay warp 0).
__global__ void __launch_bounds__(64) resident_relay_kernel(ResidentCtl* c) {
  __shared__ volatile unsigned long long s_stop_at;  // seq of the STOP command (0: none yet)
  if (threadIdx.x == 0) s_stop_at = 0;
  __syncthreads();
  if ((threadIdx.x & 31) != 0) return;
  if (threadIdx.x == 0) {  // ---- completions ----
    unsigned long long next_done = 1, ctas = 0, t0 = res_now();
    for (unsigned it = 0;; ++it) {
      if (!ctas) ctas = *reinterpret_cast<volatile unsigned long long*>(&c->ctas);
      if (ctas) {
        const unsigned long long arrived = res_ld_acquire(&c->arrive);
        while (next_done * ctas <= arrived) {
          __threadfence_system();
          c->t[3] = res_now();
          c->tlog[next_done % 64][1] = c->t[3];
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&c->done), "l"(next_done) : "memory");
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(c->host_done), "l"(next_done) : "memory");
          ++next_done;
          t0 = res_now();
        }
      }
      const unsigned long long stop_at = s_stop_at;
      if (stop_at && next_done >= stop_at) return;  // every command before the STOP published
      if ((it & 255u) == 0 && res_now() - t0 > c->idle_ns + 20000000000ull) return;  // never strand the SM
    }
  } else {  // ---- host commands ----
    unsigned long long next = 1, t0 = res_now();
    for (unsigned it = 0;; ++it) {
      const unsigned long long hb = res_ld_sys(c->host_bell);
      if (next <= hb && atomicCAS(&c->claim, next - 1, next) == next - 1) {
        const ResidentCmd v = load_host_cmd(c->host_cmd + (next % kResRing));
        write_cmd(c, v);
        __threadfence_system();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&c->bell), "l"(next) : "memory");
        if (v.op != 0) {
          s_stop_at = next;
          return;
        }
        ++next;
        t0 = res_now();
      } else {
        // published by someone else (stream submitter, CTA 0's fallback)?
        unsigned long long v[8];
        issue_slot_loads(c, next, v);
        ResidentCmd cmd;
        if (slot_valid(v, next, cmd)) {
          if (cmd.op != 0) {
            s_stop_at = next;
            return;
          }
          ++next;
          t0 = res_now();
        }
      }
      if ((it & 63u) == 0 && res_now() - t0 > c->idle_ns + 20000000000ull) {
        s_stop_at = ~0ull;  // give up: the completion warp may leave too
        return;
      }
    }
  }
}

// Submit + wait in ONE kernel (stream path): claim and write the slot, then
// spin until the relay published the completion.
__global__ void resident_submit_wait_kernel(ResidentCtl* c, ResidentCmd cmd) {
  if (atomicCAS(&c->claim, cmd.seq - 1, cmd.seq) != cmd.seq - 1) {
    c->submit_failed = 1;  // the service expired (idle STOP claimed this slot)
    return;
  }
  c->t[0] = res_now();
  c->t[1] = ~0ull;
  c->t[2] = 0;
  write_cmd(c, cmd);
  __threadfence();
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&c->bell), "l"(cmd.seq) : "memory");
  const unsigned long long t0 = res_now();
  for (unsigned it = 0; res_ld_acquire(&c->done) < cmd.seq; ++it) {
    if ((it & 255u) == 0 &&
        (*reinterpret_cast<volatile int*>(&c->expired) || res_now() - t0 > 30000000000ull))
      return;  // the host reads the failure with ghc_resident_check
  }
  c->t[4] = res_now();
}

volatile unsigned long long& vol(unsigned long long* p) { return *reinterpret_cast<volatile unsigned long long*>(p); }

}  // namespace

extern "C" {

ghc_status ghc_resident_start(ghc_master* m, int64_t n, double idle_seconds, ghc_resident** out) {
  if (!m || !out) return fail(GHC_ERR_CONFIG, "resident_start: null argument");
  if (n < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");
  ghc_plan* p = m->plan;
  if (p->layered || !p->lstm) return fail(GHC_ERR_CONFIG, "resident rounds need a fused round kernel");
  auto* r = new ghc_resident();
  r->m = m;
  r->p = p;
  r->n = n;
  auto bail = [&](ghc_status s) {
    cudaFree(r->ctl);
    cudaFreeHost(r->h_cmd);
    cudaFreeHost(r->h_bell);
    cudaFreeHost(r->h_done);
    if (r->stream) cudaStreamDestroy(r->stream);
    if (r->relay_stream) cudaStreamDestroy(r->relay_stream);
    delete r;
    return s;
  };
  if (cudaSetDevice(p->ctx->device) != cudaSuccess ||
      cudaMalloc(&r->ctl, sizeof(ResidentCtl)) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&r->h_cmd), sizeof(ResidentCmd) * kResRing, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&r->h_bell), sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&r->h_done), 2 * sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&r->relay_stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(GHC_ERR_CUDA, "resident_start: allocation failed"));
  std::memset(r->h_cmd, 0, sizeof(ResidentCmd) * kResRing);
  *r->h_bell = 0;
  r->h_done[0] = r->h_done[1] = 0;
  ResidentCtl init{};
  void* dp = nullptr;
  cudaHostGetDevicePointer(&dp, r->h_cmd, 0);
  init.host_cmd = static_cast<ResidentCmd*>(dp);
  cudaHostGetDevicePointer(&dp, r->h_bell, 0);
  init.host_bell = static_cast<unsigned long long*>(dp);
  cudaHostGetDevicePointer(&dp, r->h_done, 0);
  init.host_done = static_cast<unsigned long long*>(dp);
  init.idle_ns = static_cast<unsigned long long>((idle_seconds > 0 ? idle_seconds : 2.0) * 1e9);
  if (cudaMemcpy(r->ctl, &init, sizeof(init), cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(GHC_ERR_CUDA, "resident_start: control block upload failed"));
  // CUDA lazy loading loads a kernel's module at its first launch and that
  // load waits for the running kernels — which a resident kernel never
  // ends: load every kernel that may be launched while it runs NOW
  {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(resident_submit_wait_kernel)) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(resident_relay_kernel)) != cudaSuccess ||
        ghc_preload_gate() != GHC_OK)
      return bail(fail(GHC_ERR_CUDA, "resident_start: kernel preload failed"));
  }
  // the master's state is consumed by the kernel: finish its pending work first
  if (cudaStreamSynchronize(p->ctx->stream) != cudaSuccess)
    return bail(fail(GHC_ERR_CUDA, "resident_start: context stream failed"));
  StepArgs a{};
  a.n = static_cast<int>(n);
  a.rounds = 0;
  a.w0 = m->w[0];
  a.w1 = m->w[1];
  a.v0 = m->v[0];
  a.v1 = m->v[1];
  a.lr = m->lr;
  a.mu = m->mu;
  a.ms = m->ms;
  a.mode = MODE_SGD;
  a.res = r->ctl;
  if (ghc_status s = launch_step(p, a, n, 1, r->stream)) return bail(s);
  resident_relay_kernel<<<1, 64, 0, r->relay_stream>>>(r->ctl);
  if (cudaGetLastError() != cudaSuccess) return bail(fail(GHC_ERR_CUDA, "resident_start: relay launch failed"));
  m->host_cur_known = false;
  *out = r;
  return GHC_OK;
}

ghc_status ghc_resident_submit(ghc_resident* r, const float* x, const int32_t* y, const int32_t* idx,
                               int64_t stride, int32_t rounds, float* loss_out, uint64_t* seq_out) {
  if (!r || r->stopped) return fail(GHC_ERR_CONFIG, "resident_submit: service stopped");
  if (rounds < 1 || !x) return fail(GHC_ERR_SHAPE, "resident_submit: empty command");
  if (vol(r->h_done + 1)) return fail(GHC_ERR_CUDA, "resident service expired (idle timeout)");
  const uint64_t seq = r->next++;
  const auto t0 = std::chrono::steady_clock::now();
  while (seq - vol(r->h_done) >= static_cast<uint64_t>(kResRing)) {  // ring full: wait for a slot
    if (vol(r->h_done + 1)) return fail(GHC_ERR_CUDA, "resident service expired (idle timeout)");
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
      return fail(GHC_ERR_CUDA, "resident_submit: no progress for 30 s");
  }
  ResidentCmd c{};
  c.x = x;
  c.y = y;
  c.idx = idx;
  c.stride = stride;
  c.loss_out = loss_out;
  c.rounds = rounds;
  c.op = 0;
  c.seq = seq;
  std::memcpy(static_cast<void*>(r->h_cmd + seq % kResRing), &c, sizeof(c));
  std::atomic_thread_fence(std::memory_order_seq_cst);
  vol(r->h_bell) = seq;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (seq_out) *seq_out = seq;
  return GHC_OK;
}

ghc_status ghc_resident_wait(ghc_resident* r, uint64_t seq) {
  if (!r) return fail(GHC_ERR_CONFIG, "resident_wait: null handle");
  const auto t0 = std::chrono::steady_clock::now();
  while (vol(r->h_done) < seq) {
    if (vol(r->h_done + 1)) return fail(GHC_ERR_CUDA, "resident service expired (idle timeout)");
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
      return fail(GHC_ERR_CUDA, "resident_wait: no completion for 30 s");
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return GHC_OK;
}

ghc_status ghc_resident_submit_stream(ghc_resident* r, ghc_ctx* c, const float* x, const int32_t* y,
                                      const int32_t* idx, int64_t stride, int32_t rounds, float* loss_out,
                                      uint64_t* seq_out) {
  if (!r || r->stopped || !c) return fail(GHC_ERR_CONFIG, "resident_submit_stream: service stopped");
  if (rounds < 1 || !x) return fail(GHC_ERR_SHAPE, "resident_submit_stream: empty command");
  ResidentCmd cmd{};
  cmd.x = x;
  cmd.y = y;
  cmd.idx = idx;
  cmd.stride = stride;
  cmd.loss_out = loss_out;
  cmd.rounds = rounds;
  cmd.op = 0;
  cmd.seq = r->next++;
  resident_submit_wait_kernel<<<1, 1, 0, c->stream>>>(r->ctl, cmd);
  CU(cudaGetLastError());
  c->launches += 1;
  if (seq_out) *seq_out = cmd.seq;
  return GHC_OK;
}

ghc_status ghc_resident_times(ghc_resident* r, uint64_t* t5) {
  ResidentCtl h;
  CU(cudaMemcpy(&h, r->ctl, sizeof(h), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 5; ++i) t5[i] = h.t[i];
  for (int i = 0; i < 64; ++i) {
    t5[5 + 2 * i] = h.tlog[i][0];
    t5[6 + 2 * i] = h.tlog[i][1];
  }
  return GHC_OK;
}

// A C++ caller's per-batch loop over the host doorbell (the reference is
// C++; no Python in the loop): batch k = rows [k·x_batch_stride …) of x
// (packed rows when y == NULL), one round per call, loss k → loss_out[k];
// depth d: up to d batches in flight (1 = submit + wait per batch).
// *us_per_call = host wall time / n_calls.
ghc_status ghc_resident_bench_calls(ghc_resident* r, const float* x, int64_t x_batch_stride,
                                    const int32_t* y, int64_t y_batch_stride, int32_t n_calls,
                                    int32_t depth, float* loss_out, double* us_per_call) {
  if (!r || n_calls < 1 || depth < 1 || depth >= kResRing) return fail(GHC_ERR_CONFIG, "resident_bench_calls: bad argument");
  std::vector<uint64_t> seq(static_cast<size_t>(n_calls));
  const auto t0 = std::chrono::steady_clock::now();
  for (int k = 0; k < n_calls; ++k) {
    if (ghc_status s = ghc_resident_submit(r, x + static_cast<int64_t>(k) * x_batch_stride,
                                           y ? y + static_cast<int64_t>(k) * y_batch_stride : nullptr, nullptr, 0,
                                           1, loss_out ? loss_out + k : nullptr, &seq[static_cast<size_t>(k)]))
      return s;
    if (k + 1 >= depth)
      if (ghc_status s = ghc_resident_wait(r, seq[static_cast<size_t>(k + 1 - depth)])) return s;
  }
  if (ghc_status s = ghc_resident_wait(r, seq.back())) return s;
  *us_per_call = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n_calls;
  return GHC_OK;
}

ghc_status ghc_resident_check(ghc_resident* r) {
  ResidentCtl h;
  CU(cudaMemcpy(&h, r->ctl, sizeof(h), cudaMemcpyDeviceToHost));
  if (h.expired) return fail(GHC_ERR_CUDA, "resident service expired (idle timeout)");
  if (h.submit_failed) return fail(GHC_ERR_CUDA, "resident_submit_stream: service had expired");
  return GHC_OK;
}

ghc_status ghc_resident_stop(ghc_resident* r) {
  if (!r) return GHC_OK;
  ghc_status st = GHC_OK;
  if (!vol(r->h_done + 1)) {  // still serving: STOP through the host ring
    const uint64_t seq = r->next++;
    ResidentCmd c{};
    c.op = 1;
    c.seq = seq;
    std::memcpy(static_cast<void*>(r->h_cmd + seq % kResRing), &c, sizeof(c));
    std::atomic_thread_fence(std::memory_order_seq_cst);
    vol(r->h_bell) = seq;
  }
  if (cudaStreamSynchronize(r->stream) != cudaSuccess) st = fail(GHC_ERR_CUDA, "resident kernel failed");
  if (cudaStreamSynchronize(r->relay_stream) != cudaSuccess && st == GHC_OK)
    st = fail(GHC_ERR_CUDA, "resident relay kernel failed");
  r->m->host_cur_known = false;
  cudaFree(r->ctl);
  cudaFreeHost(r->h_cmd);
  cudaFreeHost(r->h_bell);
  cudaFreeHost(r->h_done);
  cudaStreamDestroy(r->stream);
  cudaStreamDestroy(r->relay_stream);
  delete r;
  return st;
}

}  // extern "C"
