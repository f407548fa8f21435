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

#include "ghc_internal.cuh"

struct ghc_resident {
  ghc_master* m = nullptr;
  ghc_plan* p = nullptr;
  cudaStream_t stream = nullptr;
  ResidentCtl* ctl = nullptr;                // device
  ResidentCmd* h_cmd = nullptr;              // pinned, mapped
  unsigned long long* h_bell = nullptr;      // pinned, mapped
  unsigned long long* h_done = nullptr;      // pinned, mapped [2]
  uint64_t next = 1;
  int64_t n = 0;
  bool stopped = false;
};

namespace {

// Submit + wait in ONE kernel (one tiny launch per stream command instead of two).
__global__ void resident_submit_wait_kernel(ResidentCtl* c, ResidentCmd cmd) {
  if (atomicCAS(&c->claim, cmd.seq - 1, cmd.seq) != cmd.seq - 1) {
    c->submit_failed = 1;  // the service expired (idle STOP claimed this slot)
    return;
  }
  c->cmd[cmd.seq % kResRing] = cmd;
  c->t[0] = res_now();
  c->t[1] = ~0ull;
  c->t[2] = 0;
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
    delete r;
    return s;
  };
  if (cudaSetDevice(p->ctx->device) != cudaSuccess ||
      cudaMalloc(&r->ctl, sizeof(ResidentCtl)) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&r->h_cmd), sizeof(ResidentCmd) * kResRing, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&r->h_bell), sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&r->h_done), 2 * sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess)
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
  r->m->host_cur_known = false;
  cudaFree(r->ctl);
  cudaFreeHost(r->h_cmd);
  cudaFreeHost(r->h_bell);
  cudaFreeHost(r->h_done);
  cudaStreamDestroy(r->stream);
  delete r;
  return st;
}

}  // extern "C"
