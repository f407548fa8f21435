// p2p.cu — fused NVLink exchange for synchronous Downpour across GPUs.
//
// Replaces, for the sync round, the Endpoint GRADIENT/WEIGHTS round trip of
// the reference (transport.hpp:22-44) AND the NCCL
// reduce/broadcast pair of dist.cu: every rank runs the persistent round
// kernel (lstm_round.cuh) on its own batch and holds a bit-identical replica
// of the master; inside the kernel each cluster pushes its rank-local
// sub-slice of the gradient straight into every rank's receive buffer (P2P
// stores over NVLink), each value tagged with the exchange epoch in the same
// 8-byte store (no fences, no counters), and every CTA sums the ranks' rows
// of its slice in rank order once the tags match, then applies sgd_step —
// one kernel, no host round trip, no collective call.
//
// Buffers: per rank one cudaMalloc holding the tagged receive rows
// uint2[2][GX][EP] (parity double buffer) and a line that keeps the exchange
// epoch across launches.  Ranks exchange cudaIpc handles through
// the caller (bytes over torch.distributed / any bootstrap); a "virtual"
// exchange puts all GX ranks into ONE grid on one GPU (same kernel code, peer
// pointers into one allocation) — how the path is tested on a single GPU.
#include "ghc_internal.cuh"

struct ghc_p2p {
  ghc_plan* plan = nullptr;
  int rank = 0, G = 1;
  bool virt = false;
  int ep = 0;
  size_t rank_bytes = 0;
  void* own = nullptr;                 // this process's allocation
  void* opened[kMaxRanks] = {};        // IPC-opened peer allocations
  float* gpart[kMaxRanks] = {};
  unsigned* gcnt[kMaxRanks] = {};
  unsigned barrier_epoch = 0;          // ghc_p2p_barrier calls so far (equal on all ranks)
};

namespace {

// receive rows are epoch-tagged values (uint2 per element, see ClusterXchg)
size_t gpart_bytes(int G, int ep) { return ((sizeof(uint2) * 2 * G * ep) + 255) & ~size_t(255); }
// counter lines: [cs] ClusterXchg lines, [cs] the exchange epoch, [cs + 1]
// the start barrier (slot q = rank q's arrival epoch)
size_t cnt_bytes(int cs) { return sizeof(unsigned) * kFlagStride * (cs + 2); }

ghc_status p2p_new(ghc_plan* plan, int rank, int G, bool virt, ghc_p2p** out) {
  if (!out) return fail(GHC_ERR_CONFIG, "p2p: null out");
  *out = nullptr;
  if (!plan || plan->layered || !plan->lstm || !plan->use_cluster || plan->max_clusters < 1)
    return fail(GHC_ERR_CONFIG, "p2p exchange needs the fused LSTM round kernel (cluster variant)");
  if (G < 2 || G > kMaxRanks) return fail(GHC_ERR_CONFIG, "p2p: nranks must be in [2, 8]");
  if (rank < 0 || rank >= G) return fail(GHC_ERR_CONFIG, "p2p: rank out of range");
  if (virt && plan->max_clusters / G < 1)
    return fail(GHC_ERR_CONFIG, "p2p: not enough co-resident clusters for the virtual ranks");
  auto* p = new ghc_p2p;
  p->plan = plan;
  p->rank = rank;
  p->G = G;
  p->virt = virt;
  p->ep = plan->lstm->ep[plan->cs_index];
  p->rank_bytes = gpart_bytes(G, p->ep) + cnt_bytes(plan->cluster_size);
  CU(cudaSetDevice(plan->ctx->device));
  const size_t total = p->rank_bytes * (virt ? G : 1);
  CU(cudaMalloc(&p->own, total));
  CU(cudaMemset(p->own, 0, total));
  // complete before the handle leaves this process: peers' kernels store
  // into these rows as soon as they launch, and cudaMemset is not ordered
  // with respect to other processes' work
  CU(cudaDeviceSynchronize());
  auto bind = [&](int q, char* base) {
    p->gpart[q] = reinterpret_cast<float*>(base);
    p->gcnt[q] = reinterpret_cast<unsigned*>(base + gpart_bytes(G, p->ep));
  };
  if (virt)
    for (int q = 0; q < G; ++q) bind(q, static_cast<char*>(p->own) + q * p->rank_bytes);
  else
    bind(rank, static_cast<char*>(p->own));
  *out = p;
  return GHC_OK;
}

}  // namespace

ghc_status ghc_p2p_create(ghc_plan* plan, int32_t rank, int32_t nranks, ghc_p2p** out) {
  return p2p_new(plan, rank, nranks, false, out);
}

ghc_status ghc_p2p_create_virtual(ghc_plan* plan, int32_t nranks, ghc_p2p** out) {
  return p2p_new(plan, 0, nranks, true, out);
}

ghc_status ghc_p2p_export(ghc_p2p* p, uint8_t* out_handle) {
  if (!p || !out_handle) return fail(GHC_ERR_CONFIG, "p2p_export: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == GHC_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  CU(cudaSetDevice(p->plan->ctx->device));
  CU(cudaIpcGetMemHandle(&h, p->own));
  std::memcpy(out_handle, &h, sizeof(h));
  return GHC_OK;
}

ghc_status ghc_p2p_import(ghc_p2p* p, const uint8_t* handles) {
  if (!p || !handles) return fail(GHC_ERR_CONFIG, "p2p_import: null argument");
  if (p->virt) return GHC_OK;
  CU(cudaSetDevice(p->plan->ctx->device));
  for (int q = 0; q < p->G; ++q) {
    if (q == p->rank) continue;
    if (p->opened[q]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + static_cast<size_t>(q) * GHC_IPC_HANDLE_BYTES, sizeof(h));
    void* base = nullptr;
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return fail(GHC_ERR_TRANSPORT, "p2p_import: cannot map rank " + std::to_string(q) +
                                         "'s buffer (no peer access between these GPUs?)");
    }
    p->opened[q] = base;
    p->gpart[q] = static_cast<float*>(base);
    p->gcnt[q] = reinterpret_cast<unsigned*>(static_cast<char*>(base) + gpart_bytes(p->G, p->ep));
  }
  return GHC_OK;
}

void ghc_p2p_destroy(ghc_p2p* p) {
  if (!p) return;
  cudaSetDevice(p->plan->ctx->device);
  cudaStreamSynchronize(p->plan->ctx->stream);
  for (int q = 0; q < kMaxRanks; ++q)
    if (p->opened[q]) cudaIpcCloseMemHandle(p->opened[q]);
  cudaFree(p->own);
  delete p;
}

ghc_status ghc_p2p_sync_rounds(ghc_master* m, ghc_p2p* p, const float* d_x, const int32_t* d_y,
                               const int32_t* d_idx, int64_t stride, int64_t idx_vstride,
                               const int32_t* d_counts, int64_t n_max, int32_t n_rounds,
                               float* d_loss_out) {
  if (!m || !p) return fail(GHC_ERR_CONFIG, "p2p_sync_rounds: null handle");
  if (m->plan != p->plan) return fail(GHC_ERR_CONFIG, "p2p_sync_rounds: master and exchange use different plans");
  if (n_max < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");
  if (n_rounds < 1) return GHC_OK;
  for (int q = 0; q < p->G; ++q)
    if (!p->gpart[q]) return fail(GHC_ERR_TRANSPORT, "p2p_sync_rounds: peers not imported");
  if (!d_y && (p->plan->use_tc || !p->plan->use_cluster))
    return fail(GHC_ERR_CONFIG, "packed dataset rows need the SIMT cluster round kernel");
  StepArgs a{};
  a.x = d_x;
  a.y = d_y;
  a.idx = d_idx;
  a.stride = stride;
  a.counts = d_counts;
  a.n = static_cast<int>(n_max);
  a.rounds = n_rounds;
  a.w0 = m->w[0];
  a.w1 = m->w[1];
  a.v0 = m->v[0];
  a.v1 = m->v[1];
  a.lr = m->lr;
  a.mu = m->mu;
  a.ms = m->ms;
  a.loss_out = d_loss_out;
  a.mode = MODE_SGD;
  a.GX = p->G;
  a.rank0 = p->virt ? 0 : p->rank;
  a.idx_vstride = idx_vstride;
  for (int q = 0; q < p->G; ++q) {
    a.gpart[q] = p->gpart[q];
    a.gcnt[q] = p->gcnt[q];
  }
  m->host_cur_known = false;  // the round kernel flips the buffers on device
  return launch_step(m->plan, a, n_max, p->virt ? p->G : 1);
}

// ---------------------------------------------------------------- diagnostics
// The cross-process half of the fused exchange without co-resident round
// kernels (a 2-process single-GPU test must not run ranks whose kernels
// wait on each other): rank `rank` stores n (value, epoch-tag) 64-bit
// elements into row `rank` of rank `dst`'s IPC-mapped receive rows with the
// same system-scope relaxed stores the round kernel uses (ClusterRS::
// cross_rank_sum), and the owner later reads them back with the kernel's
// system-scope loads and checks value and tag.
namespace {
__device__ __forceinline__ float diag_value(int rank, int e) { return (float)(rank * 4096 + e) + 0.25f; }

__global__ void p2p_diag_push_kernel(uint2* rows, int G, int rank, int ep, int par, unsigned tag, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n && e < ep; e += gridDim.x * blockDim.x) {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(diag_value(rank, e));
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(rows) + ((long long)par * G + rank) * ep + e;
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(dst), "l"(w) : "memory");
  }
}

__global__ void p2p_diag_check_kernel(const uint2* rows, int G, int src, int ep, int par, unsigned tag,
                                      int n, int* bad) {
  int b = 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n && e < ep; e += gridDim.x * blockDim.x) {
    const unsigned long long* p =
        reinterpret_cast<const unsigned long long*>(rows) + ((long long)par * G + src) * ep + e;
    unsigned long long w;
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    b += ((unsigned)(w >> 32) != tag) || (__uint_as_float((unsigned)w) != diag_value(src, e));
  }
  if (b) atomicAdd(bad, b);
}
}  // namespace

extern "C" ghc_status ghc_p2p_diag_push(ghc_p2p* p, int32_t dst, uint32_t tag, int32_t n) {
  if (!p || dst < 0 || dst >= p->G || !p->gpart[dst]) return fail(GHC_ERR_CONFIG, "p2p_diag_push: bad rank");
  p2p_diag_push_kernel<<<8, 256, 0, p->plan->ctx->stream>>>(reinterpret_cast<uint2*>(p->gpart[dst]), p->G,
                                                          p->rank, p->ep, tag & 1u, tag, n);
  CU(cudaGetLastError());
  p->plan->ctx->launches++;
  CU(cudaStreamSynchronize(p->plan->ctx->stream));
  return GHC_OK;
}

extern "C" ghc_status ghc_p2p_diag_check(ghc_p2p* p, int32_t src, uint32_t tag, int32_t n, int32_t* h_bad) {
  if (!p || src < 0 || src >= p->G || !h_bad) return fail(GHC_ERR_CONFIG, "p2p_diag_check: bad argument");
  int* d_bad = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(int), p->plan->ctx->stream));
  CU(cudaMemsetAsync(d_bad, 0, sizeof(int), p->plan->ctx->stream));
  p2p_diag_check_kernel<<<8, 256, 0, p->plan->ctx->stream>>>(reinterpret_cast<const uint2*>(p->gpart[p->rank]),
                                                           p->G, src, p->ep, tag & 1u, tag, n, d_bad);
  CU(cudaGetLastError());
  p->plan->ctx->launches++;
  CU(cudaMemcpyAsync(h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, p->plan->ctx->stream));
  CU(cudaFreeAsync(d_bad, p->plan->ctx->stream));
  CU(cudaStreamSynchronize(p->plan->ctx->stream));
  return GHC_OK;
}

extern "C" int32_t ghc_p2p_row_elems(const ghc_p2p* p) { return p ? p->ep : 0; }

namespace {
struct BarrierPeers {
  unsigned* line[kMaxRanks];  // each rank's barrier line (peer-mapped)
};
// Lane q < G stores this rank's epoch into slot `rank` of rank q's line
// (system scope: the line lives in another GPU's memory), then waits until
// slot q of this rank's own line reaches the epoch.  Monotone epochs: a
// rank that runs ahead into the next barrier only raises its slot further.
__global__ void p2p_start_barrier_kernel(BarrierPeers peers, int rank, int G, unsigned epoch) {
  const int q = threadIdx.x;
  if (q < G) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(peers.line[q] + rank), "r"(epoch) : "memory");
    for (long long spin = 0;; ++spin) {
      unsigned v;
      asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(peers.line[rank] + q) : "memory");
      if ((int)(v - epoch) >= 0) break;
      if (spin > (1ll << 26)) __trap();  // a rank that never arrives: fail, do not hang
    }
  }
}
}  // namespace

// Device-side barrier of the G ranks on the context stream: every rank's
// stream passes it within about one NVLink round trip of the last arrival.
// Queued right before a timed launch, it aligns the ranks' start on the
// device (a host barrier leaves tens of µs of skew between the processes'
// launches).  Virtual exchanges (one grid): no-op.
extern "C" ghc_status ghc_p2p_barrier(ghc_p2p* p) {
  if (!p) return fail(GHC_ERR_CONFIG, "p2p_barrier: null handle");
  if (p->virt) return GHC_OK;
  BarrierPeers peers{};
  for (int q = 0; q < p->G; ++q) {
    if (!p->gcnt[q]) return fail(GHC_ERR_TRANSPORT, "p2p_barrier: peers not imported");
    peers.line[q] = p->gcnt[q] + (p->plan->cluster_size + 1) * kFlagStride;
  }
  ++p->barrier_epoch;
  CU(cudaSetDevice(p->plan->ctx->device));
  p2p_start_barrier_kernel<<<1, 32, 0, p->plan->ctx->stream>>>(peers, p->rank, p->G, p->barrier_epoch);
  CU(cudaGetLastError());
  p->plan->ctx->launches++;
  return GHC_OK;
}
