// dist.cu — the worker exchange across GPUs (one process per GPU) over NCCL /
// NVLink 5: the B200-native replacement of the reference's Endpoint
// send/recv pairs (transport.hpp:22-44) for the synchronous Downpour round
// and the hierarchical groups (Topology::hierarchical,
// transport.cpp:520-531 → ncclCommSplit).
//
// Rendezvous is plumbing: the caller (bench.py / the roles driver) moves the
// 128-byte NCCL unique id between processes (torch.distributed); everything
// after that is stream-ordered on the context's stream — no host sync inside
// a round.
#include <dlfcn.h>
#include <nccl.h>

#include "ghc_internal.cuh"

using namespace ghc;

// NCCL is resolved lazily with dlopen (not a load-time dependency): a process
// may already hold torch's bundled libnccl.so.2 (a newer NCCL whose symbols
// torch needs), and binding the system copy first would break a later
// `import torch`.  Preference: GHC_NCCL_LIB, an already-loaded libnccl.so.2,
// the torch-bundled wheel, then the system library.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommSplit) commSplit = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommUserRank) commUserRank = nullptr;
  decltype(&ncclCommCount) commCount = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    if (const char* e = std::getenv("GHC_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)  // the torch wheel's copy in this image (site-packages/nvidia/nccl/lib)
      h = dlopen("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                 RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return a;
    }
#define SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
    SYM(getUniqueId, "ncclGetUniqueId");
    SYM(commInitRank, "ncclCommInitRank");
    SYM(commSplit, "ncclCommSplit");
    SYM(commDestroy, "ncclCommDestroy");
    SYM(commUserRank, "ncclCommUserRank");
    SYM(commCount, "ncclCommCount");
    SYM(reduce, "ncclReduce");
    SYM(broadcast, "ncclBroadcast");
    SYM(allReduce, "ncclAllReduce");
    SYM(errorString, "ncclGetErrorString");
#undef SYM
    a.ok = a.getUniqueId && a.commInitRank && a.commSplit && a.commDestroy && a.commUserRank &&
           a.commCount && a.reduce && a.broadcast && a.allReduce && a.errorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks required symbols";
    return a;
  }();
  return api;
}
}  // namespace

#define NCCL_API()                                                 \
  const NcclApi& N_ = nccl();                                      \
  if (!N_.ok) return ghc_fail(GHC_ERR_NCCL, N_.why)

#define NC(expr)                                                                           \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return ghc_fail(GHC_ERR_NCCL, std::string(#expr) + ": " + nccl().errorString(r_));   \
  } while (0)

struct ghc_comm {
  ghc_ctx* ctx = nullptr;
  ncclComm_t nccl = nullptr;
  int rank = 0, size = 1;
  float* gbuf = nullptr;  // [P+1] this worker's pre-scaled gradient + loss sum
  float* gsum = nullptr;  // [P+1] reduced
  int64_t cap = 0;
};

namespace {

ghc_status ensure_buffers(ghc_comm* c, int64_t n) {
  if (c->cap >= n) return GHC_OK;
  cudaSetDevice(c->ctx->device);
  cudaFree(c->gbuf);
  cudaFree(c->gsum);
  const size_t bytes = sizeof(float) * static_cast<size_t>((n + 3) & ~3LL);
  CU(cudaMalloc(&c->gbuf, bytes));
  CU(cudaMalloc(&c->gsum, bytes));
  c->cap = n;
  return GHC_OK;
}

__global__ void copy_scalar_kernel(float* dst, const float* src) { *dst = *src; }

// Non-root ranks of the reduce/broadcast exchange: the root's sgd_step status
// arrived by broadcast into ms->status; keep the same version / rejected
// counters as the root (optim.cpp:49-51, 63).
__global__ void account_kernel(MasterDev* ms) {
  if (ms->status == 0) ms->version += 1ull;
  else ms->rejected += 1ull;
  ms->cur ^= 1;  // the broadcast weights landed in the other buffer, as on the root
}

}  // namespace

extern "C" {

ghc_status ghc_comm_unique_id(uint8_t* out) {
  ncclUniqueId id;
  NCCL_API();
  NC(N_.getUniqueId(&id));
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return GHC_OK;
}

ghc_status ghc_comm_init(ghc_ctx* ctx, const uint8_t* id_bytes, int32_t rank, int32_t nranks,
                         ghc_comm** out) {
  NCCL_API();
  if (nranks < 1 || rank < 0 || rank >= nranks) return ghc_fail(GHC_ERR_CONFIG, "comm: bad rank");
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
  CU(cudaSetDevice(ctx->device));
  auto* c = new ghc_comm();
  c->ctx = ctx;
  c->rank = rank;
  c->size = nranks;
  ncclResult_t r = nccl().commInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return ghc_fail(GHC_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().errorString(r));
  }
  *out = c;
  return GHC_OK;
}

ghc_status ghc_comm_split(ghc_comm* parent, int32_t color, int32_t key, ghc_comm** out) {
  auto* c = new ghc_comm();
  c->ctx = parent->ctx;
  ncclResult_t r = nccl().commSplit(parent->nccl, color, key, &c->nccl, nullptr);
  if (r != ncclSuccess) {
    delete c;
    return ghc_fail(GHC_ERR_NCCL, std::string("ncclCommSplit: ") + nccl().errorString(r));
  }
  if (c->nccl == nullptr) {  // color == NCCL_SPLIT_NOCOLOR
    delete c;
    *out = nullptr;
    return GHC_OK;
  }
  NC(nccl().commUserRank(c->nccl, &c->rank));
  NC(nccl().commCount(c->nccl, &c->size));
  *out = c;
  return GHC_OK;
}

void ghc_comm_destroy(ghc_comm* c) {
  if (!c) return;
  cudaSetDevice(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  if (c->nccl) nccl().commDestroy(c->nccl);
  cudaFree(c->gbuf);
  cudaFree(c->gsum);
  delete c;
}

int32_t ghc_comm_rank(const ghc_comm* c) { return c->rank; }
int32_t ghc_comm_size(const ghc_comm* c) { return c->size; }

ghc_status ghc_comm_reduce_sum(ghc_comm* c, const float* d_send, float* d_recv, int64_t count,
                               int32_t root) {
  NC(nccl().reduce(d_send, d_recv, static_cast<size_t>(count), ncclFloat32, ncclSum, root, c->nccl,
                c->ctx->stream));
  return GHC_OK;
}

ghc_status ghc_comm_broadcast(ghc_comm* c, float* d_buf, int64_t count, int32_t root) {
  NC(nccl().broadcast(d_buf, d_buf, static_cast<size_t>(count), ncclFloat32, root, c->nccl,
                   c->ctx->stream));
  return GHC_OK;
}

ghc_status ghc_comm_allreduce_sum(ghc_comm* c, const float* d_send, float* d_recv, int64_t count) {
  NC(nccl().allReduce(d_send, d_recv, static_cast<size_t>(count), ncclFloat32, ncclSum, c->nccl,
                   c->ctx->stream));
  return GHC_OK;
}

// Synchronous Downpour rounds across the communicator.  Rank r is worker r;
// h_counts[round*size + k] = samples of worker k in that round (0 = worker k
// already sent DONE).  Every rank knows every count (the data layer is
// deterministic), so the sample-weighted mean Σ c_k g_k / Σ c_k is formed by
// pre-scaling each worker's summed gradient with 1/Σc and summing — one
// reduction, no host sync.
ghc_status ghc_dist_sync_rounds(ghc_master* m, ghc_comm* comm, int32_t exchange, const float* d_x,
                                const int32_t* d_y, const int32_t* d_idx, int64_t stride,
                                const int32_t* h_counts, int32_t n_rounds, float* d_loss_out) {
  if (exchange != GHC_EXCHANGE_REDUCE_BCAST && exchange != GHC_EXCHANGE_ALLREDUCE)
    return ghc_fail(GHC_ERR_CONFIG, "unknown exchange");
  ghc_plan* p = m->plan;
  ghc_ctx* ctx = p->ctx;
  const int64_t P = m->P;
  if (ghc_status s = ensure_buffers(comm, P + 1)) return s;
  int cur = 0;  // the in-place update below never flips it: cached after one read
  if (ghc_status s = ghc_master_current(m, &cur)) return s;
  const bool master_here = exchange == GHC_EXCHANGE_ALLREDUCE || comm->rank == 0;
  for (int r = 0; r < n_rounds; ++r) {
    const int32_t* cnt = h_counts + static_cast<int64_t>(r) * comm->size;
    int64_t total = 0;
    for (int k = 0; k < comm->size; ++k) total += cnt[k];
    if (total == 0) break;  // every worker has sent DONE
    const int32_t mine = cnt[comm->rank];
    float* w = m->w[cur];  // this round's weights (the update flips the double buffer)
    if (mine > 0) {
      if (ghc_status s = ghc_worker_grad(p, w, d_x, d_y,
                                         d_idx ? d_idx + static_cast<int64_t>(r) * stride : nullptr,
                                         mine, static_cast<float>(1.0 / static_cast<double>(total)),
                                         comm->gbuf, comm->gbuf + P))
        return s;
    } else {
      CU(cudaMemsetAsync(comm->gbuf, 0, sizeof(float) * (P + 1), ctx->stream));
    }
    if (exchange == GHC_EXCHANGE_REDUCE_BCAST) {
      NC(nccl().reduce(comm->gbuf, comm->gsum, static_cast<size_t>(P + 1), ncclFloat32, ncclSum, 0,
                    comm->nccl, ctx->stream));
    } else {
      NC(nccl().allReduce(comm->gbuf, comm->gsum, static_cast<size_t>(P + 1), ncclFloat32, ncclSum,
                       comm->nccl, ctx->stream));
    }
    if (master_here) {
      // sgd_step with whole-update rejection (optim.cpp:39-65): one pass into
      // the other buffer (sgd_db det mode; a rejection copies the old state)
      if (ghc_status s = master_apply_det(m, comm->gsum, m->lr, m->mu)) return s;
      if (d_loss_out) {
        copy_scalar_kernel<<<1, 1, 0, ctx->stream>>>(d_loss_out + r, comm->gsum + P);
        ctx->launches++;
      }
    } else {
      m->host_cur = cur ^ 1;  // the broadcast lands in the other buffer, as on the root
    }
    cur ^= 1;
    w = m->w[cur];
    if (exchange == GHC_EXCHANGE_REDUCE_BCAST) {
      NC(nccl().broadcast(w, w, static_cast<size_t>(P), ncclFloat32, 0, comm->nccl, ctx->stream));
      // the root's accept/reject decision, so every rank's master reports
      // the same version / rejected counters
      NC(nccl().broadcast(&m->ms->status, &m->ms->status, 1, ncclInt32, 0, comm->nccl, ctx->stream));
      if (!master_here) {
        account_kernel<<<1, 1, 0, ctx->stream>>>(m->ms);
        CU(cudaGetLastError());
        ctx->launches++;
      }
    }
  }
  return GHC_OK;
}

}  // extern "C"
