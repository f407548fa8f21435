// ghc.cu — C ABI (include/ghc.h) of the B200-native Downpour/EASGD hot path.
//
// Host glue only: argument checking with the reference's error taxonomy,
// kernel selection per Architecture, launch geometry sized to the SM count,
// cooperative launches for the kernels that carry a grid barrier.  All math
// runs in the sm_100a kernels of lstm_step.cuh / update_kernels.cuh; there is
// no CPU compute path.
#include <cstdio>
#include <cstdlib>

#include "ghc_internal.cuh"

namespace {
thread_local std::string g_err;
}  // namespace

// The instantiated fused-kernel shapes: one translation unit per shape
// (inst_*.cu, see inst.cuh) so the kernels compile in parallel.
#define GHC_DECL(D, H, T, K) LstmEntry ghc_entry_##D##_##H##_##T##_##K();
#define GHC_DECL_TRUNK(D, H, T) LstmEntry ghc_trunk_##D##_##H##_##T();
GHC_DECL(5, 20, 10, 3)
GHC_DECL(5, 8, 10, 3)
GHC_DECL(3, 4, 5, 3)
GHC_DECL(2, 16, 3, 4)
GHC_DECL(5, 32, 10, 3)
GHC_DECL(4, 12, 6, 5)
GHC_DECL_TRUNK(5, 20, 10)
GHC_DECL_TRUNK(5, 8, 10)
GHC_DECL_TRUNK(3, 4, 5)

const std::vector<LstmEntry>& lstm_table() {
  static const std::vector<LstmEntry> t = {
      ghc_entry_5_20_10_3(),  // SPEC.md:109 bench net
      ghc_entry_5_8_10_3(),  ghc_entry_3_4_5_3(), ghc_entry_2_16_3_4(),
      ghc_entry_5_32_10_3(), ghc_entry_4_12_6_5(),
  };
  return t;
}

const std::vector<LstmEntry>& trunk_table() {
  static const std::vector<LstmEntry> t = {
      ghc_trunk_5_20_10(),  // wide variant
      ghc_trunk_5_8_10(),
      ghc_trunk_3_4_5(),
  };
  return t;
}

ghc_status ghc_fail(ghc_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

extern "C" {

const char* ghc_version(void) { return "gradhub-cuda 0.1 (sm_100a)"; }
const char* ghc_last_error(void) { return g_err.c_str(); }
const char* ghc_status_name(ghc_status s) {
  switch (s) {
    case GHC_OK: return "OK";
    case GHC_ERR_SHAPE: return "ShapeError";
    case GHC_ERR_NONFINITE: return "NonFiniteGradientError";
    case GHC_ERR_CACHE_MISMATCH: return "CacheMismatchError";
    case GHC_ERR_CONFIG: return "ConfigError";
    case GHC_ERR_TRANSPORT: return "TransportError";
    case GHC_ERR_PROTOCOL: return "ProtocolError";
    case GHC_ERR_CUDA: return "CudaError";
    case GHC_ERR_NCCL: return "NcclError";
  }
  return "?";
}

ghc_status ghc_device_count(int* n) {
  CU(cudaGetDeviceCount(n));
  return GHC_OK;
}

ghc_status ghc_ctx_create(int device, ghc_ctx** out) {
  int n = 0;
  CU(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(GHC_ERR_CUDA, "no such CUDA device");
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(GHC_ERR_CUDA, std::string("libghc is built for sm_100a; device is ") + prop.name);
  CU(cudaSetDevice(device));
  auto* c = new ghc_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CU(cudaEventCreate(&c->ev0));
  CU(cudaEventCreate(&c->ev1));
  *out = c;
  return GHC_OK;
}

void ghc_ctx_destroy(ghc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaEventDestroy(c->ev0);
  cudaEventDestroy(c->ev1);
  cudaStreamDestroy(c->stream);
  cudaFree(c->splitk_ws);
  cudaFree(c->scratch_ms);
  cudaFree(c->hdr_scratch);
  if (c->gate_h) cudaFreeHost(c->gate_h);
  delete c;
}

ghc_status ghc_ctx_sync(ghc_ctx* c) {
  CU(cudaStreamSynchronize(c->stream));
  return GHC_OK;
}
int ghc_ctx_num_sms(const ghc_ctx* c) { return c->num_sms; }
uint64_t ghc_ctx_launch_count(const ghc_ctx* c) { return c->launches.load(); }

ghc_status ghc_malloc(ghc_ctx* c, size_t bytes, void** d) {
  CU(cudaSetDevice(c->device));
  CU(cudaMalloc(d, bytes ? bytes : 16));
  return GHC_OK;
}
ghc_status ghc_free(ghc_ctx* c, void* d) {
  CU(cudaSetDevice(c->device));
  CU(cudaFree(d));
  return GHC_OK;
}
ghc_status ghc_host_alloc(size_t bytes, void** h) {
  CU(cudaMallocHost(h, bytes ? bytes : 16));
  return GHC_OK;
}
ghc_status ghc_host_free(void* h) {
  CU(cudaFreeHost(h));
  return GHC_OK;
}
ghc_status ghc_memcpy_h2d(ghc_ctx* c, void* d, const void* h, size_t bytes) {
  CU(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
  return GHC_OK;
}
ghc_status ghc_memcpy_d2h(ghc_ctx* c, void* h, const void* d, size_t bytes) {
  CU(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c->stream));
  return GHC_OK;
}
ghc_status ghc_memcpy_d2d(ghc_ctx* c, void* d, const void* s, size_t bytes) {
  CU(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, c->stream));
  return GHC_OK;
}
// CUDA IPC of a ghc_malloc'd buffer (the async / EASGD mailboxes of
// roles_dist.py: one process per GPU, data over NVLink P2P copies).
ghc_status ghc_ipc_handle(ghc_ctx* c, void* d_base, uint8_t* out_handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == GHC_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  CU(cudaSetDevice(c->device));
  CU(cudaIpcGetMemHandle(&h, d_base));
  std::memcpy(out_handle, &h, sizeof(h));
  return GHC_OK;
}
ghc_status ghc_ipc_open(ghc_ctx* c, const uint8_t* handle, void** d_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CU(cudaSetDevice(c->device));
  if (cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return fail(GHC_ERR_TRANSPORT, "ipc_open: cannot map the peer buffer");
  }
  return GHC_OK;
}
ghc_status ghc_ipc_close(ghc_ctx* c, void* d_ptr) {
  CU(cudaSetDevice(c->device));
  CU(cudaIpcCloseMemHandle(d_ptr));
  return GHC_OK;
}
ghc_status ghc_memset(ghc_ctx* c, void* d, int v, size_t bytes) {
  CU(cudaMemsetAsync(d, v, bytes, c->stream));
  return GHC_OK;
}
ghc_status ghc_timer_start(ghc_ctx* c) {
  CU(cudaEventRecord(c->ev0, c->stream));
  return GHC_OK;
}
// Launch-overhead-free device timing (the "blocking kernel" of nvbench):
// ghc_stream_hold queues a 1-thread kernel that spins on a pinned host flag,
// so everything the host queues behind it (the start event, the timed
// launches, the stop event) reaches the GPU before any of it runs;
// ghc_stream_release sets the flag.  The events then time the device work
// only, not the host's launch calls.  The gate gives up after 5 s (never
// hangs the stream).
static __global__ void stream_gate_kernel(const volatile int* flag) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    if (*flag) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 5000000000ull) return;
    __nanosleep(200);
  }
}
// Load the gate kernel's module now (CUDA lazy loading would otherwise
// load it at first launch, which waits for running kernels — a resident
// round kernel never finishes on its own).
ghc_status ghc_preload_gate() {
  cudaFuncAttributes fa;
  CU(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(stream_gate_kernel)));
  return GHC_OK;
}
ghc_status ghc_stream_hold(ghc_ctx* c) {
  if (!c->gate_h) {
    CU(cudaHostAlloc(reinterpret_cast<void**>(&c->gate_h), sizeof(int), cudaHostAllocMapped));
    CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->gate_d), c->gate_h, 0));
  }
  *c->gate_h = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  stream_gate_kernel<<<1, 1, 0, c->stream>>>(c->gate_d);
  CU(cudaGetLastError());
  return GHC_OK;
}
ghc_status ghc_stream_release(ghc_ctx* c) {
  if (!c->gate_h) return fail(GHC_ERR_CONFIG, "stream_release without stream_hold");
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *reinterpret_cast<volatile int*>(c->gate_h) = 1;
  return GHC_OK;
}
ghc_status ghc_timer_stop(ghc_ctx* c, float* ms) {
  CU(cudaEventRecord(c->ev1, c->stream));
  CU(cudaEventSynchronize(c->ev1));
  CU(cudaEventElapsedTime(ms, c->ev0, c->ev1));
  return GHC_OK;
}

// ---------------------------------------------------------------- plan
ghc_status ghc_plan_create(ghc_ctx* c, const char* arch_text, ghc_plan** out) {
  if (!c || !arch_text || !out) return fail(GHC_ERR_CONFIG, "null argument");
  auto* p = new ghc_plan();
  p->ctx = c;
  try {
    p->model = parse_model(arch_text);
  } catch (const std::exception& e) {
    delete p;
    return fail(GHC_ERR_CONFIG, e.what());
  }
  const auto& L = p->model.layers;
  if (L.back().b > 32) {
    const std::string txt = arch_text;
    delete p;
    return fail(GHC_ERR_CONFIG, "softmax head: at most 32 classes on the device path ('" + txt + "')");
  }
  if (L.size() == 2 && L[0].kind == LayerKind::lstm && L[1].kind == LayerKind::softmax) {
    for (const LstmEntry& e : lstm_table())
      if (e.D == L[0].a && e.H == L[0].b && e.T == L[0].c && e.K == L[1].b) p->lstm = &e;
  }
  if (!p->lstm) {
    // dense layers, or an LSTM shape outside the fused table: LSTM trunk
    // kernel (table shapes) or the generic GEMM-based LSTM (generic.cu) +
    // tcgen05 GEMMs (layered.cu)
    p->layered = true;
    if (L[0].kind == LayerKind::lstm) {
      for (const LstmEntry& e : trunk_table())
        if (e.D == L[0].a && e.H == L[0].b && e.T == L[0].c) p->trunk = &e;
      p->generic_lstm = p->trunk == nullptr;
    }
  }
  if (p->layered) {
    p->kname = p->trunk          ? std::string(p->trunk->name) + " + tcgen05 3xTF32 dense GEMMs"
               : p->generic_lstm ? std::string("lstm_gemm (per-timestep tcgen05 GEMMs + cell kernels) + "
                                               "tcgen05 3xTF32 dense GEMMs")
                                 : std::string("tcgen05 3xTF32 dense GEMMs");
    CU(cudaSetDevice(c->device));
    p->max_ctas = c->num_sms;
    if (p->trunk) {
      CU(cudaFuncSetAttribute(reinterpret_cast<const void*>(p->trunk->fn),
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(p->trunk->smem(8))));
      int per_sm = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, reinterpret_cast<const void*>(p->trunk->fn), 256, p->trunk->smem(8)));
      p->max_ctas = (per_sm < 1 ? 1 : per_sm) * c->num_sms;
      CU(cudaMalloc(&p->part, sizeof(float) * static_cast<size_t>(p->max_ctas) * p->trunk->ppad));
    }
    CU(cudaMalloc(&p->ms, sizeof(MasterDev)));
    CU(cudaMemset(p->ms, 0, sizeof(MasterDev)));
    CU(cudaMalloc(&p->err, sizeof(int)));
    CU(cudaMemset(p->err, 0, sizeof(int)));
    const size_t bar_bytes = sizeof(unsigned) * 32 * (2 + static_cast<size_t>(p->max_ctas));
    CU(cudaMalloc(&p->bar, bar_bytes));
    CU(cudaMemset(p->bar, 0, bar_bytes));
    CU(cudaDeviceSynchronize());  // legacy-stream memsets vs the non-blocking ctx->stream
    p->use_cluster = false;
    *out = p;
    return GHC_OK;
  }
  p->kname = std::string(p->lstm->name) + " [flat]";
  CU(cudaSetDevice(c->device));
  // largest block (≤ 8 warps) whose shared memory fits one SM, and the
  // co-residency of the cooperative fused kernel at that size
  int smem_optin = 0;
  CU(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  p->max_warps = 8;
  while (p->max_warps > 1 && p->lstm->smem(p->max_warps) > static_cast<size_t>(smem_optin))
    --p->max_warps;
  int per_sm = 0;
  CU(cudaFuncSetAttribute(reinterpret_cast<const void*>(p->lstm->fn),
                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(p->lstm->smem(p->max_warps))));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, reinterpret_cast<const void*>(p->lstm->fn), 32 * p->max_warps,
      p->lstm->smem(p->max_warps)));
  if (per_sm < 1) {
    delete p;
    return fail(GHC_ERR_CUDA, "fused kernel cannot be resident (smem/registers)");
  }
  p->max_ctas = per_sm * c->num_sms;
  // cluster variants: for clusters of 8 and of 4, the largest block that
  // fits and how many clusters can be co-resident (GPC-constrained; queried,
  // not assumed).  SIMT variant (default): every sample its own warp with the
  // fewest warps per CTA.  Tensor-core variant (GHC_STEP=tc): fewest passes of
  // 8 samples per CTA over the bench batch — correct on every shape but slower
  // on B200 (legacy HMMA.1688.TF32 ≈ 12.5 cycles/instr per SM sub-partition
  // with distinct operands, tools/tc_micro.cu; 3×TF32 then delivers fewer
  // fp32 FMA/clk than FFMA).  Ties → 8 (fewer rows in the
  // cross-cluster reduce).
  {
    const char* env = std::getenv("GHC_STEP");
    const std::string step = env ? env : "";
    p->use_cluster = step != "flat";
    auto max_clusters = [&](void (*fn)(StepArgs), int cs, int warps, size_t smem) {
      if (smem > static_cast<size_t>(smem_optin)) return 0;
      if (cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(32 * warps);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = cs;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(fn), &cfg) != cudaSuccess)
        ncl = 0;
      cudaGetLastError();
      // GHC_MAX_CTAS=n: a persistent grid of at most n CTAs — for processes
      // sharing one GPU (MPS), whose grids must be co-resident side by side
      // (the occupancy query sees the whole device)
      static const int cap = [] {
        const char* e = std::getenv("GHC_MAX_CTAS");
        return e ? std::atoi(e) : 0;
      }();
      if (cap > 0 && ncl > cap / cs) ncl = cap / cs;
      return ncl;
    };
    const int64_t bench_batch = 1000;  // per-worker batch of the bench config
    if (step == "tc" && p->lstm->fn_tc[0]) {
      int64_t best_passes = INT64_MAX;
      for (int ci = 1; ci >= 0; --ci) {
        const int cs = kClusterSizes[ci];
        const int ncl = max_clusters(p->lstm->fn_tc[ci], cs, 8, p->lstm->smem_tc[ci](8));
        if (ncl < 1) continue;
        const int64_t slots = static_cast<int64_t>(ncl) * cs * kTcSamples;
        const int64_t passes = (bench_batch + slots - 1) / slots;
        if (passes < best_passes) {
          best_passes = passes;
          p->cluster_size = cs;
          p->cs_index = ci;
          p->max_clusters = ncl;
          p->round_warps = 8;
          p->use_tc = true;
        }
      }
    }
    if (!p->use_tc) {
      // fewest warps per CTA for the bench batch; clusters of 2 (148 CTAs,
      // 7 warps) only when forced: the sample phase is latency-bound, so 7
      // instead of 8 warps per SM saves 0.25 µs, while 74 cluster rows per
      // sub-slice poll cost 3 µs more in the exchange (15.5 vs 12.7 µs per
      // round, measured).  GHC_CS=2|4|8 forces a cluster size (A/B runs).
      const char* fcs = std::getenv("GHC_CS");
      const int force_cs = fcs ? std::atoi(fcs) : 0;
      int best_warps = 1 << 30;
      int64_t fb_slots = 0;  // no size holds the bench batch in one pass (e.g. a
      int fb_ci = -1, fb_ncl = 0, fb_warps = 0;  // GHC_MAX_CTAS cap): the most slots, smaller clusters on ties
      for (int ci : {1, 0, 2}) {
        const int cs = kClusterSizes[ci];
        if (force_cs ? cs != force_cs : cs == 2) continue;
        int warps = 8;
        while (warps > 1 && p->lstm->smem_round[ci](warps) > static_cast<size_t>(smem_optin)) --warps;
        const int ncl = max_clusters(p->lstm->fn_round[ci], cs, warps, p->lstm->smem_round[ci](warps));
        if (ncl < 1) continue;
        const int64_t slots = static_cast<int64_t>(ncl) * cs * kSamplesPerWarp;
        const int need = static_cast<int>((bench_batch + slots - 1) / slots);
        if (need < best_warps && need <= warps) {
          best_warps = need;
          p->cluster_size = cs;
          p->cs_index = ci;
          p->max_clusters = ncl;
          p->round_warps = warps;
        }
        if (slots * warps > fb_slots || (slots * warps == fb_slots && cs < kClusterSizes[fb_ci])) {
          fb_slots = slots * warps;
          fb_ci = ci;
          fb_ncl = ncl;
          fb_warps = warps;
        }
      }
      if (best_warps == (1 << 30) && fb_ci >= 0) {
        p->cluster_size = kClusterSizes[fb_ci];
        p->cs_index = fb_ci;
        p->max_clusters = fb_ncl;
        p->round_warps = fb_warps;
      }
    }
    if (p->use_cluster && p->max_clusters > 0) {
      std::string nm = p->lstm->name;
      if (p->use_tc) nm.replace(0, std::string("lstm_round").size(), "lstm_round_tc");
      p->kname = nm + " [clusters of " + std::to_string(p->cluster_size) + "]";
    }
    if (p->max_clusters * p->cluster_size > p->max_ctas) p->max_ctas = p->max_clusters * p->cluster_size;
  }
  CU(cudaMalloc(&p->part, sizeof(float) * static_cast<size_t>(p->max_ctas) * p->lstm->ppad));
  {  // tagged rows of the exchange: [2][clusters][EP] + weights [ranks][2][EP], tags start at 0
    const size_t ep = static_cast<size_t>(std::max({p->lstm->ep[0], p->lstm->ep[1], p->lstm->ep[2]}));
    const size_t n = 2 * static_cast<size_t>(p->max_ctas) * ep + 2 * kMaxRanks * ep;  // + weights per rank
    CU(cudaMalloc(&p->tpart, sizeof(unsigned long long) * n));
    CU(cudaMemset(p->tpart, 0, sizeof(unsigned long long) * n));
    p->tw = p->tpart + 2 * static_cast<size_t>(p->max_ctas) * ep;
  }
  CU(cudaMalloc(&p->ms, sizeof(MasterDev)));
  CU(cudaMemset(p->ms, 0, sizeof(MasterDev)));
  CU(cudaMalloc(&p->err, sizeof(int)));
  CU(cudaMemset(p->err, 0, sizeof(int)));
  const size_t bar_bytes = sizeof(unsigned) * 32 * (2 + static_cast<size_t>(p->max_ctas));
  CU(cudaMalloc(&p->bar, bar_bytes));
  CU(cudaMemset(p->bar, 0, bar_bytes));
  // the legacy-stream memsets above are not ordered with ctx->stream
  // (non-blocking): complete them before any kernel can use the plan
  CU(cudaDeviceSynchronize());
  *out = p;
  return GHC_OK;
}

ghc_status ghc_plan_set_probe(ghc_plan* p, uint64_t* d_probe) {
  p->probe = reinterpret_cast<unsigned long long*>(d_probe);
  return GHC_OK;
}

void ghc_plan_destroy(ghc_plan* p) {
  if (!p) return;
  cudaSetDevice(p->ctx->device);
  cudaStreamSynchronize(p->ctx->stream);
  cudaFree(p->part);
  cudaFree(p->tpart);
  cudaFree(p->ms);
  cudaFree(p->err);
  cudaFree(p->bar);
  layered_free(p->ws);
  generic_lstm_free(p->gws);
  delete p;
}

ghc_status ghc_plan_check_error(ghc_plan* p) {
  if (!p) return fail(GHC_ERR_CONFIG, "null plan");
  int err = 0;
  CU(cudaMemcpyAsync(&err, p->err, sizeof(int), cudaMemcpyDeviceToHost, p->ctx->stream));
  CU(cudaStreamSynchronize(p->ctx->stream));
  if (err) {
    CU(cudaMemsetAsync(p->err, 0, sizeof(int), p->ctx->stream));
    CU(cudaStreamSynchronize(p->ctx->stream));
    return fail(GHC_ERR_SHAPE, "loss: label out of range [0," + std::to_string(p->model.n_classes) + ")");
  }
  return GHC_OK;
}

int64_t ghc_plan_n_params(const ghc_plan* p) { return p->model.n_params; }
int64_t ghc_plan_input_width(const ghc_plan* p) { return p->model.input_width; }
int32_t ghc_plan_n_classes(const ghc_plan* p) { return p->model.n_classes; }
const char* ghc_plan_kernel_name(const ghc_plan* p) {
  return p->kname.c_str();
}
int32_t ghc_plan_max_clusters(const ghc_plan* p) { return p->use_cluster ? p->max_clusters : 0; }
int32_t ghc_plan_cluster_size(const ghc_plan* p) { return p->use_cluster ? p->cluster_size : 0; }

ghc_status ghc_plan_tensors(const ghc_plan* p, int64_t* off, int64_t* d0, int64_t* d1, int cap,
                            int* nt) {
  *nt = static_cast<int>(p->model.tensors.size());
  for (int i = 0; i < *nt && i < cap; ++i) {
    off[i] = p->model.tensors[i].offset;
    d0[i] = p->model.tensors[i].dim0;
    d1[i] = p->model.tensors[i].dim1;
  }
  return GHC_OK;
}

ghc_status ghc_arch_info(const char* text, int64_t* n_params, int64_t* input_width,
                         int32_t* n_classes) {
  try {
    const Model m = parse_model(text ? text : "");
    if (n_params) *n_params = m.n_params;
    if (input_width) *input_width = m.input_width;
    if (n_classes) *n_classes = m.n_classes;
  } catch (const std::exception& e) {
    return fail(GHC_ERR_CONFIG, e.what());
  }
  return GHC_OK;
}

ghc_status ghc_init_weights_text(const char* text, uint64_t seed, double* h_w) {
  try {
    init_weights(parse_model(text ? text : ""), seed, h_w);
  } catch (const std::exception& e) {
    return fail(GHC_ERR_CONFIG, e.what());
  }
  return GHC_OK;
}

ghc_status ghc_init_weights(const ghc_plan* p, uint64_t seed, double* h_w) {
  init_weights(p->model, seed, h_w);
  return GHC_OK;
}

// ---------------------------------------------------------------- worker step
ghc_status ghc_worker_grad(ghc_plan* p, const float* d_w, const float* d_x, const int32_t* d_y,
                           const int32_t* d_idx, int64_t n, float grad_scale, float* d_grad,
                           float* d_loss_sum) {
  if (n < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");  // nn.cpp:104
  if (!d_w || !d_x || !d_y || !d_grad) return fail(GHC_ERR_CONFIG, "null device pointer");
  if (p->layered) return layered_step(p, d_w, d_x, d_y, d_idx, n, grad_scale, d_grad, d_loss_sum, nullptr);
  StepArgs a{};
  a.x = d_x;
  a.y = d_y;
  a.idx = d_idx;
  a.n = static_cast<int>(n);
  a.rounds = 1;
  a.grad_scale = grad_scale;
  a.w_in = d_w;
  a.ms = p->ms;
  a.g_out = d_grad;
  a.loss_out = d_loss_sum;
  a.mode = MODE_GRAD;
  return launch_step(p, a, n);
}

ghc_status ghc_worker_grads(ghc_plan* p, int32_t W, const float* d_w, int64_t w_stride, const float* d_x,
                            const int32_t* d_y, const int32_t* const* h_idx, const int32_t* h_n,
                            float* d_grad, int64_t g_stride, float* d_loss) {
  if (W < 1 || W > kMaxRanks) return fail(GHC_ERR_CONFIG, "worker_grads: n_workers must be in [1, 8]");
  if (!p || !d_w || !d_x || !h_idx || !h_n || !d_grad) return fail(GHC_ERR_CONFIG, "worker_grads: null argument");
  int64_t n_max = 0;
  for (int k = 0; k < W; ++k) {
    if (h_n[k] < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");  // nn.cpp:104
    n_max = std::max<int64_t>(n_max, h_n[k]);
  }
  const bool fused = !p->layered && p->lstm && p->use_cluster && !p->use_tc && p->max_clusters / W >= 1 &&
                     p->lstm->fn_multi[p->cs_index] != nullptr;
  if (!fused || W == 1) {
    for (int k = 0; k < W; ++k)
      if (ghc_status s = ghc_worker_grad(p, d_w + k * w_stride, d_x, d_y, h_idx[k], h_n[k],
                                         1.0f / static_cast<float>(h_n[k]), d_grad + k * g_stride,
                                         d_loss ? d_loss + k : nullptr))
        return s;
    return GHC_OK;
  }
  StepArgs a{};
  a.x = d_x;
  a.y = d_y;
  a.n = static_cast<int>(n_max);
  a.rounds = 1;
  a.w_in = d_w;
  a.ms = p->ms;
  a.g_out = d_grad;
  a.loss_out = d_loss;
  a.mode = MODE_GRAD;
  a.w_vstride = w_stride;
  a.g_vstride = g_stride;
  for (int k = 0; k < W; ++k) {
    a.idx_v[k] = h_idx[k];
    a.n_v[k] = static_cast<int>(h_n[k]);
  }
  return launch_step(p, a, n_max, W, nullptr, true);
}

ghc_status ghc_forward(ghc_plan* p, const float* d_w, const float* d_x, const int32_t* d_y,
                       const int32_t* d_idx, int64_t n, float* d_probs, float* d_loss_sum) {
  if (n < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");
  if (p->layered) return layered_step(p, d_w, d_x, d_y, d_idx, n, 1.0f, nullptr, d_loss_sum, d_probs);
  StepArgs a{};
  a.x = d_x;
  a.y = d_y;
  a.idx = d_idx;
  a.n = static_cast<int>(n);
  a.rounds = 1;
  a.w_in = d_w;
  a.ms = p->ms;
  a.loss_out = d_loss_sum;
  a.probs_out = d_probs;
  a.mode = MODE_FWD;
  return launch_step(p, a, n);
}

// ---------------------------------------------------------------- validate
// argmax_k probs (lowest k on ties) == label, counted exactly (integer atomics
// are order-independent, so the count is deterministic).
static __global__ void argmax_correct_kernel(const float* __restrict__ probs,
                                             const int32_t* __restrict__ y, long long n, int K,
                                             unsigned long long* correct) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float* p = probs + i * K;
    int best = 0;
    for (int k = 1; k < K; ++k)
      if (p[k] > p[best]) best = k;
    c += best == __ldg(y + i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(correct, c);
}

ghc_status ghc_validate(ghc_plan* p, const float* d_w, const float* d_x, const int32_t* d_y,
                        int64_t n, int64_t* h_correct, double* h_loss_mean) {
  // "empty held-out set → configuration error"
  if (n < 1) return fail(GHC_ERR_CONFIG, "validate: empty held-out set");
  ghc_ctx* c = p->ctx;
  const int K = p->model.n_classes;
  char* ws = nullptr;
  const size_t pb = (sizeof(float) * static_cast<size_t>(n) * K + 255) & ~size_t(255);
  CU(cudaMallocAsync(reinterpret_cast<void**>(&ws), pb + 256, c->stream));
  float* probs = reinterpret_cast<float*>(ws);
  float* loss = reinterpret_cast<float*>(ws + pb);
  auto* cnt = reinterpret_cast<unsigned long long*>(ws + pb + 128);
  CU(cudaMemsetAsync(ws + pb, 0, 256, c->stream));
  ghc_status st = ghc_forward(p, d_w, d_x, d_y, nullptr, n, probs, loss);
  if (st == GHC_OK) {
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4L * c->num_sms));
    argmax_correct_kernel<<<grid, 256, 0, c->stream>>>(probs, d_y, n, K, cnt);
    c->launches++;
    CU(cudaGetLastError());
    float lsum = 0.0f;
    unsigned long long ok = 0;
    CU(cudaMemcpyAsync(&lsum, loss, sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(&ok, cnt, sizeof(ok), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    st = ghc_plan_check_error(p);
    if (h_correct) *h_correct = static_cast<int64_t>(ok);
    if (h_loss_mean) *h_loss_mean = static_cast<double>(lsum) / static_cast<double>(n);
  }
  CU(cudaFreeAsync(ws, c->stream));
  return st;
}

// ---------------------------------------------------------------- algo
static ghc_status validate_sgd(float lr, float mu) {  // optim.cpp:20-29
  if (!(lr > 0.0f)) return fail(GHC_ERR_CONFIG, "learning_rate must be > 0");
  if (!(mu >= 0.0f && mu < 1.0f)) return fail(GHC_ERR_CONFIG, "momentum must be in [0,1)");
  return GHC_OK;
}
static ghc_status validate_alpha(float alpha) {  // optim.cpp:31-37
  if (!(alpha > 0.0f && alpha < 1.0f)) return fail(GHC_ERR_CONFIG, "elastic_alpha must be in (0,1)");
  return GHC_OK;
}

namespace {
// Barrier state of the cooperative context-level kernels (sgd_apply,
// easgd_worker): owned by the context, allocated on first use, freed in
// ghc_ctx_destroy.
MasterDev* ctx_scratch_ms(ghc_ctx* c) {
  if (c->scratch_ms) return c->scratch_ms;
  MasterDev* m = nullptr;
  cudaSetDevice(c->device);
  if (cudaMalloc(&m, sizeof(MasterDev)) != cudaSuccess) return nullptr;
  if (cudaMemset(m, 0, sizeof(MasterDev)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(m);
    return nullptr;
  }
  c->scratch_ms = m;
  return m;
}
}  // namespace

ghc_status ghc_sgd_apply(ghc_ctx* c, float* d_w, float* d_v, const float* d_g, int64_t P, float lr,
                         float mu, int32_t* d_status, uint64_t* d_version) {
  if (ghc_status s = validate_sgd(lr, mu)) return s;
  if (P < 1) return fail(GHC_ERR_SHAPE, "sgd_step: empty weight set");
  MasterDev* ms = ctx_scratch_ms(c);
  if (!ms) return fail(GHC_ERR_CUDA, "scratch allocation failed");
  int vec = aligned16(d_w) && aligned16(d_v) && aligned16(d_g);
  long long PP = P;
  unsigned long long* ver = reinterpret_cast<unsigned long long*>(d_version);
  int* st = d_status;
  unsigned long long* rj = nullptr;
  void* args[] = {&d_w, &d_v, &d_g, &PP, &vec, &lr, &mu, &ms, &st, &ver, &rj};
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(sgd_apply_kernel), 256);
  CU(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sgd_apply_kernel), dim3(grid), dim3(256),
                                 args, 0, c->stream));
  c->launches++;
  return GHC_OK;
}

namespace {
bool overlaps(const void* a, const void* b, int64_t bytes) {
  const char* x = static_cast<const char*>(a);
  const char* y = static_cast<const char*>(b);
  return x < y + bytes && y < x + bytes;
}
}  // namespace

ghc_status ghc_sgd_step_out(ghc_ctx* c, const float* d_w, const float* d_v, const float* d_g,
                            float* d_w_out, float* d_v_out, int64_t P, float lr, float mu,
                            int32_t* d_status, uint64_t* d_version) {
  if (ghc_status s = validate_sgd(lr, mu)) return s;
  if (P < 1) return fail(GHC_ERR_SHAPE, "sgd_step: empty weight set");
  const int64_t b = 4 * P;
  if (overlaps(d_w_out, d_w, b) || overlaps(d_w_out, d_v, b) || overlaps(d_w_out, d_g, b) ||
      overlaps(d_v_out, d_w, b) || overlaps(d_v_out, d_v, b) || overlaps(d_v_out, d_g, b) ||
      overlaps(d_w_out, d_v_out, b))
    return fail(GHC_ERR_CONFIG, "sgd_step_out: outputs must not overlap the inputs (use ghc_sgd_apply)");
  MasterDev* ms = ctx_scratch_ms(c);
  if (!ms) return fail(GHC_ERR_CUDA, "scratch allocation failed");
  const int vec = aligned16(d_w) && aligned16(d_v) && aligned16(d_g) && aligned16(d_w_out) &&
                  aligned16(d_v_out);
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(sgd_out_kernel), 256);
  sgd_out_kernel<<<grid, 256, 0, c->stream>>>(d_w, d_v, d_g, d_w_out, d_v_out, P, vec, lr, mu, ms,
                                              d_status,
                                              reinterpret_cast<unsigned long long*>(d_version));
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_easgd_worker_step_out(ghc_ctx* c, const float* d_w, const float* d_c,
                                     const float* d_g, float* d_w_out, int64_t P, float lr,
                                     float alpha, uint64_t tau, uint64_t batch_index,
                                     int32_t* d_status) {
  if (!(lr > 0.0f)) return fail(GHC_ERR_CONFIG, "learning_rate must be > 0");
  if (ghc_status s = validate_alpha(alpha)) return s;
  if (tau < 1) return fail(GHC_ERR_CONFIG, "elastic_tau must be >= 1");
  const int64_t b = 4 * P;
  if (overlaps(d_w_out, d_w, b) || overlaps(d_w_out, d_c, b) || overlaps(d_w_out, d_g, b))
    return fail(GHC_ERR_CONFIG,
                "easgd_worker_step_out: output must not overlap the inputs (use ghc_easgd_worker_step)");
  MasterDev* ms = ctx_scratch_ms(c);
  if (!ms) return fail(GHC_ERR_CUDA, "scratch allocation failed");
  const int vec = aligned16(d_w) && aligned16(d_c) && aligned16(d_g) && aligned16(d_w_out);
  const int pull = (batch_index % tau) == 0;
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(easgd_worker_out_kernel), 256);
  easgd_worker_out_kernel<<<grid, 256, 0, c->stream>>>(d_w, d_c, d_g, d_w_out, P, vec, lr, alpha, pull,
                                                       ms, d_status);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_elastic_pull(ghc_ctx* c, float* d_w, const float* d_c, int64_t P, float alpha) {
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(elastic_kernel), 256);
  elastic_kernel<<<grid, 256, 0, c->stream>>>(d_w, d_c, P, aligned16(d_w) && aligned16(d_c), alpha,
                                              1, nullptr);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_easgd_worker_step(ghc_ctx* c, float* d_w, const float* d_c, const float* d_g,
                                 int64_t P, float lr, float alpha, uint64_t tau,
                                 uint64_t batch_index, int32_t* d_status) {
  if (!(lr > 0.0f)) return fail(GHC_ERR_CONFIG, "learning_rate must be > 0");
  if (ghc_status s = validate_alpha(alpha)) return s;
  if (tau < 1) return fail(GHC_ERR_CONFIG, "elastic_tau must be >= 1");
  MasterDev* ms = ctx_scratch_ms(c);
  if (!ms) return fail(GHC_ERR_CUDA, "scratch allocation failed");
  int vec = aligned16(d_w) && aligned16(d_c) && aligned16(d_g);
  int pull = (batch_index % tau) == 0;
  long long PP = P;
  int* st = d_status;
  void* args[] = {&d_w, &d_c, &d_g, &PP, &vec, &lr, &alpha, &pull, &ms, &st};
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(easgd_worker_kernel), 256);
  CU(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(easgd_worker_kernel), dim3(grid),
                                 dim3(256), args, 0, c->stream));
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_easgd_center_step(ghc_ctx* c, float* d_c, const float* d_w, int64_t P, float alpha,
                                 uint64_t* d_version) {
  if (ghc_status s = validate_alpha(alpha)) return s;
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(elastic_kernel), 256);
  elastic_kernel<<<grid, 256, 0, c->stream>>>(d_c, d_w, P, aligned16(d_c) && aligned16(d_w), alpha,
                                              0, reinterpret_cast<unsigned long long*>(d_version));
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_weighted_mean(ghc_ctx* c, float* d_out, const float* d_slots, const double* h_counts,
                             int32_t W, int64_t P) {
  if (W < 1 || W > kMaxSlots) return fail(GHC_ERR_CONFIG, "weighted_mean: 1..64 slots");
  SlotWeights cw{};
  double total = 0.0;
  for (int i = 0; i < W; ++i) {
    if (!(h_counts[i] >= 1.0)) return fail(GHC_ERR_PROTOCOL, "GRADIENT sample_count must be >= 1");
    cw.c[i] = static_cast<float>(h_counts[i]);
    total += h_counts[i];
  }
  const int vec = aligned16(d_out) && aligned16(d_slots) && (P % 4 == 0);
  const int grid = occupancy_grid(c, reinterpret_cast<const void*>(weighted_mean_kernel), 256);
  weighted_mean_kernel<<<grid, 256, 0, c->stream>>>(d_out, d_slots, W, P, P, vec, cw,
                                                    static_cast<float>(1.0 / total));
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

// ---------------------------------------------------------------- master
ghc_status ghc_master_create(ghc_plan* p, const double* h_w0, float lr, float mu, ghc_master** out) {
  if (ghc_status s = validate_sgd(lr, mu)) return s;
  auto* m = new ghc_master();
  m->plan = p;
  m->lr = lr;
  m->mu = mu;
  m->P = p->model.n_params;
  CU(cudaSetDevice(p->ctx->device));
  const size_t bytes = sizeof(float) * static_cast<size_t>((m->P + 3) & ~3LL);
  std::vector<float> w32(static_cast<size_t>(m->P));
  for (int64_t i = 0; i < m->P; ++i) w32[static_cast<size_t>(i)] = static_cast<float>(h_w0[i]);
  for (int b = 0; b < 2; ++b) {
    CU(cudaMalloc(&m->w[b], bytes));
    CU(cudaMalloc(&m->v[b], bytes));
    CU(cudaMemset(m->v[b], 0, bytes));
    CU(cudaMemcpy(m->w[b], w32.data(), sizeof(float) * m->P, cudaMemcpyHostToDevice));
  }
  CU(cudaMalloc(&m->ms, sizeof(MasterDev)));
  CU(cudaMemset(m->ms, 0, sizeof(MasterDev)));
  CU(cudaMalloc(&m->ms_apply, sizeof(MasterDev)));
  CU(cudaMemset(m->ms_apply, 0, sizeof(MasterDev)));
  CU(cudaMalloc(&m->ms_db, sizeof(MasterDev)));
  CU(cudaMemset(m->ms_db, 0, sizeof(MasterDev)));
  {
    float* h[4] = {m->w[0], m->w[1], m->v[0], m->v[1]};
    CU(cudaMalloc(&m->bufs, sizeof(h)));
    CU(cudaMemcpy(m->bufs, h, sizeof(h), cudaMemcpyHostToDevice));
  }
  *out = m;
  return GHC_OK;
}

void ghc_master_destroy(ghc_master* m) {
  if (!m) return;
  cudaSetDevice(m->plan->ctx->device);
  cudaStreamSynchronize(m->plan->ctx->stream);
  for (int b = 0; b < 2; ++b) {
    cudaFree(m->w[b]);
    cudaFree(m->v[b]);
  }
  cudaFree(m->ms);
  cudaFree(m->ms_apply);
  cudaFree(m->ms_db);
  cudaFree(m->bufs);
  cudaFree(m->g_scratch);
  delete m;
}

ghc_status ghc_master_current(ghc_master* m, int* cur) {
  if (!m->host_cur_known) {
    MasterDev h;
    CU(cudaMemcpyAsync(&h, m->ms, sizeof(h), cudaMemcpyDeviceToHost, m->plan->ctx->stream));
    CU(cudaStreamSynchronize(m->plan->ctx->stream));
    m->host_cur = h.cur;
    m->host_cur_known = true;
  }
  *cur = m->host_cur;
  return GHC_OK;
}
static ghc_status master_cur(ghc_master* m, int& cur) { return ghc_master_current(m, &cur); }

ghc_status ghc_master_weights(ghc_master* m, float** d_w, float** d_v) {
  int cur = 0;
  if (ghc_status s = master_cur(m, cur)) return s;
  if (d_w) *d_w = m->w[cur];
  if (d_v) *d_v = m->v[cur];
  return GHC_OK;
}

ghc_status ghc_master_read(ghc_master* m, float* h_w, float* h_v, uint64_t* version,
                           uint64_t* rejected) {
  MasterDev h;
  cudaStream_t s = m->plan->ctx->stream;
  CU(cudaMemcpyAsync(&h, m->ms, sizeof(h), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h_w) CU(cudaMemcpyAsync(h_w, m->w[h.cur], sizeof(float) * m->P, cudaMemcpyDeviceToHost, s));
  if (h_v) CU(cudaMemcpyAsync(h_v, m->v[h.cur], sizeof(float) * m->P, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (version) *version = h.version;
  if (rejected) *rejected = h.rejected;
  return ghc_plan_check_error(m->plan);
}

// Layered rounds: the round's samples count only for an accepted update
// (the fused round kernels do this in their publish step).
static __global__ void count_accepted_kernel(MasterDev* ms, int n) {
  if (ms->status == 0) ms->samples += static_cast<unsigned long long>(n);
}

// Packed dataset rows (d_y == NULL): the SIMT cluster round kernel only.
static ghc_status check_packed(const ghc_plan* p, const int32_t* d_y) {
  if (d_y) return GHC_OK;
  if (p->layered || !p->lstm || !p->use_cluster || p->max_clusters < 1 || p->use_tc)
    return fail(GHC_ERR_CONFIG, "packed dataset rows (labels == NULL) need the SIMT cluster round kernel");
  return GHC_OK;
}

__global__ void pack_rows_kernel(float* __restrict__ out, const float* __restrict__ x,
                                 const int32_t* __restrict__ y, long long rows, int width, int stride) {
  const long long tot = rows * stride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / stride;
    const int c = static_cast<int>(i - r * stride);
    out[i] = c < width ? x[r * width + c] : (c == width ? __int_as_float(y[r]) : 0.0f);
  }
}

int32_t ghc_packed_row_floats(int32_t width) { return (width + 1 + 31) & ~31; }

ghc_status ghc_dataset_pack(ghc_ctx* c, const float* d_x, const int32_t* d_y, int64_t rows, int32_t width,
                            float* d_out) {
  if (!c || !d_x || !d_y || !d_out || rows < 0 || width < 1) return fail(GHC_ERR_CONFIG, "dataset_pack: bad argument");
  const int stride = ghc_packed_row_floats(width);
  const long long tot = rows * stride;
  const int grid = static_cast<int>(std::min<long long>((tot + 255) / 256, 8LL * c->num_sms));
  pack_rows_kernel<<<grid > 0 ? grid : 1, 256, 0, c->stream>>>(d_out, d_x, d_y, rows, width, stride);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_master_sync_rounds(ghc_master* m, const float* d_x, const int32_t* d_y,
                                  const int32_t* d_idx, int64_t stride, const int32_t* d_counts,
                                  int64_t n, int32_t n_rounds, float* d_loss_out) {
  if (n < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");
  if (n_rounds < 1) return GHC_OK;
  if (ghc_status s = check_packed(m->plan, d_y)) return s;
  if (m->plan->layered) {
    // layered archs: per round the layered worker step (scale 1/n_r) then the
    // rejecting in-place sgd_step on the master's current buffers
    ghc_ctx* c = m->plan->ctx;
    std::vector<int32_t> cnt(static_cast<size_t>(n_rounds), static_cast<int32_t>(n));
    if (d_counts) {
      CU(cudaMemcpyAsync(cnt.data(), d_counts, sizeof(int32_t) * n_rounds, cudaMemcpyDeviceToHost,
                         c->stream));
      CU(cudaStreamSynchronize(c->stream));
    }
    if (!m->g_scratch) CU(cudaMalloc(&m->g_scratch, sizeof(float) * static_cast<size_t>((m->P + 4) & ~3LL)));
    int cur = 0;
    if (ghc_status s = master_cur(m, cur)) return s;
    for (int r = 0; r < n_rounds; ++r) {
      const int32_t nr = cnt[static_cast<size_t>(r)];
      const int64_t roff = d_idx ? 0 : static_cast<int64_t>(r) * stride;  // no table: rows r*stride+s
      if (ghc_status s = layered_step(m->plan, m->w[cur], d_x + roff * m->plan->model.input_width,
                                      d_y + roff,
                                      d_idx ? d_idx + static_cast<int64_t>(r) * stride : nullptr, nr,
                                      1.0f / static_cast<float>(nr), m->g_scratch,
                                      d_loss_out ? d_loss_out + r : nullptr, nullptr))
        return s;
      // one-pass double-buffered sgd_step (optim.cpp:39-65); the buffers flip
      if (ghc_status s = master_apply_det(m, m->g_scratch, m->lr, m->mu)) return s;
      cur ^= 1;
      count_accepted_kernel<<<1, 1, 0, c->stream>>>(m->ms, nr);
      CU(cudaGetLastError());
      c->launches += 1;
    }
    return GHC_OK;
  }
  StepArgs a{};
  a.x = d_x;
  a.y = d_y;
  a.idx = d_idx;
  a.stride = stride;
  a.counts = d_counts;
  a.n = static_cast<int>(n);
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
  m->host_cur_known = false;  // the round kernel flips the buffers on device
  return launch_step(m->plan, a, n);
}

ghc_status master_apply_det(ghc_master* m, const float* d_g, float lr, float mu) {
  ghc_ctx* c = m->plan->ctx;
  int cur = 0;
  if (ghc_status s = ghc_master_current(m, &cur)) return s;
  const int vec = aligned16(d_g);
  const int grid = std::min<long long>(occupancy_grid(c, reinterpret_cast<const void*>(sgd_db_kernel), 256),
                                       (m->P / 4 + 255) / 256 + 1);
  sgd_db_kernel<<<grid, 256, 0, c->stream>>>(m->bufs, m->bufs + 2, d_g, m->P, vec, lr, mu, m->ms, m->ms_db, 1);
  CU(cudaGetLastError());
  db_fixup_kernel<<<grid, 256, 0, c->stream>>>(m->bufs, m->bufs + 2, m->P, m->ms, m->ms_db);
  CU(cudaGetLastError());
  c->launches += 2;
  m->host_cur = cur ^ 1;  // flips on every call (det mode)
  m->host_cur_known = true;
  return GHC_OK;
}

ghc_status ghc_master_apply(ghc_master* m, const float* d_g) {
  // One pass into the other buffer; the device flips `cur` (no host sync).
  ghc_ctx* c = m->plan->ctx;
  const int vec = aligned16(d_g);  // w[], v[] are cudaMalloc-aligned; the tail is scalar
  const int grid = std::min<long long>(occupancy_grid(c, reinterpret_cast<const void*>(sgd_db_kernel), 256),
                                       (m->P / 4 + 255) / 256 + 1);
  m->host_cur_known = false;  // the last CTA flips ms->cur (or rejects)
  sgd_db_kernel<<<grid, 256, 0, c->stream>>>(m->bufs, m->bufs + 2, d_g, m->P, vec, m->lr, m->mu,
                                             m->ms, m->ms_db);
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

// ---------------------------------------------------------------- data
ghc_status ghc_data_generate(const ghc_data_spec* s, int32_t f0, int32_t nf, float* h_x,
                             int32_t* h_y) {
  DataSpec d{s->n_files, s->samples_per_file, s->seq_len, s->input_dim, s->n_classes, 0, s->delta,
             s->seed};
  if (f0 < 0 || nf < 0 || f0 + nf > s->n_files) return fail(GHC_ERR_CONFIG, "file range");
  generate_files(d, f0, nf, h_x, h_y);
  return GHC_OK;
}

ghc_status ghc_data_shard(int32_t n_files, int32_t W, int32_t k, int32_t* f0, int32_t* nf) {
  try {
    int a = 0, b = 0;
    shard_files(n_files, W, k, a, b);
    *f0 = a;
    *nf = b;
  } catch (const std::exception& e) {
    return fail(GHC_ERR_CONFIG, e.what());
  }
  return GHC_OK;
}

ghc_status ghc_data_epoch_indices(const ghc_data_spec* s, int32_t W, int32_t k, int32_t epoch,
                                  uint64_t seed, int32_t shuffle, int64_t* out, int64_t* count) {
  DataSpec d{s->n_files, s->samples_per_file, s->seq_len, s->input_dim, s->n_classes, 0, s->delta,
             s->seed};
  try {
    const auto idx = epoch_indices(d, W, k, epoch, seed, shuffle != 0);
    std::memcpy(out, idx.data(), idx.size() * sizeof(int64_t));
    *count = static_cast<int64_t>(idx.size());
  } catch (const std::exception& e) {
    return fail(GHC_ERR_CONFIG, e.what());
  }
  return GHC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- diagnostics
// GHC_SEGV_TRACE=1: print a native backtrace on SIGSEGV (debug aid for
// crashes that happen outside any Python frame, e.g. in finalizers).
#include <execinfo.h>
#include <csignal>
#include <unistd.h>
namespace {
void ghc_segv_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "libghc: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof(msg) - 1);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
__attribute__((constructor)) void ghc_install_segv_trace() {
  const char* e = std::getenv("GHC_SEGV_TRACE");
  if (e && e[0] == '1') signal(SIGSEGV, ghc_segv_handler);
}
}  // namespace
