// session.cu — the SPEC master/worker roles driving the
// sm_100a kernels: the C++ host code of the drop-in, written against the
// reference semantics the oracle restates (oracle/gh_oracle.c gho_run_*):
//
//   sync Downpour     SPEC.md:358-366  every round = ONE fused launch over the
//                                      round's concatenated worker batches
//                                      (Σ c_i g_i / Σ c_i ≡ one sum scaled 1/C)
//   async Downpour    SPEC.md:349-357  replayed arrival order: per step the
//                                      worker's gradient on ITS weight copy,
//                                      sgd_step at the master, reply to it
//   EASGD             SPEC.md:149-166  local steps; every τ batches the worker
//                                      exchanges with the center (updated-
//                                      center ordering)
//   hierarchical      SPEC.md:367-375  sync group masters + flush every K to a
//                                      top master (pseudo-gradient = snapshot −
//                                      current, DESIGN.md Appendix-A decision)
//
// All workers of a session live on this device ("virtual workers"); the
// across-GPU exchange of the same protocol is ghc_dist_sync_rounds (dist.cu).
// Host work per step is launch bookkeeping only; no host sync inside run().
#include "ghc_internal.cuh"

using namespace ghc;

namespace {

// Cooperative: reject-on-non-finite g, then w1 = w - lr*g; on exchange steps
// c' = c + α(w1 - c) (optim.cpp:118, version+1) and w = w1 - α(w1 - c')
// (optim.cpp:76 against the UPDATED center).
__global__ void __launch_bounds__(256) easgd_exchange_kernel(float* __restrict__ w,
                                                             float* __restrict__ c,
                                                             const float* __restrict__ g,
                                                             long long P, float lr, float alpha,
                                                             int exchange, MasterDev* ms,
                                                             int* err, unsigned long long* cver) {
  // An earlier step already met a non-finite gradient: the reference worker
  // aborted there (optim.cpp:90-92, oracle gho_run_replay), so nothing after
  // it may change the center or any worker (err is stream-ordered: every CTA
  // reads the same value and returns before the grid barrier).
  if (__ldcg(err) & 2) return;
  const int rej = check_finite_all(g, P, 0, ms);
  if (!rej) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long i = tid; i < P; i += nth) {
      float w1 = w[i];
      w1 -= lr * __ldcg(g + i);
      if (exchange) {
        float cv = c[i];
        cv += alpha * (w1 - cv);
        c[i] = cv;
        w1 -= alpha * (w1 - cv);
      }
      w[i] = w1;
    }
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicOr(err, 2);  // GHC_ERR_NONFINITE: the worker aborts (optim.cpp:90-92)
  }
  finish_rejecting(ms, rej, nullptr, (exchange && !rej) ? cver : nullptr, nullptr);
}

// One replayed async Downpour step's master side in ONE single-CTA launch for
// small P (replay_pre + sgd_db + db_fixup + replay_post + the reply copy were
// five stream operations of a few µs each): staleness against the sender's
// basis, the whole-update reject on a non-finite gradient (optim.cpp:49-53),
// sgd_step (optim.cpp:59-60: v = μv − ηg, w += v — the arithmetic of
// sgd_pass) into the other double buffer (a reject copies the old state
// there, as db_fixup does; the buffers flip either way, det mode), the
// version / rejected / status counters, the sender's new basis and samples,
// and the reply: the new weights into the sender's copy wk.
__global__ void __launch_bounds__(1024) replay_apply_kernel(float* const* __restrict__ wb,
                                                            float* const* __restrict__ vb,
                                                            const float* __restrict__ g, long long P,
                                                            float lr, float mu, MasterDev* ms,
                                                            unsigned long long* basis, int k,
                                                            long long* stale_out, unsigned long long* samples,
                                                            int n, float* __restrict__ wk) {
  __shared__ int s_cur;
  if (threadIdx.x == 0) {
    s_cur = ms->cur;
    *stale_out = (long long)(ms->version - basis[k]);
  }
  __syncthreads();
  const int cur = s_cur;
  const float* w = wb[cur];
  const float* v = vb[cur];
  float* w2 = wb[cur ^ 1];
  float* v2 = vb[cur ^ 1];
  int bad = 0;
  for (long long i = threadIdx.x; i < P; i += blockDim.x) bad |= isfinite(g[i]) ? 0 : 1;
  bad = __syncthreads_or(bad);
  for (long long i = threadIdx.x; i < P; i += blockDim.x) {
    if (bad) {
      const float wi = w[i];
      w2[i] = wi;
      v2[i] = v[i];
      wk[i] = wi;
    } else {
      const float vn = fmaf(mu, v[i], -lr * g[i]);
      const float wn = w[i] + vn;
      v2[i] = vn;
      w2[i] = wn;
      wk[i] = wn;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ms->cur = cur ^ 1;
    if (bad) {
      ms->rejected += 1ull;
      ms->status = 2;  // GHC_ERR_NONFINITE
    } else {
      ms->version += 1ull;
      ms->status = 0;
      *samples += (unsigned long long)n;
    }
    basis[k] = ms->version;
  }
}

// One sync EASGD round's exchanges (workers 0..R-1 in rank order) in ONE
// single-CTA launch for small P (the bench net: 2,143 parameters — the R
// cooperative easgd_exchange_kernel launches were ~10 µs of launch each):
// the same per-element arithmetic in the same order, the center's updates
// ordered by a CTA barrier between workers; a non-finite gradient stops the
// round at that worker (err bit 2), as the per-worker kernels do.
__global__ void __launch_bounds__(1024) easgd_round_kernel(float* __restrict__ ww, long long w_stride,
                                                           float* __restrict__ c, const float* __restrict__ g0,
                                                           long long g_stride, long long P, float lr,
                                                           float alpha, unsigned exch_mask, int R, int* err,
                                                           unsigned long long* cver) {
  if (__ldcg(err) & 2) return;
  for (int k = 0; k < R; ++k) {
    const float* g = g0 + k * g_stride;
    float* w = ww + k * w_stride;
    int bad = 0;
    for (long long i = threadIdx.x; i < P; i += blockDim.x) bad |= is_finite_f(__ldcg(g + i)) ? 0 : 1;
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) atomicOr(err, 2);  // GHC_ERR_NONFINITE: the worker aborts (optim.cpp:90-92)
      return;
    }
    const bool exchange = (exch_mask >> k) & 1u;
    for (long long i = threadIdx.x; i < P; i += blockDim.x) {
      float w1 = w[i];
      w1 -= lr * __ldcg(g + i);
      if (exchange) {
        float cv = c[i];
        cv += alpha * (w1 - cv);
        c[i] = cv;
        w1 -= alpha * (w1 - cv);
      }
      w[i] = w1;
    }
    __syncthreads();  // this worker's center update before the next worker's
    if (exchange && threadIdx.x == 0) ++*cver;
  }
}

// out = a - b (hierarchical pseudo-gradient: snapshot - current)
__global__ void sub_kernel(float* __restrict__ out, const float* __restrict__ a,
                           const float* __restrict__ b, long long P) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

// Async Downpour replay bookkeeping on the device (oracle
// gho_run_replay): staleness = accepted master updates since the sender's
// basis, taken before the apply; after it the sender's basis is the current
// version and its samples count only if the update was accepted — a rejected
// (non-finite) gradient advances neither (optim.cpp:49-51).
__global__ void replay_pre_kernel(const MasterDev* ms, const unsigned long long* basis, int k,
                                  long long* stale_out) {
  *stale_out = (long long)(ms->version - basis[k]);
}
__global__ void replay_post_kernel(const MasterDev* ms, unsigned long long* basis, int k,
                                   unsigned long long* samples, int n) {
  basis[k] = ms->version;
  if (ms->status == 0) *samples += (unsigned long long)n;
}

struct Batch {
  int64_t off;  // into the worker's index stream
  int32_t n;
};

}  // namespace

struct ghc_session {
  ghc_plan* plan = nullptr;
  ghc_train_config cfg{};
  ghc_data_spec spec{};
  int64_t P = 0;
  int W = 0;
  // data
  float* X = nullptr;
  int32_t* Y = nullptr;
  int32_t* streams = nullptr;                // all workers' index streams, concatenated
  std::vector<int64_t> stream_off;           // per worker
  std::vector<std::vector<Batch>> batches;   // per worker
  std::vector<size_t> cursor;                // per worker: next batch
  // state
  ghc_master* master = nullptr;              // Downpour master / top master (hier)
  std::vector<ghc_master*> group;            // hierarchical sub-masters
  float* worker_w = nullptr;                 // [W][P] worker copies (async / EASGD)
  float* center = nullptr;                   // EASGD center
  float* scratch_g = nullptr;                // [P+1] one worker gradient (+ loss)
  float* multi_g = nullptr;                  // [W][Pp] one round's worker gradients (sync EASGD)
  float* multi_l = nullptr;                  // [W] their loss sums
  float* snap = nullptr;                     // [G][P] flush snapshots
  float* pseudo = nullptr;                   // [G][P]
  float* comb = nullptr;                     // [P]
  unsigned long long* cver = nullptr;        // EASGD center version
  unsigned long long* d_basis = nullptr;     // [W] async Downpour: sender basis versions
  unsigned long long* d_samples = nullptr;   // accepted samples (async Downpour replay)
  MasterDev* ms = nullptr;                   // barrier scratch for cooperative kernels
  int* err = nullptr;
  std::vector<int64_t> basis;                // per worker basis version (host mirror)
  std::vector<uint64_t> bidx;                // per worker batch counter (EASGD)
  // accounting
  int64_t updates = 0, samples = 0, rounds = 0;
  uint64_t rejected_groups = 0;  // hierarchical: rejected group-master updates
  int64_t trace_cap = 0;  // entries of the caller's loss / staleness buffers
  // the master's serial validation
  float* Xv = nullptr;
  int32_t* Yv = nullptr;
  int64_t nv = 0;
  int32_t v_every = 0;
  struct VRec {
    uint64_t version;
    double accuracy, loss;
  };
  std::vector<VRec> vrec;
};

namespace {

ghc_status coop(ghc_ctx* c, const void* fn, void** args) {
  const int grid = occupancy_grid(c, fn, 256);
  CU(cudaLaunchCooperativeKernel(const_cast<void*>(fn), dim3(grid), dim3(256), args, 0, c->stream));
  c->launches++;
  return GHC_OK;
}

ghc_status upload_data(ghc_session* s) {
  const ghc_data_spec& sp = s->spec;
  DataSpec d{sp.n_files, sp.samples_per_file, sp.seq_len, sp.input_dim, sp.n_classes, 0, sp.delta,
             sp.seed};
  const int64_t rows = static_cast<int64_t>(sp.n_files) * sp.samples_per_file;
  const int64_t width = static_cast<int64_t>(sp.seq_len) * sp.input_dim;
  std::vector<float> x(static_cast<size_t>(rows * width));
  std::vector<int32_t> y(static_cast<size_t>(rows));
  generate_files(d, 0, sp.n_files, x.data(), y.data());
  CU(cudaMalloc(&s->X, sizeof(float) * x.size()));
  CU(cudaMalloc(&s->Y, sizeof(int32_t) * y.size()));
  CU(cudaMemcpy(s->X, x.data(), sizeof(float) * x.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(s->Y, y.data(), sizeof(int32_t) * y.size(), cudaMemcpyHostToDevice));
  // per-worker epoch streams: batches never cross epochs
  std::vector<int32_t> all;
  s->stream_off.assign(static_cast<size_t>(s->W), 0);
  s->batches.assign(static_cast<size_t>(s->W), {});
  for (int k = 0; k < s->W; ++k) {
    s->stream_off[static_cast<size_t>(k)] = static_cast<int64_t>(all.size());
    int64_t local = 0;
    for (int e = 0; e < s->cfg.epochs; ++e) {
      const auto idx = epoch_indices(d, s->W, k, e, s->cfg.shuffle_seed, s->cfg.shuffle != 0);
      for (size_t i = 0; i < idx.size(); i += static_cast<size_t>(s->cfg.batch_size)) {
        const size_t n = std::min(idx.size() - i, static_cast<size_t>(s->cfg.batch_size));
        s->batches[static_cast<size_t>(k)].push_back({local + static_cast<int64_t>(i),
                                                      static_cast<int32_t>(n)});
      }
      for (int64_t v : idx) all.push_back(static_cast<int32_t>(v));
      local += static_cast<int64_t>(idx.size());
    }
  }
  CU(cudaMalloc(&s->streams, sizeof(int32_t) * (all.empty() ? 1 : all.size())));
  CU(cudaMemcpy(s->streams, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice));
  s->cursor.assign(static_cast<size_t>(s->W), 0);
  return GHC_OK;
}

// One worker gradient on weights `w` over its next batch: scratch_g = mean g,
// scratch_g[P] = loss sum.  Returns the batch size (0 = worker DONE).
ghc_status worker_step(ghc_session* s, int k, const float* w, int32_t& n_out) {
  auto& cur = s->cursor[static_cast<size_t>(k)];
  const auto& bl = s->batches[static_cast<size_t>(k)];
  if (cur >= bl.size()) {
    n_out = 0;
    return GHC_OK;
  }
  const Batch b = bl[cur++];
  n_out = b.n;
  return ghc_worker_grad(s->plan, w, s->X, s->Y,
                         s->streams + s->stream_off[static_cast<size_t>(k)] + b.off, b.n,
                         1.0f / static_cast<float>(b.n), s->scratch_g, s->scratch_g + s->P);
}

ghc_status apply_master(ghc_session* s, ghc_master* m, const float* g, float lr, float mu) {
  (void)s;
  // one pass over the master's double buffers (sgd_db det mode, ghc.cu)
  return master_apply_det(m, g, lr, mu);
}

// The master's current weights (the double buffer flips on every apply).
float* master_w(ghc_master* m) {
  int cur = 0;
  ghc_master_current(m, &cur);  // known on the host: never a device read here
  return m->w[cur];
}

// VALIDATE_RESULT of the current master weights (EASGD: the center), appended
// to the run log; a second request at the same version is not repeated.
ghc_status validate_now(ghc_session* s) {
  if (s->nv < 1) return GHC_OK;
  const float* w = nullptr;
  uint64_t version = 0;
  if (s->cfg.algo == GHC_ALGO_EASGD && s->cfg.groups == 0) {
    w = s->center;
    CU(cudaMemcpy(&version, s->cver, sizeof(version), cudaMemcpyDeviceToHost));
  } else {
    float* dw = nullptr;
    if (ghc_status st = ghc_master_weights(s->master, &dw, nullptr)) return st;
    w = dw;
    CU(cudaMemcpy(&version, &s->master->ms->version, sizeof(version), cudaMemcpyDeviceToHost));
  }
  if (!s->vrec.empty() && s->vrec.back().version == version) return GHC_OK;
  int64_t correct = 0;
  double loss = 0.0;
  if (ghc_status st = ghc_validate(s->plan, w, s->Xv, s->Yv, s->nv, &correct, &loss)) return st;
  s->vrec.push_back({version, static_cast<double>(correct) / static_cast<double>(s->nv), loss});
  return GHC_OK;
}

ghc_status run_sync(ghc_session* s, float* h_loss) {
  // Round r = one fused launch over the active workers' batches, rank order.
  const int B = s->cfg.batch_size;
  const int64_t stride = static_cast<int64_t>(s->W) * B;
  std::vector<int32_t> table, counts;
  std::vector<int32_t> host_streams;
  {
    size_t total = 0;
    for (auto& v : s->batches) total += v.size();
    (void)total;
  }
  // gather host copies of the streams to build the round table
  int64_t all = 0;
  for (int k = 0; k < s->W; ++k) {
    int64_t len = 0;
    for (auto& b : s->batches[static_cast<size_t>(k)]) len = std::max(len, b.off + b.n);
    all = std::max(all, s->stream_off[static_cast<size_t>(k)] + len);
  }
  host_streams.resize(static_cast<size_t>(all));
  CU(cudaMemcpy(host_streams.data(), s->streams, sizeof(int32_t) * all, cudaMemcpyDeviceToHost));
  for (int64_t r = 0;; ++r) {
    if (s->cfg.max_updates > 0 && r >= s->cfg.max_updates) break;
    int32_t cnt = 0;
    const size_t base = table.size();
    table.resize(base + static_cast<size_t>(stride), 0);
    for (int k = 0; k < s->W; ++k) {
      auto& cur = s->cursor[static_cast<size_t>(k)];
      if (cur >= s->batches[static_cast<size_t>(k)].size()) continue;
      const Batch b = s->batches[static_cast<size_t>(k)][cur++];
      const int32_t* src = host_streams.data() + s->stream_off[static_cast<size_t>(k)] + b.off;
      std::copy(src, src + b.n, table.begin() + static_cast<int64_t>(base) + cnt);
      cnt += b.n;
    }
    if (cnt == 0) {
      table.resize(base);
      break;
    }
    counts.push_back(cnt);
  }
  const int R = static_cast<int>(counts.size());
  if (R == 0) return GHC_OK;
  int32_t *d_table = nullptr, *d_counts = nullptr;
  float* d_loss = nullptr;
  CU(cudaMalloc(&d_table, sizeof(int32_t) * table.size()));
  CU(cudaMalloc(&d_counts, sizeof(int32_t) * counts.size()));
  CU(cudaMalloc(&d_loss, sizeof(float) * counts.size()));
  CU(cudaMemcpy(d_table, table.data(), sizeof(int32_t) * table.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_counts, counts.data(), sizeof(int32_t) * counts.size(), cudaMemcpyHostToDevice));
  // samples of the ACCEPTED rounds only (oracle gho_run_sync): the round
  // kernel counts them on the device next to version / rejected
  MasterDev before{};
  CU(cudaMemcpy(&before, s->master->ms, sizeof(before), cudaMemcpyDeviceToHost));
  // one persistent launch for all rounds, or chunks of V rounds with the
  // master's serial validation in between (split launches are bit-identical)
  ghc_status st = GHC_OK;
  const int V = s->nv > 0 && s->v_every > 0 ? s->v_every : R;
  for (int r0 = 0; r0 < R && st == GHC_OK; r0 += V) {
    const int nr = std::min(V, R - r0);
    st = ghc_master_sync_rounds(s->master, s->X, s->Y, d_table + static_cast<int64_t>(r0) * stride,
                                stride, d_counts + r0, stride, nr, d_loss + r0);
    if (st == GHC_OK && V < R) st = validate_now(s);
  }
  if (st == GHC_OK && h_loss) {
    std::vector<float> lo(static_cast<size_t>(R));
    CU(cudaMemcpyAsync(lo.data(), d_loss, sizeof(float) * R, cudaMemcpyDeviceToHost,
                       s->plan->ctx->stream));
    CU(cudaStreamSynchronize(s->plan->ctx->stream));
    for (int r = 0; r < R && r < s->trace_cap; ++r)
      h_loss[r] = lo[static_cast<size_t>(r)] / static_cast<float>(counts[static_cast<size_t>(r)]);
  }
  cudaStreamSynchronize(s->plan->ctx->stream);
  MasterDev after{};
  CU(cudaMemcpy(&after, s->master->ms, sizeof(after), cudaMemcpyDeviceToHost));
  s->samples += static_cast<int64_t>(after.samples - before.samples);
  cudaFree(d_table);
  cudaFree(d_counts);
  cudaFree(d_loss);
  s->rounds += R;
  return st;
}

// sync_rounds: `order` is the sync EASGD round-robin (each round every active
// worker once, in rank order).  A worker's gradient then depends only on its
// own weights, fixed since its previous step, so a round's gradients are
// computed up front in ONE launch (ghc_worker_grads) when the round's
// workers are 0..R-1 (contiguous weight rows); the exchanges stay serial in
// rank order.
ghc_status run_replay(ghc_session* s, const int32_t* order, int64_t n_order, float* h_loss,
                      int64_t* h_stale, bool sync_rounds = false) {
  ghc_ctx* c = s->plan->ctx;
  const int64_t P = s->P;
  std::vector<float*> loss_dst;
  float* d_loss = nullptr;
  CU(cudaMalloc(&d_loss, sizeof(float) * (n_order > 0 ? n_order : 1)));
  std::vector<int32_t> counts;
  int64_t version = 0;  // EASGD: center exchanges (host mirror of cver)
  const bool downpour = s->cfg.algo == GHC_ALGO_DOWNPOUR;
  long long* d_stale = nullptr;
  unsigned long long samples0 = 0;
  if (downpour) {
    CU(cudaMalloc(&d_stale, sizeof(long long) * (n_order > 0 ? n_order : 1)));
    CU(cudaMemcpy(&samples0, s->d_samples, sizeof(samples0), cudaMemcpyDeviceToHost));
  }
  const int64_t Pp = (P + 4) & ~3LL;  // multi_g row stride (16-B rows)
  int64_t round_end = 0, round_begin = 0;
  bool round_multi = false;
  std::vector<int32_t> round_n;
  for (int64_t step = 0; step < n_order; ++step) {
    const int k = order[step];
    if (k < 0 || k >= s->W) return fail(GHC_ERR_PROTOCOL, "replay order names an unknown worker");
    float* wk = s->worker_w + static_cast<int64_t>(k) * P;
    if (sync_rounds && !downpour && step == round_end) {
      // the next round: the run of strictly increasing worker ids from here
      round_begin = step;
      round_end = step;
      while (round_end < n_order && (round_end == step || order[round_end] > order[round_end - 1])) ++round_end;
      const int R = static_cast<int>(round_end - round_begin);
      round_multi = R > 1 && R <= kMaxRanks;
      for (int i = 0; i < R && round_multi; ++i) round_multi = order[round_begin + i] == i;  // workers 0..R-1
      if (round_multi) {
        std::vector<const int32_t*> idx(static_cast<size_t>(R));
        round_n.assign(static_cast<size_t>(R), 0);
        for (int i = 0; i < R; ++i) {
          auto& cur = s->cursor[static_cast<size_t>(i)];
          const auto& bl = s->batches[static_cast<size_t>(i)];
          if (cur >= bl.size()) return fail(GHC_ERR_PROTOCOL, "replay order uses a worker that already sent DONE");
          const Batch b = bl[cur++];
          idx[static_cast<size_t>(i)] = s->streams + s->stream_off[static_cast<size_t>(i)] + b.off;
          round_n[static_cast<size_t>(i)] = b.n;
        }
        if (!s->multi_g) {
          CU(cudaMalloc(&s->multi_g, sizeof(float) * static_cast<size_t>(kMaxRanks * Pp)));
          CU(cudaMalloc(&s->multi_l, sizeof(float) * kMaxRanks));
        }
        if (ghc_status st = ghc_worker_grads(s->plan, R, s->worker_w, P, s->X, s->Y, idx.data(),
                                             round_n.data(), s->multi_g, Pp, s->multi_l))
          return st;
      }
    }
    if (round_multi && step == round_begin && P <= (1LL << 16)) {
      // the whole round's host bookkeeping, then ONE exchange launch — unless
      // a validation falls inside the round (it must see the center between
      // two workers' exchanges): then the per-worker path below
      const int R = static_cast<int>(round_end - round_begin);
      unsigned mask = 0;
      int64_t v = version;
      bool val_inside = false;
      for (int i = 0; i < R; ++i) {
        const uint64_t bi = s->bidx[static_cast<size_t>(i)];
        if ((bi % static_cast<uint64_t>(s->cfg.tau)) == 0) {
          mask |= 1u << i;
          ++v;
          if (s->v_every > 0 && v % s->v_every == 0) val_inside = true;
        }
      }
      if (!val_inside) {
        for (int i = 0; i < R; ++i) {
          const int64_t st_i = round_begin + i;
          const int32_t ni = round_n[static_cast<size_t>(i)];
          counts.push_back(ni);
          CU(cudaMemcpyAsync(d_loss + st_i, s->multi_l + i, sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
          s->samples += ni;
          s->bidx[static_cast<size_t>(i)]++;
          const bool exch = (mask >> i) & 1u;
          if (h_stale && st_i < s->trace_cap) h_stale[st_i] = exch ? version - s->basis[static_cast<size_t>(i)] : 0;
          if (exch) {
            ++version;
            s->basis[static_cast<size_t>(i)] = version;
          }
        }
        easgd_round_kernel<<<1, 1024, 0, c->stream>>>(s->worker_w, P, s->center, s->multi_g, Pp, P, s->cfg.lr,
                                                      s->cfg.alpha, mask, R, s->err, s->cver);
        CU(cudaGetLastError());
        c->launches++;
        step = round_end - 1;
        continue;
      }
    }
    int32_t n = 0;
    const float* g_step = s->scratch_g;
    if (round_multi) {
      const int i = static_cast<int>(step - round_begin);
      n = round_n[static_cast<size_t>(i)];
      g_step = s->multi_g + i * Pp;
      CU(cudaMemcpyAsync(d_loss + step, s->multi_l + i, sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    } else {
      if (ghc_status st = worker_step(s, k, wk, n)) return st;
      if (n == 0) return fail(GHC_ERR_PROTOCOL, "replay order uses a worker that already sent DONE");
      CU(cudaMemcpyAsync(d_loss + step, s->scratch_g + P, sizeof(float), cudaMemcpyDeviceToDevice,
                         c->stream));
    }
    counts.push_back(n);
    if (downpour) {
      // sgd_step at the master, reply to the sender only;
      // staleness / basis / samples follow the device's accepted count
      if (P <= (1LL << 16)) {
        ghc_master* m = s->master;
        int cur = 0;
        if (ghc_status st = ghc_master_current(m, &cur)) return st;
        replay_apply_kernel<<<1, 1024, 0, c->stream>>>(m->bufs, m->bufs + 2, s->scratch_g, P, s->cfg.lr,
                                                       s->cfg.mu, m->ms, s->d_basis, k, d_stale + step,
                                                       s->d_samples, n, wk);
        CU(cudaGetLastError());
        c->launches++;
        m->host_cur = cur ^ 1;  // the buffers flip on every step (det mode)
        m->host_cur_known = true;
      } else {
        replay_pre_kernel<<<1, 1, 0, c->stream>>>(s->master->ms, s->d_basis, k, d_stale + step);
        if (ghc_status st = apply_master(s, s->master, s->scratch_g, s->cfg.lr, s->cfg.mu))
          return st;
        replay_post_kernel<<<1, 1, 0, c->stream>>>(s->master->ms, s->d_basis, k, s->d_samples, n);
        c->launches += 2;
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(wk, master_w(s->master), sizeof(float) * P, cudaMemcpyDeviceToDevice,
                           c->stream));
      }
      if (s->v_every > 0) {  // the cadence needs the accepted count (serial)
        uint64_t ver = 0;
        CU(cudaMemcpyAsync(&ver, &s->master->ms->version, sizeof(ver), cudaMemcpyDeviceToHost,
                           c->stream));
        CU(cudaStreamSynchronize(c->stream));
        if (ver % static_cast<uint64_t>(s->v_every) == 0)
          if (ghc_status st = validate_now(s)) return st;
      }
    } else {
      s->samples += n;
      const uint64_t bi = s->bidx[static_cast<size_t>(k)]++;
      int exch = (bi % static_cast<uint64_t>(s->cfg.tau)) == 0;
      if (h_stale && step < s->trace_cap)
        h_stale[step] = exch ? version - s->basis[static_cast<size_t>(k)] : 0;
      float* cc = s->center;
      const float* g = g_step;
      long long PP = P;
      float lr = s->cfg.lr, alpha = s->cfg.alpha;
      MasterDev* ms = s->ms;
      int* err = s->err;
      unsigned long long* cv = s->cver;
      void* args[] = {&wk, &cc, &g, &PP, &lr, &alpha, &exch, &ms, &err, &cv};
      if (ghc_status st = coop(c, reinterpret_cast<const void*>(easgd_exchange_kernel), args))
        return st;
      if (exch) {
        ++version;
        s->basis[static_cast<size_t>(k)] = version;
        if (s->v_every > 0 && version % s->v_every == 0)
          if (ghc_status st = validate_now(s)) return st;
      }
    }
  }
  if (h_loss && n_order > 0) {
    std::vector<float> lo(static_cast<size_t>(n_order));
    CU(cudaMemcpyAsync(lo.data(), d_loss, sizeof(float) * n_order, cudaMemcpyDeviceToHost,
                       c->stream));
    CU(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < n_order && i < s->trace_cap; ++i)
      h_loss[i] = lo[static_cast<size_t>(i)] / counts[static_cast<size_t>(i)];
  }
  CU(cudaStreamSynchronize(c->stream));
  if (downpour) {
    if (h_stale && n_order > 0) {
      const int64_t nt = std::min(n_order, s->trace_cap);
      CU(cudaMemcpy(h_stale, d_stale, sizeof(long long) * nt, cudaMemcpyDeviceToHost));
    }
    unsigned long long samples1 = 0;
    CU(cudaMemcpy(&samples1, s->d_samples, sizeof(samples1), cudaMemcpyDeviceToHost));
    s->samples += static_cast<int64_t>(samples1 - samples0);
    cudaFree(d_stale);
  }
  cudaFree(d_loss);
  s->rounds += n_order;
  return GHC_OK;
}

ghc_status run_hier(ghc_session* s, float* h_loss) {
  ghc_ctx* c = s->plan->ctx;
  const int G = s->cfg.groups, Wg = s->W / G;
  const int64_t P = s->P;
  const int B = s->cfg.batch_size;
  std::vector<int64_t> absorbed(static_cast<size_t>(G), 0), since(static_cast<size_t>(G), 0);
  int32_t* d_idx = nullptr;
  float* d_lsum = nullptr;
  const int64_t stride = static_cast<int64_t>(Wg) * B;
  CU(cudaMalloc(&d_idx, sizeof(int32_t) * stride * G));
  CU(cudaMalloc(&d_lsum, sizeof(float) * G));
  // host copy of streams for building each group's round index list
  int64_t all = 0;
  for (int k = 0; k < s->W; ++k)
    for (auto& b : s->batches[static_cast<size_t>(k)])
      all = std::max(all, s->stream_off[static_cast<size_t>(k)] + b.off + b.n);
  std::vector<int32_t> hs(static_cast<size_t>(all));
  CU(cudaMemcpy(hs.data(), s->streams, sizeof(int32_t) * all, cudaMemcpyDeviceToHost));
  std::vector<int32_t> tab(static_cast<size_t>(stride * G));
  std::vector<float> lsum(static_cast<size_t>(G));
  std::vector<int> gstat(static_cast<size_t>(G), 0);
  for (int64_t r = 0;; ++r) {
    if (s->cfg.max_updates > 0 && r >= s->cfg.max_updates) break;
    bool any_group = false;
    std::vector<int32_t> cnt(static_cast<size_t>(G), 0);
    std::vector<int> flushing(static_cast<size_t>(G), 0);
    for (int q = 0; q < G; ++q) {
      for (int j = 0; j < Wg; ++j) {
        const int k = q * Wg + j;
        auto& cur = s->cursor[static_cast<size_t>(k)];
        if (cur >= s->batches[static_cast<size_t>(k)].size()) continue;
        const Batch b = s->batches[static_cast<size_t>(k)][cur++];
        const int32_t* src = hs.data() + s->stream_off[static_cast<size_t>(k)] + b.off;
        std::copy(src, src + b.n, tab.begin() + q * stride + cnt[static_cast<size_t>(q)]);
        cnt[static_cast<size_t>(q)] += b.n;
      }
    }
    CU(cudaMemcpyAsync(d_idx, tab.data(), sizeof(int32_t) * tab.size(), cudaMemcpyHostToDevice,
                       c->stream));
    double rl = 0.0, rc = 0.0;
    for (int q = 0; q < G; ++q) {
      if (cnt[static_cast<size_t>(q)] == 0) {
        if (absorbed[static_cast<size_t>(q)] > 0) flushing[static_cast<size_t>(q)] = 1;
        continue;
      }
      any_group = true;
      // group round: fused sync step of the group's workers (rank order)
      if (ghc_status st = ghc_master_sync_rounds(s->group[static_cast<size_t>(q)], s->X, s->Y,
                                                 d_idx + q * stride, stride, nullptr,
                                                 cnt[static_cast<size_t>(q)], 1, d_lsum + q))
        return st;
      CU(cudaMemcpyAsync(&gstat[static_cast<size_t>(q)], &s->group[static_cast<size_t>(q)]->ms->status,
                         sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    }
    CU(cudaMemcpyAsync(lsum.data(), d_lsum, sizeof(float) * G, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    // a group update counts toward absorbed / the flush cadence only if the
    // group master accepted it (oracle gho_run_hier; optim.cpp:49-51)
    for (int q = 0; q < G; ++q) {
      if (cnt[static_cast<size_t>(q)] == 0) continue;
      if (gstat[static_cast<size_t>(q)] == 0) {
        absorbed[static_cast<size_t>(q)] += cnt[static_cast<size_t>(q)];
        since[static_cast<size_t>(q)] += 1;
      } else {
        ++s->rejected_groups;
      }
      if (since[static_cast<size_t>(q)] >= s->cfg.flush_k) flushing[static_cast<size_t>(q)] = 1;
    }
    for (int q = 0; q < G; ++q)
      if (cnt[static_cast<size_t>(q)] > 0) {
        rl += lsum[static_cast<size_t>(q)];
        rc += cnt[static_cast<size_t>(q)];
      }
    if (h_loss && rc > 0 && r < s->trace_cap) h_loss[r] = static_cast<float>(rl / rc);
    // top master: sync combine over flushing groups (group order)
    std::vector<double> wts;
    int nfl = 0;
    for (int q = 0; q < G; ++q) {
      if (!flushing[static_cast<size_t>(q)]) continue;
      float* gw = nullptr;
      if (ghc_status st = ghc_master_weights(s->group[static_cast<size_t>(q)], &gw, nullptr))
        return st;
      sub_kernel<<<64, 256, 0, c->stream>>>(s->pseudo + static_cast<int64_t>(nfl) * P,
                                           s->snap + static_cast<int64_t>(q) * P, gw, P);
      c->launches++;
      wts.push_back(static_cast<double>(absorbed[static_cast<size_t>(q)]));
      ++nfl;
    }
    if (nfl > 0) {
      if (ghc_status st = ghc_weighted_mean(c, s->comb, s->pseudo, wts.data(), nfl, P)) return st;
      if (ghc_status st = apply_master(s, s->master, s->comb, s->cfg.parent_lr, s->cfg.parent_mu))
        return st;
      float* tw = master_w(s->master);  // the top master's new (or, rejected, unchanged) weights
      int tstat = 0;  // the top master's samples count only an accepted update
      CU(cudaMemcpyAsync(&tstat, &s->master->ms->status, sizeof(int), cudaMemcpyDeviceToHost,
                         c->stream));
      CU(cudaStreamSynchronize(c->stream));
      if (tstat == 0)
        for (double v : wts) s->samples += static_cast<int64_t>(v);
      for (int q = 0; q < G; ++q) {
        if (!flushing[static_cast<size_t>(q)]) continue;
        float* gw = nullptr;
        if (ghc_status st = ghc_master_weights(s->group[static_cast<size_t>(q)], &gw, nullptr))
          return st;
        CU(cudaMemcpyAsync(gw, tw, sizeof(float) * P, cudaMemcpyDeviceToDevice, c->stream));
        CU(cudaMemcpyAsync(s->snap + static_cast<int64_t>(q) * P, tw, sizeof(float) * P,
                           cudaMemcpyDeviceToDevice, c->stream));
        absorbed[static_cast<size_t>(q)] = 0;
        since[static_cast<size_t>(q)] = 0;
      }
    }
    ++s->rounds;
    if (!any_group) break;
  }
  CU(cudaStreamSynchronize(c->stream));
  cudaFree(d_idx);
  cudaFree(d_lsum);
  return GHC_OK;
}

}  // namespace

extern "C" {

ghc_status ghc_session_create(ghc_plan* p, const ghc_train_config* cfg, const ghc_data_spec* spec,
                              ghc_session** out) {
  if (!p || !cfg || !spec || !out) return fail(GHC_ERR_CONFIG, "null argument");
  if (cfg->n_workers < 1 || cfg->batch_size < 1 || cfg->epochs < 0)
    return fail(GHC_ERR_CONFIG, "session: workers, batch_size must be >= 1");
  if (spec->n_files < cfg->n_workers)
    return fail(GHC_ERR_CONFIG, "shard_files: more workers than files; reduce workers");
  if (static_cast<int64_t>(spec->seq_len) * spec->input_dim != p->model.input_width ||
      spec->n_classes != p->model.n_classes)
    return fail(GHC_ERR_SHAPE, "session: dataset shape does not match the architecture");
  if (!(cfg->lr > 0.0f) || !(cfg->mu >= 0.0f && cfg->mu < 1.0f))
    return fail(GHC_ERR_CONFIG, "learning_rate must be > 0 and momentum in [0,1)");
  if (cfg->algo == GHC_ALGO_EASGD && (!(cfg->alpha > 0.0f && cfg->alpha < 1.0f) || cfg->tau < 1))
    return fail(GHC_ERR_CONFIG, "elastic_alpha must be in (0,1) and elastic_tau >= 1");
  if (cfg->groups > 0 && (cfg->n_workers % cfg->groups != 0 || cfg->flush_k < 1))
    return fail(GHC_ERR_CONFIG, "hierarchical: workers must split evenly into groups, K >= 1");
  auto* s = new ghc_session();
  s->plan = p;
  s->cfg = *cfg;
  s->spec = *spec;
  s->P = p->model.n_params;
  s->W = cfg->n_workers;
  CU(cudaSetDevice(p->ctx->device));
  if (ghc_status st = upload_data(s)) {
    delete s;
    return st;
  }
  std::vector<double> w0(static_cast<size_t>(s->P));
  init_weights(p->model, cfg->weight_seed, w0.data());
  if (ghc_status st = ghc_master_create(p, w0.data(), cfg->lr, cfg->mu, &s->master)) return st;
  const size_t pb = sizeof(float) * static_cast<size_t>((s->P + 3) & ~3LL);
  CU(cudaMalloc(&s->scratch_g, pb + 16));
  CU(cudaMalloc(&s->ms, sizeof(MasterDev)));
  CU(cudaMemset(s->ms, 0, sizeof(MasterDev)));
  CU(cudaMalloc(&s->err, sizeof(int)));
  CU(cudaMemset(s->err, 0, sizeof(int)));
  CU(cudaMalloc(&s->cver, sizeof(unsigned long long)));
  CU(cudaMemset(s->cver, 0, sizeof(unsigned long long)));
  CU(cudaMalloc(&s->d_basis, sizeof(unsigned long long) * static_cast<size_t>(s->W)));
  CU(cudaMemset(s->d_basis, 0, sizeof(unsigned long long) * static_cast<size_t>(s->W)));
  CU(cudaMalloc(&s->d_samples, sizeof(unsigned long long)));
  CU(cudaMemset(s->d_samples, 0, sizeof(unsigned long long)));
  std::vector<float> w32(static_cast<size_t>(s->P));
  for (int64_t i = 0; i < s->P; ++i) w32[static_cast<size_t>(i)] = static_cast<float>(w0[static_cast<size_t>(i)]);
  // every worker starts from the initial WEIGHTS message (f32 wire)
  CU(cudaMalloc(&s->worker_w, sizeof(float) * static_cast<size_t>(s->P) * s->W));
  for (int k = 0; k < s->W; ++k)
    CU(cudaMemcpy(s->worker_w + static_cast<int64_t>(k) * s->P, w32.data(), sizeof(float) * s->P,
                  cudaMemcpyHostToDevice));
  CU(cudaMalloc(&s->center, pb));
  CU(cudaMemcpy(s->center, w32.data(), sizeof(float) * s->P, cudaMemcpyHostToDevice));
  if (cfg->groups > 0) {
    const int G = cfg->groups;
    s->group.resize(static_cast<size_t>(G));
    for (int q = 0; q < G; ++q)
      if (ghc_status st = ghc_master_create(p, w0.data(), cfg->lr, cfg->mu, &s->group[static_cast<size_t>(q)]))
        return st;
    // the top master uses the pass-through parent settings
    s->master->lr = cfg->parent_lr;
    s->master->mu = cfg->parent_mu;
    CU(cudaMalloc(&s->snap, sizeof(float) * static_cast<size_t>(s->P) * G));
    CU(cudaMalloc(&s->pseudo, sizeof(float) * static_cast<size_t>(s->P) * G));
    CU(cudaMalloc(&s->comb, pb));
    for (int q = 0; q < G; ++q)
      CU(cudaMemcpy(s->snap + static_cast<int64_t>(q) * s->P, w32.data(), sizeof(float) * s->P,
                    cudaMemcpyHostToDevice));
  }
  s->basis.assign(static_cast<size_t>(s->W), 0);
  s->bidx.assign(static_cast<size_t>(s->W), 0);
  *out = s;
  return GHC_OK;
}

void ghc_session_destroy(ghc_session* s) {
  if (!s) return;
  cudaSetDevice(s->plan->ctx->device);
  cudaStreamSynchronize(s->plan->ctx->stream);
  ghc_master_destroy(s->master);
  for (auto* g : s->group) ghc_master_destroy(g);
  cudaFree(s->X);
  cudaFree(s->Y);
  cudaFree(s->streams);
  cudaFree(s->worker_w);
  cudaFree(s->center);
  cudaFree(s->scratch_g);
  cudaFree(s->multi_g);
  cudaFree(s->multi_l);
  cudaFree(s->snap);
  cudaFree(s->pseudo);
  cudaFree(s->comb);
  cudaFree(s->cver);
  cudaFree(s->d_basis);
  cudaFree(s->d_samples);
  cudaFree(s->ms);
  cudaFree(s->err);
  cudaFree(s->Xv);
  cudaFree(s->Yv);
  delete s;
}

ghc_status ghc_session_run(ghc_session* s, const int32_t* h_order, int64_t n_order, float* h_loss,
                           int64_t* h_staleness, int64_t trace_cap) {
  s->trace_cap = trace_cap < 0 ? 0 : trace_cap;
  ghc_status st;
  std::vector<int32_t> rr;
  bool sync_order = false;  // rr: the sync EASGD round-robin (run_replay batches each round's gradients)
  if (s->cfg.groups > 0) {
    st = run_hier(s, h_loss);
  } else if (s->cfg.mode == GHC_MODE_SYNC && s->cfg.algo == GHC_ALGO_DOWNPOUR) {
    st = run_sync(s, h_loss);
  } else {
    if (!h_order) {
      if (s->cfg.mode != GHC_MODE_SYNC)
        return fail(GHC_ERR_CONFIG, "replay mode needs the worker arrival order");
      // sync EASGD: every worker runs one batch per round, exchanges in rank order
      std::vector<size_t> left(static_cast<size_t>(s->W));
      for (int k = 0; k < s->W; ++k) left[static_cast<size_t>(k)] = s->batches[static_cast<size_t>(k)].size() - s->cursor[static_cast<size_t>(k)];
      for (bool any = true; any;) {
        any = false;
        for (int k = 0; k < s->W; ++k)
          if (left[static_cast<size_t>(k)] > 0) {
            --left[static_cast<size_t>(k)];
            rr.push_back(k);
            any = true;
          }
      }
      h_order = rr.data();
      n_order = static_cast<int64_t>(rr.size());
      sync_order = true;
    }
    st = run_replay(s, h_order, n_order, h_loss, h_staleness, sync_order);
  }
  if (st != GHC_OK) return st;
  int err = 0;
  CU(cudaMemcpy(&err, s->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err & 2) return fail(GHC_ERR_NONFINITE, "easgd_worker_step: gradient has NaN/Inf entries");
  return validate_now(s);  // "and once at end"
}

ghc_status ghc_session_load_data(ghc_session* s, const float* h_x, const int32_t* h_y,
                                 int64_t rows) {
  if (!s || !h_x || !h_y) return fail(GHC_ERR_CONFIG, "session: null argument");
  const int64_t want = static_cast<int64_t>(s->spec.n_files) * s->spec.samples_per_file;
  if (rows != want) return fail(GHC_ERR_SHAPE, "session_load_data: rows != n_files*samples_per_file");
  const int64_t width = s->plan->model.input_width;
  CU(cudaMemcpy(s->X, h_x, sizeof(float) * rows * width, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(s->Y, h_y, sizeof(int32_t) * rows, cudaMemcpyHostToDevice));
  return GHC_OK;
}

ghc_status ghc_session_set_validation(ghc_session* s, const float* h_x, const int32_t* h_y,
                                      int64_t n, int32_t every) {
  if (!s) return fail(GHC_ERR_CONFIG, "session: null handle");
  if (n < 1 || !h_x || !h_y) return fail(GHC_ERR_CONFIG, "validate: empty held-out set");
  if (every < 0) return fail(GHC_ERR_CONFIG, "validation cadence must be >= 0");
  const int64_t width = s->plan->model.input_width;
  cudaFree(s->Xv);
  cudaFree(s->Yv);
  s->Xv = nullptr;
  s->Yv = nullptr;
  CU(cudaMalloc(&s->Xv, sizeof(float) * n * width));
  CU(cudaMalloc(&s->Yv, sizeof(int32_t) * n));
  CU(cudaMemcpy(s->Xv, h_x, sizeof(float) * n * width, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(s->Yv, h_y, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  s->nv = n;
  s->v_every = every;
  return GHC_OK;
}

ghc_status ghc_session_validations(ghc_session* s, int64_t cap, uint64_t* versions,
                                   double* accuracy, double* loss, int64_t* count) {
  if (!s) return fail(GHC_ERR_CONFIG, "session: null handle");
  const int64_t n = static_cast<int64_t>(s->vrec.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const auto& v = s->vrec[static_cast<size_t>(i)];
    if (versions) versions[i] = v.version;
    if (accuracy) accuracy[i] = v.accuracy;
    if (loss) loss[i] = v.loss;
  }
  if (count) *count = n;
  return GHC_OK;
}

ghc_status ghc_session_read(ghc_session* s, float* h_w, float* h_v, float* h_worker_w,
                            float* h_group_w, uint64_t* stats) {
  const int64_t P = s->P;
  uint64_t ver = 0, rej = 0;
  if (s->cfg.algo == GHC_ALGO_EASGD && s->cfg.groups == 0) {
    if (h_w) CU(cudaMemcpy(h_w, s->center, sizeof(float) * P, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&ver, s->cver, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  } else {
    if (ghc_status st = ghc_master_read(s->master, h_w, h_v, &ver, &rej)) return st;
  }
  if (h_worker_w)
    CU(cudaMemcpy(h_worker_w, s->worker_w, sizeof(float) * P * s->W, cudaMemcpyDeviceToHost));
  if (h_group_w)
    for (size_t q = 0; q < s->group.size(); ++q)
      if (ghc_status st = ghc_master_read(s->group[q], h_group_w + q * P, nullptr, nullptr, nullptr))
        return st;
  if (stats) {
    stats[0] = ver;
    stats[1] = rej + s->rejected_groups;
    stats[2] = static_cast<uint64_t>(s->samples);
    stats[3] = static_cast<uint64_t>(s->rounds);
  }
  return GHC_OK;
}

}  // extern "C"
