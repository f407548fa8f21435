// ref_roles.cpp — CPU ORACLE / CPU BASELINE (TEST INFRASTRUCTURE ONLY).
//
// Runs the UNMODIFIED reference library (nn.cpp, optim.cpp, proto.cpp,
// transport.cpp, tensor.cpp, arch.cpp from /root/reference/proj/src, compiled
// by oracle/Makefile into oracle/_ref/) and adds the SPEC-only layers the
// reference describes but does not ship: the data layer and
// the master/worker roles, one std::thread per rank over the
// reference's own InprocHub transport (transport.cpp:25-177).  This is the
// "reference MPI CPU run" of BASELINE.md §2 and the pin for the C restatement
// in gh_oracle.c.
//
// Exposed as a C API (ghr_*) for ctypes; no reference types cross it.
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

#include "gh_oracle.h"
#include "gradhub/arch.hpp"
#include "gradhub/errors.hpp"
#include "gradhub/nn.hpp"
#include "gradhub/optim.hpp"
#include "gradhub/proto.hpp"
#include "gradhub/rng.hpp"
#include "gradhub/tensor.hpp"
#include "gradhub/transport.hpp"

using namespace gradhub;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ShapeError*>(&e)) return GHO_SHAPE;
  if (dynamic_cast<const NonFiniteGradientError*>(&e)) return GHO_NONFINITE;
  if (dynamic_cast<const CacheMismatchError*>(&e)) return GHO_CACHE_MISMATCH;
  if (dynamic_cast<const ConfigError*>(&e)) return GHO_CONFIG;
  if (dynamic_cast<const TransportError*>(&e)) return GHO_TRANSPORT;
  if (dynamic_cast<const ProtocolError*>(&e)) return GHO_PROTOCOL;
  return GHO_CONFIG;
}

#define GUARD_BEGIN try {
#define GUARD_END                         \
  }                                       \
  catch (const std::exception& e) {       \
    return status_of(e);                  \
  }                                       \
  return GHO_OK;

WeightSet to_ws(const Architecture& arch, const double* flat, std::uint64_t version = 0) {
  WeightSet w;
  const std::vector<Tensor> shape = arch.zero_weights();
  const std::size_t p = arch.n_params();
  w.tensors = unflatten(shape, std::vector<double>(flat, flat + p));
  w.version = version;
  return w;
}

void from_tensors(const std::vector<Tensor>& ts, double* out) {
  const std::vector<double> f = flatten(ts);
  std::memcpy(out, f.data(), f.size() * sizeof(double));
}

// ---- SPEC data layer over the reference Rng (same decisions as gh_oracle.c) ----
constexpr std::uint64_t kMeanStream = 0x6d65616eULL;
constexpr std::uint64_t kFileStream = 0x66696c65ULL;

void generate_files(const gho_data_spec& s, int f0, int nf, double* x, std::int32_t* y) {
  const std::size_t width = static_cast<std::size_t>(s.seq_len) * s.input_dim;
  std::vector<double> means(static_cast<std::size_t>(s.n_classes) * width);
  Rng mr(mix_seed(s.seed, kMeanStream));
  for (double& m : means) m = mr.normal();
  for (int f = f0; f < f0 + nf; ++f) {
    Rng fr(mix_seed(mix_seed(s.seed, kFileStream), static_cast<std::uint64_t>(f)));
    for (int i = 0; i < s.samples_per_file; ++i) {
      const std::size_t row = static_cast<std::size_t>(f - f0) * s.samples_per_file + i;
      const int lab = static_cast<int>((static_cast<long long>(i) + f) % s.n_classes);
      y[row] = lab;
      for (std::size_t j = 0; j < width; ++j) {
        const double v = s.delta * means[static_cast<std::size_t>(lab) * width + j] + fr.normal();
        x[row * width + j] = static_cast<double>(static_cast<float>(v));
      }
    }
  }
}

void shard_of(int n_files, int W, int k, int& f0, int& nf) {
  if (n_files < W) throw ConfigError("shard_files: more workers than files");
  const int base = n_files / W, extra = n_files % W;
  nf = base + (k < extra ? 1 : 0);
  f0 = k * base + (k < extra ? k : extra);
}

std::vector<std::int64_t> epoch_indices(const gho_data_spec& s, int W, int k, int epoch,
                                        std::uint64_t shuffle_seed, bool shuffle) {
  int f0, nf;
  shard_of(s.n_files, W, k, f0, nf);
  std::vector<std::int64_t> idx(static_cast<std::size_t>(nf) * s.samples_per_file);
  for (std::size_t j = 0; j < idx.size(); ++j)
    idx[j] = static_cast<std::int64_t>(f0) * s.samples_per_file + static_cast<std::int64_t>(j);
  if (shuffle) {
    Rng r(mix_seed(mix_seed(shuffle_seed, static_cast<std::uint64_t>(k)),
                   static_cast<std::uint64_t>(epoch)));
    r.shuffle(idx);
  }
  return idx;
}

// A worker's batch stream: epochs × shuffled shard, short last batch.
struct Stream {
  const gho_data_spec* s;
  const gho_train_cfg* cfg;
  int k;
  int epoch = 0;
  std::size_t pos = 0;
  std::vector<std::int64_t> idx;
  bool done = false;
  // rows of this worker's data: either the full dataset (base_row = 0) or its shard
  const double* x;
  const std::int32_t* y;
  std::int64_t base_row;

  void init() {
    idx = epoch_indices(*s, cfg->n_workers, k, 0, cfg->shuffle_seed, cfg->shuffle != 0);
    done = cfg->epochs < 1;
  }
  bool next(Batch& b) {
    if (done) return false;
    const std::size_t width = static_cast<std::size_t>(s->seq_len) * s->input_dim;
    const std::size_t nb = std::min<std::size_t>(cfg->batch_size, idx.size() - pos);
    b.n_samples = nb;
    b.inputs.resize(nb * width);
    b.labels.resize(nb);
    for (std::size_t j = 0; j < nb; ++j) {
      const std::int64_t g = idx[pos + j] - base_row;
      std::memcpy(&b.inputs[j * width], x + g * static_cast<std::int64_t>(width),
                  width * sizeof(double));
      b.labels[j] = y[g];
    }
    pos += nb;
    if (pos >= idx.size()) {
      if (++epoch >= cfg->epochs) {
        done = true;
      } else {
        idx = epoch_indices(*s, cfg->n_workers, k, epoch, cfg->shuffle_seed, cfg->shuffle != 0);
        pos = 0;
      }
    }
    return true;
  }
};

WirePrecision wire_of(const gho_train_cfg& c) {
  return c.wire_f64 ? WirePrecision::f64 : WirePrecision::f32;
}

// ---- Synchronous Downpour over InprocHub, one thread per rank -----------------
struct SyncResult {
  WeightSet w;
  OptimState s;
  gho_run_stats st{};
  std::vector<std::vector<double>> loss;   // [round][worker]
  std::vector<std::vector<double>> count;  // [round][worker]
  double seconds_timed = 0.0;
};

void run_sync_threads(const Architecture& arch, const gho_data_spec& spec,
                      const gho_train_cfg& cfg, const double* x, const std::int32_t* y,
                      bool full_dataset, int warmup_rounds, SyncResult& res) {
  const int W = cfg.n_workers;
  auto eps = establish(Topology::flat(W), "inproc", wire_of(cfg));
  WeightSet w0 = init_weights(arch, cfg.weight_seed);
  OptimState st0 = OptimState::for_weights(w0, cfg.lr, cfg.mu);
  const std::int64_t max_rounds = cfg.max_updates > 0 ? cfg.max_updates : INT64_MAX;
  std::vector<std::vector<double>> loss_rw, cnt_rw;
  std::mutex log_mu;
  std::exception_ptr err;
  std::mutex err_mu;
  auto record_err = [&](std::exception_ptr e) {
    std::lock_guard<std::mutex> lk(err_mu);
    if (!err) err = e;
  };

  // Per-worker shard data when the caller did not pass the full dataset.
  std::vector<std::vector<double>> shard_x(static_cast<std::size_t>(W));
  std::vector<std::vector<std::int32_t>> shard_y(static_cast<std::size_t>(W));
  std::vector<std::int64_t> base(static_cast<std::size_t>(W), 0);

  std::chrono::steady_clock::time_point t_start{}, t_end{};

  std::thread master([&] {
    try {
      Endpoint& ep = *eps[0];
      WeightSet w = w0;
      OptimState s = st0;
      std::vector<bool> active(static_cast<std::size_t>(W) + 1, true);
      int n_active = W;
      for (int r = 1; r <= W; ++r) ep.send(r, WeightsMsg{w.tensors, w.version});
      std::int64_t round = 0;
      while (n_active > 0) {
        if (round == warmup_rounds) t_start = std::chrono::steady_clock::now();
        if (round >= max_rounds) break;
        std::map<int, GradientMsg> buf;
        std::vector<bool> pending = active;
        int n_pending = n_active;
        while (n_pending > 0) {
          auto in = ep.recv();
          if (!in) throw TransportError("master: session ended early");
          const int from = in->from;
          if (std::holds_alternative<DoneMsg>(in->msg)) {
            if (active[from]) {
              active[from] = false;
              --n_active;
            }
            if (pending[from]) {
              pending[from] = false;
              --n_pending;
            }
          } else if (auto* g = std::get_if<GradientMsg>(&in->msg)) {
            if (buf.count(from)) throw ProtocolError("duplicate gradient in sync round");
            buf.emplace(from, std::move(*g));
            pending[from] = false;
            --n_pending;
          }
        }
        if (buf.empty()) break;
        // Σ c_i g_i / Σ c_i, rank order.
        std::vector<Tensor> comb = arch.zero_weights();
        double total = 0.0;
        for (auto& [r, g] : buf) {
          const double c = static_cast<double>(g.sample_count);
          for (std::size_t t = 0; t < comb.size(); ++t)
            for (std::size_t j = 0; j < comb[t].values.size(); ++j)
              comb[t].values[j] += c * g.tensors[t].values[j];
          total += c;
        }
        for (Tensor& t : comb)
          for (double& v : t.values) v = v / total;
        Gradient gr;
        gr.tensors = std::move(comb);
        gr.basis_version = w.version;
        try {
          auto [nw, ns] = sgd_step(w, gr, s);
          w = std::move(nw);
          s = std::move(ns);
          res.st.updates += 1;
          res.st.samples += static_cast<std::int64_t>(total);
        } catch (const NonFiniteGradientError&) {
          res.st.rejected += 1;
        }
        for (auto& [r, g] : buf) ep.send(r, WeightsMsg{w.tensors, w.version});
        ++round;
      }
      t_end = std::chrono::steady_clock::now();
      for (int r = 1; r <= W; ++r) {
        if (!active[r]) continue;
        try {
          ep.send(r, ShutdownMsg{});
        } catch (const TransportError&) {
          // the worker finished and closed before seeing the cap
        }
      }
      while (ep.recv()) {
        // drain gradients / DONEs sent before the workers saw SHUTDOWN
      }
      res.w = w;
      res.s = s;
      res.st.version = w.version;
      ep.close();
    } catch (...) {
      record_err(std::current_exception());
      eps[0]->close();
    }
  });

  std::vector<std::thread> workers;
  for (int r = 1; r <= W; ++r) {
    workers.emplace_back([&, r] {
      const int k = r - 1;
      try {
        Endpoint& ep = *eps[static_cast<std::size_t>(r)];
        Stream st{&spec, &cfg, k};
        if (full_dataset) {
          st.x = x;
          st.y = y;
          st.base_row = 0;
        } else {
          int f0, nf;
          shard_of(spec.n_files, W, k, f0, nf);
          const std::size_t width = static_cast<std::size_t>(spec.seq_len) * spec.input_dim;
          const std::size_t rows = static_cast<std::size_t>(nf) * spec.samples_per_file;
          shard_x[k].resize(rows * width);
          shard_y[k].resize(rows);
          generate_files(spec, f0, nf, shard_x[k].data(), shard_y[k].data());
          st.x = shard_x[k].data();
          st.y = shard_y[k].data();
          st.base_row = static_cast<std::int64_t>(f0) * spec.samples_per_file;
        }
        st.init();
        auto in = ep.recv();
        if (!in) throw TransportError("worker: no initial weights");
        auto* wm = std::get_if<WeightsMsg>(&in->msg);
        if (!wm) throw ProtocolError("worker: expected WEIGHTS");
        WeightSet w;
        w.tensors = std::move(wm->tensors);
        w.version = wm->version;
        Batch b;
        std::size_t round = 0;
        bool stop = false;
        while (!stop && st.next(b)) {
          ForwardResult fr = forward(w, arch, b);
          const double lo = loss(fr.probs, b.labels);
          Gradient g = backward(w, arch, fr.cache, b.labels);
          {
            std::lock_guard<std::mutex> lk(log_mu);
            if (loss_rw.size() <= round) {
              loss_rw.resize(round + 1, std::vector<double>(static_cast<std::size_t>(W), 0.0));
              cnt_rw.resize(round + 1, std::vector<double>(static_cast<std::size_t>(W), 0.0));
            }
            loss_rw[round][static_cast<std::size_t>(k)] = lo;
            cnt_rw[round][static_cast<std::size_t>(k)] = static_cast<double>(b.n_samples);
          }
          ep.send(0, GradientMsg{std::move(g.tensors), g.basis_version, b.n_samples});
          auto rep = ep.recv();
          if (!rep) throw TransportError("worker: master vanished");
          if (std::holds_alternative<ShutdownMsg>(rep->msg)) {
            stop = true;
            break;
          }
          auto* nw = std::get_if<WeightsMsg>(&rep->msg);
          if (!nw) throw ProtocolError("worker: expected WEIGHTS");
          w.tensors = std::move(nw->tensors);
          w.version = nw->version;
          ++round;
        }
        if (!stop) ep.send(0, DoneMsg{static_cast<std::uint32_t>(r)});
        ep.close();
      } catch (...) {
        record_err(std::current_exception());
        eps[static_cast<std::size_t>(r)]->close();
      }
    });
  }
  master.join();
  for (auto& t : workers) t.join();
  if (err) std::rethrow_exception(err);
  res.loss = std::move(loss_rw);
  res.count = std::move(cnt_rw);
  if (t_start.time_since_epoch().count() != 0)
    res.seconds_timed = std::chrono::duration<double>(t_end - t_start).count();
}

}  // namespace

extern "C" {

const char* ghr_last_error(void) { return g_err.c_str(); }

int ghr_n_params(const char* arch_text, std::int64_t* out) {
  GUARD_BEGIN
  *out = static_cast<std::int64_t>(parse_architecture(arch_text).n_params());
  GUARD_END
}

int ghr_init_weights(const char* arch_text, std::uint64_t seed, double* w) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  from_tensors(init_weights(arch, seed).tensors, w);
  GUARD_END
}

int ghr_checksum(const char* arch_text, const double* w, std::uint64_t* out) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  *out = weights_checksum(to_ws(arch, w));
  GUARD_END
}

// forward (nn.cpp:100) + loss (nn.cpp:234) + backward (nn.cpp:250).
int ghr_forward_backward(const char* arch_text, const double* w, const double* x,
                         const std::int32_t* y, std::int64_t n, double* grad,
                         double* probs, double* loss_out) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  const WeightSet ws = to_ws(arch, w);
  Batch b;
  b.n_samples = static_cast<std::size_t>(n);
  b.inputs.assign(x, x + n * static_cast<std::int64_t>(arch.input_width()));
  b.labels.assign(y, y + n);
  ForwardResult fr = forward(ws, arch, b);
  if (probs) std::memcpy(probs, fr.probs.p.data(), fr.probs.p.size() * sizeof(double));
  if (loss_out) *loss_out = loss(fr.probs, b.labels);
  if (grad) from_tensors(backward(ws, arch, fr.cache, b.labels).tensors, grad);
  GUARD_END
}

// Cache guard (nn.cpp:253-260): backward against weights that changed after forward.
int ghr_stale_cache_probe(const char* arch_text, const double* w, const double* x,
                          const std::int32_t* y, std::int64_t n) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  WeightSet ws = to_ws(arch, w);
  Batch b;
  b.n_samples = static_cast<std::size_t>(n);
  b.inputs.assign(x, x + n * static_cast<std::int64_t>(arch.input_width()));
  b.labels.assign(y, y + n);
  ForwardResult fr = forward(ws, arch, b);
  ws.tensors[0].values[0] += 1.0;
  backward(ws, arch, fr.cache, b.labels);
  GUARD_END
}

int ghr_finite_diff(const char* arch_text, const double* w, const double* x,
                    const std::int32_t* y, std::int64_t n, double eps, double* grad) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  Batch b;
  b.n_samples = static_cast<std::size_t>(n);
  b.inputs.assign(x, x + n * static_cast<std::int64_t>(arch.input_width()));
  b.labels.assign(y, y + n);
  from_tensors(finite_diff_gradient(to_ws(arch, w), arch, b, eps).tensors, grad);
  GUARD_END
}

// sgd_step (optim.cpp:39-65): w, v updated in place only on success.
int ghr_sgd_step(const char* arch_text, double* w, double* v, const double* g,
                 double lr, double mu, std::uint64_t* version) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  WeightSet ws = to_ws(arch, w, version ? *version : 0);
  OptimState s;
  s.velocity = to_ws(arch, v).tensors;
  s.learning_rate = lr;
  s.momentum = mu;
  Gradient gr;
  gr.tensors = to_ws(arch, g).tensors;
  auto [nw, ns] = sgd_step(ws, gr, s);
  from_tensors(nw.tensors, w);
  from_tensors(ns.velocity, v);
  if (version) *version = nw.version;
  GUARD_END
}

int ghr_elastic_pull(const char* arch_text, double* w, const double* c, double alpha) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  from_tensors(elastic_pull(to_ws(arch, w), to_ws(arch, c), alpha).tensors, w);
  GUARD_END
}

int ghr_easgd_worker_step(const char* arch_text, double* w, const double* c,
                          const double* g, double lr, double alpha, std::uint64_t tau,
                          std::uint64_t batch_index) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  OptimState s;
  s.learning_rate = lr;
  s.momentum = 0.0;
  ElasticConfig e;
  e.alpha = alpha;
  e.tau = tau;
  Gradient gr;
  gr.tensors = to_ws(arch, g).tensors;
  from_tensors(easgd_worker_step(to_ws(arch, w), to_ws(arch, c), gr, s, e, batch_index).tensors,
               w);
  GUARD_END
}

int ghr_easgd_center_step(const char* arch_text, double* c, const double* w, double alpha,
                          std::uint64_t* version) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  ElasticConfig e;
  e.alpha = alpha;
  e.tau = 1;
  WeightSet out = easgd_center_step(to_ws(arch, c, version ? *version : 0), to_ws(arch, w), e);
  from_tensors(out.tensors, c);
  if (version) *version = out.version;
  GUARD_END
}

// proto.cpp encode of WEIGHTS / GRADIENT / SHUTDOWN frames (golden vectors).
int ghr_encode(int kind, const char* arch_text, const double* w, std::uint64_t version,
               std::uint64_t sample_count, int wire_f64, std::uint8_t* out,
               std::int64_t cap, std::int64_t* len) {
  GUARD_BEGIN
  Message m;
  if (kind == 0) {
    m = ShutdownMsg{};
  } else {
    const Architecture arch = parse_architecture(arch_text);
    if (kind == 1) m = WeightsMsg{to_ws(arch, w).tensors, version};
    else m = GradientMsg{to_ws(arch, w).tensors, version, sample_count};
  }
  const auto bytes = encode(m, wire_f64 ? WirePrecision::f64 : WirePrecision::f32);
  *len = static_cast<std::int64_t>(bytes.size());
  if (static_cast<std::int64_t>(bytes.size()) > cap) throw ShapeError("encode: buffer too small");
  std::memcpy(out, bytes.data(), bytes.size());
  GUARD_END
}

// SPEC data layer over the reference Rng.
int ghr_generate(const gho_data_spec* s, double* x, std::int32_t* y) {
  GUARD_BEGIN
  generate_files(*s, 0, s->n_files, x, y);
  GUARD_END
}

int ghr_epoch_indices(const gho_data_spec* s, std::int32_t W, std::int32_t k, std::int32_t epoch,
                      std::uint64_t shuffle_seed, std::int32_t shuffle, std::int64_t* out,
                      std::int64_t* count) {
  GUARD_BEGIN
  const auto idx = epoch_indices(*s, W, k, epoch, shuffle_seed, shuffle != 0);
  std::memcpy(out, idx.data(), idx.size() * sizeof(std::int64_t));
  *count = static_cast<std::int64_t>(idx.size());
  GUARD_END
}

// Threaded sync Downpour over the reference InprocHub.  x/y = full dataset
// (nullable: then every worker generates its own shard, as in a real run).
int ghr_run_sync(const char* arch_text, const gho_data_spec* spec, const double* x,
                 const std::int32_t* y, const gho_train_cfg* cfg, double* w_out,
                 double* v_out, double* loss_trace, gho_run_stats* stats) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  SyncResult res;
  run_sync_threads(arch, *spec, *cfg, x, y, x != nullptr, -1, res);
  from_tensors(res.w.tensors, w_out);
  if (v_out) from_tensors(res.s.velocity, v_out);
  if (loss_trace) {
    for (std::size_t r = 0; r < res.loss.size(); ++r) {
      double num = 0.0, den = 0.0;
      for (std::size_t k = 0; k < res.loss[r].size(); ++k) {
        num += res.count[r][k] * res.loss[r][k];
        den += res.count[r][k];
      }
      if (r < static_cast<std::size_t>(res.st.updates + res.st.rejected)) loss_trace[r] = num / den;
    }
  }
  if (stats) *stats = res.st;
  GUARD_END
}

// CPU baseline: threaded sync Downpour, `warmup` untimed rounds then `timed`
// rounds; wall seconds of the timed rounds.  Workers generate their shards.
int ghr_bench_sync(const char* arch_text, const gho_data_spec* spec, const gho_train_cfg* cfg,
                   std::int32_t warmup, std::int32_t timed, double* seconds,
                   std::int64_t* samples) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  gho_train_cfg c = *cfg;
  c.max_updates = warmup + timed;
  SyncResult res;
  run_sync_threads(arch, *spec, c, nullptr, nullptr, false, warmup, res);
  *seconds = res.seconds_timed;
  std::int64_t n = 0;
  for (std::size_t r = static_cast<std::size_t>(warmup); r < res.count.size(); ++r)
    for (double v : res.count[r]) n += static_cast<std::int64_t>(v);
  *samples = n;
  GUARD_END
}

// Single-thread forward+backward micro-benchmark.
int ghr_bench_fwd_bwd(const char* arch_text, std::int64_t n, std::int32_t reps, double* seconds) {
  GUARD_BEGIN
  const Architecture arch = parse_architecture(arch_text);
  const WeightSet w = init_weights(arch, 7);
  Batch b;
  b.n_samples = static_cast<std::size_t>(n);
  b.inputs.resize(static_cast<std::size_t>(n) * arch.input_width());
  b.labels.resize(static_cast<std::size_t>(n));
  Rng r(1);
  for (double& v : b.inputs) v = r.normal();
  for (std::size_t i = 0; i < b.labels.size(); ++i)
    b.labels[i] = static_cast<int>(i % arch.n_classes());
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) {
    ForwardResult fr = forward(w, arch, b);
    Gradient g = backward(w, arch, fr.cache, b.labels);
    (void)g;
  }
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  GUARD_END
}

}  // extern "C"
