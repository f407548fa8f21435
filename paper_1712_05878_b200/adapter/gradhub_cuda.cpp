// gradhub_cuda.cpp — see gradhub_cuda.hpp.
#include "gradhub_cuda.hpp"

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <variant>

#include "gradhub/errors.hpp"

namespace gradhub::cuda {

namespace {

[[noreturn]] void rethrow(ghc_status s, const char* what) {
  const std::string msg = std::string(what) + ": " + ghc_last_error();
  switch (s) {
    case GHC_ERR_SHAPE: throw ShapeError(msg);
    case GHC_ERR_NONFINITE: throw NonFiniteGradientError(msg);
    case GHC_ERR_CACHE_MISMATCH: throw CacheMismatchError(msg);
    case GHC_ERR_CONFIG: throw ConfigError(msg);
    case GHC_ERR_TRANSPORT: throw TransportError(msg);
    case GHC_ERR_PROTOCOL: throw ProtocolError(msg);
    default: throw std::runtime_error(msg);
  }
}

void check(ghc_status s, const char* what) {
  if (s != GHC_OK) rethrow(s, what);
}

struct Thread {
  ghc_ctx* ctx = nullptr;
  std::map<std::string, ghc_plan*> plans;
  ~Thread() {
    for (auto& [k, p] : plans) ghc_plan_destroy(p);
    if (ctx) ghc_ctx_destroy(ctx);
  }
};
thread_local Thread t_state;

ghc_plan* plan_for(const Architecture& arch) {
  const std::string text = format_architecture(arch);
  auto it = t_state.plans.find(text);
  if (it != t_state.plans.end()) return it->second;
  ghc_plan* p = nullptr;
  check(ghc_plan_create(thread_context(), text.c_str(), &p), "parse_architecture");
  t_state.plans.emplace(text, p);
  return p;
}

// Device buffer owned for the duration of one call (on a given context).
struct Dev {
  ghc_ctx* c = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
  explicit Dev(size_t b, ghc_ctx* ctx = nullptr) : c(ctx ? ctx : thread_context()), bytes(b) {
    check(ghc_malloc(c, b ? b : 16, &p), "alloc");
  }
  Dev(const Dev&) = delete;
  Dev(Dev&& o) noexcept : c(o.c), p(o.p), bytes(o.bytes) { o.p = nullptr; }
  ~Dev() {
    if (p) ghc_free(c, p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void put(const void* h, size_t b) { check(ghc_memcpy_h2d(c, p, h, b), "h2d"); }
  void get(void* h, size_t b) const {
    check(ghc_memcpy_d2h(c, h, p, b), "d2h");
    check(ghc_ctx_sync(c), "sync");
  }
};

std::vector<double> flat64(const std::vector<Tensor>& ts) {
  std::vector<double> out;
  for (const Tensor& t : ts) out.insert(out.end(), t.values.begin(), t.values.end());
  return out;
}

std::vector<Tensor> from_f32(const std::vector<Tensor>& shape, const std::vector<float>& f) {
  std::vector<Tensor> out = shape;
  size_t k = 0;
  for (Tensor& t : out)
    for (double& v : t.values) v = static_cast<double>(f[k++]);
  return out;
}

// The reference's f64 tensors on the device as f32 (one upload of the f64
// values, rounded on the GPU) — optionally with the stale-cache token.
struct DevWeights {
  Dev w32;
  uint64_t token = 0;
  DevWeights(const std::vector<Tensor>& ts, bool want_token)
      : w32(sizeof(float) * count(ts)) {
    const std::vector<double> f = flat64(ts);
    Dev w64(sizeof(double) * f.size()), h(sizeof(uint64_t));
    w64.put(f.data(), sizeof(double) * f.size());
    check(ghc_weights_import_f64(thread_context(), w32.as<float>(), w64.as<double>(),
                                 static_cast<int64_t>(f.size()), want_token ? h.as<uint64_t>() : nullptr),
          "weights upload");
    if (want_token) h.get(&token, sizeof(token));
    else check(ghc_ctx_sync(thread_context()), "sync");
  }
  static size_t count(const std::vector<Tensor>& ts) {
    size_t n = 0;
    for (const Tensor& t : ts) n += t.values.size();
    return n;
  }
};

Dev upload_f32(const std::vector<Tensor>& ts) {
  DevWeights d(ts, false);
  return std::move(d.w32);
}

std::vector<float> download(const Dev& d, size_t n) {
  std::vector<float> v(n);
  d.get(v.data(), n * sizeof(float));
  return v;
}

void check_batch(const Architecture& arch, const Batch& batch) {
  if (batch.n_samples < 1) throw ShapeError("batch: n_samples must be >= 1");
  if (batch.inputs.size() != batch.n_samples * arch.input_width())
    throw ShapeError("batch: inputs size != n_samples*width");
  if (batch.labels.size() != batch.n_samples) throw ShapeError("batch: labels size != n_samples");
}

}  // namespace

ghc_ctx* thread_context(int device) {
  if (!t_state.ctx) check(ghc_ctx_create(device, &t_state.ctx), "ghc_ctx_create");
  return t_state.ctx;
}

WeightSet init_weights(const Architecture& arch, std::uint64_t seed) {
  arch.validate();
  WeightSet w;
  w.tensors = arch.zero_weights();
  std::vector<double> flat(arch.n_params());
  check(ghc_init_weights(plan_for(arch), seed, flat.data()), "init_weights");
  size_t k = 0;
  for (Tensor& t : w.tensors)
    for (double& v : t.values) v = flat[k++];
  return w;
}

ForwardResult forward(const WeightSet& w, const Architecture& arch, const Batch& batch) {
  arch.validate();
  if (!shape_congruent(w.tensors, arch.zero_weights()))
    throw ShapeError("weight set does not match the architecture");
  check_batch(arch, batch);
  ghc_plan* p = plan_for(arch);
  const size_t n = batch.n_samples, K = arch.n_classes();
  std::vector<float> x(batch.inputs.begin(), batch.inputs.end());
  std::vector<int32_t> y(batch.labels.begin(), batch.labels.end());
  for (int32_t& l : y)
    if (l < 0 || static_cast<size_t>(l) >= K) l = 0;  // forward ignores labels (nn.cpp:100)
  DevWeights dw(w.tensors, true);
  Dev dx(n * arch.input_width() * 4), dy(n * sizeof(int32_t)), dp(n * K * 4), dl(4);
  dx.put(x.data(), x.size() * 4);
  dy.put(y.data(), n * sizeof(int32_t));
  check(ghc_forward(p, dw.w32.as<float>(), dx.as<float>(), dy.as<int32_t>(), nullptr,
                    static_cast<int64_t>(n), dp.as<float>(), dl.as<float>()),
        "forward");
  const std::vector<float> probs = download(dp, n * K);
  ForwardResult out;
  out.probs.rows = n;
  out.probs.cols = K;
  out.probs.p.assign(probs.begin(), probs.end());
  // The fused kernel recomputes the activations in backward; the cache keeps
  // the batch and the guard: version + the device-computed weight token.
  out.cache.n_samples = n;
  out.cache.weights_version = w.version;
  out.cache.weights_checksum = dw.token;
  out.cache.arch_signature = format_architecture(arch);
  out.cache.layers.resize(arch.layers.size());
  out.cache.layers[0].x = batch.inputs;
  out.cache.layers.back().probs = out.probs.p;
  if (const auto* l0 = std::get_if<LstmSpec>(&arch.layers[0])) {
    // the LSTM LayerCache (nn.hpp:15-23) from the generic GEMM-based forward
    const size_t T = l0->seq_len, H = l0->hidden_dim, nT = n * T;
    Dev dg(nT * 4 * H * 4), dc(nT * H * 4), dt(nT * H * 4), dh(nT * H * 4);
    check(ghc_forward_cache(p, dw.w32.as<float>(), dx.as<float>(), static_cast<int64_t>(n), dg.as<float>(),
                            dc.as<float>(), dt.as<float>(), dh.as<float>()),
          "forward cache");
    LayerCache& lc = out.cache.layers[0];
    auto fill = [](std::vector<double>& dst, const std::vector<float>& src) { dst.assign(src.begin(), src.end()); };
    fill(lc.gates, download(dg, nT * 4 * H));
    fill(lc.cell, download(dc, nT * H));
    fill(lc.tanh_c, download(dt, nT * H));
    fill(lc.hidden, download(dh, nT * H));
    if (arch.layers.size() == 2) {  // the softmax layer's input is h_T
      LayerCache& sc = out.cache.layers[1];
      sc.x.resize(n * H);
      for (size_t s = 0; s < n; ++s)
        for (size_t u = 0; u < H; ++u) sc.x[s * H + u] = lc.hidden[(s * T + T - 1) * H + u];
    }
  }
  return out;
}

double loss(const ProbMatrix& probs, const std::vector<int>& labels) {
  if (labels.size() != probs.rows) throw ShapeError("loss: labels size != probability rows");
  const size_t n = probs.rows;
  if (n == 0) return 0.0 / 0.0;  // the reference divides 0 by 0 too
  std::vector<int32_t> y(labels.begin(), labels.end());
  Dev dp(probs.p.size() * sizeof(double)), dy(n * sizeof(int32_t));
  dp.put(probs.p.data(), probs.p.size() * sizeof(double));
  dy.put(y.data(), n * sizeof(int32_t));
  double s = 0.0;
  check(ghc_nll_sum(thread_context(), dp.as<double>(), dy.as<int32_t>(), static_cast<int64_t>(n),
                    static_cast<int32_t>(probs.cols), &s),
        "loss");
  return s / static_cast<double>(n);
}

double batch_loss(const WeightSet& w, const Architecture& arch, const Batch& batch) {
  arch.validate();
  if (!shape_congruent(w.tensors, arch.zero_weights()))
    throw ShapeError("weight set does not match the architecture");
  check_batch(arch, batch);
  const size_t K = arch.n_classes();
  for (int l : batch.labels)
    if (l < 0 || static_cast<size_t>(l) >= K)
      throw ShapeError("loss: label " + std::to_string(l) + " out of range [0," + std::to_string(K) + ")");
  ghc_plan* p = plan_for(arch);
  const size_t n = batch.n_samples;
  std::vector<float> x(batch.inputs.begin(), batch.inputs.end());
  std::vector<int32_t> y(batch.labels.begin(), batch.labels.end());
  Dev dw = upload_f32(w.tensors), dx(x.size() * 4), dy(n * 4), dl(4);
  dx.put(x.data(), x.size() * 4);
  dy.put(y.data(), n * 4);
  check(ghc_forward(p, dw.as<float>(), dx.as<float>(), dy.as<int32_t>(), nullptr, static_cast<int64_t>(n),
                    nullptr, dl.as<float>()),
        "batch_loss");
  float lsum = 0.0f;
  dl.get(&lsum, 4);
  check(ghc_plan_check_error(p), "batch_loss");
  return static_cast<double>(lsum) / static_cast<double>(n);
}

Gradient backward(const WeightSet& w, const Architecture& arch, const ForwardCache& cache,
                  const std::vector<int>& labels) {
  // nn.cpp:252-262 guards, unchanged semantics
  if (!shape_congruent(w.tensors, arch.zero_weights()))
    throw ShapeError("weight set does not match the architecture");
  if (cache.arch_signature != format_architecture(arch) ||
      cache.layers.size() != arch.layers.size())
    throw CacheMismatchError("backward: cache built for a different architecture");
  DevWeights dw(w.tensors, true);  // the upload recomputes the token on the device
  if (cache.weights_checksum != dw.token || cache.weights_version != w.version)
    throw CacheMismatchError("backward: cache is stale (weights changed since forward)");
  const size_t n = cache.n_samples, K = arch.n_classes();
  if (labels.size() != n) throw ShapeError("backward: labels size != cached batch");
  for (int l : labels)
    if (l < 0 || static_cast<size_t>(l) >= K) throw ShapeError("backward: label out of range");
  ghc_plan* p = plan_for(arch);
  std::vector<float> x(cache.layers[0].x.begin(), cache.layers[0].x.end());
  std::vector<int32_t> y(labels.begin(), labels.end());
  const size_t P = arch.n_params();
  Dev dx(x.size() * 4), dy(n * 4), dg(P * 4), dl(4);
  dx.put(x.data(), x.size() * 4);
  dy.put(y.data(), n * 4);
  check(ghc_worker_grad(p, dw.w32.as<float>(), dx.as<float>(), dy.as<int32_t>(), nullptr,
                        static_cast<int64_t>(n), 1.0f / static_cast<float>(n), dg.as<float>(),
                        dl.as<float>()),
        "backward");
  Gradient g;
  g.tensors = from_f32(arch.zero_weights(), download(dg, P));
  g.basis_version = w.version;
  return g;
}

std::pair<WeightSet, OptimState> sgd_step(const WeightSet& w, const Gradient& g,
                                          const OptimState& s) {
  s.validate();
  if (!shape_congruent(w.tensors, g.tensors)) throw ShapeError("sgd_step: gradient shape mismatch");
  if (!shape_congruent(w.tensors, s.velocity)) throw ShapeError("sgd_step: velocity shape mismatch");
  const size_t P = DevWeights::count(w.tensors);
  Dev dw = upload_f32(w.tensors), dv = upload_f32(s.velocity), dg = upload_f32(g.tensors), ds(4);
  Dev dw2(P * 4), dv2(P * 4);  // value semantics: one pass into new buffers
  int32_t st = 0;
  ds.put(&st, 4);
  check(ghc_sgd_step_out(thread_context(), dw.as<float>(), dv.as<float>(), dg.as<float>(),
                         dw2.as<float>(), dv2.as<float>(), static_cast<int64_t>(P),
                         static_cast<float>(s.learning_rate), static_cast<float>(s.momentum),
                         ds.as<int32_t>(), nullptr),
        "sgd_step");
  ds.get(&st, 4);
  if (st == GHC_ERR_NONFINITE)
    throw NonFiniteGradientError("sgd_step: gradient has NaN/Inf entries; update rejected");
  WeightSet out;
  out.tensors = from_f32(w.tensors, download(dw2, P));
  out.version = w.version + 1;
  OptimState ns = s;
  ns.velocity = from_f32(s.velocity, download(dv2, P));
  return {std::move(out), std::move(ns)};
}

WeightSet elastic_pull(const WeightSet& w, const WeightSet& center, double alpha) {
  if (!shape_congruent(w.tensors, center.tensors))
    throw ShapeError("elastic_pull: worker/center shapes differ");
  const size_t P = DevWeights::count(w.tensors);
  Dev dw = upload_f32(w.tensors), dc = upload_f32(center.tensors);
  check(ghc_elastic_pull(thread_context(), dw.as<float>(), dc.as<float>(), static_cast<int64_t>(P),
                         static_cast<float>(alpha)),
        "elastic_pull");
  WeightSet out = w;
  out.tensors = from_f32(w.tensors, download(dw, P));
  return out;
}

WeightSet easgd_worker_step(const WeightSet& w, const WeightSet& center, const Gradient& g,
                            const OptimState& s, const ElasticConfig& e,
                            std::uint64_t batch_index) {
  s.validate();
  e.validate();
  if (!shape_congruent(w.tensors, g.tensors))
    throw ShapeError("easgd_worker_step: gradient shape does not match weights");
  const size_t P = DevWeights::count(w.tensors);
  Dev dw = upload_f32(w.tensors), dc = upload_f32(center.tensors), dg = upload_f32(g.tensors), ds(4);
  Dev dw2(P * 4);
  int32_t st = 0;
  ds.put(&st, 4);
  check(ghc_easgd_worker_step_out(thread_context(), dw.as<float>(), dc.as<float>(), dg.as<float>(),
                                  dw2.as<float>(), static_cast<int64_t>(P),
                                  static_cast<float>(s.learning_rate), static_cast<float>(e.alpha),
                                  e.tau, batch_index, ds.as<int32_t>()),
        "easgd_worker_step");
  ds.get(&st, 4);
  if (st == GHC_ERR_NONFINITE)
    throw NonFiniteGradientError("easgd_worker_step: gradient has NaN/Inf entries");
  WeightSet out = w;
  out.tensors = from_f32(w.tensors, download(dw2, P));
  return out;
}

WeightSet easgd_center_step(const WeightSet& center, const WeightSet& worker,
                            const ElasticConfig& e) {
  e.validate();
  if (!shape_congruent(center.tensors, worker.tensors))
    throw ShapeError("easgd_center_step: worker/center shapes differ");
  const size_t P = DevWeights::count(center.tensors);
  Dev dc = upload_f32(center.tensors), dw = upload_f32(worker.tensors);
  check(ghc_easgd_center_step(thread_context(), dc.as<float>(), dw.as<float>(),
                              static_cast<int64_t>(P), static_cast<float>(e.alpha), nullptr),
        "easgd_center_step");
  WeightSet out;
  out.tensors = from_f32(center.tensors, download(dc, P));
  out.version = center.version + 1;
  return out;
}

// ===========================================================================
// "nvlink" backend: in-process Endpoints with device mailboxes
// ===========================================================================
namespace {

// A queued message: the control record (message with value-less tensors)
// plus the mailbox slot holding its payload on the receiver's device.
struct Rec {
  int from = -1;
  Message msg;
  int slot = -1;       // -1: no payload
  size_t count = 0;    // values in the slot
};

struct NvHub {
  struct Link {  // sender → receiver: `cap` payload slots on the receiver's device
    std::vector<void*> slot;
    std::vector<size_t> bytes;
    std::vector<bool> busy;
  };
  struct Box {  // per receiver
    std::mutex mu;
    std::condition_variable nonempty, space;
    std::deque<Rec> q;
    std::vector<size_t> inflight;  // per sender: slots / records outstanding
  };
  int n = 0, ndev = 1;
  WirePrecision wire = WirePrecision::f32;
  size_t cap = 16;
  std::vector<std::unique_ptr<Box>> boxes;
  std::vector<std::vector<Link>> links;  // [to][from]
  std::vector<ghc_ctx*> alloc_ctx;       // per device: mailbox allocations
  std::mutex state_mu;
  std::vector<bool> closed;
  int open_count = 0;

  NvHub(int n_, WirePrecision w, size_t c) : n(n_), wire(w), cap(c ? c : 1) {
    int nd = 0;
    check(ghc_device_count(&nd), "device count");
    ndev = nd > 0 ? nd : 1;
    alloc_ctx.assign(static_cast<size_t>(ndev), nullptr);
    for (int d = 0; d < ndev && d < n; ++d) check(ghc_ctx_create(d, &alloc_ctx[static_cast<size_t>(d)]), "ctx");
    for (int r = 0; r < n; ++r) {
      boxes.push_back(std::make_unique<Box>());
      boxes.back()->inflight.assign(static_cast<size_t>(n), 0);
    }
    links.assign(static_cast<size_t>(n), std::vector<Link>(static_cast<size_t>(n)));
    for (auto& row : links)
      for (Link& l : row) {
        l.slot.assign(cap, nullptr);
        l.bytes.assign(cap, 0);
        l.busy.assign(cap, false);
      }
    closed.assign(static_cast<size_t>(n), false);
    open_count = n;
  }
  ~NvHub() {
    for (int to = 0; to < n; ++to)
      for (auto& l : links[static_cast<size_t>(to)])
        for (void* p : l.slot)
          if (p) ghc_free(alloc_ctx[static_cast<size_t>(device_of(to))], p);
    for (ghc_ctx* c : alloc_ctx)
      if (c) ghc_ctx_destroy(c);
  }
  int device_of(int r) const { return r % ndev; }

  int open_others(int self) {
    std::lock_guard<std::mutex> lk(state_mu);
    return open_count - (closed[static_cast<size_t>(self)] ? 0 : 1);
  }
  bool is_closed(int r) {
    std::lock_guard<std::mutex> lk(state_mu);
    return closed[static_cast<size_t>(r)];
  }
  void mark_closed(int r) {
    {
      std::lock_guard<std::mutex> lk(state_mu);
      if (closed[static_cast<size_t>(r)]) return;
      closed[static_cast<size_t>(r)] = true;
      --open_count;
    }
    for (auto& b : boxes) {
      std::lock_guard<std::mutex> lk(b->mu);
      b->nonempty.notify_all();
      b->space.notify_all();
    }
  }

  // Wait for link space (backpressure, as transport.cpp:68-81) and reserve a
  // slot of at least `bytes` on the receiver's device (-1: no payload).
  int reserve(int from, int to, size_t bytes) {
    Box& box = *boxes[static_cast<size_t>(to)];
    std::unique_lock<std::mutex> lk(box.mu);
    box.space.wait(lk, [&] {
      return box.inflight[static_cast<size_t>(from)] < cap || is_closed(to) || is_closed(from);
    });
    if (is_closed(to)) throw TransportError("send: rank " + std::to_string(to) + " is closed");
    if (is_closed(from)) throw TransportError("send after shutdown");
    ++box.inflight[static_cast<size_t>(from)];
    if (bytes == 0) return -1;
    Link& l = links[static_cast<size_t>(to)][static_cast<size_t>(from)];
    for (size_t s = 0; s < cap; ++s)
      if (!l.busy[s]) {
        l.busy[s] = true;
        if (l.bytes[s] < bytes) {
          ghc_ctx* ac = alloc_ctx[static_cast<size_t>(device_of(to))];
          if (l.slot[s]) ghc_free(ac, l.slot[s]);
          l.slot[s] = nullptr;
          l.bytes[s] = 0;
          check(ghc_malloc(ac, bytes, &l.slot[s]), "mailbox alloc");
          l.bytes[s] = bytes;
        }
        return static_cast<int>(s);
      }
    throw TransportError("nvlink: no free mailbox slot");  // unreachable: inflight < cap
  }
  void push(int to, Rec r) {
    Box& box = *boxes[static_cast<size_t>(to)];
    std::lock_guard<std::mutex> lk(box.mu);
    box.q.push_back(std::move(r));
    box.nonempty.notify_one();
  }
  void release(int to, int from, int slot) {
    Box& box = *boxes[static_cast<size_t>(to)];
    std::lock_guard<std::mutex> lk(box.mu);
    if (slot >= 0) links[static_cast<size_t>(to)][static_cast<size_t>(from)].busy[static_cast<size_t>(slot)] = false;
    --box.inflight[static_cast<size_t>(from)];
    box.space.notify_all();
  }
  void* slot_ptr(int to, int from, int slot) {
    return links[static_cast<size_t>(to)][static_cast<size_t>(from)].slot[static_cast<size_t>(slot)];
  }
};

// Value-less copy of the tensors (dims travel in the control record).
std::vector<Tensor> dims_only(const std::vector<Tensor>& ts, size_t& count) {
  std::vector<Tensor> out;
  count = 0;
  for (const Tensor& t : ts) {
    out.emplace_back(t.dims, std::vector<double>{});
    count += t.values.size();
  }
  return out;
}

void refill(std::vector<Tensor>& ts, const double* v) {
  for (Tensor& t : ts) {
    size_t m = 1;
    for (size_t d : t.dims) m *= d;
    t.values.assign(v, v + m);
    v += m;
  }
}

class NvEndpoint final : public Endpoint, public DeviceEndpoint {
 public:
  NvEndpoint(std::shared_ptr<NvHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {
    check(ghc_ctx_create(hub_->device_of(rank_), &ctx_), "ghc_ctx_create");
  }
  ~NvEndpoint() override {
    close();
    drop_held();
    if (stage_) ghc_free(ctx_, stage_);
    ghc_ctx_destroy(ctx_);
  }
  int rank() const override { return rank_; }
  int device() const override { return hub_->device_of(rank_); }

  void send(int to, const Message& m) override {
    precheck(to);
    Rec r;
    r.from = rank_;
    const std::vector<Tensor>* ts = nullptr;
    if (auto* w = std::get_if<WeightsMsg>(&m)) {
      ts = &w->tensors;
      WeightsMsg c;
      c.tensors = dims_only(w->tensors, r.count);
      c.version = w->version;
      r.msg = std::move(c);
    } else if (auto* g = std::get_if<GradientMsg>(&m)) {
      ts = &g->tensors;
      GradientMsg c;
      c.tensors = dims_only(g->tensors, r.count);
      c.basis_version = g->basis_version;
      c.sample_count = g->sample_count;
      r.msg = std::move(c);
    } else {
      r.msg = m;
    }
    if (ts) {
      // stage the values (wire precision) on this rank's GPU, one peer copy
      const size_t es = hub_->wire == WirePrecision::f64 ? 8 : 4;
      const size_t bytes = r.count * es;
      std::vector<unsigned char> host(bytes);
      size_t k = 0;
      for (const Tensor& t : *ts)
        for (double v : t.values) {
          if (es == 4) {
            const float f = static_cast<float>(v);
            std::memcpy(&host[4 * k], &f, 4);
          } else {
            std::memcpy(&host[8 * k], &v, 8);
          }
          ++k;
        }
      ensure_stage(bytes);
      check(ghc_memcpy_h2d(ctx_, stage_, host.data(), bytes), "h2d");
      r.slot = hub_->reserve(rank_, to, bytes ? bytes : 16);
      move_payload(to, r.slot, stage_, bytes);
    } else {
      r.slot = hub_->reserve(rank_, to, 0);
    }
    hub_->push(to, std::move(r));
    ++sent_;
  }

  void send_device(int to, int kind, const float* d_values, std::size_t count,
                   const std::vector<Tensor>& shape, std::uint64_t version,
                   std::uint64_t sample_count) override {
    precheck(to);
    if (hub_->wire != WirePrecision::f32) throw ConfigError("send_device: f32 wire only");
    Rec r;
    r.from = rank_;
    r.count = count;
    size_t cnt = 0;
    if (kind == 2) {
      WeightsMsg c;
      c.tensors = dims_only(shape, cnt);
      c.version = version;
      r.msg = std::move(c);
    } else if (kind == 3) {
      GradientMsg c;
      c.tensors = dims_only(shape, cnt);
      c.basis_version = version;
      c.sample_count = sample_count;
      r.msg = std::move(c);
    } else {
      throw ProtocolError("send_device: WEIGHTS (2) or GRADIENT (3) only");
    }
    r.slot = hub_->reserve(rank_, to, count * 4 ? count * 4 : 16);
    move_payload(to, r.slot, d_values, count * 4);
    hub_->push(to, std::move(r));
    ++sent_;
  }

  std::optional<Incoming> recv() override {
    drop_held();
    std::optional<Rec> r = pop();
    if (!r) return std::nullopt;
    if (r->slot >= 0) {
      const size_t es = hub_->wire == WirePrecision::f64 ? 8 : 4;
      std::vector<unsigned char> host(r->count * es);
      check(ghc_memcpy_d2h(ctx_, host.data(), hub_->slot_ptr(rank_, r->from, r->slot), host.size()), "d2h");
      check(ghc_ctx_sync(ctx_), "sync");
      std::vector<double> v(r->count);
      for (size_t i = 0; i < r->count; ++i) {
        if (es == 4) {
          float f;
          std::memcpy(&f, &host[4 * i], 4);
          v[i] = static_cast<double>(f);
        } else {
          std::memcpy(&v[i], &host[8 * i], 8);
        }
      }
      if (auto* w = std::get_if<WeightsMsg>(&r->msg)) refill(w->tensors, v.data());
      if (auto* g = std::get_if<GradientMsg>(&r->msg)) refill(g->tensors, v.data());
    }
    hub_->release(rank_, r->from, r->slot);
    ++received_;
    return Incoming{r->from, std::move(r->msg)};
  }

  std::optional<Incoming> recv_device(const float** d_values, std::size_t* count) override {
    drop_held();
    std::optional<Rec> r = pop();
    if (!r) return std::nullopt;
    if (d_values) *d_values = r->slot >= 0 ? static_cast<const float*>(hub_->slot_ptr(rank_, r->from, r->slot)) : nullptr;
    if (count) *count = r->count;
    held_from_ = r->from;  // the slot stays reserved until the next recv
    held_slot_ = r->slot;
    ++received_;
    return Incoming{r->from, std::move(r->msg)};
  }

  void close() override { hub_->mark_closed(rank_); }

 private:
  void precheck(int to) {
    if (to < 0 || to >= hub_->n || to == rank_) throw TransportError("send: unknown rank " + std::to_string(to));
    if (hub_->is_closed(rank_)) throw TransportError("send after shutdown");
    if (hub_->is_closed(to)) throw TransportError("send: rank " + std::to_string(to) + " is closed");
  }
  void ensure_stage(size_t bytes) {
    if (stage_bytes_ >= bytes && stage_) return;
    if (stage_) ghc_free(ctx_, stage_);
    stage_ = nullptr;
    check(ghc_malloc(ctx_, bytes ? bytes : 16, &stage_), "stage alloc");
    stage_bytes_ = bytes;
  }
  // sender GPU → receiver GPU mailbox slot (NVLink peer copy), completed
  // before the control record is published
  void move_payload(int to, int slot, const void* src, size_t bytes) {
    if (bytes)
      check(ghc_memcpy_peer(ctx_, hub_->slot_ptr(to, rank_, slot), hub_->device_of(to), src,
                            hub_->device_of(rank_), bytes),
            "peer copy");
    check(ghc_ctx_sync(ctx_), "sync");
  }
  std::optional<Rec> pop() {
    NvHub::Box& box = *hub_->boxes[static_cast<size_t>(rank_)];
    std::unique_lock<std::mutex> lk(box.mu);
    box.nonempty.wait(lk, [&] { return !box.q.empty() || hub_->open_others(rank_) == 0; });
    if (box.q.empty()) return std::nullopt;  // all peers closed and drained
    Rec r = std::move(box.q.front());
    box.q.pop_front();
    return r;
  }
  void drop_held() {
    if (held_from_ >= 0) hub_->release(rank_, held_from_, held_slot_);
    held_from_ = held_slot_ = -1;
  }

  std::shared_ptr<NvHub> hub_;
  int rank_;
  ghc_ctx* ctx_ = nullptr;
  void* stage_ = nullptr;
  size_t stage_bytes_ = 0;
  int held_from_ = -1, held_slot_ = -1;
};

}  // namespace

std::vector<std::unique_ptr<Endpoint>> establish(const Topology& topo, const std::string& backend,
                                                 WirePrecision wire, std::size_t link_capacity) {
  if (backend != "nvlink") return gradhub::establish(topo, backend, wire, link_capacity);
  topo.validate();
  const int n = topo.n_ranks();
  auto hub = std::make_shared<NvHub>(n, wire, link_capacity);
  std::vector<std::unique_ptr<Endpoint>> eps;
  for (int r = 0; r < n; ++r) eps.push_back(std::make_unique<NvEndpoint>(hub, r));
  return eps;
}

}  // namespace gradhub::cuda
