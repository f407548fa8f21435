// gradhub_cuda.cpp — see gradhub_cuda.hpp.
#include "gradhub_cuda.hpp"

#include <cstring>
#include <map>
#include <string>

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

// Device buffer owned for the duration of one call.
struct Dev {
  void* p = nullptr;
  size_t bytes = 0;
  explicit Dev(size_t b) : bytes(b) { check(ghc_malloc(thread_context(), b ? b : 16, &p), "alloc"); }
  ~Dev() { ghc_free(thread_context(), p); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void put(const void* h, size_t b) { check(ghc_memcpy_h2d(thread_context(), p, h, b), "h2d"); }
  void get(void* h, size_t b) const {
    check(ghc_memcpy_d2h(thread_context(), h, p, b), "d2h");
    check(ghc_ctx_sync(thread_context()), "sync");
  }
};

std::vector<float> to_f32(const std::vector<Tensor>& ts) {
  std::vector<float> out;
  for (const Tensor& t : ts)
    for (double v : t.values) out.push_back(static_cast<float>(v));  // f32 wire rounding
  return out;
}

std::vector<Tensor> from_f32(const std::vector<Tensor>& shape, const std::vector<float>& f) {
  std::vector<Tensor> out = shape;
  size_t k = 0;
  for (Tensor& t : out)
    for (double& v : t.values) v = static_cast<double>(f[k++]);
  return out;
}

Dev upload(const std::vector<float>& v) {
  Dev d(v.size() * sizeof(float));
  d.put(v.data(), v.size() * sizeof(float));
  return d;
}

std::vector<float> download(const Dev& d, size_t n) {
  std::vector<float> v(n);
  d.get(v.data(), n * sizeof(float));
  return v;
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
  if (batch.n_samples < 1) throw ShapeError("batch: n_samples must be >= 1");
  if (batch.inputs.size() != batch.n_samples * arch.input_width())
    throw ShapeError("batch: inputs size != n_samples*width");
  if (batch.labels.size() != batch.n_samples) throw ShapeError("batch: labels size != n_samples");
  ghc_plan* p = plan_for(arch);
  const size_t n = batch.n_samples, K = arch.n_classes();
  std::vector<float> x(batch.inputs.begin(), batch.inputs.end());
  std::vector<int32_t> y(batch.labels.begin(), batch.labels.end());
  for (int32_t& l : y)
    if (l < 0 || static_cast<size_t>(l) >= K) l = 0;  // forward ignores labels (nn.cpp:100)
  Dev dw = upload(to_f32(w.tensors)), dx = upload(x), dy(n * sizeof(int32_t)), dp(n * K * 4),
      dl(4);
  dy.put(y.data(), n * sizeof(int32_t));
  check(ghc_forward(p, dw.as<float>(), dx.as<float>(), dy.as<int32_t>(), nullptr,
                    static_cast<int64_t>(n), dp.as<float>(), dl.as<float>()),
        "forward");
  const std::vector<float> probs = download(dp, n * K);
  ForwardResult out;
  out.probs.rows = n;
  out.probs.cols = K;
  out.probs.p.assign(probs.begin(), probs.end());
  // The fused kernel recomputes activations in backward; the cache keeps the
  // batch plus the reference's stale-cache guard (nn.cpp:116-119).
  out.cache.n_samples = n;
  out.cache.weights_version = w.version;
  out.cache.weights_checksum = weights_checksum(w);
  out.cache.arch_signature = format_architecture(arch);
  out.cache.layers.resize(arch.layers.size());
  out.cache.layers[0].x = batch.inputs;
  return out;
}

double loss(const ProbMatrix& probs, const std::vector<int>& labels) {
  return gradhub::loss(probs, labels);  // O(n·K) host reduction of device probs
}

Gradient backward(const WeightSet& w, const Architecture& arch, const ForwardCache& cache,
                  const std::vector<int>& labels) {
  // nn.cpp:252-262 guards, unchanged semantics
  if (!shape_congruent(w.tensors, arch.zero_weights()))
    throw ShapeError("weight set does not match the architecture");
  if (cache.arch_signature != format_architecture(arch) ||
      cache.layers.size() != arch.layers.size())
    throw CacheMismatchError("backward: cache built for a different architecture");
  if (cache.weights_checksum != weights_checksum(w) || cache.weights_version != w.version)
    throw CacheMismatchError("backward: cache is stale (weights changed since forward)");
  const size_t n = cache.n_samples, K = arch.n_classes();
  if (labels.size() != n) throw ShapeError("backward: labels size != cached batch");
  for (int l : labels)
    if (l < 0 || static_cast<size_t>(l) >= K) throw ShapeError("backward: label out of range");
  ghc_plan* p = plan_for(arch);
  std::vector<float> x(cache.layers[0].x.begin(), cache.layers[0].x.end());
  std::vector<int32_t> y(labels.begin(), labels.end());
  const size_t P = arch.n_params();
  Dev dw = upload(to_f32(w.tensors)), dx = upload(x), dy(n * 4), dg(P * 4), dl(4);
  dy.put(y.data(), n * 4);
  check(ghc_worker_grad(p, dw.as<float>(), dx.as<float>(), dy.as<int32_t>(), nullptr,
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
  const std::vector<float> wf = to_f32(w.tensors);
  const size_t P = wf.size();
  Dev dw = upload(wf), dv = upload(to_f32(s.velocity)), dg = upload(to_f32(g.tensors)), ds(4);
  int32_t st = 0;
  ds.put(&st, 4);
  check(ghc_sgd_apply(thread_context(), dw.as<float>(), dv.as<float>(), dg.as<float>(),
                      static_cast<int64_t>(P), static_cast<float>(s.learning_rate),
                      static_cast<float>(s.momentum), ds.as<int32_t>(), nullptr),
        "sgd_step");
  ds.get(&st, 4);
  if (st == GHC_ERR_NONFINITE)
    throw NonFiniteGradientError("sgd_step: gradient has NaN/Inf entries; update rejected");
  WeightSet out;
  out.tensors = from_f32(w.tensors, download(dw, P));
  out.version = w.version + 1;
  OptimState ns = s;
  ns.velocity = from_f32(s.velocity, download(dv, P));
  return {std::move(out), std::move(ns)};
}

WeightSet elastic_pull(const WeightSet& w, const WeightSet& center, double alpha) {
  if (!shape_congruent(w.tensors, center.tensors))
    throw ShapeError("elastic_pull: worker/center shapes differ");
  const std::vector<float> wf = to_f32(w.tensors);
  Dev dw = upload(wf), dc = upload(to_f32(center.tensors));
  check(ghc_elastic_pull(thread_context(), dw.as<float>(), dc.as<float>(),
                         static_cast<int64_t>(wf.size()), static_cast<float>(alpha)),
        "elastic_pull");
  WeightSet out = w;
  out.tensors = from_f32(w.tensors, download(dw, wf.size()));
  return out;
}

WeightSet easgd_worker_step(const WeightSet& w, const WeightSet& center, const Gradient& g,
                            const OptimState& s, const ElasticConfig& e,
                            std::uint64_t batch_index) {
  s.validate();
  e.validate();
  if (!shape_congruent(w.tensors, g.tensors))
    throw ShapeError("easgd_worker_step: gradient shape does not match weights");
  const std::vector<float> wf = to_f32(w.tensors);
  Dev dw = upload(wf), dc = upload(to_f32(center.tensors)), dg = upload(to_f32(g.tensors)),
      ds(4);
  int32_t st = 0;
  ds.put(&st, 4);
  check(ghc_easgd_worker_step(thread_context(), dw.as<float>(), dc.as<float>(), dg.as<float>(),
                              static_cast<int64_t>(wf.size()),
                              static_cast<float>(s.learning_rate), static_cast<float>(e.alpha),
                              e.tau, batch_index, ds.as<int32_t>()),
        "easgd_worker_step");
  ds.get(&st, 4);
  if (st == GHC_ERR_NONFINITE)
    throw NonFiniteGradientError("easgd_worker_step: gradient has NaN/Inf entries");
  WeightSet out = w;
  out.tensors = from_f32(w.tensors, download(dw, wf.size()));
  return out;
}

WeightSet easgd_center_step(const WeightSet& center, const WeightSet& worker,
                            const ElasticConfig& e) {
  e.validate();
  if (!shape_congruent(center.tensors, worker.tensors))
    throw ShapeError("easgd_center_step: worker/center shapes differ");
  const std::vector<float> cf = to_f32(center.tensors);
  Dev dc = upload(cf), dw = upload(to_f32(worker.tensors));
  check(ghc_easgd_center_step(thread_context(), dc.as<float>(), dw.as<float>(),
                              static_cast<int64_t>(cf.size()), static_cast<float>(e.alpha),
                              nullptr),
        "easgd_center_step");
  WeightSet out;
  out.tensors = from_f32(center.tensors, download(dc, cf.size()));
  out.version = center.version + 1;
  return out;
}

}  // namespace gradhub::cuda
