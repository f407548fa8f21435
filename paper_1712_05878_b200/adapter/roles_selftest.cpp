// roles_selftest.cpp — the reference-facing drop-in end to end: the SPEC
// master/worker role loops (the same loop shape as
// oracle/ref_roles.cpp) written ONCE against the reference API (Endpoint,
// Message, forward / loss / backward / sgd_step) and run three ways:
//
//   ref   : gradhub::establish(…, "inproc") + gradhub:: compute (the reference)
//   xport : gradhub::cuda::establish(…, "nvlink") + gradhub:: compute
//           → must be BIT-identical to `ref` (the transport moves values
//             exactly at the wire precision)
//   gpu   : gradhub::cuda::establish(…, "nvlink") + gradhub::cuda:: compute
//           → weights within 1e-5 relative of `ref`; versions, staleness and
//             every endpoint's message counts exact
//
// for synchronous Downpour (rank-order combine) and asynchronous Downpour
// with a replayed arrival order (workers take turns; staleness arises from
// the interleaving).  Prints one line per check and "ROLES OK"; exit 1 on a
// mismatch.  Run by tests/test_gpu_adapter.py on the GPU box.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <map>
#include <thread>

#include "gradhub/arch.hpp"
#include "gradhub/errors.hpp"
#include "gradhub/rng.hpp"
#include "gradhub_cuda.hpp"

using namespace gradhub;

namespace {

struct RefApi {
  static ForwardResult forward(const WeightSet& w, const Architecture& a, const Batch& b) {
    return gradhub::forward(w, a, b);
  }
  static Gradient backward(const WeightSet& w, const Architecture& a, const ForwardCache& c,
                           const std::vector<int>& l) {
    return gradhub::backward(w, a, c, l);
  }
  static double loss(const ProbMatrix& p, const std::vector<int>& l) { return gradhub::loss(p, l); }
  static std::pair<WeightSet, OptimState> sgd_step(const WeightSet& w, const Gradient& g,
                                                   const OptimState& s) {
    return gradhub::sgd_step(w, g, s);
  }
};
struct CudaApi {
  static ForwardResult forward(const WeightSet& w, const Architecture& a, const Batch& b) {
    return gradhub::cuda::forward(w, a, b);
  }
  static Gradient backward(const WeightSet& w, const Architecture& a, const ForwardCache& c,
                           const std::vector<int>& l) {
    return gradhub::cuda::backward(w, a, c, l);
  }
  static double loss(const ProbMatrix& p, const std::vector<int>& l) {
    return gradhub::cuda::loss(p, l);
  }
  static std::pair<WeightSet, OptimState> sgd_step(const WeightSet& w, const Gradient& g,
                                                   const OptimState& s) {
    return gradhub::cuda::sgd_step(w, g, s);
  }
};

struct Run {
  WeightSet w;
  std::vector<std::uint64_t> stale;
  std::vector<double> loss;
  std::vector<std::uint64_t> sent, recvd;
  std::uint64_t updates = 0;
};

// batch j of worker k: fixed synthetic rows (reference Rng)
Batch make_batch(const Architecture& arch, int k, int j, std::size_t B) {
  Batch b;
  b.n_samples = B;
  Rng r(mix_seed(mix_seed(1234, static_cast<std::uint64_t>(k)), static_cast<std::uint64_t>(j)));
  for (std::size_t i = 0; i < B; ++i) {
    const int y = static_cast<int>(r.below(arch.n_classes()));
    b.labels.push_back(y);
    for (std::size_t c = 0; c < arch.input_width(); ++c)
      b.inputs.push_back(static_cast<double>(static_cast<float>(r.normal() + 1.5 * (y - 1.0))));
  }
  return b;
}

template <class Api>
Run run_sync(const Architecture& arch, std::vector<std::unique_ptr<Endpoint>> eps, int W, int R,
             std::size_t B) {
  Run out;
  std::vector<std::thread> th;
  th.emplace_back([&] {
    Endpoint& ep = *eps[0];
    WeightSet w = init_weights(arch, 7);
    OptimState s = OptimState::for_weights(w, 0.05, 0.9);
    for (int k = 1; k <= W; ++k) ep.send(k, WeightsMsg{w.tensors, w.version});
    for (int r = 0; r < R; ++r) {
      std::map<int, GradientMsg> buf;
      while (static_cast<int>(buf.size()) < W) {
        auto in = ep.recv();
        if (!in) throw TransportError("master: session ended early");
        auto* g = std::get_if<GradientMsg>(&in->msg);
        if (!g) throw ProtocolError("master: expected GRADIENT");
        buf.emplace(in->from, std::move(*g));
      }
      std::vector<Tensor> comb = arch.zero_weights();  // Σ c_i g_i / Σ c_i, rank order
      double total = 0.0;
      for (auto& [k, g] : buf) {
        const double c = static_cast<double>(g.sample_count);
        for (std::size_t t = 0; t < comb.size(); ++t)
          for (std::size_t j = 0; j < comb[t].values.size(); ++j) comb[t].values[j] += c * g.tensors[t].values[j];
        total += c;
      }
      for (Tensor& t : comb)
        for (double& v : t.values) v /= total;
      Gradient gr;
      gr.tensors = std::move(comb);
      gr.basis_version = w.version;
      auto [nw, ns] = Api::sgd_step(w, gr, s);
      w = std::move(nw);
      s = std::move(ns);
      ++out.updates;
      for (int k = 1; k <= W; ++k) ep.send(k, WeightsMsg{w.tensors, w.version});
    }
    for (int k = 1; k <= W; ++k) ep.send(k, ShutdownMsg{});
    while (ep.recv()) {
    }
    out.w = w;
    ep.close();
  });
  std::vector<std::vector<double>> losses(static_cast<std::size_t>(W));
  for (int k = 1; k <= W; ++k)
    th.emplace_back([&, k] {
      Endpoint& ep = *eps[static_cast<std::size_t>(k)];
      for (int j = 0;; ++j) {
        auto in = ep.recv();
        if (!in || std::holds_alternative<ShutdownMsg>(in->msg)) break;
        auto* wm = std::get_if<WeightsMsg>(&in->msg);
        if (!wm) throw ProtocolError("worker: expected WEIGHTS");
        WeightSet w;
        w.tensors = std::move(wm->tensors);
        w.version = wm->version;
        const Batch b = make_batch(arch, k, j, B + static_cast<std::size_t>(k));  // ragged batches
        ForwardResult fr = Api::forward(w, arch, b);
        losses[static_cast<std::size_t>(k - 1)].push_back(Api::loss(fr.probs, b.labels));
        Gradient g = Api::backward(w, arch, fr.cache, b.labels);
        ep.send(0, GradientMsg{std::move(g.tensors), g.basis_version, b.n_samples});
      }
      ep.send(0, DoneMsg{static_cast<std::uint32_t>(k)});
      ep.close();
    });
  for (auto& t : th) t.join();
  for (auto& l : losses) out.loss.insert(out.loss.end(), l.begin(), l.end());
  for (auto& e : eps) {
    out.sent.push_back(e->messages_sent());
    out.recvd.push_back(e->messages_received());
  }
  return out;
}

// Async Downpour, replayed arrival order: worker order[i] sends the i-th
// gradient the master applies; the master replies WEIGHTS
// to the sender only.  Staleness = master version − gradient basis version.
template <class Api>
Run run_async(const Architecture& arch, std::vector<std::unique_ptr<Endpoint>> eps, int W,
              const std::vector<int>& order, std::size_t B) {
  Run out;
  std::atomic<std::size_t> turn{0};
  std::vector<std::thread> th;
  th.emplace_back([&] {
    Endpoint& ep = *eps[0];
    WeightSet w = init_weights(arch, 7);
    OptimState s = OptimState::for_weights(w, 0.05, 0.9);
    for (int k = 1; k <= W; ++k) ep.send(k, WeightsMsg{w.tensors, w.version});
    for (std::size_t i = 0; i < order.size(); ++i) {
      auto in = ep.recv();
      if (!in) throw TransportError("master: session ended early");
      auto* g = std::get_if<GradientMsg>(&in->msg);
      if (!g || in->from != order[i]) throw ProtocolError("master: out-of-order gradient");
      out.stale.push_back(w.version - g->basis_version);
      Gradient gr;
      gr.tensors = std::move(g->tensors);
      gr.basis_version = g->basis_version;
      auto [nw, ns] = Api::sgd_step(w, gr, s);
      w = std::move(nw);
      s = std::move(ns);
      ++out.updates;
      ep.send(in->from, WeightsMsg{w.tensors, w.version});
      turn.store(i + 1);
    }
    for (int k = 1; k <= W; ++k) ep.send(k, ShutdownMsg{});
    while (ep.recv()) {
    }
    out.w = w;
    ep.close();
  });
  for (int k = 1; k <= W; ++k)
    th.emplace_back([&, k] {
      Endpoint& ep = *eps[static_cast<std::size_t>(k)];
      std::size_t next = 0;  // next position of this worker in `order`
      for (int j = 0;; ++j) {
        auto in = ep.recv();
        if (!in || std::holds_alternative<ShutdownMsg>(in->msg)) break;
        auto* wm = std::get_if<WeightsMsg>(&in->msg);
        WeightSet w;
        w.tensors = std::move(wm->tensors);
        w.version = wm->version;
        while (next < order.size() && order[next] != k) ++next;
        if (next >= order.size()) continue;  // no more turns: wait for SHUTDOWN
        const Batch b = make_batch(arch, k, j, B);
        ForwardResult fr = Api::forward(w, arch, b);
        Gradient g = Api::backward(w, arch, fr.cache, b.labels);
        while (turn.load() != next) std::this_thread::yield();  // replayed arrival
        ep.send(0, GradientMsg{std::move(g.tensors), g.basis_version, b.n_samples});
        ++next;
      }
      ep.close();
    });
  for (auto& t : th) t.join();
  for (auto& e : eps) {
    out.sent.push_back(e->messages_sent());
    out.recvd.push_back(e->messages_received());
  }
  return out;
}

int failures = 0;
void expect(bool ok, const char* what, double v) {
  std::printf("%-52s %s (%.3e)\n", what, ok ? "ok" : "FAIL", v);
  if (!ok) ++failures;
}
double rel(const WeightSet& a, const WeightSet& b) {
  double num = 0, den = 0;
  for (std::size_t t = 0; t < a.tensors.size(); ++t)
    for (std::size_t j = 0; j < a.tensors[t].values.size(); ++j) {
      const double d = a.tensors[t].values[j] - b.tensors[t].values[j];
      num += d * d;
      den += b.tensors[t].values[j] * b.tensors[t].values[j];
    }
  return std::sqrt(num / (den > 0 ? den : 1));
}
void compare(const char* tag, const Run& a, const Run& ref, double tol) {
  char buf[128];
  const double r = rel(a.w, ref.w);
  std::snprintf(buf, sizeof buf, "%s weights rel", tag);
  expect(tol == 0 ? r == 0.0 : r <= tol, buf, r);
  std::snprintf(buf, sizeof buf, "%s version / updates exact", tag);
  expect(a.w.version == ref.w.version && a.updates == ref.updates, buf, static_cast<double>(a.w.version));
  std::snprintf(buf, sizeof buf, "%s staleness exact", tag);
  expect(a.stale == ref.stale, buf, static_cast<double>(a.stale.size()));
  std::snprintf(buf, sizeof buf, "%s message counts exact", tag);
  expect(a.sent == ref.sent && a.recvd == ref.recvd, buf, static_cast<double>(a.sent.size()));
  double dl = 0;
  for (std::size_t i = 0; i < a.loss.size() && i < ref.loss.size(); ++i)
    dl = std::fmax(dl, std::fabs(a.loss[i] - ref.loss[i]) / ref.loss[i]);
  std::snprintf(buf, sizeof buf, "%s losses rel", tag);
  expect(a.loss.size() == ref.loss.size() && (tol == 0 ? dl == 0 : dl <= 1e-4), buf, dl);
}

}  // namespace

int main() {
  const Architecture arch = parse_architecture("lstm(5,20,10),softmax(20,3)");
  const int W = 4, R = 12;
  const std::size_t B = 64;
  for (WirePrecision wp : {WirePrecision::f32, WirePrecision::f64}) {
    const char* wn = wp == WirePrecision::f32 ? "f32" : "f64";
    std::printf("-- sync Downpour, %d workers, %d rounds, %s wire\n", W, R, wn);
    const Run ref = run_sync<RefApi>(arch, establish(Topology::flat(W), "inproc", wp), W, R, B);
    const Run xp = run_sync<RefApi>(arch, cuda::establish(Topology::flat(W), "nvlink", wp), W, R, B);
    compare("sync nvlink transport (reference math)", xp, ref, 0.0);
    if (wp == WirePrecision::f32) {
      const Run gpu = run_sync<CudaApi>(arch, cuda::establish(Topology::flat(W), "nvlink", wp), W, R, B);
      compare("sync nvlink + GPU math", gpu, ref, 1e-5);
    }
  }
  std::vector<int> order;
  {
    Rng r(99);
    for (int i = 0; i < 40; ++i) order.push_back(1 + static_cast<int>(r.below(W)));
  }
  std::printf("-- async Downpour, %d workers, %zu replayed arrivals\n", W, order.size());
  const Run ref = run_async<RefApi>(arch, establish(Topology::flat(W), "inproc"), W, order, B);
  const Run xp = run_async<RefApi>(arch, cuda::establish(Topology::flat(W), "nvlink"), W, order, B);
  compare("async nvlink transport (reference math)", xp, ref, 0.0);
  const Run gpu = run_async<CudaApi>(arch, cuda::establish(Topology::flat(W), "nvlink"), W, order, B);
  compare("async nvlink + GPU math", gpu, ref, 1e-5);
  std::uint64_t smax = 0;
  for (auto s : ref.stale) smax = std::max(smax, s);
  expect(smax > 0, "async replay produced staleness > 0", static_cast<double>(smax));

  // transport error semantics (transport.cpp:86-96)
  {
    auto eps = cuda::establish(Topology::flat(2), "nvlink");
    bool threw = false;
    try {
      eps[1]->send(7, DoneMsg{});
    } catch (const TransportError&) {
      threw = true;
    }
    expect(threw, "send to unknown rank -> TransportError", 0);
    eps[2]->close();
    threw = false;
    try {
      eps[1]->send(2, DoneMsg{});
    } catch (const TransportError&) {
      threw = true;
    }
    expect(threw, "send to closed rank -> TransportError", 0);
    eps[0]->close();
    eps[1]->close();
    expect(!eps[1]->recv().has_value(), "recv after every peer closed -> nullopt", 0);
  }
  // device-resident path: a payload sent from device memory arrives in the
  // receiver's device mailbox without a host copy
  {
    auto eps = cuda::establish(Topology::flat(1), "nvlink");
    auto* d0 = dynamic_cast<cuda::DeviceEndpoint*>(eps[0].get());
    auto* d1 = dynamic_cast<cuda::DeviceEndpoint*>(eps[1].get());
    const WeightSet w = init_weights(arch, 3);
    std::vector<float> h;
    for (const Tensor& t : w.tensors)
      for (double v : t.values) h.push_back(static_cast<float>(v));
    void* dsrc = nullptr;
    ghc_ctx* c = nullptr;  // the sender's device (rank 1 → device 1 mod count)
    ghc_ctx_create(d1->device(), &c);
    ghc_malloc(c, h.size() * 4, &dsrc);
    ghc_memcpy_h2d(c, dsrc, h.data(), h.size() * 4);
    ghc_ctx_sync(c);
    d1->send_device(0, 3, static_cast<const float*>(dsrc), h.size(), w.tensors, 5, 17);
    const float* dv = nullptr;
    std::size_t cnt = 0;
    auto in = d0->recv_device(&dv, &cnt);
    std::vector<float> back(cnt);
    ghc_ctx* c0 = nullptr;  // the receiver's device
    ghc_ctx_create(d0->device(), &c0);
    ghc_memcpy_d2h(c0, back.data(), dv, cnt * 4);
    ghc_ctx_sync(c0);
    ghc_ctx_destroy(c0);
    auto* g = in ? std::get_if<GradientMsg>(&in->msg) : nullptr;
    expect(g && g->basis_version == 5 && g->sample_count == 17 && back == h,
           "send_device / recv_device payload exact", static_cast<double>(cnt));
    ghc_free(c, dsrc);
    ghc_ctx_destroy(c);
    eps[0]->close();
    eps[1]->close();
  }
  std::printf(failures ? "ROLES FAIL\n" : "ROLES OK\n");
  return failures ? 1 : 0;
}
