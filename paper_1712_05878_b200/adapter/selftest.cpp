// selftest.cpp — drop-in check: the reference's own C++ API (gradhub::,
// compiled from /root/reference/proj/src) vs the GPU backend with the same
// signatures (gradhub::cuda::, this directory), on identical inputs.
// Prints one line per check and "ADAPTER OK" at the end; exit code 1 on a
// mismatch.  Run by tests/test_gpu_adapter.py on the GPU box.
#include <cmath>
#include <cstdio>

#include "gradhub/arch.hpp"
#include "gradhub/errors.hpp"
#include "gradhub/rng.hpp"
#include "gradhub_cuda.hpp"

using namespace gradhub;

static int failures = 0;

static double rel(const std::vector<Tensor>& a, const std::vector<Tensor>& b) {
  double num = 0, den = 0;
  for (size_t t = 0; t < a.size(); ++t)
    for (size_t j = 0; j < a[t].values.size(); ++j) {
      const double d = a[t].values[j] - b[t].values[j];
      num += d * d;
      den += b[t].values[j] * b[t].values[j];
    }
  return std::sqrt(num / (den > 0 ? den : 1));
}

static void expect(bool ok, const char* what, double v) {
  std::printf("%-44s %s (%.3e)\n", what, ok ? "ok" : "FAIL", v);
  if (!ok) ++failures;
}

int main() {
  const Architecture arch = parse_architecture("lstm(5,20,10),softmax(20,3)");
  // init_weights: bit-identical host draw (nn.cpp:83-98)
  const WeightSet w = init_weights(arch, 7);
  const WeightSet wc = cuda::init_weights(arch, 7);
  expect(rel(wc.tensors, w.tensors) == 0.0, "init_weights bit-identical", rel(wc.tensors, w.tensors));

  Batch b;
  b.n_samples = 500;
  Rng r(42);
  for (size_t i = 0; i < b.n_samples * arch.input_width(); ++i)
    b.inputs.push_back(static_cast<double>(static_cast<float>(2.0 * r.normal())));
  for (size_t i = 0; i < b.n_samples; ++i) b.labels.push_back(static_cast<int>(r.below(3)));
  // the device consumes f32 weights (the reference's f32 wire, proto.cpp:125)
  WeightSet w32 = w;
  for (Tensor& t : w32.tensors)
    for (double& v : t.values) v = static_cast<double>(static_cast<float>(v));

  const ForwardResult fr = forward(w32, arch, b);
  const ForwardResult fc = cuda::forward(w32, arch, b);
  double pd = 0;
  for (size_t i = 0; i < fr.probs.p.size(); ++i) pd = std::fmax(pd, std::fabs(fr.probs.p[i] - fc.probs.p[i]));
  expect(pd <= 2e-6, "forward probs max|dp|", pd);
  {  // the LSTM LayerCache (nn.hpp:15-23): gates, cell, tanh_c, hidden
    const LayerCache &a = fr.cache.layers[0], &c = fc.cache.layers[0];
    double m = 0;
    bool sized = a.gates.size() == c.gates.size() && a.cell.size() == c.cell.size() &&
                 a.tanh_c.size() == c.tanh_c.size() && a.hidden.size() == c.hidden.size();
    if (sized) {
      for (size_t i = 0; i < a.gates.size(); ++i) m = std::fmax(m, std::fabs(a.gates[i] - c.gates[i]));
      for (size_t i = 0; i < a.cell.size(); ++i) m = std::fmax(m, std::fabs(a.cell[i] - c.cell[i]));
      for (size_t i = 0; i < a.tanh_c.size(); ++i) m = std::fmax(m, std::fabs(a.tanh_c[i] - c.tanh_c[i]));
      for (size_t i = 0; i < a.hidden.size(); ++i) m = std::fmax(m, std::fabs(a.hidden[i] - c.hidden[i]));
    }
    expect(sized && m <= 2e-6, "forward LayerCache (gates/cell/tanh/hidden) max|d|", sized ? m : -1.0);
    const LayerCache &as = fr.cache.layers[1], &cs = fc.cache.layers[1];
    double ms = 0;
    for (size_t i = 0; i < as.x.size() && i < cs.x.size(); ++i) ms = std::fmax(ms, std::fabs(as.x[i] - cs.x[i]));
    expect(as.x.size() == cs.x.size() && ms <= 2e-6, "softmax layer input h_T max|d|", ms);
  }
  const double lr_ = loss(fr.probs, b.labels), lc = cuda::loss(fc.probs, b.labels);
  expect(std::fabs(lr_ - lc) / lr_ <= 1e-5, "loss rel", std::fabs(lr_ - lc) / lr_);

  const Gradient gr = backward(w32, arch, fr.cache, b.labels);
  const Gradient gc = cuda::backward(w32, arch, fc.cache, b.labels);
  expect(rel(gc.tensors, gr.tensors) <= 2e-5, "backward grad rel", rel(gc.tensors, gr.tensors));

  // stale cache → CacheMismatchError (nn.cpp:257-260)
  bool thrown = false;
  try {
    WeightSet w2 = w32;
    w2.version += 1;
    cuda::backward(w2, arch, fc.cache, b.labels);
  } catch (const CacheMismatchError&) {
    thrown = true;
  }
  expect(thrown, "stale cache -> CacheMismatchError", 0);
  // a value change below f32 resolution with the same version: the device
  // token hashes the f64 bits, like the reference's FNV checksum (nn.cpp:66-81)
  thrown = false;
  try {
    WeightSet w3 = w32;
    w3.tensors[2].values[5] = std::nextafter(w3.tensors[2].values[5], 1.0);
    cuda::backward(w3, arch, fc.cache, b.labels);
  } catch (const CacheMismatchError&) {
    thrown = true;
  }
  expect(thrown, "f64 value change -> CacheMismatchError", 0);
  // batch_loss: the fused forward's device loss sum (nn.hpp:68-69)
  const double bl = batch_loss(w32, arch, b), blc = cuda::batch_loss(w32, arch, b);
  expect(std::fabs(bl - blc) / bl <= 1e-5, "batch_loss rel", std::fabs(bl - blc) / bl);
  thrown = false;
  try {
    std::vector<int> bad_labels = b.labels;
    bad_labels[7] = 3;
    cuda::loss(fc.probs, bad_labels);
  } catch (const ShapeError&) {
    thrown = true;
  }
  expect(thrown, "loss label out of range -> ShapeError", 0);

  // sgd_step + serial training loop (optim.cpp:39-65)
  OptimState s = OptimState::for_weights(w32, 0.05, 0.9);
  OptimState sc = s;
  WeightSet wr = w32, wg = w32;
  for (int it = 0; it < 20; ++it) {
    Batch bb = b;
    const ForwardResult f1 = forward(wr, arch, bb);
    auto [nw, ns] = sgd_step(wr, backward(wr, arch, f1.cache, bb.labels), s);
    wr = nw;
    s = ns;
    const ForwardResult f2 = cuda::forward(wg, arch, bb);
    auto [ng, nsc] = cuda::sgd_step(wg, cuda::backward(wg, arch, f2.cache, bb.labels), sc);
    wg = ng;
    sc = nsc;
  }
  expect(wg.version == wr.version, "version after 20 steps", static_cast<double>(wg.version));
  expect(rel(wg.tensors, wr.tensors) <= 1e-5, "20 serial SGD steps w rel", rel(wg.tensors, wr.tensors));

  thrown = false;
  try {
    Gradient bad = gr;
    bad.tensors[1].values[3] = std::nan("");
    cuda::sgd_step(w32, bad, OptimState::for_weights(w32, 0.1, 0.0));
  } catch (const NonFiniteGradientError&) {
    thrown = true;
  }
  expect(thrown, "NaN gradient -> NonFiniteGradientError", 0);

  // EASGD (optim.cpp:67-123)
  ElasticConfig e;
  e.alpha = 0.5;
  e.tau = 10;
  const WeightSet ce = easgd_center_step(w32, wr, e), cc = cuda::easgd_center_step(w32, wr, e);
  expect(rel(cc.tensors, ce.tensors) <= 1e-6 && cc.version == ce.version, "easgd_center_step",
         rel(cc.tensors, ce.tensors));
  const WeightSet we = easgd_worker_step(wr, w32, gr, s, e, 20);
  const WeightSet wce = cuda::easgd_worker_step(wr, w32, gr, s, e, 20);
  expect(rel(wce.tensors, we.tensors) <= 1e-6, "easgd_worker_step (pull batch)", rel(wce.tensors, we.tensors));
  const WeightSet pe = elastic_pull(wr, w32, 0.25), pc = cuda::elastic_pull(wr, w32, 0.25);
  expect(rel(pc.tensors, pe.tensors) <= 1e-6, "elastic_pull", rel(pc.tensors, pe.tensors));

  thrown = false;
  try {
    ElasticConfig e1;
    e1.alpha = 1.0;
    cuda::easgd_center_step(w32, wr, e1);
  } catch (const ConfigError&) {
    thrown = true;
  }
  expect(thrown, "alpha = 1 -> ConfigError (optim.cpp:32)", 0);

  std::printf(failures ? "ADAPTER FAILED (%d)\n" : "ADAPTER OK\n", failures);
  return failures ? 1 : 0;
}
