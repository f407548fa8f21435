// gradhub_cuda.hpp — drop-in GPU backend for the reference's Model / Algo API.
//
// The functions below have the SAME signatures and semantics as the
// reference's nn.hpp / optim.hpp (namespace gradhub) and live in
// gradhub::cuda, so a caller switches by changing the namespace (or by the
// one-line `using` shown in INTEGRATION.md).  Each call converts the
// reference's f64 value types to the flat f32 layout of include/ghc.h
// (weight-set order, arch.cpp:95-112), runs the sm_100a kernels, converts
// back, and rethrows ghc_status as the reference exception class
// (errors.hpp:10-45).  Compiled against the reference headers at build time
// (paper_1712_05878_b200/adapter/Makefile); nothing of the reference is copied.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "ghc.h"
#include "gradhub/nn.hpp"
#include "gradhub/optim.hpp"

namespace gradhub::cuda {

// One CUDA context (device + stream) per host thread; plans cached per
// architecture text.
ghc_ctx* thread_context(int device = 0);

// nn.hpp:53-65 ------------------------------------------------------------
WeightSet init_weights(const Architecture& arch, std::uint64_t seed);
ForwardResult forward(const WeightSet& w, const Architecture& arch, const Batch& batch);
double loss(const ProbMatrix& probs, const std::vector<int>& labels);
Gradient backward(const WeightSet& w, const Architecture& arch, const ForwardCache& cache,
                  const std::vector<int>& labels);

// optim.hpp:33-48 ---------------------------------------------------------
std::pair<WeightSet, OptimState> sgd_step(const WeightSet& w, const Gradient& g,
                                          const OptimState& s);
WeightSet elastic_pull(const WeightSet& w, const WeightSet& center, double alpha);
WeightSet easgd_worker_step(const WeightSet& w, const WeightSet& center, const Gradient& g,
                            const OptimState& s, const ElasticConfig& e,
                            std::uint64_t batch_index);
WeightSet easgd_center_step(const WeightSet& center, const WeightSet& worker,
                            const ElasticConfig& e);

}  // namespace gradhub::cuda
