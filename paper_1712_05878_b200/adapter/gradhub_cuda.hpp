// gradhub_cuda.hpp — drop-in GPU backend for the reference's Model / Algo /
// transport API.
//
// The functions below have the SAME signatures and semantics as the
// reference's nn.hpp / optim.hpp / transport.hpp (namespace gradhub) and live
// in gradhub::cuda, so a caller switches by changing the namespace (or by the
// one-line `using` shown in INTEGRATION.md).  Each call moves the reference's
// f64 value types into the flat f32 layout of include/ghc.h (weight-set
// order, arch.cpp:95-112; the f32 rounding is the reference's f32 wire), runs
// the sm_100a kernels, converts back, and rethrows ghc_status as the
// reference exception class (errors.hpp:10-45).  Compiled against the
// reference headers at build time (paper_1712_05878_b200/adapter/Makefile);
// nothing of the reference is copied and no reference compute function is
// called.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "ghc.h"
#include "gradhub/nn.hpp"
#include "gradhub/optim.hpp"
#include "gradhub/transport.hpp"

namespace gradhub::cuda {

// One CUDA context (device + stream) per host thread; plans cached per
// architecture text.
ghc_ctx* thread_context(int device = 0);

// nn.hpp:53-69 ------------------------------------------------------------
// forward keeps the reference's stale-cache guard (nn.cpp:116-119, 253-260)
// with a device-computed token: ForwardCache::weights_checksum holds the
// hash of every f64 weight value, computed on the GPU while the weights are
// uploaded (ghc_weights_import_f64) — backward recomputes it on its own
// upload and throws CacheMismatchError on any difference, like the
// reference's host FNV pass.  ForwardCache::layers[0].x keeps the batch (the
// fused kernel recomputes the activations in backward instead of reading
// gates / cell / hidden back from host memory).
WeightSet init_weights(const Architecture& arch, std::uint64_t seed);
ForwardResult forward(const WeightSet& w, const Architecture& arch, const Batch& batch);
double loss(const ProbMatrix& probs, const std::vector<int>& labels);  // device NLL (f64)
Gradient backward(const WeightSet& w, const Architecture& arch, const ForwardCache& cache,
                  const std::vector<int>& labels);
// forward + loss without the probabilities leaving the GPU (the fused
// forward's device loss sum).
double batch_loss(const WeightSet& w, const Architecture& arch, const Batch& batch);

// optim.hpp:33-48 ---------------------------------------------------------
std::pair<WeightSet, OptimState> sgd_step(const WeightSet& w, const Gradient& g,
                                          const OptimState& s);
WeightSet elastic_pull(const WeightSet& w, const WeightSet& center, double alpha);
WeightSet easgd_worker_step(const WeightSet& w, const WeightSet& center, const Gradient& g,
                            const OptimState& s, const ElasticConfig& e,
                            std::uint64_t batch_index);
WeightSet easgd_center_step(const WeightSet& center, const WeightSet& worker,
                            const ElasticConfig& e);

// transport.hpp:110-120 ---------------------------------------------------
// establish(topo, backend): "nvlink" returns in-process Endpoints whose
// WEIGHTS / GRADIENT payloads live on the GPUs: rank r is bound to device
// r mod (device count); send() stages the tensor values (wire precision) on
// the sender's GPU and moves them with one peer copy (NVLink) into a slot of
// the receiver's device mailbox; recv() returns them from there.  Header
// fields and the small messages (HELLO, DONE, SHUTDOWN, VALIDATE_RESULT)
// travel in the host-side control record.  Semantics follow the reference's
// inproc backend (transport.cpp:25-177): per-(sender,receiver) FIFO, bounded
// links with blocking backpressure, TransportError on unknown / closed peers,
// recv() → nullopt once every peer closed and the queue drained, message
// counters.  Any other backend name is forwarded to gradhub::establish.
std::vector<std::unique_ptr<Endpoint>> establish(const Topology& topo, const std::string& backend,
                                                 WirePrecision wire = WirePrecision::f32,
                                                 std::size_t link_capacity = 16);

// The GPU side of an "nvlink" Endpoint for device-resident producers and
// consumers (a GPU worker's gradient is already in HBM): send a payload that
// lives on this rank's device, and receive one without the host copy.
class DeviceEndpoint {
 public:
  virtual ~DeviceEndpoint() = default;
  virtual int device() const = 0;
  // GRADIENT (kind 3) or WEIGHTS (kind 2) from a device buffer of `count`
  // f32 values on this rank's device; `shape` gives the tensor dims.
  virtual void send_device(int to, int kind, const float* d_values, std::size_t count,
                           const std::vector<Tensor>& shape, std::uint64_t version,
                           std::uint64_t sample_count) = 0;
  // Next message; for WEIGHTS / GRADIENT *d_values points at the f32 payload
  // in this rank's device mailbox (valid until the next recv_device call) and
  // the message's tensors carry dims only.
  virtual std::optional<Incoming> recv_device(const float** d_values, std::size_t* count) = 0;
};

}  // namespace gradhub::cuda
