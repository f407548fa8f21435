// host_model.hpp — host-side model/data layer of libghc (C++, no CUDA).
//
// The reference's Architecture grammar and validation (arch.cpp:26-73,
// 173-214), parameter layout (arch.cpp:95-112), deterministic init
// (nn.cpp:83-98 over rng.hpp:13-74) and the SPEC-only data layer
// (SPEC.md:416-481).  Bit-identical to the reference: std::mt19937_64 words
// with the reference's own 53-bit / Box–Muller / rejection constructions.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

namespace ghc {

enum class LayerKind { dense, lstm, softmax };
enum class Act { tanh = 0, relu = 1, identity = 2 };

struct Layer {
  LayerKind kind;
  int a = 0, b = 0, c = 0;  // dense(in,out), lstm(D,H,T), softmax(in,K)
  Act act = Act::tanh;
};

struct TensorInfo {
  int64_t offset, dim0, dim1;  // dim1 == 0 for 1-D
  int64_t size() const { return dim0 * (dim1 ? dim1 : 1); }
};

struct Model {
  std::vector<Layer> layers;
  std::vector<TensorInfo> tensors;
  int64_t n_params = 0;
  int64_t input_width = 0;
  int n_classes = 0;
};

// Throws std::invalid_argument with a ConfigError-style message.
Model parse_model(const std::string& text);

// Reference Rng semantics (rng.hpp:13-74).
class HostRng {
 public:
  explicit HostRng(uint64_t seed) : gen_(seed) {}
  uint64_t u64() { return gen_(); }
  double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  double normal();
  uint64_t below(uint64_t n);
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) {
      const size_t j = static_cast<size_t>(below(i));
      std::swap(v[i - 1], v[j]);
    }
  }

 private:
  std::mt19937_64 gen_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

uint64_t mix_seed(uint64_t a, uint64_t b);

void init_weights(const Model& m, uint64_t seed, double* w);

struct DataSpec {
  int32_t n_files, samples_per_file, seq_len, input_dim, n_classes, pad_;
  double delta;
  uint64_t seed;
};

void generate_files(const DataSpec& s, int f0, int nf, float* x, int32_t* y);
void shard_files(int n_files, int n_workers, int worker, int& f0, int& nf);
std::vector<int64_t> epoch_indices(const DataSpec& s, int n_workers, int worker, int epoch,
                                   uint64_t shuffle_seed, bool shuffle);

}  // namespace ghc
