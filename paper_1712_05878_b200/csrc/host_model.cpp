// host_model.cpp — see host_model.hpp.
#include "host_model.hpp"

#include <cctype>
#include <stdexcept>

namespace ghc {

namespace {

struct Cursor {
  const std::string& s;
  size_t pos = 0;
  void ws() {
    while (pos < s.size() && std::isspace(static_cast<unsigned char>(s[pos]))) ++pos;
  }
  bool eat(char c) {
    ws();
    if (pos < s.size() && s[pos] == c) {
      ++pos;
      return true;
    }
    return false;
  }
  std::string word() {
    ws();
    const size_t b = pos;
    while (pos < s.size() && (std::isalnum(static_cast<unsigned char>(s[pos])) || s[pos] == '_'))
      ++pos;
    return s.substr(b, pos - b);
  }
  int num() {
    ws();
    const size_t b = pos;
    long long v = 0;
    while (pos < s.size() && std::isdigit(static_cast<unsigned char>(s[pos]))) {
      v = v * 10 + (s[pos] - '0');
      if (v > 0x7fffffff) throw std::invalid_argument("architecture: number too large");
      ++pos;
    }
    if (pos == b) throw std::invalid_argument("architecture: expected number at " + std::to_string(b));
    return static_cast<int>(v);
  }
};

int out_of(const Layer& l) { return l.b; }
int in_of(const Layer& l) { return l.a; }

// arch.cpp:26-73 — LSTM only first, softmax exactly last, dims chain.
void validate(const std::vector<Layer>& L) {
  if (L.empty()) throw std::invalid_argument("architecture: no layers");
  for (size_t i = 0; i < L.size(); ++i) {
    const bool last = i + 1 == L.size();
    const std::string at = "architecture: layer " + std::to_string(i) + ": ";
    switch (L[i].kind) {
      case LayerKind::softmax:
        if (L[i].a < 1 || L[i].b < 1) throw std::invalid_argument(at + "softmax dims must be >= 1");
        if (!last) throw std::invalid_argument(at + "softmax output must be the last layer");
        break;
      case LayerKind::lstm:
        if (L[i].a < 1 || L[i].b < 1 || L[i].c < 1)
          throw std::invalid_argument(at + "lstm dims and seq_len must be >= 1");
        if (i != 0) throw std::invalid_argument(at + "lstm must be the first layer");
        break;
      case LayerKind::dense:
        if (L[i].a < 1 || L[i].b < 1) throw std::invalid_argument(at + "dense dims must be >= 1");
        if (last) throw std::invalid_argument("architecture: last layer must be a softmax output");
        break;
    }
    if (i > 0 && in_of(L[i]) != out_of(L[i - 1]))
      throw std::invalid_argument(at + "in dim does not chain with previous out dim");
  }
  if (L.back().kind != LayerKind::softmax)
    throw std::invalid_argument("architecture: last layer must be a softmax output");
}

}  // namespace

Model parse_model(const std::string& text) {
  Model m;
  Cursor p{text};
  for (;;) {
    const std::string kind = p.word();
    if (kind.empty()) throw std::invalid_argument("architecture: expected layer in '" + text + "'");
    if (!p.eat('(')) throw std::invalid_argument("architecture: expected '(' after " + kind);
    Layer l;
    if (kind == "dense") {
      l.kind = LayerKind::dense;
      l.a = p.num();
      if (!p.eat(',')) throw std::invalid_argument("architecture: dense needs 3 args");
      l.b = p.num();
      if (!p.eat(',')) throw std::invalid_argument("architecture: dense needs 3 args");
      const std::string act = p.word();
      if (act == "tanh") l.act = Act::tanh;
      else if (act == "relu") l.act = Act::relu;
      else if (act == "identity") l.act = Act::identity;
      else throw std::invalid_argument("architecture: unknown activation '" + act + "'");
    } else if (kind == "lstm") {
      l.kind = LayerKind::lstm;
      l.a = p.num();
      if (!p.eat(',')) throw std::invalid_argument("architecture: lstm needs 3 args");
      l.b = p.num();
      if (!p.eat(',')) throw std::invalid_argument("architecture: lstm needs 3 args");
      l.c = p.num();
    } else if (kind == "softmax") {
      l.kind = LayerKind::softmax;
      l.a = p.num();
      if (!p.eat(',')) throw std::invalid_argument("architecture: softmax needs 2 args");
      l.b = p.num();
    } else {
      throw std::invalid_argument("architecture: unknown layer kind '" + kind + "'");
    }
    if (!p.eat(')')) throw std::invalid_argument("architecture: expected ')'");
    m.layers.push_back(l);
    if (!p.eat(',')) break;
  }
  p.ws();
  if (p.pos != text.size())
    throw std::invalid_argument("architecture: trailing input at " + std::to_string(p.pos));
  validate(m.layers);
  int64_t off = 0;
  auto push = [&](int64_t d0, int64_t d1) {
    m.tensors.push_back({off, d0, d1});
    off += d0 * (d1 ? d1 : 1);
  };
  for (const Layer& l : m.layers) {
    if (l.kind == LayerKind::lstm) {
      push(4LL * l.b, l.a);
      push(4LL * l.b, l.b);
      push(4LL * l.b, 0);
    } else {
      push(l.b, l.a);
      push(l.b, 0);
    }
  }
  m.n_params = off;
  const Layer& f = m.layers.front();
  m.input_width = f.kind == LayerKind::lstm ? static_cast<int64_t>(f.a) * f.c : f.a;
  m.n_classes = m.layers.back().b;
  return m;
}

double HostRng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1 = uniform01();
  const double u2 = uniform01();
  while (u1 <= 0.0) u1 = uniform01();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
  spare_ = r * std::sin(th);
  has_spare_ = true;
  return r * std::cos(th);
}

uint64_t HostRng::below(uint64_t n) {
  if (n == 0) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x = gen_();
  while (x >= limit) x = gen_();
  return x % n;
}

uint64_t mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void init_weights(const Model& m, uint64_t seed, double* w) {
  for (size_t ti = 0; ti < m.tensors.size(); ++ti) {
    const TensorInfo& t = m.tensors[ti];
    const double fan_out = static_cast<double>(t.dim0);
    const double fan_in = t.dim1 ? static_cast<double>(t.dim1) : fan_out;
    const double bound = std::sqrt(6.0 / (fan_in + fan_out));
    HostRng r(mix_seed(seed, ti));
    for (int64_t j = 0; j < t.size(); ++j) w[t.offset + j] = r.uniform(-bound, bound);
  }
}

// ---- data layer: SPEC.md:416-481, generator formula per DESIGN.md ----
namespace {
constexpr uint64_t kMeanStream = 0x6d65616eULL;  // "mean"
constexpr uint64_t kFileStream = 0x66696c65ULL;  // "file"
}  // namespace

void generate_files(const DataSpec& s, int f0, int nf, float* x, int32_t* y) {
  const int64_t width = static_cast<int64_t>(s.seq_len) * s.input_dim;
  std::vector<double> means(static_cast<size_t>(s.n_classes * width));
  HostRng mr(mix_seed(s.seed, kMeanStream));
  for (double& v : means) v = mr.normal();
  for (int f = f0; f < f0 + nf; ++f) {
    HostRng fr(mix_seed(mix_seed(s.seed, kFileStream), static_cast<uint64_t>(f)));
    for (int i = 0; i < s.samples_per_file; ++i) {
      const int64_t row = static_cast<int64_t>(f - f0) * s.samples_per_file + i;
      const int lab = static_cast<int>((static_cast<int64_t>(i) + f) % s.n_classes);
      y[row] = lab;
      const double* mu = means.data() + static_cast<int64_t>(lab) * width;
      for (int64_t j = 0; j < width; ++j)
        x[row * width + j] = static_cast<float>(s.delta * mu[j] + fr.normal());
    }
  }
}

void shard_files(int n_files, int n_workers, int worker, int& f0, int& nf) {
  if (n_workers < 1 || worker < 0 || worker >= n_workers)
    throw std::invalid_argument("shard_files: bad worker index");
  if (n_files < n_workers)
    throw std::invalid_argument("shard_files: more workers than files; reduce workers");
  const int base = n_files / n_workers, extra = n_files % n_workers;
  nf = base + (worker < extra ? 1 : 0);
  f0 = worker * base + (worker < extra ? worker : extra);
}

std::vector<int64_t> epoch_indices(const DataSpec& s, int n_workers, int worker, int epoch,
                                   uint64_t shuffle_seed, bool shuffle) {
  int f0, nf;
  shard_files(s.n_files, n_workers, worker, f0, nf);
  std::vector<int64_t> idx(static_cast<size_t>(nf) * s.samples_per_file);
  for (size_t j = 0; j < idx.size(); ++j)
    idx[j] = static_cast<int64_t>(f0) * s.samples_per_file + static_cast<int64_t>(j);
  if (shuffle) {
    HostRng r(mix_seed(mix_seed(shuffle_seed, static_cast<uint64_t>(worker)),
                       static_cast<uint64_t>(epoch)));
    r.shuffle(idx);
  }
  return idx;
}

}  // namespace ghc
