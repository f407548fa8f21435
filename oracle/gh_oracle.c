/*
 * gh_oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see gh_oracle.h).
 *
 * Double-precision restatement of /root/reference/proj (gradhub) for the hot
 * path, written to reproduce the reference's floating-point operation order so
 * that results are bit-identical to the reference build in oracle/_ref (the
 * tests check this).  The SPEC-only layers (data, roles) follow SPEC.md and
 * the decisions recorded in DESIGN.md §"Oracle decisions".
 *
 * Never linked into the product.  Compile with -O2 -ffp-contract=off and no
 * -march flags (matches the reference build recipe in oracle/Makefile).
 */
#include "gh_oracle.h"

#include <ctype.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ====================================================================== */
/* rng.hpp:13-74 — mt19937_64 words, 53-bit uniforms, Box-Muller, below,   */
/* Fisher-Yates, splitmix64 seed mixing.                                   */
/* ====================================================================== */

#define MT_N 312
#define MT_M 156

void gho_rng_seed(gho_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    const uint64_t prev = r->mt[i - 1];
    r->mt[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

static void mt_twist(gho_rng* r) {
  static const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  static const uint64_t mag = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= mag;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->mti = 0;
}

uint64_t gho_rng_u64(gho_rng* r) {
  if (r->mti >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:21-23 */
double gho_rng_uniform01(gho_rng* r) {
  return (double)(gho_rng_u64(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:25 */
double gho_rng_uniform(gho_rng* r, double lo, double hi) {
  return lo + (hi - lo) * gho_rng_uniform01(r);
}

/* rng.hpp:27-40: the second draw happens before the u1 retry loop. */
double gho_rng_normal(gho_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = gho_rng_uniform01(r);
  const double u2 = gho_rng_uniform01(r);
  while (u1 <= 0.0) u1 = gho_rng_uniform01(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
  r->spare = rad * sin(theta);
  r->has_spare = 1;
  return rad * cos(theta);
}

/* rng.hpp:43-49 */
uint64_t gho_rng_below(gho_rng* r, uint64_t n) {
  if (n == 0) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x = gho_rng_u64(r);
  while (x >= limit) x = gho_rng_u64(r);
  return x % n;
}

/* rng.hpp:53-59 */
void gho_rng_shuffle_i64(gho_rng* r, int64_t* v, int64_t n) {
  for (int64_t i = n; i > 1; --i) {
    const int64_t j = (int64_t)gho_rng_below(r, (uint64_t)i);
    const int64_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

/* rng.hpp:68-74 */
uint64_t gho_mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* ====================================================================== */
/* arch.cpp                                                                */
/* ====================================================================== */

static int32_t layer_in(const gho_arch* a, int i) { return a->a[i]; }
static int32_t layer_out(const gho_arch* a, int i) {
  return a->kind[i] == GHO_DENSE ? a->b[i]
         : a->kind[i] == GHO_LSTM ? a->b[i]
                                  : a->b[i];
}

/* arch.cpp:26-73 */
int gho_arch_validate(const gho_arch* a) {
  if (a->n_layers < 1 || a->n_layers > GHO_MAX_LAYERS) return GHO_CONFIG;
  for (int i = 0; i < a->n_layers; ++i) {
    const int last = (i + 1 == a->n_layers);
    switch (a->kind[i]) {
      case GHO_SOFTMAX:
        if (a->a[i] < 1 || a->b[i] < 1 || !last) return GHO_CONFIG;
        break;
      case GHO_LSTM:
        if (a->a[i] < 1 || a->b[i] < 1 || a->c[i] < 1 || i != 0) return GHO_CONFIG;
        break;
      case GHO_DENSE:
        if (a->a[i] < 1 || a->b[i] < 1 || last) return GHO_CONFIG;
        if (a->c[i] < GHO_TANH || a->c[i] > GHO_IDENTITY) return GHO_CONFIG;
        break;
      default:
        return GHO_CONFIG;
    }
    if (i > 0 && layer_in(a, i) != layer_out(a, i - 1)) return GHO_CONFIG;
  }
  if (a->kind[a->n_layers - 1] != GHO_SOFTMAX) return GHO_CONFIG;
  return GHO_OK;
}

/* arch.cpp:75-81 */
int64_t gho_arch_input_width(const gho_arch* a) {
  if (a->kind[0] == GHO_LSTM) return (int64_t)a->a[0] * a->c[0];
  return a->a[0];
}

int32_t gho_arch_n_classes(const gho_arch* a) { return a->b[a->n_layers - 1]; }

/* arch.cpp:95-112: dense → W[out×in], b[out]; lstm → Wx[4H×D], Wh[4H×H],
 * b[4H]; softmax → W[K×in], b[K]. */
int gho_arch_tensors(const gho_arch* a, int64_t* offset, int64_t* size,
                     int64_t* dim0, int64_t* dim1, int cap) {
  int nt = 0;
  int64_t off = 0;
#define PUSH(d0, d1)                                   \
  do {                                                 \
    if (nt < cap) {                                    \
      offset[nt] = off;                                \
      dim0[nt] = (d0);                                 \
      dim1[nt] = (d1);                                 \
      size[nt] = (int64_t)(d0) * ((d1) ? (d1) : 1);    \
    }                                                  \
    off += (int64_t)(d0) * ((d1) ? (d1) : 1);          \
    ++nt;                                              \
  } while (0)
  for (int i = 0; i < a->n_layers; ++i) {
    if (a->kind[i] == GHO_LSTM) {
      const int64_t H = a->b[i], D = a->a[i];
      PUSH(4 * H, D);
      PUSH(4 * H, H);
      PUSH(4 * H, 0);
    } else {
      PUSH(a->b[i], a->a[i]);
      PUSH(a->b[i], 0);
    }
  }
#undef PUSH
  return nt;
}

int64_t gho_arch_n_params(const gho_arch* a) {
  int64_t off[3 * GHO_MAX_LAYERS], sz[3 * GHO_MAX_LAYERS], d0[3 * GHO_MAX_LAYERS],
      d1[3 * GHO_MAX_LAYERS];
  const int nt = gho_arch_tensors(a, off, sz, d0, d1, 3 * GHO_MAX_LAYERS);
  return off[nt - 1] + sz[nt - 1];
}

/* Grammar arch.hpp:54-57 / parser arch.cpp:173-214. */
typedef struct {
  const char* s;
  size_t pos;
} ps_t;

static void ps_ws(ps_t* p) {
  while (p->s[p->pos] && isspace((unsigned char)p->s[p->pos])) ++p->pos;
}
static int ps_eat(ps_t* p, char c) {
  ps_ws(p);
  if (p->s[p->pos] == c) {
    ++p->pos;
    return 1;
  }
  return 0;
}
static size_t ps_ident(ps_t* p, char* buf, size_t cap) {
  ps_ws(p);
  size_t n = 0;
  while (p->s[p->pos] && (isalnum((unsigned char)p->s[p->pos]) || p->s[p->pos] == '_')) {
    if (n + 1 < cap) buf[n++] = p->s[p->pos];
    ++p->pos;
  }
  buf[n] = 0;
  return n;
}
static int ps_num(ps_t* p, int32_t* out) {
  ps_ws(p);
  const size_t start = p->pos;
  long long v = 0;
  while (isdigit((unsigned char)p->s[p->pos])) {
    v = v * 10 + (p->s[p->pos] - '0');
    if (v > 0x7fffffff) return 0;
    ++p->pos;
  }
  if (p->pos == start) return 0;
  *out = (int32_t)v;
  return 1;
}

int gho_arch_parse(const char* text, gho_arch* out) {
  memset(out, 0, sizeof(*out));
  ps_t p = {text, 0};
  char kind[32];
  for (;;) {
    if (!ps_ident(&p, kind, sizeof kind)) return GHO_CONFIG;
    if (!ps_eat(&p, '(')) return GHO_CONFIG;
    const int i = out->n_layers;
    if (i >= GHO_MAX_LAYERS) return GHO_CONFIG;
    if (strcmp(kind, "dense") == 0) {
      char act[32];
      out->kind[i] = GHO_DENSE;
      if (!ps_num(&p, &out->a[i]) || !ps_eat(&p, ',') || !ps_num(&p, &out->b[i]) ||
          !ps_eat(&p, ','))
        return GHO_CONFIG;
      ps_ident(&p, act, sizeof act);
      if (strcmp(act, "tanh") == 0) out->c[i] = GHO_TANH;
      else if (strcmp(act, "relu") == 0) out->c[i] = GHO_RELU;
      else if (strcmp(act, "identity") == 0) out->c[i] = GHO_IDENTITY;
      else return GHO_CONFIG;
    } else if (strcmp(kind, "lstm") == 0) {
      out->kind[i] = GHO_LSTM;
      if (!ps_num(&p, &out->a[i]) || !ps_eat(&p, ',') || !ps_num(&p, &out->b[i]) ||
          !ps_eat(&p, ',') || !ps_num(&p, &out->c[i]))
        return GHO_CONFIG;
    } else if (strcmp(kind, "softmax") == 0) {
      out->kind[i] = GHO_SOFTMAX;
      if (!ps_num(&p, &out->a[i]) || !ps_eat(&p, ',') || !ps_num(&p, &out->b[i]))
        return GHO_CONFIG;
    } else {
      return GHO_CONFIG;
    }
    if (!ps_eat(&p, ')')) return GHO_CONFIG;
    out->n_layers = i + 1;
    if (!ps_eat(&p, ',')) break;
  }
  ps_ws(&p);
  if (p.s[p.pos] != 0) return GHO_CONFIG;
  return gho_arch_validate(out);
}

/* ====================================================================== */
/* nn.cpp                                                                  */
/* ====================================================================== */

/* nn.cpp:66-81: FNV-1a over (rank, dims, raw f64 bits) per tensor. */
uint64_t gho_weights_checksum(const gho_arch* a, const double* w) {
  int64_t off[48], sz[48], d0[48], d1[48];
  const int nt = gho_arch_tensors(a, off, sz, d0, d1, 48);
  uint64_t h = 1469598103934665603ULL;
#define MIX(val)                                          \
  do {                                                    \
    const uint64_t v_ = (uint64_t)(val);                  \
    for (int k_ = 0; k_ < 8; ++k_) {                      \
      h ^= (v_ >> (8 * k_)) & 0xff;                       \
      h *= 1099511628211ULL;                              \
    }                                                     \
  } while (0)
  for (int t = 0; t < nt; ++t) {
    MIX(d1[t] ? 2 : 1);
    MIX(d0[t]);
    if (d1[t]) MIX(d1[t]);
    for (int64_t j = 0; j < sz[t]; ++j) {
      uint64_t bits;
      memcpy(&bits, &w[off[t] + j], 8);
      MIX(bits);
    }
  }
#undef MIX
  return h;
}

/* nn.cpp:83-98: tensor ti drawn from Rng(mix_seed(seed, ti)) uniformly in
 * ±sqrt(6/(fan_in+fan_out)); fan_out = dims[0], fan_in = dims[1] or fan_out. */
void gho_init_weights(const gho_arch* a, uint64_t seed, double* w) {
  int64_t off[48], sz[48], d0[48], d1[48];
  const int nt = gho_arch_tensors(a, off, sz, d0, d1, 48);
  gho_rng r;
  for (int t = 0; t < nt; ++t) {
    const double fan_out = (double)d0[t];
    const double fan_in = d1[t] ? (double)d1[t] : fan_out;
    const double bound = sqrt(6.0 / (fan_in + fan_out));
    gho_rng_seed(&r, gho_mix_seed(seed, (uint64_t)t));
    for (int64_t j = 0; j < sz[t]; ++j) w[off[t] + j] = gho_rng_uniform(&r, -bound, bound);
  }
}

static double sigm(double v) { return 1.0 / (1.0 + exp(-v)); }

/* nn.cpp:17-24 */
static double act_fn(double z, int act) {
  if (act == GHO_TANH) return tanh(z);
  if (act == GHO_RELU) return z > 0.0 ? z : 0.0;
  return z;
}
/* nn.cpp:26-36 */
static double act_grad(double z, int act) {
  if (act == GHO_TANH) {
    const double t = tanh(z);
    return 1.0 - t * t;
  }
  if (act == GHO_RELU) return z > 0.0 ? 1.0 : 0.0;
  return 1.0;
}

typedef struct {
  double* x;      /* layer input */
  double* z;      /* dense preactivation */
  double* gates;  /* lstm n×T×4H */
  double* cell;   /* lstm n×T×H */
  double* tanh_c; /* lstm n×T×H */
  double* hidden; /* lstm n×T×H */
  double* probs;  /* softmax n×K */
} lcache;

int gho_forward_backward(const gho_arch* a, const double* w, const double* x,
                         const int32_t* y, int64_t n, double* grad,
                         double* probs, double* loss_out) {
  if (gho_arch_validate(a) != GHO_OK) return GHO_CONFIG;
  if (n < 1) return GHO_SHAPE; /* nn.cpp:104 */
  const int L = a->n_layers;
  const int32_t K = gho_arch_n_classes(a);
  for (int64_t s = 0; s < n; ++s)
    if (y[s] < 0 || y[s] >= K) return GHO_SHAPE; /* nn.cpp:241-244 */

  int64_t toff[48], tsz[48], td0[48], td1[48];
  gho_arch_tensors(a, toff, tsz, td0, td1, 48);

  lcache lc[GHO_MAX_LAYERS];
  memset(lc, 0, sizeof lc);

  /* ---------------- forward (nn.cpp:100-232) ---------------- */
  const int64_t width = gho_arch_input_width(a);
  double* cur = (double*)malloc(sizeof(double) * (size_t)(n * width));
  memcpy(cur, x, sizeof(double) * (size_t)(n * width));
  int ti = 0;
  for (int li = 0; li < L; ++li) {
    lc[li].x = cur; /* cache owns the layer input */
    if (a->kind[li] == GHO_DENSE) { /* nn.cpp:129-145 */
      const int64_t in = a->a[li], out = a->b[li];
      const double* W = w + toff[ti];
      const double* b = w + toff[ti + 1];
      ti += 2;
      lc[li].z = (double*)malloc(sizeof(double) * (size_t)(n * out));
      double* yv = (double*)malloc(sizeof(double) * (size_t)(n * out));
      for (int64_t s = 0; s < n; ++s) {
        const double* xs = cur + s * in;
        for (int64_t o = 0; o < out; ++o) {
          double acc = b[o];
          const double* Wr = W + o * in;
          for (int64_t i = 0; i < in; ++i) acc += Wr[i] * xs[i];
          lc[li].z[s * out + o] = acc;
          yv[s * out + o] = act_fn(acc, a->c[li]);
        }
      }
      cur = yv;
    } else if (a->kind[li] == GHO_LSTM) { /* nn.cpp:146-201 */
      const int64_t D = a->a[li], H = a->b[li], T = a->c[li];
      const double* Wx = w + toff[ti];
      const double* Wh = w + toff[ti + 1];
      const double* b = w + toff[ti + 2];
      ti += 3;
      lc[li].gates = (double*)calloc((size_t)(n * T * 4 * H), sizeof(double));
      lc[li].cell = (double*)calloc((size_t)(n * T * H), sizeof(double));
      lc[li].tanh_c = (double*)calloc((size_t)(n * T * H), sizeof(double));
      lc[li].hidden = (double*)calloc((size_t)(n * T * H), sizeof(double));
      double* yv = (double*)malloc(sizeof(double) * (size_t)(n * H));
      double* pre = (double*)malloc(sizeof(double) * (size_t)(4 * H));
      for (int64_t s = 0; s < n; ++s) {
        const double* seq = cur + s * T * D;
        for (int64_t t = 0; t < T; ++t) {
          const double* xt = seq + t * D;
          const double* hp = t > 0 ? lc[li].hidden + (s * T + t - 1) * H : NULL;
          const double* cp = t > 0 ? lc[li].cell + (s * T + t - 1) * H : NULL;
          for (int64_t r = 0; r < 4 * H; ++r) {
            double acc = b[r];
            for (int64_t d = 0; d < D; ++d) acc += Wx[r * D + d] * xt[d];
            if (hp)
              for (int64_t k = 0; k < H; ++k) acc += Wh[r * H + k] * hp[k];
            pre[r] = acc;
          }
          double* g = lc[li].gates + (s * T + t) * 4 * H;
          double* ct = lc[li].cell + (s * T + t) * H;
          double* tc = lc[li].tanh_c + (s * T + t) * H;
          double* ht = lc[li].hidden + (s * T + t) * H;
          for (int64_t k = 0; k < H; ++k) {
            const double ig = sigm(pre[k]);
            const double fg = sigm(pre[H + k]);
            const double gg = tanh(pre[2 * H + k]);
            const double og = sigm(pre[3 * H + k]);
            g[k] = ig;
            g[H + k] = fg;
            g[2 * H + k] = gg;
            g[3 * H + k] = og;
            const double cprev = cp ? cp[k] : 0.0;
            ct[k] = fg * cprev + ig * gg;
            tc[k] = tanh(ct[k]);
            ht[k] = og * tc[k];
          }
        }
        for (int64_t k = 0; k < H; ++k) yv[s * H + k] = lc[li].hidden[(s * T + T - 1) * H + k];
      }
      free(pre);
      cur = yv;
    } else { /* softmax nn.cpp:202-229 */
      const int64_t in = a->a[li];
      const double* W = w + toff[ti];
      const double* b = w + toff[ti + 1];
      ti += 2;
      lc[li].probs = (double*)malloc(sizeof(double) * (size_t)(n * K));
      double* z = (double*)malloc(sizeof(double) * (size_t)K);
      for (int64_t s = 0; s < n; ++s) {
        const double* xs = cur + s * in;
        double zmax = -1e300;
        for (int64_t k = 0; k < K; ++k) {
          double acc = b[k];
          for (int64_t i = 0; i < in; ++i) acc += W[k * in + i] * xs[i];
          z[k] = acc;
          zmax = zmax > acc ? zmax : acc;
        }
        double denom = 0.0;
        for (int64_t k = 0; k < K; ++k) denom += exp(z[k] - zmax);
        for (int64_t k = 0; k < K; ++k) lc[li].probs[s * K + k] = exp(z[k] - zmax) / denom;
      }
      free(z);
      /* `cur` (the softmax input) is owned by lc[li].x already */
    }
  }
  const double* P = lc[L - 1].probs;
  if (probs) memcpy(probs, P, sizeof(double) * (size_t)(n * K));

  /* loss nn.cpp:234-248 */
  if (loss_out) {
    double total = 0.0;
    for (int64_t s = 0; s < n; ++s) total += -log(P[s * K + y[s]]);
    *loss_out = total / (double)n;
  }

  /* ---------------- backward (nn.cpp:250-399) ---------------- */
  if (grad) {
    const int64_t np = gho_arch_n_params(a);
    memset(grad, 0, sizeof(double) * (size_t)np);
    double* dy = NULL;
    ti = 3 * GHO_MAX_LAYERS; /* unused sentinel */
    int tcur = 0;
    for (int li = 0; li < L; ++li) tcur += a->kind[li] == GHO_LSTM ? 3 : 2;
    for (int li = L - 1; li >= 0; --li) {
      const double* lx = lc[li].x;
      if (a->kind[li] == GHO_SOFTMAX) { /* nn.cpp:276-311 */
        tcur -= 2;
        const int64_t in = a->a[li];
        const double* W = w + toff[tcur];
        double* dW = grad + toff[tcur];
        double* db = grad + toff[tcur + 1];
        double* dz = (double*)malloc(sizeof(double) * (size_t)(n * K));
        const double inv_n = 1.0 / (double)n;
        for (int64_t s = 0; s < n; ++s)
          for (int64_t k = 0; k < K; ++k) {
            double v = P[s * K + k];
            if (k == y[s]) v -= 1.0;
            dz[s * K + k] = v * inv_n;
          }
        dy = (double*)calloc((size_t)(n * in), sizeof(double));
        for (int64_t s = 0; s < n; ++s) {
          const double* xs = lx + s * in;
          for (int64_t k = 0; k < K; ++k) {
            const double d = dz[s * K + k];
            db[k] += d;
            for (int64_t i = 0; i < in; ++i) {
              dW[k * in + i] += d * xs[i];
              dy[s * in + i] += W[k * in + i] * d;
            }
          }
        }
        free(dz);
      } else if (a->kind[li] == GHO_DENSE) { /* nn.cpp:312-334 */
        tcur -= 2;
        const int64_t in = a->a[li], out = a->b[li];
        const double* W = w + toff[tcur];
        double* dW = grad + toff[tcur];
        double* db = grad + toff[tcur + 1];
        double* dx = (double*)calloc((size_t)(n * in), sizeof(double));
        for (int64_t s = 0; s < n; ++s) {
          const double* xs = lx + s * in;
          for (int64_t o = 0; o < out; ++o) {
            const double d = dy[s * out + o] * act_grad(lc[li].z[s * out + o], a->c[li]);
            db[o] += d;
            for (int64_t i = 0; i < in; ++i) {
              dW[o * in + i] += d * xs[i];
              dx[s * in + i] += W[o * in + i] * d;
            }
          }
        }
        free(dy);
        dy = dx;
      } else { /* lstm BPTT nn.cpp:335-396 */
        tcur -= 3;
        const int64_t D = a->a[li], H = a->b[li], T = a->c[li];
        const double* Wh = w + toff[tcur + 1];
        double* dWx = grad + toff[tcur];
        double* dWh = grad + toff[tcur + 1];
        double* db = grad + toff[tcur + 2];
        double* dh = (double*)malloc(sizeof(double) * (size_t)H);
        double* dc = (double*)malloc(sizeof(double) * (size_t)H);
        double* dz = (double*)malloc(sizeof(double) * (size_t)(4 * H));
        double* dhp = (double*)malloc(sizeof(double) * (size_t)H);
        for (int64_t s = 0; s < n; ++s) {
          for (int64_t k = 0; k < H; ++k) {
            dh[k] = dy[s * H + k];
            dc[k] = 0.0;
          }
          for (int64_t t = T - 1; t >= 0; --t) {
            const double* g = lc[li].gates + (s * T + t) * 4 * H;
            const double* tc = lc[li].tanh_c + (s * T + t) * H;
            const double* cp = t > 0 ? lc[li].cell + (s * T + t - 1) * H : NULL;
            const double* hp = t > 0 ? lc[li].hidden + (s * T + t - 1) * H : NULL;
            const double* xt = lx + (s * T + t) * D;
            for (int64_t k = 0; k < H; ++k) {
              const double ig = g[k], fg = g[H + k], gg = g[2 * H + k], og = g[3 * H + k];
              const double dout = dh[k] * tc[k];
              dc[k] += dh[k] * og * (1.0 - tc[k] * tc[k]);
              const double di = dc[k] * gg;
              const double dg = dc[k] * ig;
              const double df = dc[k] * (cp ? cp[k] : 0.0);
              dz[k] = di * ig * (1.0 - ig);
              dz[H + k] = df * fg * (1.0 - fg);
              dz[2 * H + k] = dg * (1.0 - gg * gg);
              dz[3 * H + k] = dout * og * (1.0 - og);
            }
            for (int64_t r = 0; r < 4 * H; ++r) {
              const double d = dz[r];
              db[r] += d;
              for (int64_t q = 0; q < D; ++q) dWx[r * D + q] += d * xt[q];
              if (hp)
                for (int64_t k = 0; k < H; ++k) dWh[r * H + k] += d * hp[k];
            }
            for (int64_t k = 0; k < H; ++k) dhp[k] = 0.0;
            for (int64_t r = 0; r < 4 * H; ++r) {
              const double d = dz[r];
              for (int64_t k = 0; k < H; ++k) dhp[k] += Wh[r * H + k] * d;
            }
            for (int64_t k = 0; k < H; ++k) {
              dh[k] = dhp[k];
              dc[k] *= g[H + k];
            }
          }
        }
        free(dh);
        free(dc);
        free(dz);
        free(dhp);
        free(dy);
        dy = NULL;
      }
    }
    free(dy);
  }

  for (int li = 0; li < L; ++li) {
    free(lc[li].x);
    free(lc[li].z);
    free(lc[li].gates);
    free(lc[li].cell);
    free(lc[li].tanh_c);
    free(lc[li].hidden);
    free(lc[li].probs);
  }
  return GHO_OK;
}

/* nn.cpp:407-426 */
/* validate — SPEC.md:376-384 (no reference code: the roles are SPEC-only). */
int gho_validate(const gho_arch* a, const double* w, const double* x, const int32_t* y,
                 int64_t n, int64_t* correct, double* loss_mean) {
  if (n < 1) return GHO_CONFIG;
  const int32_t K = gho_arch_n_classes(a);
  double* probs = (double*)malloc(sizeof(double) * (size_t)n * (size_t)K);
  if (!probs) return GHO_CONFIG;
  int rc = gho_forward_backward(a, w, x, y, n, NULL, probs, loss_mean);
  if (rc == GHO_OK) {
    int64_t ok = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double* p = probs + i * K;
      int32_t best = 0;
      for (int32_t k = 1; k < K; ++k)
        if (p[k] > p[best]) best = k;  /* strict: ties keep the lowest index */
      ok += best == y[i];
    }
    *correct = ok;
  }
  free(probs);
  return rc;
}

int gho_finite_diff(const gho_arch* a, const double* w, const double* x,
                    const int32_t* y, int64_t n, double eps, double* grad) {
  if (!(eps > 0.0)) return GHO_CONFIG;
  const int64_t np = gho_arch_n_params(a);
  double* probe = (double*)malloc(sizeof(double) * (size_t)np);
  memcpy(probe, w, sizeof(double) * (size_t)np);
  int rc = GHO_OK;
  for (int64_t j = 0; j < np && rc == GHO_OK; ++j) {
    const double saved = probe[j];
    double lp = 0.0, lm = 0.0;
    probe[j] = saved + eps;
    rc = gho_forward_backward(a, probe, x, y, n, NULL, NULL, &lp);
    probe[j] = saved - eps;
    if (rc == GHO_OK) rc = gho_forward_backward(a, probe, x, y, n, NULL, NULL, &lm);
    probe[j] = saved;
    grad[j] = (lp - lm) / (2.0 * eps);
  }
  free(probe);
  return rc;
}

/* ====================================================================== */
/* optim.cpp                                                               */
/* ====================================================================== */

static int all_finite(const double* g, int64_t p) { /* tensor.cpp:29-36 */
  for (int64_t j = 0; j < p; ++j)
    if (!isfinite(g[j])) return 0;
  return 1;
}

/* optim.cpp:20-29 + 39-65.  On NONFINITE nothing is modified. */
int gho_sgd_step(double* w, double* v, const double* g, int64_t p, double lr,
                 double mu) {
  if (!(lr > 0.0)) return GHO_CONFIG;
  if (!(mu >= 0.0 && mu < 1.0)) return GHO_CONFIG;
  if (!all_finite(g, p)) return GHO_NONFINITE;
  for (int64_t j = 0; j < p; ++j) {
    v[j] = mu * v[j] - lr * g[j];
    w[j] += v[j];
  }
  return GHO_OK;
}

/* optim.cpp:67-80 */
void gho_elastic_pull(double* w, const double* center, int64_t p, double alpha) {
  for (int64_t j = 0; j < p; ++j) w[j] -= alpha * (w[j] - center[j]);
}

static int elastic_validate(double alpha, uint64_t tau) { /* optim.cpp:31-37 */
  if (!(alpha > 0.0 && alpha < 1.0)) return GHO_CONFIG;
  if (tau < 1) return GHO_CONFIG;
  return GHO_OK;
}

/* optim.cpp:82-105 */
int gho_easgd_worker_step(double* w, const double* center, const double* g,
                          int64_t p, double lr, double alpha, uint64_t tau,
                          uint64_t batch_index) {
  if (!(lr > 0.0)) return GHO_CONFIG;
  if (elastic_validate(alpha, tau) != GHO_OK) return GHO_CONFIG;
  if (!all_finite(g, p)) return GHO_NONFINITE;
  for (int64_t j = 0; j < p; ++j) w[j] -= lr * g[j];
  if (batch_index % tau == 0) gho_elastic_pull(w, center, p, alpha);
  return GHO_OK;
}

/* optim.cpp:107-123 */
int gho_easgd_center_step(double* c, const double* worker, int64_t p,
                          double alpha) {
  if (elastic_validate(alpha, 1) != GHO_OK) return GHO_CONFIG;
  for (int64_t j = 0; j < p; ++j) c[j] += alpha * (worker[j] - c[j]);
  return GHO_OK;
}

/* proto.cpp:125 (f64→f32 round-to-nearest) then proto.cpp:79 (widen). */
void gho_wire_round(double* dst, const double* src, int64_t p, int wire_f64) {
  if (wire_f64) {
    if (dst != src) memmove(dst, src, sizeof(double) * (size_t)p);
    return;
  }
  for (int64_t j = 0; j < p; ++j) dst[j] = (double)(float)src[j];
}

/* ====================================================================== */
/* data.  Generator formula: DESIGN.md "Data layer".     */
/* ====================================================================== */

#define GHO_MEAN_STREAM 0x6d65616eULL /* "mean" */
#define GHO_FILE_STREAM 0x66696c65ULL /* "file" */

static void class_means(const gho_data_spec* s, double* means) {
  gho_rng r;
  gho_rng_seed(&r, gho_mix_seed(s->seed, GHO_MEAN_STREAM));
  const int64_t m = (int64_t)s->n_classes * s->seq_len * s->input_dim;
  for (int64_t j = 0; j < m; ++j) means[j] = gho_rng_normal(&r);
}

void gho_generate_files(const gho_data_spec* s, int32_t f0, int32_t nf,
                        double* x, int32_t* y) {
  const int64_t width = (int64_t)s->seq_len * s->input_dim;
  double* means = (double*)malloc(sizeof(double) * (size_t)(s->n_classes * width));
  class_means(s, means);
  gho_rng r;
  for (int32_t f = f0; f < f0 + nf; ++f) {
    gho_rng_seed(&r, gho_mix_seed(gho_mix_seed(s->seed, GHO_FILE_STREAM), (uint64_t)f));
    for (int32_t i = 0; i < s->samples_per_file; ++i) {
      const int64_t row = (int64_t)(f - f0) * s->samples_per_file + i;
      const int32_t lab = (int32_t)(((int64_t)i + f) % s->n_classes);
      y[row] = lab;
      const double* m = means + (int64_t)lab * width;
      for (int64_t j = 0; j < width; ++j) {
        const double v = s->delta * m[j] + gho_rng_normal(&r);
        x[row * width + j] = (double)(float)v; /* files hold f32 */
      }
    }
  }
  free(means);
}

void gho_generate(const gho_data_spec* s, double* x, int32_t* y) {
  gho_generate_files(s, 0, s->n_files, x, y);
}

/* contiguous blocks in rank order, sizes differ by ≤1,
 * the first (n_files mod W) workers get the extra file. */
int gho_shard_files(int32_t n_files, int32_t n_workers, int32_t worker,
                    int32_t* first_file, int32_t* n_files_out) {
  if (n_workers < 1 || worker < 0 || worker >= n_workers) return GHO_CONFIG;
  if (n_files < n_workers) return GHO_CONFIG;
  const int32_t base = n_files / n_workers, extra = n_files % n_workers;
  *n_files_out = base + (worker < extra ? 1 : 0);
  *first_file = worker * base + (worker < extra ? worker : extra);
  return GHO_OK;
}

/* SPEC.md:449-457 with Appendix-A decision 3: the epoch permutation of the
 * worker's shard is Rng(mix_seed(mix_seed(shuffle_seed, worker), epoch)). */
int64_t gho_epoch_indices(const gho_data_spec* s, int32_t n_workers,
                          int32_t worker, int32_t epoch, uint64_t shuffle_seed,
                          int32_t shuffle, int64_t* out) {
  int32_t f0 = 0, nf = 0;
  if (gho_shard_files(s->n_files, n_workers, worker, &f0, &nf) != GHO_OK) return -1;
  const int64_t cnt = (int64_t)nf * s->samples_per_file;
  for (int64_t j = 0; j < cnt; ++j) out[j] = (int64_t)f0 * s->samples_per_file + j;
  if (shuffle) {
    gho_rng r;
    gho_rng_seed(&r, gho_mix_seed(gho_mix_seed(shuffle_seed, (uint64_t)worker), (uint64_t)epoch));
    gho_rng_shuffle_i64(&r, out, cnt);
  }
  return cnt;
}

/* ====================================================================== */
/* roles                                                 */
/* ====================================================================== */

/* Per-worker batch cursor: epochs × ceil(shard/B) batches. */
typedef struct {
  int32_t worker;
  int32_t epoch;
  int64_t pos;
  int64_t count;
  int64_t* idx;
  int32_t done;
} cursor_t;

static void cursor_init(cursor_t* c, const gho_data_spec* s,
                        const gho_train_cfg* cfg, int32_t worker) {
  int32_t f0, nf;
  gho_shard_files(s->n_files, cfg->n_workers, worker, &f0, &nf);
  c->worker = worker;
  c->epoch = 0;
  c->pos = 0;
  c->idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)((int64_t)nf * s->samples_per_file));
  c->count = gho_epoch_indices(s, cfg->n_workers, worker, 0, cfg->shuffle_seed,
                               cfg->shuffle, c->idx);
  c->done = cfg->epochs < 1;
}

/* Gathers the next batch into xb/yb; returns its sample_count (0 = DONE). */
static int64_t cursor_next(cursor_t* c, const gho_data_spec* s,
                           const gho_train_cfg* cfg, const double* x,
                           const int32_t* y, double* xb, int32_t* yb) {
  if (c->done) return 0;
  const int64_t width = (int64_t)s->seq_len * s->input_dim;
  int64_t nb = c->count - c->pos;
  if (nb > cfg->batch_size) nb = cfg->batch_size;
  for (int64_t j = 0; j < nb; ++j) {
    const int64_t g = c->idx[c->pos + j];
    memcpy(xb + j * width, x + g * width, sizeof(double) * (size_t)width);
    yb[j] = y[g];
  }
  c->pos += nb;
  if (c->pos >= c->count) {
    c->epoch += 1;
    if (c->epoch >= cfg->epochs) {
      c->done = 1;
    } else {
      c->count = gho_epoch_indices(s, cfg->n_workers, c->worker, c->epoch,
                                   cfg->shuffle_seed, cfg->shuffle, c->idx);
      c->pos = 0;
    }
  }
  return nb;
}

static int check_cfg(const gho_arch* a, const gho_data_spec* s,
                     const gho_train_cfg* cfg) {
  if (gho_arch_validate(a) != GHO_OK) return GHO_CONFIG;
  if (cfg->n_workers < 1 || cfg->batch_size < 1) return GHO_CONFIG;
  if (s->n_files < cfg->n_workers) return GHO_CONFIG;
  if (gho_arch_input_width(a) != (int64_t)s->seq_len * s->input_dim) return GHO_SHAPE;
  if (gho_arch_n_classes(a) != s->n_classes) return GHO_SHAPE;
  if (!(cfg->lr > 0.0) || !(cfg->mu >= 0.0 && cfg->mu < 1.0)) return GHO_CONFIG;
  return GHO_OK;
}

/* Synchronous Downpour.  Each round: every active worker computes its
 * gradient on the broadcast weights (wire-rounded), sends it wire-rounded
 * with its sample count; the master forms Σ c_i g_i / Σ c_i in worker
 * (rank) order, applies sgd_step and broadcasts.  DONE workers drop out
 * (SPEC.md:327).  A non-finite combined gradient is rejected and the
 * current weights are re-sent. */
int gho_run_sync(const gho_arch* a, const gho_data_spec* s, const double* x,
                 const int32_t* y, const gho_train_cfg* cfg, double* w_out,
                 double* v_out, double* loss_trace, gho_run_stats* st) {
  int rc = check_cfg(a, s, cfg);
  if (rc != GHO_OK) return rc;
  const int32_t W = cfg->n_workers;
  const int64_t P = gho_arch_n_params(a);
  const int64_t width = gho_arch_input_width(a);
  double* w = w_out;
  double* v = v_out;
  gho_init_weights(a, cfg->weight_seed, w);
  memset(v, 0, sizeof(double) * (size_t)P);
  double* ww = (double*)malloc(sizeof(double) * (size_t)P);   /* broadcast copy */
  double* g = (double*)malloc(sizeof(double) * (size_t)P);
  double* acc = (double*)malloc(sizeof(double) * (size_t)P);
  double* xb = (double*)malloc(sizeof(double) * (size_t)(cfg->batch_size * width));
  int32_t* yb = (int32_t*)malloc(sizeof(int32_t) * (size_t)cfg->batch_size);
  cursor_t* cur = (cursor_t*)calloc((size_t)W, sizeof(cursor_t));
  for (int32_t k = 0; k < W; ++k) cursor_init(&cur[k], s, cfg, k);
  gho_run_stats stats = {0, 0, 0, 0};
  uint64_t version = 0;
  gho_wire_round(ww, w, P, cfg->wire_f64);
  for (int64_t round = 0;; ++round) {
    if (cfg->max_updates > 0 && round >= cfg->max_updates) break;
    memset(acc, 0, sizeof(double) * (size_t)P);
    double total = 0.0, wloss = 0.0;
    int any = 0;
    for (int32_t k = 0; k < W; ++k) {
      const int64_t nb = cursor_next(&cur[k], s, cfg, x, y, xb, yb);
      if (nb == 0) continue;
      any = 1;
      double lo = 0.0;
      rc = gho_forward_backward(a, ww, xb, yb, nb, g, NULL, &lo);
      if (rc != GHO_OK) goto out;
      gho_wire_round(g, g, P, cfg->wire_f64);
      const double c = (double)nb;
      for (int64_t j = 0; j < P; ++j) acc[j] += c * g[j];
      total += c;
      wloss += c * lo;
    }
    if (!any) break;
    for (int64_t j = 0; j < P; ++j) acc[j] = acc[j] / total;
    if (loss_trace) loss_trace[round] = wloss / total;
    rc = gho_sgd_step(w, v, acc, P, cfg->lr, cfg->mu);
    if (rc == GHO_OK) {
      ++version;
      ++stats.updates;
      stats.samples += (int64_t)total;
    } else if (rc == GHO_NONFINITE) {
      ++stats.rejected;
      rc = GHO_OK;
    } else {
      goto out;
    }
    gho_wire_round(ww, w, P, cfg->wire_f64);
  }
out:
  stats.version = version;
  if (st) *st = stats;
  for (int32_t k = 0; k < W; ++k) free(cur[k].idx);
  free(cur);
  free(ww);
  free(g);
  free(acc);
  free(xb);
  free(yb);
  return rc;
}

int gho_run_replay(const gho_arch* a, const gho_data_spec* s, const double* x,
                   const int32_t* y, const gho_train_cfg* cfg,
                   const int32_t* order, int64_t n_order, double* w_out,
                   double* v_out, double* worker_w, int64_t* staleness,
                   double* loss_trace, gho_run_stats* st) {
  int rc = check_cfg(a, s, cfg);
  if (rc != GHO_OK) return rc;
  if (cfg->algo == GHO_EASGD && elastic_validate(cfg->alpha, (uint64_t)cfg->tau) != GHO_OK)
    return GHO_CONFIG;
  const int32_t W = cfg->n_workers;
  const int64_t P = gho_arch_n_params(a);
  const int64_t width = gho_arch_input_width(a);
  double* w = w_out; /* master weights (Downpour) or center (EASGD) */
  double* v = v_out;
  gho_init_weights(a, cfg->weight_seed, w);
  memset(v, 0, sizeof(double) * (size_t)P);
  double* lw = (double*)malloc(sizeof(double) * (size_t)(P * W)); /* worker-local weights */
  uint64_t* basis = (uint64_t*)calloc((size_t)W, sizeof(uint64_t));
  uint64_t* bidx = (uint64_t*)calloc((size_t)W, sizeof(uint64_t));
  double* g = (double*)malloc(sizeof(double) * (size_t)P);
  double* msg = (double*)malloc(sizeof(double) * (size_t)P);
  double* xb = (double*)malloc(sizeof(double) * (size_t)(cfg->batch_size * width));
  int32_t* yb = (int32_t*)malloc(sizeof(int32_t) * (size_t)cfg->batch_size);
  cursor_t* cur = (cursor_t*)calloc((size_t)W, sizeof(cursor_t));
  for (int32_t k = 0; k < W; ++k) {
    cursor_init(&cur[k], s, cfg, k);
    gho_wire_round(lw + (int64_t)k * P, w, P, cfg->wire_f64); /* initial WEIGHTS */
  }
  gho_run_stats stats = {0, 0, 0, 0};
  uint64_t version = 0;
  for (int64_t step = 0; step < n_order; ++step) {
    const int32_t k = order[step];
    if (k < 0 || k >= W) {
      rc = GHO_PROTOCOL;
      goto out;
    }
    const int64_t nb = cursor_next(&cur[k], s, cfg, x, y, xb, yb);
    if (nb == 0) { /* the worker already sent DONE */
      rc = GHO_PROTOCOL;
      goto out;
    }
    double* mine = lw + (int64_t)k * P;
    double lo = 0.0;
    rc = gho_forward_backward(a, mine, xb, yb, nb, g, NULL, &lo);
    if (rc != GHO_OK) goto out;
    if (loss_trace) loss_trace[step] = lo;
    if (cfg->algo == GHO_DOWNPOUR) {
      /* GRADIENT up, sgd_step, WEIGHTS to sender. */
      gho_wire_round(msg, g, P, cfg->wire_f64);
      if (staleness) staleness[step] = (int64_t)(version - basis[k]);
      rc = gho_sgd_step(w, v, msg, P, cfg->lr, cfg->mu);
      if (rc == GHO_OK) {
        ++version;
        ++stats.updates;
        stats.samples += nb;
      } else if (rc == GHO_NONFINITE) {
        ++stats.rejected;
        rc = GHO_OK;
      } else {
        goto out;
      }
      gho_wire_round(mine, w, P, cfg->wire_f64);
      basis[k] = version;
    } else {
      /* EASGD (optim.cpp:82-123; DESIGN.md ordering): local step w1 = w - ηg;
       * on batch_index % tau == 0 the worker sends w1, the master applies
       * the center step and replies with the UPDATED center c', and the
       * worker pulls toward c' — gap factor (1-α)^2. */
      if (!all_finite(g, P)) {
        rc = GHO_NONFINITE;
        goto out;
      }
      const uint64_t bi = bidx[k]++;
      if (bi % (uint64_t)cfg->tau == 0) {
        for (int64_t j = 0; j < P; ++j) msg[j] = mine[j];
        for (int64_t j = 0; j < P; ++j) msg[j] -= cfg->lr * g[j]; /* optim.cpp:97-98 */
        gho_wire_round(msg, msg, P, cfg->wire_f64);
        gho_easgd_center_step(w, msg, P, cfg->alpha);
        ++version;
        ++stats.updates;
        if (staleness) staleness[step] = (int64_t)(version - 1 - basis[k]);
        gho_wire_round(msg, w, P, cfg->wire_f64);
        basis[k] = version;
        rc = gho_easgd_worker_step(mine, msg, g, P, cfg->lr, cfg->alpha,
                                   (uint64_t)cfg->tau, bi);
      } else {
        if (staleness) staleness[step] = 0;
        rc = gho_easgd_worker_step(mine, w /*unused*/, g, P, cfg->lr, cfg->alpha,
                                   (uint64_t)cfg->tau, bi);
      }
      stats.samples += nb;
      if (rc != GHO_OK) goto out;
    }
  }
out:
  stats.version = version;
  if (st) *st = stats;
  if (worker_w) memcpy(worker_w, lw, sizeof(double) * (size_t)(P * W));
  for (int32_t k = 0; k < W; ++k) free(cur[k].idx);
  free(cur);
  free(lw);
  free(basis);
  free(bidx);
  free(g);
  free(msg);
  free(xb);
  free(yb);
  return rc;
}

int gho_run_hier(const gho_arch* a, const gho_data_spec* s, const double* x,
                 const int32_t* y, const gho_train_cfg* cfg, double* w_out,
                 double* group_w_out, double* loss_trace, gho_run_stats* st) {
  int rc = check_cfg(a, s, cfg);
  if (rc != GHO_OK) return rc;
  const int32_t G = cfg->groups, W = cfg->n_workers;
  if (G < 1 || W % G != 0 || cfg->flush_k < 1) return GHO_CONFIG;
  if (!(cfg->parent_lr > 0.0) || !(cfg->parent_mu >= 0.0 && cfg->parent_mu < 1.0))
    return GHO_CONFIG;
  const int32_t Wg = W / G;
  const int64_t P = gho_arch_n_params(a);
  const int64_t width = gho_arch_input_width(a);
  double* top = w_out;
  double* vtop = (double*)calloc((size_t)P, sizeof(double));
  gho_init_weights(a, cfg->weight_seed, top);
  double* gw = (double*)malloc(sizeof(double) * (size_t)(P * G));   /* group weights */
  double* gv = (double*)calloc((size_t)(P * G), sizeof(double));    /* group velocity */
  double* snap = (double*)malloc(sizeof(double) * (size_t)(P * G)); /* flush snapshot */
  double* pseudo = (double*)malloc(sizeof(double) * (size_t)(P * G));
  int64_t* absorbed = (int64_t*)calloc((size_t)G, sizeof(int64_t));
  int64_t* since = (int64_t*)calloc((size_t)G, sizeof(int64_t));
  int32_t* flushing = (int32_t*)calloc((size_t)G, sizeof(int32_t));
  double* ww = (double*)malloc(sizeof(double) * (size_t)P);
  double* g = (double*)malloc(sizeof(double) * (size_t)P);
  double* acc = (double*)malloc(sizeof(double) * (size_t)P);
  double* xb = (double*)malloc(sizeof(double) * (size_t)(cfg->batch_size * width));
  int32_t* yb = (int32_t*)malloc(sizeof(int32_t) * (size_t)cfg->batch_size);
  cursor_t* cur = (cursor_t*)calloc((size_t)W, sizeof(cursor_t));
  for (int32_t k = 0; k < W; ++k) cursor_init(&cur[k], s, cfg, k);
  for (int32_t q = 0; q < G; ++q) {
    gho_wire_round(gw + (int64_t)q * P, top, P, cfg->wire_f64);
    memcpy(snap + (int64_t)q * P, gw + (int64_t)q * P, sizeof(double) * (size_t)P);
  }
  gho_run_stats stats = {0, 0, 0, 0};
  uint64_t version = 0;
  for (int64_t round = 0;; ++round) {
    if (cfg->max_updates > 0 && round >= cfg->max_updates) break;
    int any_group = 0;
    double rl = 0.0, rc_tot = 0.0;
    for (int32_t q = 0; q < G; ++q) {
      double* wq = gw + (int64_t)q * P;
      flushing[q] = 0;
      memset(acc, 0, sizeof(double) * (size_t)P);
      double total = 0.0;
      int any = 0;
      gho_wire_round(ww, wq, P, cfg->wire_f64);
      for (int32_t j = 0; j < Wg; ++j) {
        const int32_t k = q * Wg + j;
        const int64_t nb = cursor_next(&cur[k], s, cfg, x, y, xb, yb);
        if (nb == 0) continue;
        any = 1;
        double lo = 0.0;
        rc = gho_forward_backward(a, ww, xb, yb, nb, g, NULL, &lo);
        if (rc != GHO_OK) goto out;
        gho_wire_round(g, g, P, cfg->wire_f64);
        const double c = (double)nb;
        for (int64_t p = 0; p < P; ++p) acc[p] += c * g[p];
        total += c;
        rl += c * lo;
        rc_tot += c;
      }
      if (!any) {
        if (absorbed[q] > 0) flushing[q] = 1; /* final flush of a finished group */
        continue;
      }
      any_group = 1;
      for (int64_t p = 0; p < P; ++p) acc[p] = acc[p] / total;
      rc = gho_sgd_step(wq, gv + (int64_t)q * P, acc, P, cfg->lr, cfg->mu);
      if (rc == GHO_OK) {
        absorbed[q] += (int64_t)total;
        since[q] += 1;
      } else if (rc == GHO_NONFINITE) {
        ++stats.rejected;
        rc = GHO_OK;
      } else {
        goto out;
      }
      if (since[q] >= cfg->flush_k) flushing[q] = 1;
    }
    if (loss_trace && rc_tot > 0) loss_trace[round] = rl / rc_tot;
    /* Top master: synchronous combine over the flushing groups, group order. */
    int nflush = 0;
    for (int32_t q = 0; q < G; ++q) nflush += flushing[q];
    if (nflush > 0) {
      memset(acc, 0, sizeof(double) * (size_t)P);
      double total = 0.0;
      for (int32_t q = 0; q < G; ++q) {
        if (!flushing[q]) continue;
        double* ps = pseudo + (int64_t)q * P;
        for (int64_t p = 0; p < P; ++p) ps[p] = snap[(int64_t)q * P + p] - gw[(int64_t)q * P + p];
        gho_wire_round(ps, ps, P, cfg->wire_f64);
        const double c = (double)absorbed[q];
        for (int64_t p = 0; p < P; ++p) acc[p] += c * ps[p];
        total += c;
      }
      for (int64_t p = 0; p < P; ++p) acc[p] = acc[p] / total;
      rc = gho_sgd_step(top, vtop, acc, P, cfg->parent_lr, cfg->parent_mu);
      if (rc == GHO_OK) {
        ++version;
        ++stats.updates;
        stats.samples += (int64_t)total;
      } else if (rc == GHO_NONFINITE) {
        ++stats.rejected;
        rc = GHO_OK;
      } else {
        goto out;
      }
      for (int32_t q = 0; q < G; ++q) {
        if (!flushing[q]) continue;
        gho_wire_round(gw + (int64_t)q * P, top, P, cfg->wire_f64);
        memcpy(snap + (int64_t)q * P, gw + (int64_t)q * P, sizeof(double) * (size_t)P);
        absorbed[q] = 0;
        since[q] = 0;
      }
    }
    if (!any_group) break;
  }
out:
  stats.version = version;
  if (st) *st = stats;
  if (group_w_out) memcpy(group_w_out, gw, sizeof(double) * (size_t)(P * G));
  for (int32_t k = 0; k < W; ++k) free(cur[k].idx);
  free(cur);
  free(vtop);
  free(gw);
  free(gv);
  free(snap);
  free(pseudo);
  free(absorbed);
  free(since);
  free(flushing);
  free(ww);
  free(g);
  free(acc);
  free(xb);
  free(yb);
  return rc;
}

/* ==================================================================== */
/* proto.cpp frames — restated (encode proto.cpp:214-272, decode 288-386) */
/* ==================================================================== */
#define GHO_MAX_T 64
static void le_put(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t le_get(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

int64_t gho_frame_size(const gho_arch* a, int kind, int wire_f64) {
  if (kind == 0) return 15;
  int64_t off[GHO_MAX_T], sz[GHO_MAX_T], d0[GHO_MAX_T], d1[GHO_MAX_T];
  const int nt = gho_arch_tensors(a, off, sz, d0, d1, GHO_MAX_T);
  const int64_t es = wire_f64 ? 8 : 4;
  int64_t block = 4;
  for (int t = 0; t < nt; ++t) block += 1 + 4 * (d1[t] ? 2 : 1) + es * sz[t];
  return 15 + (kind == 1 ? 8 : 16) + block;
}

int gho_encode_frame(const gho_arch* a, int kind, const double* w, uint64_t version,
                     uint64_t sample_count, int wire_f64, uint8_t* out, int64_t cap,
                     int64_t* len) {
  if (kind < 0 || kind > 2) return GHO_CONFIG;
  if (kind == 2 && sample_count < 1) return GHO_CONFIG; /* proto.cpp:231-233 */
  const int64_t n = gho_frame_size(a, kind, wire_f64);
  *len = n;
  if (n > cap) return GHO_SHAPE;
  uint8_t type = kind == 0 ? 0x06 : (kind == 1 ? 0x02 : 0x03);
  if (kind != 0 && wire_f64) type |= 0x40;
  uint8_t* p = out;
  p[0] = 'G'; p[1] = 'H'; p[2] = 'U'; p[3] = 'B';
  le_put(p + 4, 1, 2);
  p[6] = type;
  le_put(p + 7, (uint64_t)(n - 15), 8);
  p += 15;
  if (kind == 0) return GHO_OK;
  le_put(p, version, 8);
  p += 8;
  if (kind == 2) {
    le_put(p, sample_count, 8);
    p += 8;
  }
  int64_t off[GHO_MAX_T], sz[GHO_MAX_T], d0[GHO_MAX_T], d1[GHO_MAX_T];
  const int nt = gho_arch_tensors(a, off, sz, d0, d1, GHO_MAX_T);
  le_put(p, (uint64_t)nt, 4);
  p += 4;
  for (int t = 0; t < nt; ++t) {
    const int rank = d1[t] ? 2 : 1;
    *p++ = (uint8_t)rank;
    le_put(p, (uint64_t)d0[t], 4);
    p += 4;
    if (rank == 2) {
      le_put(p, (uint64_t)d1[t], 4);
      p += 4;
    }
    for (int64_t i = 0; i < sz[t]; ++i) {
      const double v = w[off[t] + i];
      if (wire_f64) {
        uint64_t b;
        memcpy(&b, &v, 8);
        le_put(p, b, 8);
        p += 8;
      } else {
        const float f = (float)v;
        uint32_t b;
        memcpy(&b, &f, 4);
        le_put(p, b, 4);
        p += 4;
      }
    }
  }
  return GHO_OK;
}

int gho_decode_frame(const gho_arch* a, const uint8_t* in, int64_t len, int* kind, double* w,
                     uint64_t* version, uint64_t* sample_count, int* wire_f64, int* status) {
  *status = 0;
  if (len < 4) { *status = 3; return GHO_PROTOCOL; }
  if (memcmp(in, "GHUB", 4) != 0) { *status = 1; return GHO_PROTOCOL; }
  if (len < 15) { *status = 3; return GHO_PROTOCOL; }
  if (le_get(in + 4, 2) != 1) { *status = 2; return GHO_PROTOCOL; }
  const uint8_t type = in[6], base = type & (uint8_t)~0x40;
  const int f64 = (type & 0x40) != 0;
  if (!(base >= 0x01 && base <= 0x06) || (f64 && base != 0x02 && base != 0x03)) {
    *status = 5;
    return GHO_PROTOCOL;
  }
  const uint64_t plen = le_get(in + 7, 8);
  if (plen > (1ull << 40)) { *status = 4; return GHO_PROTOCOL; }
  if (plen > (uint64_t)(len - 15)) { *status = 3; return GHO_PROTOCOL; }
  const uint8_t* p = in + 15;
  uint64_t rem = plen;
#define NEED(n) do { if (rem < (uint64_t)(n)) { *status = 6; return GHO_PROTOCOL; } } while (0)
  *wire_f64 = f64;
  if (base != 0x02 && base != 0x03) {
    /* HELLO/VALIDATE_RESULT/DONE/SHUTDOWN: not parameter frames */
    *kind = base == 0x06 ? 0 : -(int)base;
    const uint64_t want = base == 0x01 ? 5 : base == 0x04 ? 24 : base == 0x05 ? 4 : 0;
    if (rem != want) { *status = 6; return GHO_PROTOCOL; }
    return GHO_OK;
  }
  *kind = base == 0x02 ? 1 : 2;
  NEED(8);
  *version = le_get(p, 8); p += 8; rem -= 8;
  *sample_count = 0;
  if (base == 0x03) {
    NEED(8);
    *sample_count = le_get(p, 8); p += 8; rem -= 8;
    if (*sample_count < 1) { *status = 6; return GHO_PROTOCOL; }
  }
  NEED(4);
  const uint64_t count = le_get(p, 4); p += 4; rem -= 4;
  if (count > rem) { *status = 6; return GHO_PROTOCOL; }
  int64_t off[GHO_MAX_T], sz[GHO_MAX_T], d0[GHO_MAX_T], d1[GHO_MAX_T];
  const int nt = gho_arch_tensors(a, off, sz, d0, d1, GHO_MAX_T);
  int shape_ok = (int64_t)count == nt;
  const int es = f64 ? 8 : 4;
  for (uint64_t t = 0; t < count; ++t) {
    NEED(1);
    const int rank = *p++; rem -= 1;
    if (rank == 0) { *status = 6; return GHO_PROTOCOL; }
    uint64_t elems = 1, dims[2] = {0, 0};
    for (int r = 0; r < rank; ++r) {
      NEED(4);
      const uint64_t d = le_get(p, 4); p += 4; rem -= 4;
      if (d == 0) { *status = 6; return GHO_PROTOCOL; }
      if (r < 2) dims[r] = d;
      if (elems > (1ull << 40) / d) { *status = 6; return GHO_PROTOCOL; }
      elems *= d;
    }
    if (elems * (uint64_t)es > rem) { *status = 6; return GHO_PROTOCOL; }
    if (shape_ok && (int)t < nt) {
      const int want_rank = d1[t] ? 2 : 1;
      shape_ok = rank == want_rank && (int64_t)dims[0] == d0[t] &&
                 (want_rank == 1 || (int64_t)dims[1] == d1[t]);
    }
    for (uint64_t i = 0; i < elems; ++i) {
      double v;
      if (f64) {
        const uint64_t b = le_get(p, 8);
        memcpy(&v, &b, 8);
      } else {
        const uint32_t b = (uint32_t)le_get(p, 4);
        float f;
        memcpy(&f, &b, 4);
        v = (double)f;
      }
      if (shape_ok && w) w[off[t] + (int64_t)i] = v;
      p += es;
      rem -= (uint64_t)es;
    }
  }
#undef NEED
  if (rem != 0) { *status = 6; return GHO_PROTOCOL; }
  return shape_ok ? GHO_OK : GHO_SHAPE;
}
