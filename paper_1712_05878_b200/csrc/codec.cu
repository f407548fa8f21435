// codec.cu — GHUB wire frames on the device.
//
// The reference encodes every WEIGHTS / GRADIENT message byte by byte on the
// host (proto.cpp:214-272, decode 288-386).  For a multi-node / TCP transport
// the frame of a 16.9 M-parameter gradient is 67.5 MB (f32) — an HBM-bound
// byte-shuffling job, done here where the parameters already live:
//
//   pack:   one thread per ALIGNED 16-byte chunk of the output frame; value
//           bytes start at arbitrary byte offsets (15-byte header, 1-byte
//           ranks), so each chunk is assembled from ≤ 5 source words with
//           funnel shifts and written with one 16-byte store (coalesced);
//           the few chunks that touch header bytes take a bytewise path.
//   unpack: one thread per value, two/three aligned 32-bit loads + funnel
//           shift; the header is parsed and validated on the host first with
//           the reference's DecodeStatus taxonomy.
//
// Layout (little-endian): "GHUB" | u16 format 1 | u8 type (0x02 WEIGHTS,
// 0x03 GRADIENT, | 0x40 for f64 values, 0x06 SHUTDOWN) | u64 payload length |
// WEIGHTS: u64 version | GRADIENT: u64 basis_version, u64 sample_count |
// u32 tensor count | per tensor: u8 rank, u32 dims[rank], values.
#include "ghc_internal.cuh"

namespace {

constexpr int kMaxT = 16;       // parameter tensors of an arch (5 for the bench net)
constexpr int kHdrMax = 256;    // header bytes of a frame (fixed part + tensor headers)

struct FrameMap {
  long long total;              // frame bytes
  int es;                       // value bytes: 4 (f32) or 8 (f64)
  int nt;                       // tensors
  long long dst[kMaxT];         // byte offset of tensor t's first value
  long long src[kMaxT];         // parameter offset of tensor t
  long long n[kMaxT];           // values of tensor t
  int hdr_len;                  // header bytes (all non-value bytes, in order)
  long long hdr_dst[kMaxT + 1]; // frame offset of header piece i
  int hdr_off[kMaxT + 2];       // piece i = hdr[hdr_off[i] .. hdr_off[i+1])
  unsigned char hdr[kHdrMax];
};

void put_le(unsigned char* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

ghc_status build_map(const ghc_plan* p, int kind, int f64, uint64_t version, uint64_t count,
                     FrameMap& m) {
  if (kind < 0 || kind > 2) return fail(GHC_ERR_CONFIG, "frame kind must be 0 (SHUTDOWN), 1 (WEIGHTS) or 2 (GRADIENT)");
  if (kind == 2 && count < 1) return fail(GHC_ERR_CONFIG, "GRADIENT sample_count must be >= 1");
  int64_t off[kMaxT], d0[kMaxT], d1[kMaxT];
  int nt = 0;
  if (ghc_status s = ghc_plan_tensors(p, off, d0, d1, kMaxT, &nt)) return s;
  if (nt > kMaxT) return fail(GHC_ERR_CONFIG, "frame: too many tensors");
  m = FrameMap{};
  m.es = f64 ? 8 : 4;
  unsigned char* h = m.hdr;
  int hl = 0;
  long long pos = 0;
  auto piece = [&](int i) {  // start header piece i at frame offset pos
    m.hdr_dst[i] = pos;
    m.hdr_off[i] = hl;
  };
  piece(0);
  unsigned char type = kind == 0 ? 0x06 : (kind == 1 ? 0x02 : 0x03);
  if (kind != 0 && f64) type |= 0x40;
  h[0] = 'G'; h[1] = 'H'; h[2] = 'U'; h[3] = 'B';
  put_le(h + 4, 1, 2);
  h[6] = type;
  hl = 15;  // payload length patched below
  if (kind != 0) {
    put_le(h + hl, version, 8);
    hl += 8;
    if (kind == 2) {
      put_le(h + hl, count, 8);
      hl += 8;
    }
    put_le(h + hl, static_cast<uint64_t>(nt), 4);
    hl += 4;
  }
  pos = hl;
  m.nt = kind == 0 ? 0 : nt;
  for (int t = 0; t < m.nt; ++t) {
    if (t > 0) piece(t);
    const int rank = d1[t] ? 2 : 1;
    const int start = hl;
    h[hl++] = static_cast<unsigned char>(rank);
    put_le(h + hl, static_cast<uint64_t>(d0[t]), 4);
    hl += 4;
    if (rank == 2) {
      put_le(h + hl, static_cast<uint64_t>(d1[t]), 4);
      hl += 4;
    }
    pos += hl - start;
    m.dst[t] = pos;
    m.src[t] = off[t];
    m.n[t] = d0[t] * (d1[t] ? d1[t] : 1);
    pos += m.n[t] * m.es;
  }
  m.hdr_off[m.nt > 0 ? m.nt : 1] = hl;
  m.hdr_len = hl;
  m.total = pos;
  put_le(h + 7, static_cast<uint64_t>(pos - 15), 8);
  return GHC_OK;
}

__device__ __forceinline__ unsigned frame_byte(const FrameMap& m, const float* __restrict__ w,
                                               long long b) {
  for (int t = 0; t < m.nt; ++t) {
    const long long lo = m.dst[t], hi = lo + m.n[t] * m.es;
    if (b >= lo && b < hi) {
      const long long k = (b - lo) / m.es;
      const int o = static_cast<int>((b - lo) % m.es);
      const float v = __ldg(w + m.src[t] + k);
      const unsigned long long bits =
          m.es == 8 ? static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(v)))
                    : __float_as_uint(v);
      return static_cast<unsigned>((bits >> (8 * o)) & 0xff);
    }
  }
  // header byte: piece i covers [hdr_dst[i], hdr_dst[i] + len_i)
  const int np = m.nt > 0 ? m.nt : 1;
  for (int i = 0; i < np; ++i) {
    const long long lo = m.hdr_dst[i];
    const int len = m.hdr_off[i + 1] - m.hdr_off[i];
    if (b >= lo && b < lo + len) return m.hdr[m.hdr_off[i] + (b - lo)];
  }
  return 0;
}

// 32-bit word j of the value stream of tensor t (f64: low/high halves)
__device__ __forceinline__ unsigned value_word(const FrameMap& m, const float* __restrict__ w, int t,
                                               long long j) {
  if (m.es == 4) return __float_as_uint(__ldg(w + m.src[t] + j));
  const double d = static_cast<double>(__ldg(w + m.src[t] + (j >> 1)));
  const long long bits = __double_as_longlong(d);
  return (j & 1) ? static_cast<unsigned>(bits >> 32) : static_cast<unsigned>(bits);
}

__global__ void pack_frame_kernel(const FrameMap m, const float* __restrict__ w,
                                  unsigned char* __restrict__ out) {
  const long long nchunk = (m.total + 15) / 16;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunk;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c0 = c * 16;
    int seg = -1;
    for (int t = 0; t < m.nt; ++t)
      if (c0 >= m.dst[t] && c0 + 16 <= m.dst[t] + m.n[t] * m.es) seg = t;
    if (seg >= 0) {  // whole chunk inside one tensor's values: funnel-shifted words
      const long long b = c0 - m.dst[seg];
      const long long j0 = b >> 2;
      const int r = static_cast<int>(b & 3);
      const long long nw = m.n[seg] * (m.es / 4);
      unsigned wd[5];
      const long long a = j0 & ~3LL;  // f32: two aligned 16-B loads cover words j0..j0+4
      if (m.es == 4 && ((m.src[seg] + a) & 3) == 0 && a + 8 <= nw) {
        const uint4* q = reinterpret_cast<const uint4*>(w + m.src[seg] + a);
        const uint4 q0 = __ldg(q), q1 = __ldg(q + 1);
        const unsigned v8[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        switch (static_cast<int>(j0 - a)) {  // static register indices per case
          case 0: wd[0] = v8[0]; wd[1] = v8[1]; wd[2] = v8[2]; wd[3] = v8[3]; wd[4] = v8[4]; break;
          case 1: wd[0] = v8[1]; wd[1] = v8[2]; wd[2] = v8[3]; wd[3] = v8[4]; wd[4] = v8[5]; break;
          case 2: wd[0] = v8[2]; wd[1] = v8[3]; wd[2] = v8[4]; wd[3] = v8[5]; wd[4] = v8[6]; break;
          default: wd[0] = v8[3]; wd[1] = v8[4]; wd[2] = v8[5]; wd[3] = v8[6]; wd[4] = v8[7]; break;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 5; ++k) wd[k] = (k < 4 || r) && j0 + k < nw ? value_word(m, w, seg, j0 + k) : 0u;
      }
      uint4 o;
      o.x = r ? __funnelshift_r(wd[0], wd[1], 8 * r) : wd[0];
      o.y = r ? __funnelshift_r(wd[1], wd[2], 8 * r) : wd[1];
      o.z = r ? __funnelshift_r(wd[2], wd[3], 8 * r) : wd[2];
      o.w = r ? __funnelshift_r(wd[3], wd[4], 8 * r) : wd[3];
      reinterpret_cast<uint4*>(out + c0)[0] = o;
    } else {  // header bytes / segment edges / frame tail: bytewise
      for (int i = 0; i < 16 && c0 + i < m.total; ++i)
        out[c0 + i] = static_cast<unsigned char>(frame_byte(m, w, c0 + i));
    }
  }
}

__global__ void unpack_frame_kernel(const FrameMap m, const unsigned char* __restrict__ in,
                                    long long len, float* __restrict__ w) {
  long long total = 0;
  for (int t = 0; t < m.nt; ++t) total += m.n[t];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int t = 0;
    long long k = i;
    while (k >= m.n[t]) k -= m.n[t++];
    const long long b = m.dst[t] + k * m.es;
    const long long a0 = b & ~3LL;
    const int r = static_cast<int>(b & 3);
    const int words = m.es / 4 + (r ? 1 : 0);
    unsigned wd[3];
    if (a0 + 4 * words <= len) {
#pragma unroll
      for (int q = 0; q < 3; ++q)
        wd[q] = q < words ? __ldg(reinterpret_cast<const unsigned*>(in + a0) + q) : 0u;
    } else {  // last value of the frame: never read past its end
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        unsigned v = 0;
        for (int y = 0; y < 4; ++y) {
          const long long p = a0 + 4 * q + y;
          if (p < len) v |= static_cast<unsigned>(in[p]) << (8 * y);
        }
        wd[q] = v;
      }
    }
    const unsigned lo = r ? __funnelshift_r(wd[0], wd[1], 8 * r) : wd[0];
    float v;
    if (m.es == 4) {
      v = __uint_as_float(lo);
    } else {
      const unsigned hi = r ? __funnelshift_r(wd[1], wd[2], 8 * r) : wd[1];
      v = __double2float_rn(__longlong_as_double(
          static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo)));
    }
    w[m.src[t] + k] = v;
  }
}

const char* decode_name(int s) {
  static const char* names[] = {"ok",        "bad magic",       "unsupported format version",
                                "truncated frame", "payload length overflow",
                                "unknown message type", "malformed payload"};
  return s >= 0 && s <= 6 ? names[s] : "?";
}

int grid_for(ghc_ctx* c, long long work) {
  const long long g = (work + 255) / 256;
  const long long cap = 8LL * c->num_sms;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

ghc_status ghc_frame_size(const ghc_plan* p, int32_t kind, int32_t wire_f64, int64_t* bytes) {
  FrameMap m;
  if (ghc_status s = build_map(p, kind, wire_f64, 0, 1, m)) return s;
  if (bytes) *bytes = m.total;
  return GHC_OK;
}

ghc_status ghc_encode_frame(ghc_plan* p, int32_t kind, int32_t wire_f64, const float* d_w,
                            uint64_t version, uint64_t sample_count, uint8_t* d_out, int64_t cap,
                            int64_t* len) {
  FrameMap m;
  if (ghc_status s = build_map(p, kind, wire_f64, version, sample_count, m)) return s;
  if (len) *len = m.total;
  if (m.total > cap) return fail(GHC_ERR_SHAPE, "encode: frame buffer too small");
  if (reinterpret_cast<uintptr_t>(d_out) & 15) return fail(GHC_ERR_CONFIG, "encode: output must be 16-byte aligned");
  if (kind != 0 && !d_w) return fail(GHC_ERR_CONFIG, "encode: null parameters");
  ghc_ctx* c = p->ctx;
  pack_frame_kernel<<<grid_for(c, (m.total + 15) / 16), 256, 0, c->stream>>>(m, d_w, d_out);
  c->launches++;
  CU(cudaGetLastError());
  return GHC_OK;
}

ghc_status ghc_decode_frame(ghc_plan* p, const uint8_t* d_frame, int64_t len, int32_t* kind,
                            float* d_w, uint64_t* version, uint64_t* sample_count,
                            int32_t* wire_f64, int32_t* decode_status) {
  ghc_ctx* c = p->ctx;
  auto bad = [&](int s) {
    if (decode_status) *decode_status = s;
    return fail(GHC_ERR_PROTOCOL, std::string("decode: ") + decode_name(s));
  };
  if (decode_status) *decode_status = 0;
  // header bytes → host (at most kHdrMax + the value regions we skip)
  auto fetch = [&](int64_t off, int64_t n, unsigned char* dst) -> ghc_status {
    CU(cudaMemcpyAsync(dst, d_frame + off, static_cast<size_t>(n), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return GHC_OK;
  };
  unsigned char h[32];
  if (len < 4) return bad(3);
  if (ghc_status s = fetch(0, std::min<int64_t>(len, 15), h)) return s;
  if (std::memcmp(h, "GHUB", 4) != 0) return bad(1);
  if (len < 15) return bad(3);
  if ((h[4] | (h[5] << 8)) != 1) return bad(2);
  const unsigned char type = h[6], base = type & 0xBF;
  const bool f64 = (type & 0x40) != 0;
  if (!(base >= 0x01 && base <= 0x06) || (f64 && base != 0x02 && base != 0x03)) return bad(5);
  uint64_t plen = 0;
  for (int i = 0; i < 8; ++i) plen |= static_cast<uint64_t>(h[7 + i]) << (8 * i);
  if (plen > (1ULL << 40)) return bad(4);
  if (plen > static_cast<uint64_t>(len - 15)) return bad(3);
  if (wire_f64) *wire_f64 = f64;
  if (base != 0x02 && base != 0x03) {
    const uint64_t want = base == 0x01 ? 5 : base == 0x04 ? 24 : base == 0x05 ? 4 : 0;
    if (plen != want) return bad(6);
    if (kind) *kind = base == 0x06 ? 0 : -static_cast<int>(base);
    return GHC_OK;
  }
  // WEIGHTS / GRADIENT: walk the payload (small host fetches for the headers)
  int64_t pos = 15;
  uint64_t rem = plen;
  auto take = [&](int n, uint64_t& v) -> int {
    if (rem < static_cast<uint64_t>(n)) return 6;
    unsigned char b[8];
    if (fetch(pos, n, b) != GHC_OK) return -1;
    v = 0;
    for (int i = 0; i < n; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    pos += n;
    rem -= static_cast<uint64_t>(n);
    return 0;
  };
  uint64_t ver = 0, cnt = 0, ntens = 0;
  if (int e = take(8, ver)) return e < 0 ? GHC_ERR_CUDA : bad(e);
  if (base == 0x03) {
    if (int e = take(8, cnt)) return e < 0 ? GHC_ERR_CUDA : bad(e);
    if (cnt < 1) return bad(6);
  }
  if (int e = take(4, ntens)) return e < 0 ? GHC_ERR_CUDA : bad(e);
  if (ntens > rem) return bad(6);
  FrameMap want;
  if (ghc_status s = build_map(p, base == 0x02 ? 1 : 2, f64, ver, base == 0x03 ? cnt : 1, want)) return s;
  int64_t toff[kMaxT], td0[kMaxT], td1[kMaxT];
  int tn = 0;
  if (ghc_status s = ghc_plan_tensors(p, toff, td0, td1, kMaxT, &tn)) return s;
  // the arch check the roles do when they rebuild a WeightSet (ShapeError)
  bool shape_ok = static_cast<int>(ntens) == want.nt;
  FrameMap m = want;
  const int es = f64 ? 8 : 4;
  for (uint64_t t = 0; t < ntens; ++t) {
    uint64_t rank = 0;
    if (int e = take(1, rank)) return e < 0 ? GHC_ERR_CUDA : bad(e);
    if (rank == 0) return bad(6);
    uint64_t elems = 1, dims[2] = {0, 0};
    for (uint64_t q = 0; q < rank; ++q) {
      uint64_t d = 0;
      if (int e = take(4, d)) return e < 0 ? GHC_ERR_CUDA : bad(e);
      if (d == 0) return bad(6);
      if (q < 2) dims[q] = d;
      if (elems > (1ULL << 40) / d) return bad(6);
      elems *= d;
    }
    if (elems * es > rem) return bad(6);
    if (shape_ok && static_cast<int>(t) < want.nt) {
      const uint64_t want_rank = td1[t] ? 2 : 1;
      shape_ok = rank == want_rank && dims[0] == static_cast<uint64_t>(td0[t]) &&
                 (want_rank == 1 || dims[1] == static_cast<uint64_t>(td1[t]));
    }
    if (static_cast<int>(t) < kMaxT) m.dst[t] = pos;
    pos += static_cast<int64_t>(elems) * es;
    rem -= elems * es;
  }
  if (rem != 0) return bad(6);
  if (!shape_ok) return fail(GHC_ERR_SHAPE, "decode: frame tensors do not match the architecture");
  if (kind) *kind = base == 0x02 ? 1 : 2;
  if (version) *version = ver;
  if (sample_count) *sample_count = cnt;
  if (d_w) {
    unpack_frame_kernel<<<grid_for(c, want.src[want.nt - 1] + want.n[want.nt - 1]), 256, 0,
                          c->stream>>>(m, d_frame, len, d_w);
    c->launches++;
    CU(cudaGetLastError());
  }
  return GHC_OK;
}
