// codec.cu — GHUB wire frames on the device.
//
// The reference encodes every WEIGHTS / GRADIENT message byte by byte on the
// host (proto.cpp:214-272, decode 288-386).  For a multi-node / TCP transport
// the frame of a 16.9 M-parameter gradient is 67.5 MB (f32) — an HBM-bound
// byte-shuffling job, done here where the parameters already live:
//
//   pack:   per tensor, blocks of 1024 ALIGNED 16-byte output chunks; value
//           bytes start at arbitrary byte offsets (15-byte header, 1-byte
//           ranks), so the block stages the value words in shared memory
//           (coalesced loads) and each chunk is assembled from ≤ 5 staged
//           words with funnel shifts and written with one 16-byte store
//           (coalesced); the few chunks that touch header bytes or region
//           boundaries take a bytewise path in block 0.
//   unpack: per tensor, blocks of 16 KB of value bytes staged as aligned
//           words (uint4 loads), four values per thread, one 16-byte store;
//           the header pieces are gathered in one launch + one copy and
//           validated on the host with the reference's DecodeStatus taxonomy.
// Flat grids (every block has work).  Measured: DESIGN.md §8 f4.
//
// Layout (little-endian): "GHUB" | u16 format 1 | u8 type (0x02 WEIGHTS,
// 0x03 GRADIENT, | 0x40 for f64 values, 0x06 SHUTDOWN) | u64 payload length |
// WEIGHTS: u64 version | GRADIENT: u64 basis_version, u64 sample_count |
// u32 tensor count | per tensor: u8 rank, u32 dims[rank], values.
#include "ghc_internal.cuh"

namespace {

constexpr int kMaxT = 16;       // parameter tensors of an arch (5 for the bench net)
constexpr int kHdrMax = 256;    // header bytes of a frame (fixed part + tensor headers)
constexpr int kMaxEdge = 3 * kMaxT + kHdrMax / 16 + 4;  // edge chunks: ≤ 2 per boundary + header + tail
constexpr int kPackChunks = 1024;   // output chunks (16 B) per pack block: 16 KB
constexpr int kUnpackBytes = 16384; // frame bytes per unpack block

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
  int nedge;                    // 16-B output chunks not inside one tensor's values
  long long edge[kMaxEdge];     // (header pieces, region boundaries, frame tail)
  int blk0[kMaxT + 1];          // launch: tensor t owns blocks [blk0[t], blk0[t+1]) (flat grid)
};

// Flat grid: block → (tensor, block within the tensor).  No empty blocks
// (a grid of (blocks of the largest tensor) × tensors launched ~36 k idle
// blocks for the wide net, ≈ 30 µs of block scheduling).
__device__ __forceinline__ int block_tensor(const FrameMap& m, int b, int& bx) {
  int t = 0;
  while (t < m.nt && b >= m.blk0[t + 1]) ++t;
  bx = b - m.blk0[t];
  return t;
}

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
  // chunks the interior pass of the pack kernel does not write: every chunk
  // that is not wholly inside one tensor's value bytes
  const long long nch = (pos + 15) / 16;
  long long c = 0;
  for (int t = 0; t <= m.nt; ++t) {
    const long long stop = t < m.nt ? (m.dst[t] + 15) / 16 : nch;  // first interior chunk of t
    for (; c < stop; ++c) {
      if (m.nedge >= kMaxEdge) return fail(GHC_ERR_CONFIG, "frame: too many edge chunks");
      m.edge[m.nedge++] = c;
    }
    if (t < m.nt) c = std::max(c, (m.dst[t] + m.n[t] * m.es) / 16);  // past t's interior chunks
  }
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

// Pack.  Blocks of tensor t (block_tensor): the 16-B output chunks wholly
// inside t's value bytes, kPackChunks per block: the block stages the value words it
// needs in shared memory (coalesced loads of the f32 parameters; f64 frames:
// the widened doubles' halves), then each thread assembles consecutive
// chunks from five staged words (funnel shift by the region's byte
// misalignment) and stores them as coalesced 16-B stores.  Block 0: the
// edge chunks (headers, region boundaries, tail), bytewise.
__global__ void __launch_bounds__(256) pack_frame_kernel(const FrameMap m, const float* __restrict__ w,
                                                          unsigned char* __restrict__ out) {
  // f32: 4·kPackChunks + 5 staged words (+ ≤ 3 of alignment); f64: the
  // 2·kPackChunks + 3 floats are staged above the words they widen into
  constexpr int kF64Stage = 4 * kPackChunks + 8;  // ≥ 2·nf: widened words never overwrite staged floats
  __shared__ __align__(16) unsigned sw[kF64Stage + 2 * kPackChunks + 16];
  if (blockIdx.x == 0) {  // block 0: the edge chunks, one byte per thread (its
    // loads overlap the bulk instead of trailing it as the last block)
    for (int e = threadIdx.x; e < 16 * m.nedge; e += blockDim.x) {
      const long long b = m.edge[e >> 4] * 16 + (e & 15);
      if (b < m.total) out[b] = static_cast<unsigned char>(frame_byte(m, w, b));
    }
    return;
  }
  int bx;
  const int t = block_tensor(m, static_cast<int>(blockIdx.x) - 1, bx);
  if (t >= m.nt) return;
  const long long L = m.dst[t], H = L + m.n[t] * m.es;
  const long long cfirst = (L + 15) / 16, cend = H / 16;  // interior chunks [cfirst, cend)
  const long long c0 = cfirst + static_cast<long long>(bx) * kPackChunks;
  if (c0 >= cend) return;
  const int nc = static_cast<int>(min(static_cast<long long>(kPackChunks), cend - c0));
  const long long nwords = m.n[t] * (m.es / 4);
  const int r = static_cast<int>((16 * c0 - L) & 3);   // byte misalignment (same for every chunk)
  long long j_lo = (16 * c0 - L) >> 2;                  // first value word of chunk c0
  if (m.es == 8) j_lo &= ~1LL;                          // whole doubles
  const long long j_hi = min(nwords, ((16 * (c0 + nc) - L) >> 2) + 1);  // one past the last word needed
  const int nw = static_cast<int>(j_hi - j_lo);
  // staged floats: [g0, g0 + nf) of the parameter array, loaded as aligned
  // float4s from A = g0 & ~3 (all of a thread's loads in flight before its
  // shared-memory stores); word j of the value stream is sw[(j - j_lo) + d]
  // (f32) or a half of the double widened from staged float (j - j_lo) / 2
  const long long pend = m.src[m.nt - 1] + m.n[m.nt - 1];  // end of the parameter array
  const long long g0 = m.src[t] + (m.es == 4 ? j_lo : (j_lo >> 1));
  const int nf = m.es == 4 ? nw : (nw + 1) / 2;
  const long long A = g0 & ~3LL;
  const int d = static_cast<int>(g0 - A);
  const int nv = (d + nf + 3) / 4;
  float* sf = reinterpret_cast<float*>(sw);  // f64: floats first, widened below
  for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * blockDim.x) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      const long long e = A + 4LL * i;
      if (i < nv && e + 4 <= pend) {
        v[u] = __ldg(reinterpret_cast<const float4*>(w + e));
      } else {
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < nv) {
          if (e < pend) v[u].x = __ldg(w + e);
          if (e + 1 < pend) v[u].y = __ldg(w + e + 1);
          if (e + 2 < pend) v[u].z = __ldg(w + e + 2);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nv) {
        if (m.es == 4) {
          reinterpret_cast<float4*>(sf)[i] = v[u];
        } else {  // f64: staged above the ≤ 2·nf words they widen into
          reinterpret_cast<float4*>(sf + kF64Stage)[i] = v[u];
        }
      }
    }
  }
  if (m.es == 8) {  // floats staged at sf[kF64Stage + d + k] → double k = words 2k, 2k+1
    __syncthreads();
    for (int k = threadIdx.x; k < nf; k += blockDim.x) {
      const long long bits = __double_as_longlong(static_cast<double>(sf[kF64Stage + d + k]));
      sw[2 * k] = static_cast<unsigned>(bits);
      sw[2 * k + 1] = static_cast<unsigned>(bits >> 32);
    }
  }
  const int wo = m.es == 4 ? d : 0;  // word j ↔ sw[j - j_lo + wo]
  __syncthreads();
  const int a0 = static_cast<int>(((16 * c0 - L) >> 2) - j_lo) + wo;  // staged word of chunk c0's first byte
  for (int q = threadIdx.x; q < nc; q += blockDim.x) {
    const long long c = c0 + q;
    const int a = a0 + 4 * q;
    // two aligned LDS.128 (consecutive lanes, consecutive 16 B: no bank
    // conflicts; five scalar loads at a 4-word lane stride were 4-way)
    const uint4* sw4 = reinterpret_cast<const uint4*>(sw) + (a >> 2);
    const uint4 u0 = sw4[0], u1 = sw4[1];
    unsigned wd[5];
    switch (a & 3) {  // static register indices per case
      case 0: wd[0] = u0.x; wd[1] = u0.y; wd[2] = u0.z; wd[3] = u0.w; wd[4] = u1.x; break;
      case 1: wd[0] = u0.y; wd[1] = u0.z; wd[2] = u0.w; wd[3] = u1.x; wd[4] = u1.y; break;
      case 2: wd[0] = u0.z; wd[1] = u0.w; wd[2] = u1.x; wd[3] = u1.y; wd[4] = u1.z; break;
      default: wd[0] = u0.w; wd[1] = u1.x; wd[2] = u1.y; wd[3] = u1.z; wd[4] = u1.w; break;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) wd[k] = a + k < nw + wo ? wd[k] : 0u;
    uint4 o;
    o.x = r ? __funnelshift_r(wd[0], wd[1], 8 * r) : wd[0];
    o.y = r ? __funnelshift_r(wd[1], wd[2], 8 * r) : wd[1];
    o.z = r ? __funnelshift_r(wd[2], wd[3], 8 * r) : wd[2];
    o.w = r ? __funnelshift_r(wd[3], wd[4], 8 * r) : wd[3];
    reinterpret_cast<uint4*>(out + 16 * c)[0] = o;
  }
}

// Unpack.  Blocks of tensor t (block_tensor), each a span of
// kUnpackBytes / es values: the block stages the frame words covering their bytes in shared
// memory (coalesced 4-B loads), then each thread funnel-shifts a value out of
// its staged words and stores it (coalesced).  Never reads past `len`.
__global__ void __launch_bounds__(256) unpack_frame_kernel(const FrameMap m, const unsigned char* __restrict__ in,
                                                            long long len, float* __restrict__ w) {
  __shared__ __align__(16) unsigned sw[kUnpackBytes / 4 + 16];
  int bx;
  const int t = block_tensor(m, static_cast<int>(blockIdx.x), bx);
  if (t >= m.nt) return;
  const int per = kUnpackBytes / m.es;
  const long long k0 = static_cast<long long>(bx) * per;
  if (k0 >= m.n[t]) return;
  const int nk = static_cast<int>(min(static_cast<long long>(per), m.n[t] - k0));
  const long long b0 = m.dst[t] + k0 * m.es;              // first byte of the block's values
  const long long w_lo = b0 >> 2;
  const long long w_hi = (b0 + static_cast<long long>(nk) * m.es + 3) / 4 + 1;  // + the funnel's extra word
  const int nw = static_cast<int>(w_hi - w_lo);
  // aligned 16-B loads from word A = w_lo & ~3 (16-B aligned frames; else
  // 4-B loads), all of a thread's loads in flight before its smem stores;
  // word wi ↔ sw[wi - w_lo + d]
  const bool vec = (reinterpret_cast<uintptr_t>(in) & 15u) == 0;
  const long long A = vec ? (w_lo & ~3LL) : w_lo;
  const int d = static_cast<int>(w_lo - A);
  const int nv = vec ? (d + nw + 3) / 4 : nw;
  auto word = [&](long long wi) {
    if (4 * wi + 4 <= len) return __ldg(reinterpret_cast<const unsigned*>(in) + wi);
    unsigned v = 0;  // the frame's last word: bytes before `len` only
    for (int y = 0; y < 4; ++y)
      if (4 * wi + y < len) v |= static_cast<unsigned>(in[4 * wi + y]) << (8 * y);
    return v;
  };
  for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * blockDim.x) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i >= nv) continue;
      if (!vec) {
        v[u].x = word(A + i);
      } else if (16 * (A / 4 + i) + 16 <= len) {
        v[u] = __ldg(reinterpret_cast<const uint4*>(in) + A / 4 + i);
      } else {
        v[u] = make_uint4(word(A + 4 * i), word(A + 4 * i + 1), word(A + 4 * i + 2), word(A + 4 * i + 3));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i >= nv) continue;
      if (vec) reinterpret_cast<uint4*>(sw)[i] = v[u];
      else sw[i] = v[u].x;
    }
  }
  __syncthreads();
  float* dst = w + m.src[t] + k0;
  const int r = static_cast<int>(b0 & 3);  // the same byte misalignment for every value
  const int ab = static_cast<int>((b0 >> 2) - w_lo) + d;  // staged word of the first value
  int q0 = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    // four values per thread: their (es/4)·4 + 1 words from aligned LDS.128s
    // (consecutive lanes, consecutive 16 B) and one 16-B store
    const int nq = nk / 4;
    const uint4* sw4 = reinterpret_cast<const uint4*>(sw);
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      const int a = ab + (m.es / 4) * 4 * q;  // ≡ ab (mod 4)
      unsigned wv[12];
      const uint4 u0 = sw4[a >> 2], u1 = sw4[(a >> 2) + 1];
      wv[0] = u0.x; wv[1] = u0.y; wv[2] = u0.z; wv[3] = u0.w;
      wv[4] = u1.x; wv[5] = u1.y; wv[6] = u1.z; wv[7] = u1.w;
      if (m.es == 8) {
        const uint4 u2 = sw4[(a >> 2) + 2];
        wv[8] = u2.x; wv[9] = u2.y; wv[10] = u2.z; wv[11] = u2.w;
      } else {
        wv[8] = wv[9] = wv[10] = wv[11] = 0u;
      }
      unsigned x[9];  // words a .. a+8 (shift by a & 3, static register indices)
      switch (a & 3) {
        case 0:
#pragma unroll
          for (int i = 0; i < 9; ++i) x[i] = wv[i];
          break;
        case 1:
#pragma unroll
          for (int i = 0; i < 9; ++i) x[i] = wv[i + 1];
          break;
        case 2:
#pragma unroll
          for (int i = 0; i < 9; ++i) x[i] = wv[i + 2];
          break;
        default:
#pragma unroll
          for (int i = 0; i < 9; ++i) x[i] = wv[i + 3];
          break;
      }
      float4 o;
      float* ov = &o.x;
      if (m.es == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) ov[i] = __uint_as_float(r ? __funnelshift_r(x[i], x[i + 1], 8 * r) : x[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const unsigned lo = r ? __funnelshift_r(x[2 * i], x[2 * i + 1], 8 * r) : x[2 * i];
          const unsigned hi = r ? __funnelshift_r(x[2 * i + 1], x[2 * i + 2], 8 * r) : x[2 * i + 1];
          ov[i] = __double2float_rn(__longlong_as_double(
              static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo)));
        }
      }
      reinterpret_cast<float4*>(dst)[q] = o;
    }
    q0 = 4 * nq;
  }
  for (int q = q0 + threadIdx.x; q < nk; q += blockDim.x) {  // the rest, one value per thread
    const long long b = b0 + static_cast<long long>(q) * m.es;
    const int a = static_cast<int>((b >> 2) - w_lo) + d;
    const unsigned lo = r ? __funnelshift_r(sw[a], sw[a + 1], 8 * r) : sw[a];
    float v;
    if (m.es == 4) {
      v = __uint_as_float(lo);
    } else {
      const unsigned hi = r ? __funnelshift_r(sw[a + 1], sw[a + 2], 8 * r) : sw[a + 1];
      v = __double2float_rn(__longlong_as_double(
          static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo)));
    }
    dst[q] = v;
  }
}

const char* decode_name(int s) {
  static const char* names[] = {"ok",        "bad magic",       "unsupported format version",
                                "truncated frame", "payload length overflow",
                                "unknown message type", "malformed payload"};
  return s >= 0 && s <= 6 ? names[s] : "?";
}

// The header bytes decode expects, gathered on the device in ONE launch and
// brought to the host in ONE copy: the first 64 bytes (fixed header + first
// tensor header) and every later tensor header at its position in a WEIGHTS /
// GRADIENT frame of this architecture, f32 and f64 — instead of one
// synchronous copy per header field (≈ 20 round trips per decode).
constexpr int kMaxPieces = 4 * kMaxT + 1;
constexpr int kHdrScratch = 64 + 4 * kMaxT * 16;  // piece bytes: first 64 + ≤ 9 per tensor header
struct Pieces {
  int n;
  long long off[kMaxPieces];
  int len[kMaxPieces];
  int out[kMaxPieces];
};
__global__ void gather_pieces_kernel(const unsigned char* __restrict__ in, long long len, const Pieces p,
                                     unsigned char* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= p.n) return;
  for (int b = threadIdx.x; b < p.len[i]; b += blockDim.x)
    out[p.out[i] + b] = p.off[i] + b < len ? in[p.off[i] + b] : 0;
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
  long long nb = 0;  // flat grid: each tensor's interior chunk blocks, then one edge block
  for (int t = 0; t < m.nt; ++t) {
    m.blk0[t] = static_cast<int>(nb);
    nb += std::max(0LL, ((m.dst[t] + m.n[t] * m.es) / 16 - (m.dst[t] + 15) / 16 + kPackChunks - 1) / kPackChunks);
  }
  m.blk0[m.nt] = static_cast<int>(nb);
  pack_frame_kernel<<<static_cast<unsigned>(nb + 1), 256, 0, c->stream>>>(m, d_w, d_out);
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
  // header bytes → host: the expected header pieces in one gather + copy;
  // a read outside them (a frame of another layout) falls back to its own copy
  Pieces pc{};
  auto add = [&](long long off, int n) {
    if (pc.n >= kMaxPieces || n <= 0 || off >= len) return;
    pc.off[pc.n] = off;
    pc.len[pc.n] = n;
    pc.out[pc.n] = pc.n ? pc.out[pc.n - 1] + pc.len[pc.n - 1] : 0;
    ++pc.n;
  };
  add(0, 64);
  for (int kind_ : {1, 2})
    for (int f64_ : {0, 1}) {
      FrameMap mm;
      if (build_map(p, kind_, f64_, 0, 1, mm) != GHC_OK) continue;
      for (int t = 1; t < mm.nt; ++t) add(mm.hdr_dst[t], mm.hdr_off[t + 1] - mm.hdr_off[t]);
    }
  std::vector<unsigned char> cache;
  if (pc.n > 0) {
    const int total = pc.n ? pc.out[pc.n - 1] + pc.len[pc.n - 1] : 0;
    cache.resize(static_cast<size_t>(total));
    // a context-owned scratch (a stream-ordered allocation per call costs
    // a pool remap after every synchronisation: ≈ 0.3 ms per decode)
    if (total > kHdrScratch) return fail(GHC_ERR_CONFIG, "decode: header pieces exceed the scratch");
    if (!c->hdr_scratch) CU(cudaMalloc(reinterpret_cast<void**>(&c->hdr_scratch), kHdrScratch));
    gather_pieces_kernel<<<pc.n, 64, 0, c->stream>>>(d_frame, len, pc, c->hdr_scratch);
    c->launches++;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(cache.data(), c->hdr_scratch, static_cast<size_t>(total), cudaMemcpyDeviceToHost,
                       c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  auto fetch = [&](int64_t off, int64_t n, unsigned char* dst) -> ghc_status {
    for (int i = 0; i < pc.n; ++i)
      if (off >= pc.off[i] && off + n <= pc.off[i] + pc.len[i] && off + n <= len) {
        std::memcpy(dst, cache.data() + pc.out[i] + (off - pc.off[i]), static_cast<size_t>(n));
        return GHC_OK;
      }
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
    if (reinterpret_cast<uintptr_t>(d_frame) & 3) return fail(GHC_ERR_CONFIG, "decode: frame must be 4-byte aligned");
    long long nb = 0;  // flat grid: kUnpackBytes of values per block
    for (int t = 0; t < m.nt; ++t) {
      m.blk0[t] = static_cast<int>(nb);
      nb += (m.n[t] * es + kUnpackBytes - 1) / kUnpackBytes;
    }
    m.blk0[m.nt] = static_cast<int>(nb);
    unpack_frame_kernel<<<static_cast<unsigned>(std::max(1LL, nb)), 256, 0, c->stream>>>(m, d_frame, len, d_w);
    c->launches++;
    CU(cudaGetLastError());
  }
  return GHC_OK;
}
