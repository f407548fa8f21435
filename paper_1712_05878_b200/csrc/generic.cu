// generic.cu — the LSTM layer for ANY lstm(D,H,T) (arch.hpp:36-57 accepts
// every positive size; the fused round kernels are instantiated for a table
// of shapes only).  The recurrence is restated as GEMMs on the tcgen05
// tensor cores (dense_gemm.cuh, 3×TF32) plus one pointwise cell kernel per
// timestep, with every sample of the batch in each GEMM:
//
//   forward  (nn.cpp:146-201)
//     Gx[s,t,:]  = Wx·x[s,t] + b                one GEMM, M = n·T, K = D
//     for t:  Z  = Gx[:,t,:] + Wh·h[:,t-1]      one GEMM, M = n, K = H
//             i,f,g,o = σ,σ,tanh,σ(Z); c = f·c' + i·g; h = o·tanh(c)
//                                                  (cell kernel; gates, c,
//                                                  tanh c, h kept per (s,t):
//                                                  the reference's LayerCache)
//   backward (nn.cpp:335-396), from dh_T:
//     for t = T-1…0:  dz_t, dc ← cell-backward(dh, dc, cache)   (pointwise)
//                     dh ← Whᵀ·dz_t                            one GEMM
//     dWx = Σ_{s,t} dz ⊗ x,  dWh = Σ_{s,t≥1} dz ⊗ h_{t-1}      two split-K GEMMs,
//                                                             K = n·T
//     db  = Σ_{s,t} dz                                        fixed-order sums
//
// Deterministic: every reduction has a fixed order.  Used for LSTM trunks of
// layered architectures and for lstm→softmax shapes outside the fused table.
#include "ghc_internal.cuh"

using namespace ghc;

namespace {

__device__ __forceinline__ float sigm(float z) { return 1.0f / (1.0f + expf(-z)); }

// Gates of timestep t for every (sample, unit); G holds Wx·x + b on entry
// and the activated gates on exit.
__global__ void lstm_cell_fwd_kernel(float* __restrict__ G, const float* __restrict__ Gh,
                                     float* __restrict__ Cc, float* __restrict__ TC,
                                     float* __restrict__ Hs, int n, int T, int H, int t) {
  const long long tot = (long long)n * H;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / H), u = (int)(i % H);
    const long long st = (long long)s * T + t;
    float* g = G + st * 4 * H;
    float z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) z[q] = g[q * H + u] + (Gh ? Gh[(long long)s * 4 * H + q * H + u] : 0.0f);
    const float ig = sigm(z[0]), fg = sigm(z[1]), gg = tanhf(z[2]), og = sigm(z[3]);
    const float cp = t > 0 ? Cc[(st - 1) * H + u] : 0.0f;
    const float c = fg * cp + ig * gg;
    const float tc = tanhf(c);
    g[0 * H + u] = ig;
    g[1 * H + u] = fg;
    g[2 * H + u] = gg;
    g[3 * H + u] = og;
    Cc[st * H + u] = c;
    TC[st * H + u] = tc;
    Hs[st * H + u] = og * tc;
  }
}

// Cell backward of timestep t (nn.cpp:351-392): dh (this step's ∂ℓ/∂h_t),
// dc carried across steps (in place), dz_t written to DZ[s,t,:].
__global__ void lstm_cell_bwd_kernel(const float* __restrict__ G, const float* __restrict__ Cc,
                                     const float* __restrict__ TC, const float* __restrict__ dH,
                                     int ldh, float* __restrict__ DC, float* __restrict__ DZ, int n,
                                     int T, int H, int t) {
  const long long tot = (long long)n * H;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / H), u = (int)(i % H);
    const long long st = (long long)s * T + t;
    const float* g = G + st * 4 * H;
    const float ig = g[u], fg = g[H + u], gg = g[2 * H + u], og = g[3 * H + u];
    const float tc = TC[st * H + u];
    const float cp = t > 0 ? Cc[(st - 1) * H + u] : 0.0f;
    const float dh = dH[(long long)s * ldh + u];
    float dc = DC[i];
    const float dout = dh * tc;
    dc = fmaf(dh * og, 1.0f - tc * tc, dc);
    const float di = dc * gg, dg = dc * ig, df = dc * cp;
    float* dz = DZ + st * 4 * H;
    dz[u] = di * ig * (1.0f - ig);
    dz[H + u] = df * fg * (1.0f - fg);
    dz[2 * H + u] = dg * (1.0f - gg * gg);
    dz[3 * H + u] = dout * og * (1.0f - og);
    DC[i] = dc * fg;
  }
}

// HshT[k][s·T+t] = h[s][t-1][k] (0 at t = 0): the K-major operand of
// dWh = Σ dz_t ⊗ h_{t-1}.
__global__ void shift_transpose_kernel(float* __restrict__ out, int ldo, const float* __restrict__ Hs,
                                       int n, int T, int H) {
  __shared__ float tile[32][33];
  const long long rows = (long long)n * T;  // (s,t) index
  const long long r0 = (long long)blockIdx.y * 32;
  const int k0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long r = r0 + i;
    const int k = k0 + threadIdx.x;
    float v = 0.0f;
    if (r < rows && k < H && (r % T) != 0) v = Hs[(r - 1) * H + k];
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i;
    const long long r = r0 + threadIdx.x;
    if (k < H && r < rows) out[(long long)k * ldo + r] = tile[threadIdx.x][i];
  }
}

// out[r] = Σ_j X[r][j], one block per row, fixed order (strided, then tree).
__global__ void rowsum_kernel(float* __restrict__ out, const float* __restrict__ X, long long ld,
                              long long cols) {
  __shared__ float red[256];
  const float* x = X + (long long)blockIdx.x * ld;
  float t = 0.0f;
  for (long long j = threadIdx.x; j < cols; j += blockDim.x) t += x[j];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

struct GBuf {
  float* p = nullptr;
  size_t cap = 0;
  ghc_status ensure(size_t n) {
    if (n <= cap) return GHC_OK;
    cudaFree(p);
    p = nullptr;
    cap = 0;
    CU(cudaMalloc(&p, sizeof(float) * (n ? n : 1)));
    cap = n;
    return GHC_OK;
  }
};

int grid_for(ghc_ctx* c, long long n) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 8LL * c->num_sms)));
}

}  // namespace

struct GenericLstmWorkspace {
  GBuf G, Cc, TC, Hs, Gh, DZ, DC, dH, WhT, DZT, XT, HshT;
};

void generic_lstm_free(GenericLstmWorkspace* ws) {
  if (!ws) return;
  GBuf* all[] = {&ws->G, &ws->Cc, &ws->TC, &ws->Hs, &ws->Gh, &ws->DZ, &ws->DC, &ws->dH,
                 &ws->WhT, &ws->DZT, &ws->XT, &ws->HshT};
  for (GBuf* b : all) cudaFree(b->p);
  delete ws;
}

// Forward over n samples (rows of X, T·D floats each): caches in the
// workspace, h_T into hT_out[n×H] (nullable).
ghc_status generic_lstm_fwd(ghc_plan* p, const float* w, const float* X, int n, float* hT_out) {
  ghc_ctx* c = p->ctx;
  const Layer& L0 = p->model.layers[0];
  const int D = L0.a, H = L0.b, T = L0.c;
  if (!p->gws) p->gws = new GenericLstmWorkspace();
  GenericLstmWorkspace& ws = *p->gws;
  const long long nT = static_cast<long long>(n) * T;
  const float* Wx = w + p->model.tensors[0].offset;
  const float* Wh = w + p->model.tensors[1].offset;
  const float* b = w + p->model.tensors[2].offset;
  if (ghc_status s = ws.G.ensure(static_cast<size_t>(nT) * 4 * H)) return s;
  if (ghc_status s = ws.Cc.ensure(static_cast<size_t>(nT) * H)) return s;
  if (ghc_status s = ws.TC.ensure(static_cast<size_t>(nT) * H)) return s;
  if (ghc_status s = ws.Hs.ensure(static_cast<size_t>(nT) * H)) return s;
  if (ghc_status s = ws.Gh.ensure(static_cast<size_t>(n) * 4 * H)) return s;
  // Gx = X·Wxᵀ + b over all (s,t): X is [n·T × D] row-major (time-major rows)
  if (ghc_status s = gemm_nt_ct(c, X, Wx, ws.G.p, static_cast<int>(nT), 4 * H, D, D, D, 4 * H,
                                GHC_EPI_BIAS_ACT, 2, b, nullptr, 0, 1.0f, nullptr, 0))
    return s;
  const int grid = grid_for(c, static_cast<long long>(n) * H);
  for (int t = 0; t < T; ++t) {
    const float* gh = nullptr;
    if (t > 0) {  // Wh·h_{t-1} for every sample
      if (ghc_status s = gemm_nt_ct(c, ws.Hs.p + static_cast<long long>(t - 1) * H, Wh, ws.Gh.p, n, 4 * H, H,
                                    T * H, H, 4 * H, GHC_EPI_STORE, 2, nullptr, nullptr, 0, 1.0f, nullptr, 0))
        return s;
      gh = ws.Gh.p;
    }
    lstm_cell_fwd_kernel<<<grid, 256, 0, c->stream>>>(ws.G.p, gh, ws.Cc.p, ws.TC.p, ws.Hs.p, n, T, H, t);
    c->launches++;
    CU(cudaGetLastError());
  }
  if (hT_out) {  // h_T rows (strided copy)
    CU(cudaMemcpy2DAsync(hT_out, sizeof(float) * H, ws.Hs.p + static_cast<long long>(T - 1) * H,
                         sizeof(float) * T * H, sizeof(float) * H, n, cudaMemcpyDeviceToDevice, c->stream));
  }
  return GHC_OK;
}

// Backward from dh_T (dhT[n×H], already scaled): Wx, Wh, b gradients into
// g_out at the trunk's tensor offsets.  Needs the caches of the last
// generic_lstm_fwd on the same batch.
ghc_status generic_lstm_bwd(ghc_plan* p, const float* w, const float* X, int n, const float* dhT,
                            float* g_out) {
  ghc_ctx* c = p->ctx;
  const Layer& L0 = p->model.layers[0];
  const int D = L0.a, H = L0.b, T = L0.c;
  GenericLstmWorkspace& ws = *p->gws;
  const long long nT = static_cast<long long>(n) * T;
  const int ldk = static_cast<int>((nT + 3) & ~3LL);  // K-major operands: 16-B rows (TMA)
  const float* Wh = w + p->model.tensors[1].offset;
  if (ghc_status s = ws.DZ.ensure(static_cast<size_t>(nT) * 4 * H)) return s;
  if (ghc_status s = ws.DC.ensure(static_cast<size_t>(n) * H)) return s;
  if (ghc_status s = ws.dH.ensure(static_cast<size_t>(n) * H)) return s;
  if (ghc_status s = ws.WhT.ensure(static_cast<size_t>(H) * 4 * H)) return s;
  CU(cudaMemsetAsync(ws.DC.p, 0, sizeof(float) * n * H, c->stream));
  if (ghc_status s = ghc_transpose(c, ws.WhT.p, Wh, 4 * H, H, H, 4 * H)) return s;  // [H × 4H]
  const int grid = grid_for(c, static_cast<long long>(n) * H);
  const float* dh = dhT;
  int ldh = H;
  for (int t = T - 1; t >= 0; --t) {
    lstm_cell_bwd_kernel<<<grid, 256, 0, c->stream>>>(ws.G.p, ws.Cc.p, ws.TC.p, dh, ldh, ws.DC.p, ws.DZ.p, n,
                                                      T, H, t);
    c->launches++;
    CU(cudaGetLastError());
    if (t > 0) {  // dh_{t-1} = Whᵀ·dz_t (the reference also forms it at t = 0, unused)
      if (ghc_status s = gemm_nt_ct(c, ws.DZ.p + static_cast<long long>(t) * 4 * H, ws.WhT.p, ws.dH.p, n, H,
                                    4 * H, T * 4 * H, 4 * H, H, GHC_EPI_STORE, 2, nullptr, nullptr, 0, 1.0f,
                                    nullptr, 0))
        return s;
      dh = ws.dH.p;
      ldh = H;
    }
  }
  // weight gradients: K-major operands over the (s,t) index
  if (ghc_status s = ws.DZT.ensure(static_cast<size_t>(4 * H) * ldk)) return s;
  if (ghc_status s = ws.XT.ensure(static_cast<size_t>(D) * ldk)) return s;
  if (ghc_status s = ws.HshT.ensure(static_cast<size_t>(H) * ldk)) return s;
  if (ghc_status s = ghc_transpose(c, ws.DZT.p, ws.DZ.p, static_cast<int>(nT), 4 * H, 4 * H, ldk)) return s;
  if (ghc_status s = ghc_transpose(c, ws.XT.p, X, static_cast<int>(nT), D, D, ldk)) return s;
  {
    dim3 g2((H + 31) / 32, static_cast<unsigned>((nT + 31) / 32));
    shift_transpose_kernel<<<g2, dim3(32, 8), 0, c->stream>>>(ws.HshT.p, ldk, ws.Hs.p, n, T, H);
    c->launches++;
    CU(cudaGetLastError());
  }
  const auto& tn = p->model.tensors;
  if (ghc_status s = gemm_nt_splitk(c, ws.DZT.p, ws.XT.p, g_out + tn[0].offset, 4 * H, D, static_cast<int>(nT),
                                    ldk, ldk, D))
    return s;
  if (ghc_status s = gemm_nt_splitk(c, ws.DZT.p, ws.HshT.p, g_out + tn[1].offset, 4 * H, H,
                                    static_cast<int>(nT), ldk, ldk, H))
    return s;
  rowsum_kernel<<<4 * H, 256, 0, c->stream>>>(g_out + tn[2].offset, ws.DZT.p, ldk, nT);
  c->launches++;
  CU(cudaGetLastError());
  return GHC_OK;
}

// The reference's LayerCache of the LSTM layer (nn.hpp:15-23) for the last
// generic forward: gates [n×T×4H], cell, tanh_c, hidden [n×T×H] (nullable).
ghc_status generic_lstm_cache(ghc_plan* p, int n, float* d_gates, float* d_cell, float* d_tanh,
                              float* d_hidden) {
  ghc_ctx* c = p->ctx;
  const Layer& L0 = p->model.layers[0];
  const long long nT = static_cast<long long>(n) * L0.c;
  const int H = L0.b;
  GenericLstmWorkspace& ws = *p->gws;
  if (d_gates) CU(cudaMemcpyAsync(d_gates, ws.G.p, sizeof(float) * nT * 4 * H, cudaMemcpyDeviceToDevice, c->stream));
  if (d_cell) CU(cudaMemcpyAsync(d_cell, ws.Cc.p, sizeof(float) * nT * H, cudaMemcpyDeviceToDevice, c->stream));
  if (d_tanh) CU(cudaMemcpyAsync(d_tanh, ws.TC.p, sizeof(float) * nT * H, cudaMemcpyDeviceToDevice, c->stream));
  if (d_hidden) CU(cudaMemcpyAsync(d_hidden, ws.Hs.p, sizeof(float) * nT * H, cudaMemcpyDeviceToDevice, c->stream));
  return GHC_OK;
}

extern "C" ghc_status ghc_forward_cache(ghc_plan* p, const float* d_w, const float* d_x, int64_t n,
                                        float* d_gates, float* d_cell, float* d_tanh, float* d_hidden) {
  if (!p || !d_w || !d_x) return fail(GHC_ERR_CONFIG, "forward_cache: null argument");
  if (n < 1) return fail(GHC_ERR_SHAPE, "batch: n_samples must be >= 1");
  if (p->model.layers.empty() || p->model.layers[0].kind != LayerKind::lstm)
    return fail(GHC_ERR_CONFIG, "forward_cache: the first layer is not an LSTM");
  if (ghc_status s = generic_lstm_fwd(p, d_w, d_x, static_cast<int>(n), nullptr)) return s;
  return generic_lstm_cache(p, static_cast<int>(n), d_gates, d_cell, d_tanh, d_hidden);
}
