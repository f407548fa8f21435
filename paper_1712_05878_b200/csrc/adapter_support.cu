// adapter_support.cu — device-side pieces of the reference-facing drop-in
// (adapter/gradhub_cuda.cpp): the peer copy of the "nvlink" Endpoint, the
// weights upload with its stale-cache token, and the batch loss.
//
//  * ghc_memcpy_peer: one message payload from the sender's GPU into the
//    receiver's mailbox slot (cudaMemcpyPeerAsync: NVLink P2P on a B200 box,
//    a device copy when both ranks share a GPU).  Replaces the reference's
//    inproc mailbox byte copy (transport.cpp:25-177) for WEIGHTS / GRADIENT.
//  * ghc_weights_import_f64: the reference's WeightSet values are f64; they
//    are uploaded once, rounded to the f32 the kernels consume (the f32 wire
//    of proto.cpp) AND hashed in the same pass.  The hash is the device-side
//    replacement of weights_checksum (nn.cpp:66-81, FNV-1a over every f64
//    value): an order-independent 64-bit mix of (index, f64 bits) summed with
//    wrapping adds, so any change of any f64 value changes it (up to 2^-64)
//    and the result is deterministic.  forward() stores it in the cache,
//    backward() recomputes it while uploading — CacheMismatchError keeps the
//    reference's semantics without the host O(P) FNV pass.
//  * ghc_nll_sum: Σ_s −log p[s][y_s] in f64 with a fixed reduction order
//    (nn.cpp:234-248) and the reference's label range check.
#include "ghc_internal.cuh"

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {  // splitmix64 finaliser
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void import_f64_kernel(float* __restrict__ w32, const double* __restrict__ w64, long long P,
                                  unsigned long long* __restrict__ hash) {
  unsigned long long h = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = w64[i];
    if (w32) w32[i] = (float)v;
    h += mix64(mix64((unsigned long long)i) ^ (unsigned long long)__double_as_longlong(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && hash) atomicAdd(hash, h);  // integer adds: order-independent
}

// One block; thread t sums rows t, t+1024, … in order, then a fixed tree.
__global__ void __launch_bounds__(1024) nll_kernel(const double* __restrict__ probs, const int32_t* __restrict__ y,
                                                   long long n, int K, double* out, int* bad) {
  __shared__ double red[1024];
  double s = 0.0;
  int b = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const int l = y[i];
    if (l < 0 || l >= K) {
      b = 1;
      continue;
    }
    s += -log(probs[i * K + l]);
  }
  red[threadIdx.x] = s;
  b = __syncthreads_or(b);
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = red[0];
    *bad = b;
  }
}

}  // namespace

extern "C" {

ghc_status ghc_memcpy_peer(ghc_ctx* c, void* d_dst, int32_t dst_device, const void* d_src,
                           int32_t src_device, size_t bytes) {
  if (!c) return fail(GHC_ERR_CONFIG, "memcpy_peer: null context");
  CU(cudaSetDevice(c->device));
  CU(cudaMemcpyPeerAsync(d_dst, dst_device, d_src, src_device, bytes, c->stream));
  return GHC_OK;
}

ghc_status ghc_weights_import_f64(ghc_ctx* c, float* d_w32, const double* d_w64, int64_t P,
                                  uint64_t* d_hash) {
  if (!c || !d_w64 || P < 0) return fail(GHC_ERR_CONFIG, "weights_import_f64: bad argument");
  CU(cudaSetDevice(c->device));
  if (d_hash) CU(cudaMemsetAsync(d_hash, 0, sizeof(uint64_t), c->stream));
  const int grid = static_cast<int>(std::min<int64_t>((P + 255) / 256, 4L * c->num_sms));
  import_f64_kernel<<<grid > 0 ? grid : 1, 256, 0, c->stream>>>(
      d_w32, d_w64, P, reinterpret_cast<unsigned long long*>(d_hash));
  CU(cudaGetLastError());
  c->launches++;
  return GHC_OK;
}

ghc_status ghc_nll_sum(ghc_ctx* c, const double* d_probs, const int32_t* d_y, int64_t n, int32_t K,
                       double* h_sum) {
  if (!c || n < 1 || K < 1 || !h_sum) return fail(GHC_ERR_SHAPE, "loss: empty batch");
  CU(cudaSetDevice(c->device));
  char* ws = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&ws), 16, c->stream));
  nll_kernel<<<1, 1024, 0, c->stream>>>(d_probs, d_y, n, K, reinterpret_cast<double*>(ws),
                                        reinterpret_cast<int*>(ws + 8));
  CU(cudaGetLastError());
  c->launches++;
  double s = 0.0;
  int bad = 0;
  CU(cudaMemcpyAsync(&s, ws, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(&bad, ws + 8, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaFreeAsync(ws, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (bad) return fail(GHC_ERR_SHAPE, "loss: label out of range [0," + std::to_string(K) + ")");
  *h_sum = s;
  return GHC_OK;
}

}  // extern "C"
