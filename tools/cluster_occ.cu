// cluster_occ.cu — co-resident clusters per cluster size on this GPU
// (cudaOccupancyMaxActiveClusters), for a 256-thread CTA that fills one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occ tools/cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) k(int* p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}

int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  printf("{\"sms\": %d, \"rows\": [", pr.multiProcessorCount);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  bool first = true;
  for (int smem : {100 * 1024, 200 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = cs;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("%s{\"smem\": %d, \"cs\": %d, \"clusters\": %d, \"ctas\": %d, \"err\": \"%s\"}", first ? "" : ", ", smem,
             cs, n, n * cs, cudaGetErrorString(e));
      first = false;
      cudaGetLastError();
    }
  }
  printf("]}\n");
}
