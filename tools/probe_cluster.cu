// How many thread-block clusters of a given size fit on the GPU at once (cudaOccupancyMaxActiveClusters)
// for a 1-CTA-per-SM shared-memory footprint: sizing input for a per-(request, KV head) cluster design.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_probe() { extern __shared__ char s[]; s[threadIdx.x] = 0; }
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {100 * 1024, 150 * 1024, 200 * 1024, 220 * 1024}) {
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int cl : {2, 4, 8, 12, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl * 64); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_probe, &cfg);
      printf("sms=%d smem=%dKB cluster=%2d -> max active clusters %d (%d CTAs) %s\n", sms, smem / 1024, cl, n, n * cl,
             e ? cudaGetErrorString(e) : "");
    }
  }
  return 0;
}
