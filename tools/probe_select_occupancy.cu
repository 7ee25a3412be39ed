// Max co-resident 8-CTA select clusters (cudaOccupancyMaxActiveClusters) for the decode kernels.
#include "../paper_2410_21465_b200/csrc/decode.cu"
#include <cstdio>
using namespace skv;
template <int G, bool Z>
static void q(const char* name, size_t dyn) {
  cudaFuncSetAttribute(k_select<G, Z>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelectSmemMax);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(8 * 64); cfg.blockDim = dim3(kSelThreads); cfg.dynamicSmemBytes = dyn;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kSelCL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k_select<G, Z>, &cfg);
  int per_sm = -1; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select<G, Z>, kSelThreads, dyn);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_select<G, Z>);
  printf("%s dyn=%zu KB: max active clusters %d (%s), blocks/SM %d, regs %d, static smem %zu\n", name, dyn / 1024, n,
         cudaGetErrorString(e), per_sm, fa.numRegs, fa.sharedSizeBytes);
}
int main() {
  q<4, true>("k_select<4>", 8 * 1024);
  q<4, true>("k_select<4>", 16 * 1024);
  q<16, true>("k_select<16>", 16 * 1024);
  q<16, true>("k_select<16>", 64 * 1024);
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("SMs %d, smem/SM %zu KB, regs/SM %d\n", p.multiProcessorCount, p.sharedMemPerMultiprocessor / 1024, p.regsPerMultiprocessor);
  return 0;
}
