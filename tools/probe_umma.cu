// tcgen05.mma (kind::f16, SS operands, M=128, K=16) issue / completion cost vs N, single CTA.
// Tells whether the score kernel's per-tile MMA time (8 MMAs of N=16) is issue- or latency-bound.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__global__ void k(unsigned long long* out, int N, int ntile, int accbufs, int nwarps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  uint8_t* A = sm; uint8_t* B = sm + 32768;
  for (int i = threadIdx.x; i < (32768 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar))); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < nwarps) {
    const uint32_t tmem = tb + w * 64;
    long long c0 = clock64();
    for (int t = 0; t < ntile; ++t) {
      const uint32_t d = tmem + (t % accbufs) * 16;
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t ko = (kk >> 2) * 16384 + (kk & 3) * 32;
        const uint64_t ad = desc(su32(A) + ko), bd = desc(su32(B) + (kk >> 2) * 16384 + (kk & 3) * 32);
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
      }
    }
    long long c1 = clock64();
    long long c2 = c1;
    if (w == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" :: "r"(su32(&bar)) : "memory");
      c2 = clock64();
    }
    if (blockIdx.x == 0 && w == nwarps - 1) { out[0] = c1 - c0; }
    if (blockIdx.x == 0 && w == 0) { out[1] = c2 - c0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int grid : {1, 148})
    for (int nw : {1, 2, 4})
      for (int nt : {8, 32}) {
        k<<<grid, 128, 65536 + 1024>>>(d, 16, nt, 4, nw);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("grid=%3d warps=%d tiles/warp=%2d (MMAs/warp=%3d): last warp issue %6llu cyc (%.1f/mma/warp)  warp0 complete %6llu %s\n",
               grid, nw, nt, nt * 8, h[0], (double)h[0] / (nt * 8), h[1], e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
