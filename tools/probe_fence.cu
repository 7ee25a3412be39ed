// Probe: what does a GPU-scope fence / release operation cost on an SM whose CTA has host-link (PCIe)
// bulk reads in flight -- issued by the SAME thread, by ANOTHER warp of the same CTA, or by another CTA
// on the same SM -- and after those reads have landed?  Sizing input for merging the per-unit attention
// partials inside the sparse grid (needs a release before a per-head counter) instead of a merge grid.
// Standalone tool: not part of the product library.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChunk = 2048, kPerCta = 14;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// mode: 0 __threadfence by a warp that issued nothing; 1 __threadfence by the issuing thread;
// 2 st.release.gpu by another warp; 3 red.release.gpu.add by another warp; 4 fence after the reads landed;
// 5 atom.add.acq_rel by another warp; 6 no host reads at all (baseline fence)
__global__ void k_probe(const uint8_t* host, int nch, int mode, int* flag, long long* out) {
  __shared__ __align__(128) uint8_t buf[kPerCta * kChunk];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (mode != 6)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar)), "r"(kPerCta * kChunk) : "memory");
  }
  __syncthreads();
  if (mode != 6 && tid < kPerCta) {
    const size_t c = ((size_t)blockIdx.x * 7919u + tid * 104729u) % nch;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(su32(buf + tid * kChunk)), "l"(host + c * kChunk), "r"(kChunk), "r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  auto wait_bar = [&]() {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(su32(&bar)) : "memory");
  };
  long long t0 = 0, t1 = 0;
  const bool me = (mode == 1) ? tid == 0 : tid == 64;     // the measuring thread (warp 2 unless mode 1)
  if (mode == 4 && me) wait_bar();
  if (me) {
    flag[blockIdx.x] = 1;                                 // a global store to order
    t0 = gt();
    if (mode == 0 || mode == 1 || mode == 4 || mode == 6) __threadfence();
    else if (mode == 2) asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(flag + gridDim.x + blockIdx.x), "r"(2) : "memory");
    else if (mode == 3) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(flag + 2 * gridDim.x), "r"(1) : "memory");
    else if (mode == 5) { int o; asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(o) : "l"(flag + 2 * gridDim.x), "r"(1) : "memory"); }
    t1 = gt();
  }
  if (mode != 6 && tid == 32) wait_bar();
  __syncthreads();
  const long long tend = gt();
  if (me) { out[3 * blockIdx.x] = t1 - t0; out[3 * blockIdx.x + 1] = t0; out[3 * blockIdx.x + 2] = tend; }
}

int main() {
  const size_t host_bytes = (size_t)1 << 30;
  uint8_t* h;
  CK(cudaHostAlloc(&h, host_bytes, cudaHostAllocMapped));
  memset(h, 1, host_bytes);
  uint8_t* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* flag; long long* out;
  CK(cudaMalloc(&flag, 4 * 4096)); CK(cudaMemset(flag, 0, 4 * 4096));
  const int grid = sms;                                   // one CTA per SM (28 KB smem + few threads)
  CK(cudaMalloc(&out, 3 * 8 * 4096));
  const char* names[] = {"__threadfence, other warp, reads in flight", "__threadfence, issuing thread, reads in flight",
                         "st.release.gpu, other warp, reads in flight", "red.release.gpu, other warp, reads in flight",
                         "__threadfence after own reads landed", "atom.acq_rel.gpu, other warp, reads in flight",
                         "__threadfence, no host reads"};
  for (int mode = 0; mode < 7; ++mode) {
    for (int g : {grid, 2 * grid}) {                      // 2 CTAs per SM: the other CTA's reads in flight too
      std::vector<long long> all;
      double span_us = 0;
      for (int trial = 0; trial < 5; ++trial) {
        k_probe<<<g, 128>>>(hd, (int)(host_bytes / kChunk), mode, flag, out);
        CK(cudaDeviceSynchronize());
        std::vector<long long> o(3 * g);
        CK(cudaMemcpy(o.data(), out, 3 * g * 8, cudaMemcpyDeviceToHost));
        long long lo = o[1], hi = o[2];
        for (int i = 0; i < g; ++i) { if (trial) all.push_back(o[3 * i]); lo = std::min(lo, o[3 * i + 1]); hi = std::max(hi, o[3 * i + 2]); }
        if (trial) span_us += (hi - lo) / 1e3 / 4;
      }
      std::sort(all.begin(), all.end());
      printf("%-48s ctas/SM=%d  p50 %8.2f us  p90 %8.2f  max %8.2f  (kernel span %.1f us)\n", names[mode], g / grid,
             all[all.size() / 2] / 1e3, all[all.size() * 9 / 10] / 1e3, all.back() / 1e3, span_us);
    }
  }
  return 0;
}
