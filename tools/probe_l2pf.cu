// Probe: does the L2 cache host-mapped (pinned) memory, and can an L2 prefetch of scattered 2 KB value
// chunks (cp.async.bulk.prefetch.L2) start the PCIe transfer ahead of the consumer's bulk copies?
//   cold    : 2048 random 2 KB chunks (4 MB, one c2 layer's selection) bulk-copied host -> smem
//   pf+wait : L2 prefetch of the same chunks, a 300 us spin, then the same gather (L2 hits?)
//   pf+now  : L2 prefetch immediately followed by the gather (in-flight misses merge?)
//   pf only : the prefetch kernel alone + spin until the prefetches have landed (how fast)
// Standalone tool: not part of the product library.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChunk = 2048;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_prefetch(const uint8_t* host, const int* ids, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(host + (size_t)ids[i] * kChunk), "r"(kChunk) : "memory");
}
__global__ void k_prefetch_lines(const uint8_t* host, const int* ids, int n) {   // 16 x 128 B line prefetches
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * 16) {
    const uint8_t* p = host + (size_t)ids[i >> 4] * kChunk + (i & 15) * 128;
    asm volatile("prefetch.global.L2 [%0];" :: "l"(p) : "memory");
  }
}

// 8 chunks per CTA (threads 0..7 issue one bulk copy each), then a checksum of the smem tile
__global__ void k_gather(const uint8_t* host, const int* ids, int n, unsigned long long* sum) {
  __shared__ __align__(128) uint8_t buf[8 * kChunk];
  __shared__ __align__(8) uint64_t bar;
  const int c0 = blockIdx.x * 8, nc = min(8, n - c0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar)), "r"(nc * kChunk) : "memory");
  }
  __syncthreads();
  if (threadIdx.x < nc)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(su32(buf + threadIdx.x * kChunk)), "l"(host + (size_t)ids[c0 + threadIdx.x] * kChunk), "r"(kChunk),
                    "r"(su32(&bar)) : "memory");
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(su32(&bar)) : "memory");
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < nc * kChunk / 8; i += blockDim.x) s += reinterpret_cast<const unsigned long long*>(buf)[i];
  atomicAdd(sum, s);
}

__global__ void k_spin(long long ns) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
}

int main() {
  const size_t host_bytes = (size_t)1 << 30;             // 1 GiB pinned, mapped
  const int n = 2048;                                    // 4 MB of chunks
  uint8_t* h;
  CK(cudaHostAlloc(&h, host_bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < host_bytes / 8; ++i) reinterpret_cast<uint64_t*>(h)[i] = i * 0x9E3779B97F4A7C15ull;
  uint8_t* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  std::mt19937 rng(1);
  const int nch = (int)(host_bytes / kChunk);
  int* ids_d;
  unsigned long long* sum_d;
  CK(cudaMalloc(&ids_d, n * 4));
  CK(cudaMalloc(&sum_d, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto fresh_ids = [&]() {                                // a new random set each trial (no reuse in L2)
    std::vector<int> ids(n);
    for (int& x : ids) x = rng() % nch;
    CK(cudaMemcpy(ids_d, ids.data(), n * 4, cudaMemcpyHostToDevice));
    unsigned long long ref = 0;
    for (int x : ids) for (int j = 0; j < kChunk / 8; ++j) ref += reinterpret_cast<uint64_t*>(h + (size_t)x * kChunk)[j];
    return ref;
  };
  auto check = [&](unsigned long long ref) {
    unsigned long long s; CK(cudaMemcpy(&s, sum_d, 8, cudaMemcpyDeviceToHost)); return s == ref;
  };
  const int gb = (n + 7) / 8;
  for (int mode = 0; mode < 6; ++mode) {
    const char* name[] = {"cold gather", "pf(bulk)+300us spin, gather", "pf(bulk) then gather at once",
                          "pf(lines)+300us spin, gather", "pf(bulk) kernel alone", "pf(bulk)+spin, gather twice (2nd)"};
    float best = 1e9, worst = 0; bool ok = true;
    for (int trial = 0; trial < 6; ++trial) {
      const unsigned long long ref = fresh_ids();
      CK(cudaMemset(sum_d, 0, 8));
      CK(cudaDeviceSynchronize());
      if (mode == 1 || mode == 5) { k_prefetch<<<(n + 255) / 256, 256>>>(hd, ids_d, n); k_spin<<<1, 32>>>(300000); }
      if (mode == 3) { k_prefetch_lines<<<(n * 16 + 255) / 256, 256>>>(hd, ids_d, n); k_spin<<<1, 32>>>(300000); }
      if (mode == 5) { k_gather<<<gb, 128>>>(hd, ids_d, n, sum_d); CK(cudaMemset(sum_d, 0, 8)); }
      CK(cudaEventRecord(e0));
      if (mode == 2) k_prefetch<<<(n + 255) / 256, 256>>>(hd, ids_d, n);
      if (mode == 4) k_prefetch<<<(n + 255) / 256, 256>>>(hd, ids_d, n);
      else k_gather<<<gb, 128>>>(hd, ids_d, n, sum_d);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (trial > 0) { best = ms < best ? ms : best; worst = ms > worst ? ms : worst; }
      if (mode != 4) ok = ok && check(ref);
    }
    printf("%-36s best %8.2f us  worst %8.2f us  (%.1f GB/s at best)  checksum %s\n", name[mode], best * 1e3, worst * 1e3,
           n * (double)kChunk / (best * 1e-3) / 1e9, mode == 4 ? "n/a" : (ok ? "ok" : "MISMATCH"));
  }
  return 0;
}
