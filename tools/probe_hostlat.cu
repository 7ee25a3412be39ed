// Host-link LATENCY probe (value-cache regime): when only a few hundred scattered 2 KB
// value chunks miss the GPU cache, is the fetch bandwidth- or latency-bound?
//   (1) dependent single-chunk bulk copies (one thread): per-fetch latency, cold vs warm GPU TLB;
//   (2) N random chunks issued at once over 256 CTAs x 8 threads (the sparse kernel's issue
//       pattern): time until all have landed, for N = 32 .. 4096;
// for a plain (4 KB-page) host buffer and a 2 MB-aligned buffer advised MADV_HUGEPAGE before
// cudaHostRegister (whether larger host pages shorten the GPU's sysmem translations).
// Standalone tool: not part of the product library.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static constexpr int CB = 2048;

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
               :: "r"(su32(b)), "r"(ph) : "memory");
}

// (1) one thread, n dependent fetches; lat[i] = ns for fetch i
__global__ void k_chain(const uint8_t* host, const int* ids, int n, uint64_t* lat) {
  __shared__ __align__(128) uint8_t buf[CB];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x) return;
  mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int i = 0; i < n; ++i) {
    const uint64_t t0 = gtimer();
    expect_tx(&bar, CB);
    bulk(buf, host + (size_t)ids[i] * CB, CB, &bar);
    wait(&bar, i & 1);
    lat[i] = gtimer() - t0;
  }
}

// (2) grid of CTAs, thread t < 8 of CTA c fetches chunk c*8+t if < n; span[c] = landing time
__global__ void k_burst(const uint8_t* host, const int* ids, int n, uint64_t* t_start, uint64_t* t_end) {
  __shared__ __align__(128) uint8_t buf[8 * CB];
  __shared__ __align__(8) uint64_t bar;
  const int base = blockIdx.x * 8;
  const int cnt = min(8, n - base);
  if (cnt <= 0) return;
  if (threadIdx.x == 0) { mbar_init(&bar, cnt); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) t_start[blockIdx.x] = gtimer();
  if (threadIdx.x < cnt) {
    expect_tx(&bar, CB);
    bulk(buf + threadIdx.x * CB, host + (size_t)ids[base + threadIdx.x] * CB, CB, &bar);
  }
  wait(&bar, 0);
  if (threadIdx.x == 0) t_end[blockIdx.x] = gtimer();
}

static void run(const char* name, uint8_t* host, size_t bytes) {
  CK(cudaHostRegister(host, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  const int nchunks = (int)(bytes / CB);
  std::mt19937 rng(7);
  std::uniform_int_distribution<int> U(0, nchunks - 1);
  int* d_ids; uint64_t *d_lat, *d_t0, *d_t1;
  const int NMAX = 8192;
  CK(cudaMalloc(&d_ids, NMAX * 4)); CK(cudaMalloc(&d_lat, NMAX * 8));
  CK(cudaMalloc(&d_t0, NMAX * 8)); CK(cudaMalloc(&d_t1, NMAX * 8));
  std::vector<int> ids(NMAX);
  std::vector<uint64_t> lat(NMAX);
  // (1) cold then warm: 64 random chunks, then the same 64 again
  for (auto& x : ids) x = U(rng);
  CK(cudaMemcpy(d_ids, ids.data(), NMAX * 4, cudaMemcpyHostToDevice));
  for (int pass = 0; pass < 2; ++pass) {
    k_chain<<<1, 32>>>(host, d_ids, 64, d_lat);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(lat.data(), d_lat, 64 * 8, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> v(lat.begin(), lat.begin() + 64);
    std::sort(v.begin(), v.end());
    printf("%s chain %s: per-fetch latency p10=%.2f p50=%.2f p90=%.2f max=%.2f us\n", name, pass ? "warm" : "cold",
           v[6] / 1e3, v[32] / 1e3, v[57] / 1e3, v[63] / 1e3);
  }
  // sequential-neighbour chain: chunks inside one 2 MB region (same large page if any)
  for (int i = 0; i < 64; ++i) ids[i] = (U(rng) & ~1023) + i * 16;
  CK(cudaMemcpy(d_ids, ids.data(), 64 * 4, cudaMemcpyHostToDevice));
  k_chain<<<1, 32>>>(host, d_ids, 64, d_lat);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(lat.data(), d_lat, 64 * 8, cudaMemcpyDeviceToHost));
  {
    std::vector<uint64_t> v(lat.begin() + 1, lat.begin() + 64);
    std::sort(v.begin(), v.end());
    printf("%s chain same-2MB-region (32 KB stride): p50=%.2f max=%.2f us\n", name, v[31] / 1e3, v[62] / 1e3);
  }
  // (2) bursts
  for (int n : {32, 128, 256, 512, 1024, 2048, 4096}) {
    double best = 1e30, med_sum = 0;
    for (int rep = 0; rep < 5; ++rep) {
      for (int i = 0; i < n; ++i) ids[i] = U(rng);
      CK(cudaMemcpy(d_ids, ids.data(), n * 4, cudaMemcpyHostToDevice));
      const int grid = (n + 7) / 8;
      k_burst<<<grid, 256>>>(host, d_ids, n, d_t0, d_t1);
      CK(cudaDeviceSynchronize());
      std::vector<uint64_t> t0(grid), t1(grid);
      CK(cudaMemcpy(t0.data(), d_t0, grid * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(t1.data(), d_t1, grid * 8, cudaMemcpyDeviceToHost));
      uint64_t a = UINT64_MAX, b = 0;
      std::vector<double> per(grid);
      for (int c = 0; c < grid; ++c) { a = std::min(a, t0[c]); b = std::max(b, t1[c]); per[c] = (t1[c] - t0[c]) / 1e3; }
      std::sort(per.begin(), per.end());
      best = std::min(best, (b - a) / 1e3);
      med_sum += per[grid / 2];
    }
    printf("%s burst n=%5d (%7.1f KB): all landed after %7.2f us (best of 5) = %6.2f GB/s; per-CTA p50 %.2f us; "
           "bandwidth bound %.2f us\n", name, n, n * 2.0, best, n * 2048.0 / (best * 1e3), med_sum / 5,
           n * 2048.0 / 51.2e3);
  }
  CK(cudaHostUnregister(host));
  cudaFree(d_ids); cudaFree(d_lat); cudaFree(d_t0); cudaFree(d_t1);
}

int main() {
  const size_t bytes = (size_t)4 << 30;
  uint8_t* a = (uint8_t*)aligned_alloc(4096, bytes);
  memset(a, 1, bytes);
  run("4K-pages", a, bytes);
  free(a);
  uint8_t* h = (uint8_t*)aligned_alloc((size_t)2 << 20, bytes);
  int adv = madvise(h, bytes, MADV_HUGEPAGE);
  memset(h, 1, bytes);
  printf("madvise(MADV_HUGEPAGE) = %d\n", adv);
  run("THP", h, bytes);
  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  if (f) { char s[256] = {0}; fgets(s, sizeof s, f); printf("THP setting: %s", s); fclose(f); }
  f = fopen("/proc/meminfo", "r");
  if (f) { char s[256]; while (fgets(s, sizeof s, f)) if (strstr(s, "AnonHugePages") || strstr(s, "Hugepagesize")) printf("%s", s); fclose(f); }
  free(h);
  return 0;
}
