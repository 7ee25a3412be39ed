// Host-link probe: how fast can a B200 pull scattered 2 KB
// value chunks (8 tokens x 128 dims x bf16, "Gather values from
// CPU") out of pinned, mapped host memory?  Measures
//   (1) pinned H2D cudaMemcpyAsync (copy-engine DMA) for reference,
//   (2) zero-copy LDG.128 sequential and random-2KB gathers at several depths,
//   (3) cp.async.bulk (TMA bulk copy) from host-mapped memory into smem.
// Standalone tool: not part of the product library.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static constexpr int CHUNK_BYTES = 2048;

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// One warp moves UNROLL chunks per iteration; lane i reads 16 B at i, i+32, ...
template <int UNROLL>
__global__ void gather_ldg(const uint8_t* __restrict__ host, const int* __restrict__ ids,
                           int n, uint8_t* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int c0 = warp * UNROLL; c0 < n; c0 += nwarps * UNROLL) {
    int4 v[UNROLL][4];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int c = c0 + u;
      if (c < n) {
        const int4* src = reinterpret_cast<const int4*>(host + (size_t)ids[c] * CHUNK_BYTES);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[u][j] = ld_nc(src + lane + 32 * j);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int c = c0 + u;
      if (c < n) {
        int4* d = reinterpret_cast<int4*>(dst + (size_t)c * CHUNK_BYTES);
#pragma unroll
        for (int j = 0; j < 4; ++j) d[lane + 32 * j] = v[u][j];
      }
    }
  }
}

// cp.async.bulk global->shared, one elected thread per warp issues DEPTH chunks,
// waits on an mbarrier, then the warp writes them back to HBM.
template <int DEPTH>
__global__ void gather_bulk(const uint8_t* __restrict__ host, const int* __restrict__ ids,
                            int n, uint8_t* __restrict__ dst) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  uint8_t* buf = smem + (size_t)wib * DEPTH * CHUNK_BYTES;
  uint32_t bar_addr = (uint32_t)__cvta_generic_to_shared(&bar[wib]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  uint32_t phase = 0;
  for (int c0 = warp * DEPTH; c0 < n; c0 += nwarps * DEPTH) {
    int cnt = min(DEPTH, n - c0);
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   :: "r"(bar_addr), "r"(cnt * CHUNK_BYTES));
      for (int u = 0; u < cnt; ++u) {
        const uint8_t* src = host + (size_t)ids[c0 + u] * CHUNK_BYTES;
        uint32_t d = (uint32_t)__cvta_generic_to_shared(buf + u * CHUNK_BYTES);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(d), "l"(src), "r"(CHUNK_BYTES), "r"(bar_addr) : "memory");
      }
    }
    // wait
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}" :: "r"(bar_addr), "r"(phase) : "memory");
    phase ^= 1;
    for (int u = 0; u < cnt; ++u) {
      const int4* s = reinterpret_cast<const int4*>(buf + u * CHUNK_BYTES);
      int4* d = reinterpret_cast<int4*>(dst + (size_t)(c0 + u) * CHUNK_BYTES);
#pragma unroll
      for (int j = 0; j < 4; ++j) d[lane + 32 * j] = s[lane + 32 * j];
    }
    __syncwarp();
  }
}

static bool verify(const uint8_t* host, const std::vector<int>& ids, const uint8_t* dev_dst, int n) {
  std::vector<uint8_t> h((size_t)n * CHUNK_BYTES);
  CK(cudaMemcpy(h.data(), dev_dst, h.size(), cudaMemcpyDeviceToHost));
  for (int c = 0; c < n; c += 97)
    for (int b = 0; b < CHUNK_BYTES; b += 61)
      if (h[(size_t)c * CHUNK_BYTES + b] != host[(size_t)ids[c] * CHUNK_BYTES + b]) return false;
  return true;
}

int main(int argc, char** argv) {
  size_t host_bytes = (argc > 1 ? atoll(argv[1]) : 4096ll) << 20;   // MiB
  int n = argc > 2 ? atoi(argv[2]) : 32768;                          // chunks per launch (64 MiB)
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int canmap = 0; CK(cudaDeviceGetAttribute(&canmap, cudaDevAttrCanMapHostMemory, 0));
  int hostptr = 0; CK(cudaDeviceGetAttribute(&hostptr, cudaDevAttrCanUseHostPointerForRegisteredMem, 0));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  printf("sms=%d canMapHost=%d hostPtrForRegistered=%d L2=%d MiB host_buf=%zu MiB chunks=%d\n",
         sms, canmap, hostptr, l2 >> 20, host_bytes >> 20, n);

  uint8_t* host = nullptr;
  CK(cudaHostAlloc(&host, host_bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < host_bytes; i += 4096) host[i] = (uint8_t)(i * 2654435761u >> 13);
  for (size_t i = 0; i < host_bytes; i += 61) host[i] = (uint8_t)(i * 40503u >> 7);
  uint8_t* hdev = nullptr; CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
  printf("host=%p devptr=%p same=%d\n", host, hdev, (void*)host == (void*)hdev);

  uint8_t* dst; CK(cudaMalloc(&dst, (size_t)n * CHUNK_BYTES));
  uint8_t* big; CK(cudaMalloc(&big, 1ull << 30));
  int* dids; CK(cudaMalloc(&dids, n * sizeof(int)));
  size_t nchunks_host = host_bytes / CHUNK_BYTES;
  std::mt19937_64 rng(1234);
  std::vector<int> rnd(n), seq(n);
  for (int i = 0; i < n; ++i) { rnd[i] = (int)(rng() % nchunks_host); seq[i] = i; }

  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto time_it = [&](auto&& fn, int reps) {
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(e0)); fn(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms);
    }
    return best;
  };

  // (1) DMA H2D
  {
    float ms = time_it([&] { CK(cudaMemcpyAsync(big, host, 1ull << 30, cudaMemcpyHostToDevice)); }, 10);
    printf("DMA_H2D_1GiB: %.2f GB/s\n", (1ull << 30) / ms / 1e6);
    ms = time_it([&] { CK(cudaMemcpyAsync(host, big, 1ull << 30, cudaMemcpyDeviceToHost)); }, 5);
    printf("DMA_D2H_1GiB: %.2f GB/s\n", (1ull << 30) / ms / 1e6);
    float ms4 = time_it([&] { CK(cudaMemcpyAsync(big, host, 4u << 20, cudaMemcpyHostToDevice)); }, 20);
    printf("DMA_H2D_4MiB: %.2f GB/s (%.1f us)\n", (4u << 20) / ms4 / 1e6, ms4 * 1e3);
  }
  // re-fill host pattern for verify (D2H overwrote the first GiB)
  for (size_t i = 0; i < host_bytes; i += 61) host[i] = (uint8_t)(i * 40503u >> 7);

  for (int pattern = 0; pattern < 2; ++pattern) {
    const std::vector<int>& ids = pattern ? rnd : seq;
    const char* pname = pattern ? "random2KB" : "sequential";
    CK(cudaMemcpy(dids, ids.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    for (int bpsm : {1, 2, 4, 8}) {
      for (int threads : {128, 256, 512}) {
        int grid = sms * bpsm;
        float ms;
        ms = time_it([&] { gather_ldg<1><<<grid, threads>>>(hdev, dids, n, dst); }, 5);
        CK(cudaGetLastError());
        printf("LDG %s U1 grid=%d thr=%d: %.2f GB/s ok=%d\n", pname, grid, threads,
               (double)n * CHUNK_BYTES / ms / 1e6, verify(host, ids, dst, n));
        ms = time_it([&] { gather_ldg<2><<<grid, threads>>>(hdev, dids, n, dst); }, 5);
        printf("LDG %s U2 grid=%d thr=%d: %.2f GB/s\n", pname, grid, threads,
               (double)n * CHUNK_BYTES / ms / 1e6);
        ms = time_it([&] { gather_ldg<4><<<grid, threads>>>(hdev, dids, n, dst); }, 5);
        printf("LDG %s U4 grid=%d thr=%d: %.2f GB/s\n", pname, grid, threads,
               (double)n * CHUNK_BYTES / ms / 1e6);
      }
    }
    for (int depth_sel = 0; depth_sel < 3; ++depth_sel) {
      for (int bpsm : {1, 2, 4}) {
        int threads = 128, grid = sms * bpsm;
        float ms = 0; size_t sm = 0;
        if (depth_sel == 0) { sm = 4 * 2 * CHUNK_BYTES;
          CK(cudaFuncSetAttribute(gather_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          ms = time_it([&] { gather_bulk<2><<<grid, threads, sm>>>(hdev, dids, n, dst); }, 5); }
        if (depth_sel == 1) { sm = 4 * 4 * CHUNK_BYTES;
          CK(cudaFuncSetAttribute(gather_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          ms = time_it([&] { gather_bulk<4><<<grid, threads, sm>>>(hdev, dids, n, dst); }, 5); }
        if (depth_sel == 2) { sm = 4 * 8 * CHUNK_BYTES;
          CK(cudaFuncSetAttribute(gather_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          ms = time_it([&] { gather_bulk<8><<<grid, threads, sm>>>(hdev, dids, n, dst); }, 5); }
        cudaError_t err = cudaGetLastError();
        printf("BULK %s depth=%d grid=%d: %.2f GB/s ok=%d err=%s\n", pname, 2 << depth_sel, grid,
               (double)n * CHUNK_BYTES / ms / 1e6, err == cudaSuccess ? verify(host, ids, dst, n) : 0,
               cudaGetErrorString(err));
      }
    }
  }
  // small-launch latency: a 4 MiB gather (one c2 layer) at the best-looking config
  {
    int n4 = 2048;
    CK(cudaMemcpy(dids, rnd.data(), n4 * sizeof(int), cudaMemcpyHostToDevice));
    for (int bpsm : {1, 2, 4}) for (int threads : {128, 256, 512}) {
      float ms = time_it([&] { gather_ldg<1><<<sms * bpsm, threads>>>(hdev, dids, n4, dst); }, 20);
      printf("LDG 4MiB-layer U1 grid=%d thr=%d: %.1f us  %.2f GB/s\n", sms * bpsm, threads, ms * 1e3,
             (double)n4 * CHUNK_BYTES / ms / 1e6);
    }
    size_t sm = 4 * 4 * CHUNK_BYTES;
    for (int bpsm : {1, 2, 4}) {
      float ms = time_it([&] { gather_bulk<4><<<sms * bpsm, 128, sm>>>(hdev, dids, n4, dst); }, 20);
      printf("BULK 4MiB-layer depth4 grid=%d: %.1f us  %.2f GB/s\n", sms * bpsm, ms * 1e3,
             (double)n4 * CHUNK_BYTES / ms / 1e6);
    }
  }
  printf("done\n");
  return 0;
}
