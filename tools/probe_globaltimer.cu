// Cost of reading %globaltimer vs clock64 from one thread (tracing overhead check).
#include <cstdio>
#include <cstdint>
__global__ void k(uint64_t* out, int n) {
  if (threadIdx.x != 0) return;
  uint64_t g0, g1, c0, c1, x = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  c0 = clock64();
  for (int i = 0; i < n; ++i) { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); x += t; }
  c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  out[0] = (c1 - c0); out[1] = g1 - g0; out[2] = x;
  // distinct values seen in a tight loop: timer granularity
  uint64_t prev = 0, changes = 0, first = 0, last = 0;
  for (int i = 0; i < 20000; ++i) {
    uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { if (!first) first = t; last = t; ++changes; prev = t; }
  }
  out[3] = changes; out[4] = last - first;
}
int main() {
  uint64_t* d; cudaMalloc(&d, 64);
  uint64_t h[5];
  for (int n : {1, 16, 256}) {
    k<<<1, 32>>>(d, n); cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("n=%d reads: %.1f cycles/read, %.1f ns/read (wall %llu ns); granularity: %llu changes over %llu ns -> %.1f ns/tick\n",
           n, (double)h[0] / n, (double)h[1] / n, (unsigned long long)h[1], (unsigned long long)h[3],
           (unsigned long long)h[4], h[3] > 1 ? (double)h[4] / (h[3] - 1) : 0.0);
  }
  return 0;
}
