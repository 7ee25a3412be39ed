// Programmatic-dependent-launch release latency: primary grid P (its CTAs stamp globaltimer at exit)
// -> dependent grid D launched with the PDL attribute (stamps right after griddepcontrol.wait).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void P(uint64_t* ts, int spin_ns, int trig, const int4* host, int4* sink) {
  if (trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (host) {                                  // zero-copy read of 4 KB per CTA from pinned host memory
    int4 v = host[(size_t)blockIdx.x * 256 + threadIdx.x];
    if (v.x == 12345) sink[threadIdx.x] = v;
  }
  uint64_t t0 = gt();
  if (blockIdx.x == 0) while (gt() - t0 < (uint64_t)spin_ns) {}      // one straggler CTA
  __syncthreads();
  if (threadIdx.x == 0) atomicMax((unsigned long long*)&ts[0], (unsigned long long)gt());
}
__global__ void Dk(uint64_t* ts) {
  if (threadIdx.x == 0) atomicMin((unsigned long long*)&ts[2], (unsigned long long)gt());   // CTA started
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicMin((unsigned long long*)&ts[1], (unsigned long long)gt());
}
// middle grid: no griddepcontrol.wait, busy for spin_ns, stamps its exit
__global__ void M(uint64_t* ts, int spin_ns) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint64_t t0 = gt();
  while (gt() - t0 < (uint64_t)spin_ns) {}
  __syncthreads();
  if (threadIdx.x == 0) atomicMax((unsigned long long*)&ts[3], (unsigned long long)gt());
}
static void launch_pdl_grid(void (*k)(uint64_t*), uint64_t* ts, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.stream = st;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, ts);
}
int main() {
  uint64_t* ts; cudaMalloc(&ts, 64);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int4 *hbuf, *dbuf, *sink; cudaHostAlloc(&hbuf, 2000 * 4096, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&dbuf, hbuf, 0); cudaMalloc(&sink, 4096);
  for (int host : {0, 1})
  for (int grid : {312, 2000})
    for (int trig : {0, 1})
      for (int rep = 0; rep < 3; ++rep) {
        uint64_t init[3] = {0, ~0ull, ~0ull};
        cudaMemcpy(ts, init, 24, cudaMemcpyHostToDevice);
        P<<<grid, 256, 0, st>>>(ts, 20000, trig, host ? dbuf : nullptr, sink);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, Dk, ts);
        cudaStreamSynchronize(st);
        uint64_t h[3]; cudaMemcpy(h, ts, 24, cudaMemcpyDeviceToHost);
        printf("host=%d P grid=%4d trigger=%d: D first CTA start %+8.2f us, D wait released %+6.2f us after P's last exit\n",
               host, grid, trig, ((double)h[2] - (double)h[0]) / 1e3, ((double)h[1] - (double)h[0]) / 1e3);
      }
  printf("--- P (host reads, trigger) -> M (no wait, busy S us) -> D (wait)\n");
  for (int spin : {0, 2000, 4000, 6000})
    for (int rep = 0; rep < 2; ++rep) {
      uint64_t init[4] = {0, ~0ull, ~0ull, 0};
      cudaMemcpy(ts, init, 32, cudaMemcpyHostToDevice);
      P<<<312, 256, 0, st>>>(ts, 20000, 1, dbuf, sink);
      {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(8); cfg.blockDim = dim3(128); cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, M, ts, spin);
      }
      launch_pdl_grid(Dk, ts, st);
      cudaStreamSynchronize(st);
      uint64_t h[4]; cudaMemcpy(h, ts, 32, cudaMemcpyDeviceToHost);
      printf("M busy %d ns: M exit %+6.2f us after P exit; D released %+6.2f us after P exit (%+6.2f after M exit)\n",
             spin, ((double)h[3] - (double)h[0]) / 1e3, ((double)h[1] - (double)h[0]) / 1e3, ((double)h[1] - (double)h[3]) / 1e3);
    }
  return 0;
}
