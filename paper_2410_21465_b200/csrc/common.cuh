// Shared device helpers for the ShadowKV sm_100a kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace skv {

constexpr int kHeadDim = 128;   // d (compiled)
constexpr int kChunk = 8;       // c (compiled), P:103 / P:273

__device__ __forceinline__ float bf2f(uint16_t v) { return __uint_as_float(((uint32_t)v) << 16); }
__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// round-to-nearest-even fp32 -> bf16 bits (inputs are finite here)
__device__ __forceinline__ uint16_t f2bf(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  return (uint32_t)f2bf(lo) | ((uint32_t)f2bf(hi) << 16);
}

// 8 bf16 (16 B) -> 8 fp32
__device__ __forceinline__ void unpack8(const uint4 v, float* f) {
  f[0] = bf_lo(v.x); f[1] = bf_hi(v.x); f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
  f[4] = bf_lo(v.z); f[5] = bf_hi(v.z); f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
}

// streaming 16 B load that bypasses L1 allocation (HBM streams, host-mapped reads)
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// RoPE angle phi = fl32(fl32(t) * inv_freq) (R15) and its sine / cosine.  Positions reach 2^20, so phi
// reaches ~1e6 rad, where sincosf takes its slow (Payne-Hanek, local-memory) path.  phi is reduced
// modulo 2 pi in fp64 instead (two-term 2 pi, |k| < 2^18: error < 1e-10 rad), then the fast path
// hardware approximation runs on |r| <= pi (abs error < 1e-6, far inside the key tolerance, R23).
__device__ __forceinline__ void rope_sincos(int t, float inv_freq, float* s, float* c) {
  const float phi = __fmul_rn((float)t, inv_freq);
  const double x = (double)phi;
  const double k = rint(x * 0.15915494309189535);
  double r = fma(-k, 6.283185307179586, x);
  r = fma(-k, 2.4492935982947064e-16, r);
  __sincosf((float)r, s, c);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}

// order-preserving map float -> uint32 (larger float -> larger key); -0 canonicalised to +0
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// merge two (max, sum-of-exp) softmax partials
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  float mn = fmaxf(m, m2);
  if (mn == -INFINITY) { m = mn; s = 0.f; return; }
  s = s * expf(m - mn) + s2 * expf(m2 - mn);
  m = mn;
}

}  // namespace skv

// ---------------------------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA 1D, cp.async.bulk) helpers
// ---------------------------------------------------------------------------------------------
namespace skv {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
// Bounded polling: a flag that never arrives (a bug, or a grid that cannot become resident) aborts the
// kernel with an error after ~2 s instead of hanging the device.  Call with the spin's start time.
__device__ __forceinline__ void spin_guard(uint64_t t0) {
  if (globaltimer() - t0 > 2000000000ull) __trap();
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// Every mbarrier wait is bounded like the flag polls (spin_guard): a phase that never completes (a lost
// TMA / tcgen05 completion, a bug) traps after ~2 s -- a sticky launch error the caller sees -- instead of
// leaving the device hung.  The first try_wait (which itself suspends for a while) is the common exit.
// (the bounded loop is out of line: inlined, its timer registers raise the register pressure of the
// attention kernel)
static __device__ __noinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait(bar, parity)) spin_guard(t0);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (!mbar_try_wait(bar, parity)) mbar_wait_bounded(bar, parity);
}
// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive_plain(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
// global (device or host-mapped) -> shared, completion signalled on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// shared -> global bulk copy (bulk-group completion; bytes % 16 == 0); wait_read: the smem source may
// be reused / the CTA may exit once the copies have read it
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// G consecutive floats (16-byte aligned when G % 4 == 0) stored / loaded as vectors
template <int G>
__device__ __forceinline__ void store_row(float* dst, const float* x) {
  if constexpr (G % 4 == 0) {
#pragma unroll
    for (int i = 0; i < G; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
  } else if constexpr (G == 2) {
    *reinterpret_cast<float2*>(dst) = make_float2(x[0], x[1]);
  } else {
#pragma unroll
    for (int i = 0; i < G; ++i) dst[i] = x[i];
  }
}
template <int G>
__device__ __forceinline__ void load_row(const float* src, float* x) {
  if constexpr (G % 4 == 0) {
#pragma unroll
    for (int i = 0; i < G; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + i);
      x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
    }
  } else if constexpr (G == 2) {
    const float2 v = *reinterpret_cast<const float2*>(src);
    x[0] = v.x; x[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < G; ++i) x[i] = src[i];
  }
}

// 8-byte {value, flag} pairs (the LL-protocol idiom), accessed as ONE 64-bit relaxed.gpu scalar (single-copy
// atomic): a reader that sees the flag sees the value written with it -- no fence on the writer's side (a
// release on an SM with host reads in flight waits for all of them, tools/probe_fence.cu)
__device__ __forceinline__ void st_tagged(uint2* p, float v, unsigned tag) {
  const unsigned long long x = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ uint2 ld_tagged(const uint2* p) {
  unsigned long long x;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  return make_uint2((unsigned)x, (unsigned)(x >> 32));
}
__device__ __forceinline__ unsigned ld_volatile_u32(const int* p) {
  unsigned r;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

// programmatic dependent launch (PDL)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace skv

// ---------------------------------------------------------------------------------------------
// cluster / DSMEM helpers
// ---------------------------------------------------------------------------------------------
namespace skv {
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Split cluster barrier.  A release-arrive waits until this thread's earlier global stores are
// performed, which on an SM with PCIe reads in flight can take tens of microseconds: arrive before
// issuing global stores (or with .relaxed when only smem lifetime is at stake), wait after them.
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same smem variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank)); return r;
}
// DSMEM reads of data published before a cluster barrier (the barrier asm is the compiler fence);
// not volatile so independent remote loads can be issued back to back
__device__ __forceinline__ int ld_dsmem_i32(uint32_t a) {
  int v; asm("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a)); return v;
}
__device__ __forceinline__ void st_dsmem_i32(uint32_t a, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}
// 16 B store into a peer CTA's smem that completes 16 bytes of tx on the peer's mbarrier (both
// shared::cluster addresses from dsmem_addr)
__device__ __forceinline__ void st_async_v4(uint32_t a, int4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.s32 [%0], {%1, %2, %3, %4}, [%5];"
               :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t a) {
  float v; asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// release-ordered fetch-add (orders this thread's earlier writes, and those made visible to it by
// a CTA barrier, before the add: cumulativity) / acquire fence for the thread that observes it
__device__ __forceinline__ int atom_add_release_gpu(int* p, int v) {
  int old; asm volatile("atom.add.release.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// relaxed (coherent at gpu scope, unordered): for values that are their own payload, e.g. a
// published chunk id that a consumer polls for
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v; asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// spin (with backoff) until flag[0] != 0, then return flag[1] (read with acquire semantics by one
// thread and broadcast through shared memory, so no thread can see a stale L1 copy)
__device__ __forceinline__ int cta_wait_flag(const int* flag) {
  __shared__ int bcast;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_gpu(flag) == 0) { __nanosleep(64); spin_guard(t0); }
    bcast = ld_acquire_gpu(flag + 1);
  }
  __syncthreads();
  return bcast;
}
}  // namespace skv
