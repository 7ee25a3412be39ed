// a1 landmark scoring on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   P = Q . L^T / sqrt(d)   (Alg 2 "P <- MatMul(Q, L^T)"; scale R6)
//
// One UMMA per 16-wide k step: M = 128 landmark rows (A, K-major, SWIZZLE_128B, streamed from HBM
// by TMA in two 64-column boxes), N = 16 query heads of the GQA group (B, zero-padded, built once
// per KV head in smem), K = 128 = head_dim, fp32 accumulators in TMEM (8 x 16 columns).  Warp
// roles (608 threads): 4 epilogue groups of 4 warps (0-3, 7-10, 11-14, 15-18; TMEM lane quadrant =
// warp % 4) on tiles i % 4, warp 4 TMA producer,
// warps 5-6 MMA issuers on alternate tiles (measured: one issuing thread is paced at ~70 cycles
// per tcgen05.mma at any N <= 128, two on different sub-partitions reach ~40, the rate at which
// the tensor core reads the 4 KB A operand from smem; tools/probe_umma.cu).  The epilogue reads
// each landmark's G logits with tcgen05.ld, masks outlier chunks (R3), writes the scaled logits
// and one softmax partial (max, sum exp) per tile and query row, which k_select merges in a fixed
// order into the exact per-head log-sum-exp.  The first ring fills are issued before griddepcontrol.wait: landmarks
// are layer state that no decode-step kernel writes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdlib>

#include "append.cuh"
#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace skv {

namespace {

constexpr int kTcStages = 6;
constexpr int kTcAcc = 8;                 // TMEM accumulator buffers (16 fp32 columns each)
constexpr int kTcMaxHeads = 4;            // KV heads a CTA's contiguous tile range may touch
constexpr int kTcMaxTiles = 64;           // tiles per CTA (outlier bitmap size); the plan never exceeds it
constexpr int kTcEpiGroups = 4;         // epilogue groups of 4 warps (one per TMEM lane quadrant), alternate tiles
constexpr int kTcThreads = (4 * kTcEpiGroups + 3) * 32;   // + 1 TMA producer, 2 MMA issuers
constexpr uint32_t kTileBytes = kSTile * kHeadDim * 2;   // 32 KB: two 16 KB SW128 boxes
constexpr uint32_t kBBytes = 16 * kHeadDim * 2;          // 4 KB: B operand of one head

// Landmarks are streamed once per decode step and never re-read within it: they are loaded with an L2
// evict-first policy so that they do not push the freshly written logits (re-read by k_select) and
// the small per-step state out of L2 (c3/c5 stream 0.2-2 GB of landmarks per layer through 126 MB).

// kind::f16 instruction descriptor: A,B bf16 K-major, D fp32, M = 128, N = 16.
constexpr uint32_t kIdesc = umma_idesc_bf16(128, 16, false, false);

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool in_sorted(const int32_t* ids, int o, int j) {
  int lo = 0, hi = o;
  while (lo < hi) { int mid = (lo + hi) >> 1; if (ids[mid] < j) lo = mid + 1; else hi = mid; }
  return lo < o && ids[lo] == j;
}

__device__ uint64_t* g_trace_tc = nullptr;              // same layout as decode.cu's trace buffer
__device__ __forceinline__ void trace_tc(uint64_t* t, int ev) {
  if (t != nullptr && threadIdx.x == 0) t[(size_t)blockIdx.x * 16 + ev] = globaltimer();
}
__device__ __forceinline__ void trace_tc_any(uint64_t* t, int ev) {   // caller restricts to one thread
  if (t != nullptr) t[(size_t)blockIdx.x * 16 + ev] = globaltimer();
}


__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }
// Reduce-scatter of G values per lane over the warp (max or sum): rounds xor 16, 8, ... halve the payload
// while it has more than one value, then finish with single-value rounds.  Lane l returns the reduction of
// row (l >> (5 - log2 G)) over all 32 lanes.
template <int G, bool kMax>
__device__ __forceinline__ float rs_reduce(float (&v)[G], int lane) {
  int n = G;
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    if (n > 1) {
      const int half = n >> 1;
      const bool up = (lane & m) != 0;
#pragma unroll
      for (int i = 0; i < G / 2; ++i) {
        if (i < half) {
          const float send = up ? v[i] : v[i + half];
          const float keep = up ? v[i + half] : v[i];
          const float got = __shfl_xor_sync(0xffffffffu, send, m);
          v[i] = kMax ? fmaxf(keep, got) : keep + got;
        }
      }
      n = half;
    } else {
      const float got = __shfl_xor_sync(0xffffffffu, v[0], m);
      v[0] = kMax ? fmaxf(v[0], got) : v[0] + got;
    }
  }
  return v[0];
}
}  // namespace

cudaError_t set_trace_buffer_tc(void* p) { return cudaMemcpyToSymbol(g_trace_tc, &p, sizeof(void*)); }

template <int G>
__global__ void __launch_bounds__(kTcThreads, 1)
k_score_tc(const __grid_constant__ CUtensorMap tmap, Dims D, const int32_t* __restrict__ oids,
           const uint16_t* __restrict__ q, float* __restrict__ logits, float2* __restrict__ part,
           int tiles_per_head, float scale, const uint16_t* __restrict__ k_new,
           const uint16_t* __restrict__ v_new, uint16_t* K_win, uint16_t* V_win, int step) {
  static_assert(G <= 16, "N = 16 covers the GQA group");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* sA = smem;                                          // [stages][32 KB]
  uint8_t* sB = smem + kTcStages * kTileBytes;                 // [kTcMaxHeads][4 KB]
  __shared__ __align__(8) uint64_t full[kTcStages], empty[kTcStages], acc_full[kTcAcc], acc_empty[kTcAcc];
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t obits[kTcMaxTiles * (kSTile / 32)];
  __shared__ float2 wpart[kTcEpiGroups][2][4][16];             // [group][tile parity][warp][row]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = D.b * D.hk * tiles_per_head;
  const int t_begin = (int)((long long)blockIdx.x * total / gridDim.x);
  const int t_end = (int)((long long)(blockIdx.x + 1) * total / gridDim.x);
  const int ntile = t_end - t_begin;
  const int bh0 = t_begin / tiles_per_head;
  uint64_t* const trace_buf = g_trace_tc ? g_trace_tc + (size_t)D.trace_slot * kTraceSlot : nullptr;
  const uint64_t pol = l2_evict_first_policy();
  trace_tc(trace_buf, 0);
  // the producer thread initialises the barriers and puts the first kTcStages tiles in flight
  // before anything else, so HBM streaming starts at kernel entry
  if (tid == 4 * 32 && ntile > 0) {
    for (int s = 0; s < kTcStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < kTcAcc; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&acc_empty[s], 4); }
    fence_mbar_init();
    prefetch_tensormap(&tmap);
  }
  if (warp == 0 && ntile > 0) {                        // TMEM: 8 accumulator buffers x 16 fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // landmarks are layer state written by build_cache, never by a decode-step kernel: the first ring
  // fills do not depend on the preceding grid and stream while it drains (PDL prologue)
  if (tid == 4 * 32 && ntile > 0) {
    for (int i = 0; i < ntile && i < kTcStages; ++i) {
      const int t = t_begin + i, bh = t / tiles_per_head, tile = t - bh * tiles_per_head;
      const int row0 = bh * D.n_c + tile * kSTile;
      mbar_expect_tx(&full[i], kTileBytes);
      tma_load_2d(sA + i * kTileBytes, &tmap, 0, row0, &full[i], pol);
      tma_load_2d(sA + i * kTileBytes + kTileBytes / 2, &tmap, 64, row0, &full[i], pol);
    }
  }
  if (ntile <= 0) { pdl_wait(); return; }
  const int nheads = (t_end - 1) / tiles_per_head - bh0 + 1;          // <= kTcMaxHeads (host check)
  // outlier bitmap of this CTA's landmark rows (R3): layer state, built before the PDL wait
  const int row_begin = t_begin * kSTile;
  for (int w = tid; w < ntile * (kSTile / 32); w += kTcThreads) obits[w] = 0u;
  __syncthreads();
  for (int i = tid; i < nheads * D.o; i += kTcThreads) {
    const int bh = bh0 + i / D.o, j = oids[(size_t)bh * D.o + i % D.o];
    const int tr = bh * tiles_per_head * kSTile + j - row_begin;      // row in this CTA's tile space
    if (tr >= 0 && tr < ntile * kSTile) atomicOr(&obits[tr >> 5], 1u << (tr & 31));
  }
  pdl_wait();                                          // everything below may read the caller's inputs
  // every CTA of this grid is resident: the selector grid may launch now (its CTAs are dispatched the
  // moment ours exit; its own griddepcontrol.wait orders it after this grid's logits and partials)
  pdl_trigger();
  trace_tc(trace_buf, 15);
  // B operands (q of each KV head in range, K-major SWIZZLE_128B, rows n >= G zero) and the a7
  // window append (R18): call inputs, after the wait
  constexpr int kBChunks = kTcMaxHeads * 16 * 16;
  uint4 qv[(kBChunks + kTcThreads - 1) / kTcThreads];
#pragma unroll
  for (int u = 0; u < (kBChunks + kTcThreads - 1) / kTcThreads; ++u) {
    const int i = tid + u * kTcThreads;
    const int hi = i >> 8, n = (i >> 4) & 15, ch = i & 15;
    qv[u] = make_uint4(0, 0, 0, 0);
    if (i < nheads * 256 && n < G) {
      const int bh = bh0 + hi, b = bh / D.hk, h = bh - b * D.hk;
      qv[u] = *reinterpret_cast<const uint4*>(q + ((size_t)b * D.hq + (size_t)h * G + n) * kHeadDim + ch * 8);
    }
  }
  const int stp = D.step_dev ? min(max(ld_acquire_gpu(D.step_dev), 0), D.max_step) : step;
  window_append(D, k_new, v_new, K_win, V_win, stp, blockIdx.x * kTcThreads + tid, gridDim.x * kTcThreads);
#pragma unroll
  for (int u = 0; u < (kBChunks + kTcThreads - 1) / kTcThreads; ++u) {
    const int i = tid + u * kTcThreads;
    if (i < nheads * 256) {
      const int hi = i >> 8, n = (i >> 4) & 15, ch = i & 15;
      const int sub = ch >> 3, c16 = ch & 7;
      *reinterpret_cast<uint4*>(sB + hi * kBBytes + sub * 2048 + n * 128 + ((c16 ^ (n & 7)) << 4)) = qv[u];
    }
  }
  trace_tc(trace_buf, 6);
  fence_proxy_async();                                    // B (generic writes) -> UMMA (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  trace_tc(trace_buf, 7);                                         // setup done

  if (warp == 4) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int i = kTcStages; i < ntile; ++i) {
        const int s = i % kTcStages, ph = (i / kTcStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int t = t_begin + i, bh = t / tiles_per_head, tile = t - bh * tiles_per_head;
        const int row0 = bh * D.n_c + tile * kSTile;
        mbar_expect_tx(&full[s], kTileBytes);
        tma_load_2d(sA + s * kTileBytes, &tmap, 0, row0, &full[s], pol);
        tma_load_2d(sA + s * kTileBytes + kTileBytes / 2, &tmap, 64, row0, &full[s], pol);
      }
    }
  } else if (warp == 5 || warp == 6) {
    // ---------------- MMA issuers: one thread each on two SM sub-partitions, alternating tiles ----------
    // (a single issuing thread is paced at ~70 cycles per tcgen05.mma; two overlap to the smem-read bound)
    if (lane == 0) {
      for (int i = warp - 5; i < ntile; i += 2) {
        const int s = i % kTcStages, ph = (i / kTcStages) & 1, buf = i % kTcAcc, aph = (i / kTcAcc) & 1;
        mbar_wait(&full[s], ph);
        if (i < 4) trace_tc_any(trace_buf, 2 + i);                  // tile i landed in smem
        mbar_wait(&acc_empty[buf], aph ^ 1);
        tc_fence_after();
        const int hi = (t_begin + i) / tiles_per_head - bh0;
        const uint32_t a0 = smem_u32(sA + s * kTileBytes), b0 = smem_u32(sB + hi * kBBytes);
#pragma unroll
        for (int k = 0; k < kHeadDim / 16; ++k) {
          const uint32_t koff = (k >> 2) * (kTileBytes / 2) + (k & 3) * 32;
          const uint32_t kboff = (k >> 2) * 2048 + (k & 3) * 32;
          umma_f16(tmem + buf * 16, umma_desc_sw128(a0 + koff), umma_desc_sw128(b0 + kboff), kIdesc, k > 0);
        }
        umma_commit(&empty[s]);          // smem stage may be refilled once these MMAs retire
        umma_commit(&acc_full[buf]);     // accumulator ready for the epilogue
        if (i == 0) trace_tc_any(trace_buf, 12);                    // tile 0's MMAs issued
      }
    }
  } else {
    // ---------------- epilogue: 4 groups of 4 warps (0-3, 7-10, 11-14, 15-18), tile i -> group i % 4 ------
    // Warp w reads TMEM lane quadrant w % 4 (32 landmark rows).  Per tile and query row it writes the
    // logits and ONE softmax partial (max, sum exp) of the tile's 128 landmarks: the four warps' partials
    // meet in smem behind one named barrier of the group and warp quad 0 merges them in a fixed order.
    // A KV head's lse is then the fixed-order merge of its tiles' partials (k_select), independent of
    // how tiles are spread over CTAs: a (request, KV head)'s result does not depend on the batch it
    // runs in (batch / head sharding is bit-exact).  Log2 domain; a finite floor stands in for -inf so
    // fully masked rows never produce inf - inf.
    constexpr float kFloor = -1e30f, kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
    const int grp = warp < 4 ? 0 : (warp - 7) / 4 + 1, quad = warp & 3;
    int bh = t_begin / tiles_per_head, tile = t_begin - bh * tiles_per_head;   // advanced incrementally
    for (int k = 0; k < grp && k < ntile; ++k) { if (++tile == tiles_per_head) { tile = 0; ++bh; } }
    int cur_bh = -1;
    float* lrow = nullptr;
    float2* prow = nullptr;
    int ncb = 0;
    const int r = 32 * quad + lane;
    for (int i = grp; i < ntile; i += kTcEpiGroups) {
      const int buf = i % kTcAcc, aph = (i / kTcAcc) & 1, par = (i / kTcEpiGroups) & 1;
      if (bh != cur_bh) {
        cur_bh = bh;
        const int b = bh / D.hk, h = bh - b * D.hk;
        lrow = logits + (size_t)(b * D.hq + h * G) * D.n_c;
        prow = part + (size_t)(b * D.hq + h * G) * tiles_per_head;
        ncb = req_nc(D, b);                               // ragged batch: chunks past it are masked
      }
      mbar_wait(&acc_full[buf], aph);
      tc_fence_after();
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * quad) << 16) + buf * 16, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      const int j = tile * kSTile + r;
      const bool out = ((obits[(i * kSTile + r) >> 5] >> (r & 31)) & 1u) || j >= ncb || j >= D.n_c;
      if (warp == 0 && lane == 0 && i < 4) trace_tc_any(trace_buf, 8 + i);   // epilogue got tile i
      float xs[G];
#pragma unroll
      for (int hq = 0; hq < G; ++hq) xs[hq] = out ? -INFINITY : v[hq] * scale;
      if (j < D.n_c) store_row<G>(lrow + (size_t)j * G, xs);   // landmark-major logits [n_c][G]
      // the warp's softmax partial per query row over its 32 landmarks: a reduce-scatter of the G row
      // values (the lane ends with row r_lane's max), an all-gather of the G maxima, then a reduce-scatter
      // of the exps: 3G + 5 - log2 G shuffles instead of 10G
      {
        float x2[G], e[G];
#pragma unroll
        for (int hq = 0; hq < G; ++hq) { x2[hq] = out ? kFloor : xs[hq] * kLog2e; e[hq] = x2[hq]; }
        const float mr = rs_reduce<G, true>(e, lane);          // max of row r_lane
        constexpr int kSh = 5 - ilog2(G);                       // row r lives in lanes (r << kSh) + ...
#pragma unroll
        for (int hq = 0; hq < G; ++hq) {
          const float m = __shfl_sync(0xffffffffu, mr, hq << kSh);
          e[hq] = out ? 0.f : exp2f(x2[hq] - m);
        }
        const float sr = rs_reduce<G, false>(e, lane);         // sum of row r_lane
        if ((lane & ((1 << kSh) - 1)) == 0) wpart[grp][par][quad][lane >> kSh] = make_float2(mr, sr);
      }
      asm volatile("bar.sync %0, 128;" :: "r"(grp + 1) : "memory");   // the group's 4 warps
      if (quad == 0 && lane < G) {                        // fixed-order merge of the 4 warps (log2 domain)
        float m = kFloor;
#pragma unroll
        for (int w = 0; w < 4; ++w) m = fmaxf(m, wpart[grp][par][w][lane].x);
        float sm = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float2 pw = wpart[grp][par][w][lane];
          sm += pw.y * exp2f(pw.x - m);
        }
        prow[(size_t)lane * tiles_per_head + tile] = m > kFloor ? make_float2(m * kLn2, sm) : make_float2(-INFINITY, 0.f);
      }
      for (int st2 = 0; st2 < kTcEpiGroups; ++st2) { if (++tile == tiles_per_head) { tile = 0; ++bh; } }
    }
    if (warp == 0 && lane == 0) trace_tc_any(trace_buf, 13);     // epilogue loop done
  }
  __syncthreads();
  trace_tc(trace_buf, 1);
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tmem));
  }
}

// ---------------------------------------------------------------------------------------------
// host: tensor map over the landmark matrix viewed as [b*h_kv*n_c rows][128] bf16
// ---------------------------------------------------------------------------------------------
size_t score_tc_smem_bytes() { return 1024 + (size_t)kTcStages * kTileBytes + (size_t)kTcMaxHeads * kBBytes; }

bool score_tc_plan(const Dims& D, int tiles_per_head, int n_sm, ScorePlan* plan) {
  const long long total = (long long)D.b * D.hk * tiles_per_head;
  if (total <= 0 || total >= (1ll << 31)) return false;
  int grid = total < n_sm ? (int)total : n_sm;
  // each CTA's contiguous tile range must touch at most kTcMaxHeads KV heads and kTcMaxTiles tiles
  while (grid < total && ((total + grid - 1) / grid > (long long)(kTcMaxHeads - 1) * tiles_per_head ||
                          (total + grid - 1) / grid > kTcMaxTiles))
    grid = grid * 2 < total ? grid * 2 : (int)total;
  const int tpc = (int)((total + grid - 1) / grid);
  const int heads = (tpc + tiles_per_head - 1) / tiles_per_head + 1;     // a range may straddle one more
  if (plan) *plan = ScorePlan{grid, tpc, heads, (int)((tiles_per_head * (long long)grid + total - 1) / total)};
  return tpc <= kTcMaxTiles && heads <= kTcMaxHeads;
}

cudaError_t init_score_tc_attrs() {
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* f) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)score_tc_smem_bytes());
  };
  set((const void*)k_score_tc<1>); set((const void*)k_score_tc<2>); set((const void*)k_score_tc<4>);
  set((const void*)k_score_tc<8>); set((const void*)k_score_tc<16>);
  return e;
}

template <int G>
cudaError_t launch_score_tc(const Dims& D, const uint16_t* L, const int32_t* oids, const uint16_t* q,
                            float* logits, float2* part, int tiles_per_head, float scale,
                            const uint16_t* k_new, const uint16_t* v_new, uint16_t* K_win, uint16_t* V_win,
                            int step, const DevCtx& ctx, cudaStream_t st) {
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
  if (!enc) return cudaErrorNotSupported;
  ScorePlan pl;
  if (!score_tc_plan(D, tiles_per_head, ctx.n_sm, &pl)) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {(cuuint64_t)kHeadDim, (cuuint64_t)D.b * D.hk * D.n_c};
  const cuuint64_t gstride[1] = {(cuuint64_t)kHeadDim * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)kSTile};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(L), gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid); cfg.blockDim = dim3(kTcThreads); cfg.dynamicSmemBytes = score_tc_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;     // prologue overlaps the prior kernel
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = D.serial ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k_score_tc<G>, map, D, oids, q, logits, part, tiles_per_head, scale, k_new, v_new,
                            K_win, V_win, step);
}

#define SKV_INST(G)                                                                                       \
  template cudaError_t launch_score_tc<G>(const Dims&, const uint16_t*, const int32_t*, const uint16_t*,  \
                                          float*, float2*, int, float, const uint16_t*, const uint16_t*,  \
                                          uint16_t*, uint16_t*, int, const DevCtx&, cudaStream_t);
SKV_INST(1)
SKV_INST(2)
SKV_INST(4)
SKV_INST(8)
SKV_INST(16)
#undef SKV_INST

}  // namespace skv
