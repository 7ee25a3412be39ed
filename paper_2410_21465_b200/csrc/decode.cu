// Algorithm 2 "ShadowKV Decoding" + sparse attention on sm_100a.
//
//   k_score<G>        CUDA-core fallback of the tcgen05 scorer (score_tc.cu; SKV_NO_TC=1): a7 window
//                     append, a1 logits l = <q, L_j>/sqrt(d) over 128-landmark tiles streamed through an
//                     mbarrier ring, per-tile softmax partials over landmarks only (R3).
//   k_select<G>       a2 lse + z_j = max_group log sum_i S (R4, R5; s_q rows per q head); a3
//                     exact top-k on an 8-CTA cluster: bucket histogram relative to z_max (pushed
//                     to every rank over DSMEM), definite chunks published unordered at deterministic slots,
//                     the threshold bucket ranked exactly (ties -> lower j, R12); radix fallback.
//   k_sparse_attn<G>  a4+a5+a6 fused per unit of <= 64 tokens.  Selected-chunk units: the thread owning a
//                     chunk issues, the moment its slot is published, the chunk's factor rows A[t] (HBM,
//                     P:182) and its 2 KB of values (cp.async.bulk from pinned host memory over PCIe, P:179;
//                     or from the HBM value cache on a hit, R26).  K~ = A.B_h on the tensor cores
//                     (mma.sync), RoPE, q.K~ logits, and once the values land softmax + PV.  Outlier
//                     and window units read exact K, V from HBM; generated-token units (NEXT-4) rebuild
//                     their keys from rank-r rows.  The host fetch is in flight from the kernel's first
//                     microseconds, so rebuild and attention math hide under it (the paper's multi-stream
//                     overlap of P:40 / P:460, inside one grid).
//   k_merge           the per-unit partials of each (b, q row) are combined by log-sum-exp into the bf16
//                     output; the merge also closes the value cache's generation and re-zeroes the slots.
// Kernels after the first are launched with programmatic dependent launch (PDL).
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "append.cuh"
#include "kernels.h"
#include "topk.cuh"
#include "rope.cuh"
#include "umma.cuh"

namespace skv {



// the decode step: the launch argument, or the device counter of a graph-replayable call (written
// by the caller's stream before this call, so read with acquire semantics), clamped to the range the
// grid and the window were sized for
__device__ __forceinline__ int cur_step(const Dims& D, int step) {
  if (!D.step_dev) return step;
  return min(max(ld_acquire_gpu(D.step_dev), 0), D.max_step);
}

// optional per-CTA timeline (globaltimer ns) for tuning: [kernel][block < 4096][event < 16]
__device__ uint64_t* g_trace = nullptr;
// kernels read g_trace once (TRACE_INIT) so that disabled tracing costs no dependent loads
#define TRACE_INIT uint64_t* const trace_buf_ = g_trace ? g_trace + (size_t)D.trace_slot * kTraceSlot : nullptr
#define trace(kernel, ev)                                                                            \
  do {                                                                                               \
    if (trace_buf_ != nullptr && threadIdx.x == 0)                                                   \
      trace_buf_[((size_t)(kernel) * 4096 + blockIdx.x) * 16 + (ev)] = globaltimer();                \
  } while (0)
cudaError_t set_trace_buffer(void* p) { return cudaMemcpyToSymbol(g_trace, &p, sizeof(void*)); }

// ---------------------------------------------------------------------------------------------
// transpose-reduce over the 16 lanes of a half-warp: each lane holds N partial sums (N % 16 == 0);
// afterwards lane `sub` holds the full sums of elements [sub*N/16, (sub+1)*N/16) in v[0..N/16).
// ---------------------------------------------------------------------------------------------
template <int N, int M>
__device__ __forceinline__ void rs_stage(float* v, int sub) {
  constexpr int H = N / 2;
  const bool up = sub & M;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    float send = up ? v[i] : v[i + H];
    float keep = up ? v[i + H] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, M);
  }
}
template <int N>
__device__ __forceinline__ void reduce_scatter16(float* v, int sub) {
  rs_stage<N, 8>(v, sub); rs_stage<N / 2, 4>(v, sub); rs_stage<N / 4, 2>(v, sub); rs_stage<N / 8, 1>(v, sub);
}

// R rows (16 B of each per lane) dotted with G q heads; returns dot of row sub/G with head sub%G.
template <int G>
__device__ __forceinline__ float rows_dot_q(const uint4* v, const float (&qr)[G][8], int sub) {
  constexpr int R = 16 / G;
  float acc[16];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    float f[8];
    unpack8(v[i], f);
#pragma unroll
    for (int hq = 0; hq < G; ++hq) {
      float a = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) a = fmaf(f[e], qr[hq][e], a);
      acc[i * G + hq] = a;
    }
  }
  reduce_scatter16<16>(acc, sub);
  return acc[0];
}

template <int G>
__device__ __forceinline__ void load_q_regs(const uint16_t* qrow0, int sub, float (&qr)[G][8]) {
#pragma unroll
  for (int hq = 0; hq < G; ++hq) unpack8(*reinterpret_cast<const uint4*>(qrow0 + hq * kHeadDim + sub * 8), qr[hq]);
}

__device__ __forceinline__ bool is_outlier(const int32_t* __restrict__ ids, int o, int j) {
  int lo = 0, hi = o;                       // ids ascending (P:131 output, ABI contract)
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(ids + mid) < j) lo = mid + 1; else hi = mid;
  }
  return lo < o && __ldg(ids + lo) == j;
}

// =============================================================================================
// a1: landmark scoring
// =============================================================================================
template <int G>
__global__ void __launch_bounds__(256, G >= 16 ? 1 : 2)
k_score(Dims D, const uint16_t* __restrict__ L, const int32_t* __restrict__ oids, const uint16_t* __restrict__ q,
        float* __restrict__ logits, float2* __restrict__ part, int tiles_per_head, float scale,
        const uint16_t* __restrict__ k_new, const uint16_t* __restrict__ v_new, uint16_t* K_win,
        uint16_t* V_win, int step) {
  TRACE_INIT;
  constexpr int R = 16 / G;
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* buf = reinterpret_cast<uint16_t*>(smem);                                   // [S][128][128]
  float* P = reinterpret_cast<float*>(smem + (size_t)kSStages * kSTile * kHeadDim * 2);  // [2][G][128]
  uint32_t* obits = reinterpret_cast<uint32_t*>(P + 2 * G * kSTile);                   // outlier bitmap of the head
  __shared__ __align__(8) uint64_t full[kSStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, sub = lane & 15;
  const int total = D.b * D.hk * tiles_per_head;
  const int t_begin = (int)((long long)blockIdx.x * total / gridDim.x);
  const int t_end = (int)((long long)(blockIdx.x + 1) * total / gridDim.x);
  const int nwords = (D.n_c + 31) >> 5;
  trace(0, 0);
  pdl_trigger();                                       // let the select grid become resident early
  // a7: append the current token's K, V to the window (R18)
  const int stp = cur_step(D, step);
  window_append(D, k_new, v_new, K_win, V_win, stp, blockIdx.x * 256 + tid, gridDim.x * 256);
  if (tid == 0) {
    for (int st = 0; st < kSStages; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int it) {                           // thread 0: TMA bulk load of tile t_begin + it
    const int t = t_begin + it;
    if (t >= t_end) return;
    const int bh = t / tiles_per_head, tile = t - bh * tiles_per_head;
    const int j0 = tile * kSTile, rows = min(kSTile, D.n_c - j0);
    const int st = it % kSStages;
    mbar_expect_tx(&full[st], rows * kHeadDim * 2);
    bulk_g2s(buf + (size_t)st * kSTile * kHeadDim, L + ((size_t)bh * D.n_c + j0) * kHeadDim, rows * kHeadDim * 2, &full[st]);
  };
  if (tid == 0)
    for (int it = 0; it < kSStages - 1; ++it) issue(it);
  float qr[G][8];
  int cur_bh = -1;
  for (int it = 0; t_begin + it < t_end; ++it) {
    const int t = t_begin + it;
    if (tid == 0) { fence_proxy_async(); issue(it + kSStages - 1); }
    const int bh = t / tiles_per_head, tile = t - bh * tiles_per_head;
    const int b = bh / D.hk, h = bh - b * D.hk;
    const int j0 = tile * kSTile, rows = min(kSTile, D.n_c - j0);
    if (bh != cur_bh) {                                // new KV head: q registers + outlier bitmap
      load_q_regs<G>(q + ((size_t)b * D.hq + (size_t)h * G) * kHeadDim, sub, qr);
      __syncthreads();
      for (int w = tid; w < nwords; w += 256) obits[w] = 0u;
      __syncthreads();
      for (int i = tid; i < D.o; i += 256) {
        const int j = oids[(size_t)bh * D.o + i];
        atomicOr(&obits[j >> 5], 1u << (j & 31));
      }
      __syncthreads();
      cur_bh = bh;
    }
    const int st = it % kSStages;
    float* Pb = P + (it & 1) * G * kSTile;
    mbar_wait(&full[st], (it / kSStages) & 1);
    const uint16_t* tb = buf + (size_t)st * kSTile * kHeadDim;
#pragma unroll
    for (int rb = 0; rb < 16; rb += 2 * R) {          // warp: rows [16w, 16w+16)
      const int rl = rb + half * R;
      uint4 v[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int r = warp * 16 + rl + i;
        v[i] = (rl + i < 16 && r < rows) ? reinterpret_cast<const uint4*>(tb + (size_t)r * kHeadDim)[sub]
                                         : make_uint4(0, 0, 0, 0);
      }
      const float dot = rows_dot_q<G>(v, qr, sub);
      const int il = rl + sub / G, r = warp * 16 + il;
      if (il < 16 && r < rows) {
        const int j = j0 + r;
        Pb[(sub % G) * kSTile + r] = (((obits[j >> 5] >> (j & 31)) & 1u) || j >= req_nc(D, b)) ? -INFINITY : dot * scale;
      }
    }
    __syncthreads();                                   // Pb complete; stage `st` free for reuse
    float* lb = logits + ((size_t)b * D.hq + (size_t)h * G) * D.n_c + (size_t)j0 * G;   // [n_c][G]
    for (int idx = tid; idx < G * kSTile; idx += 256) {
      const int r = idx / G, hq = idx - r * G;
      if (r < rows) lb[idx] = Pb[hq * kSTile + r];
    }
    for (int hq = warp; hq < G; hq += 8) {           // the tile's softmax partial (per-tile: batch invariant)
      float x[kSTile / 32];
      float m = -INFINITY;
#pragma unroll
      for (int u = 0; u < kSTile / 32; ++u) { const int r = lane + 32 * u; x[u] = r < rows ? Pb[hq * kSTile + r] : -INFINITY; m = fmaxf(m, x[u]); }
      m = warp_max(m);
      float sm = 0.f;
      if (m > -INFINITY) {
#pragma unroll
        for (int u = 0; u < kSTile / 32; ++u) sm += expf(x[u] - m);
      }
      sm = warp_sum(sm);
      if (lane == 0) part[((size_t)b * D.hq + (size_t)h * G + hq) * tiles_per_head + tile] = make_float2(m, sm);
    }
  }
  trace(0, 1);
}

// =============================================================================================
// a2 + a3: normalise, group max, exact top-k
// =============================================================================================
// 0 = highest scores; 255 = catch-all.  zmax comes from the score partials' running max, which may
// sit an ulp off the largest z: clamp, so every z maps into [0, 255] the same way in every pass
__device__ __forceinline__ int zbucket(float z, float zmax) {
  return min(255, max(0, (int)floorf((zmax - z) * 32.f)));
}

// One cluster of kSelCL CTAs per (request, KV head); CTA `rank` owns landmarks
// [rank * n_per, (rank + 1) * n_per).  Cluster-wide max / histogram / candidates / prefix are
// exchanged through distributed shared memory (DSMEM).
template <int NT>
__device__ __forceinline__ int block_sum(int x, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = __reduce_add_sync(0xffffffffu, x);
  if (lane == 0) wsum[warp] = x;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) t += wsum[w];
  __syncthreads();
  return t;
}

// z_j over the G rows of a KV head = (q head, query token) pairs, SQ tokens per q head (rows hq*SQ + i):
// z = max_hq log sum_i exp(l_{hq,i} - lse_{hq,i})  (softmax, sum over s_q, group max; R4, R5);
// SQ = 1 is the plain max of (l - lse).
template <int G, int SQ>
__device__ __forceinline__ float group_z(const float* lg, const float* lse) {
  float zz = -INFINITY;
  if constexpr (SQ == 1 || G % SQ != 0) {
#pragma unroll
    for (int hq = 0; hq < G; ++hq) zz = fmaxf(zz, lg[hq] - lse[hq]);
  } else {
#pragma unroll
    for (int r0 = 0; r0 < G; r0 += SQ) {
      float m = -INFINITY;
#pragma unroll
      for (int i = 0; i < SQ; ++i) m = fmaxf(m, lg[r0 + i] - lse[r0 + i]);
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < SQ; ++i) acc += expf(lg[r0 + i] - lse[r0 + i] - m);
      zz = fmaxf(zz, m > -INFINITY ? m + logf(acc) : -INFINITY);
    }
  }
  return zz;
}

// ---------------------------------------------------------------------------------------------
// Value-chunk cache (R26): least-recently-SELECTED replacement with
// capacity C >= k slots per (request, KV head).  After a step's selection is published, one CTA per head
//   1. reads the k selected chunks and probes the directory: a chunk inserted by an earlier step and not
//      evicted since (1 <= tag <= generation) is a HIT in slot s (the sparse units probe the same way);
//   2. ranks every slot by its LRS key ((last selection generation + 1) << 32 | chunk + 1; empty = 0);
//      slots hit in this step are never victims (key = max);
//   3. gives the misses, in selection-position order, the slots with the smallest keys in order (empty
//      slots first, then the least recently selected chunk, ties -> the lower chunk id: the oracle's rule);
//   4. updates the directory (evicted chunks leave it, misses enter with tag generation + 1) and the slot
//      state (hits and misses: last selection = this generation), and publishes each miss's slot as an
//      8-byte {slot, generation + 1} pair that the unit holding the miss polls before writing its values
//      (no fence: the consumer checks the tag).
// Hits are never moved (their slot is not a victim), so no slot is read and written in one step.
struct VcArgs {
  unsigned long long* dir;      // [b*h_kv][n_c]
  unsigned long long* stats;    // [b*h_kv][4] {generation, ...}
  unsigned long long* slots;    // [b*h_kv][C + k]: slot state, then the miss -> slot assignments
  int C, Cp;                    // capacity, next power of two (bitonic sort width)
};
__host__ __device__ inline size_t vc_assign_smem_bytes(int k, int Cp) {
  return (size_t)2 * k * 4 + 8 + (size_t)Cp * 12;
}
template <int NT>
__device__ __noinline__ void vc_assign(const VcArgs vc, unsigned long long gen, const int32_t* slots_pub, size_t bh,
                                       int n, int k,
                                       uint8_t* smem, TopKSmem<NT>& tk) {
  const int tid = threadIdx.x;
  const int C = vc.C, Cp = vc.Cp;
  unsigned long long* dir = vc.dir + bh * n;
  unsigned long long* meta = vc.slots + bh * (size_t)(C + k);
  unsigned long long* assign = meta + C;
  const unsigned long long now = (gen + 1) << 32;
  int* pchunk = reinterpret_cast<int*>(smem);                   // [k] chunk id at each position
  int* pslot = pchunk + k;                                      // [k] hit slot, or -1
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem + ((2 * k * 4 + 7) & ~7));   // [Cp]
  unsigned* val = reinterpret_cast<unsigned*>(key + Cp);        // [Cp] slot index
  for (int p = tid; p < k; p += NT) {                           // 1. the whole selection (every rank has
    int v;                                                      //    published or is about to)
    const uint64_t t0 = globaltimer();
    while ((v = ld_relaxed_gpu(slots_pub + p)) == 0) { __nanosleep(32); spin_guard(t0); }
    const int j = v - 1;
    pchunk[p] = j;
    const unsigned long long e = ld_relaxed_gpu_u64(dir + j);
    const unsigned tag = (unsigned)(e >> 32);
    pslot[p] = (tag != 0u && tag <= (unsigned)gen) ? (int)(unsigned)e : -1;
  }
  for (int sl = tid; sl < Cp; sl += NT) {                       // 2. LRS keys of the slots
    key[sl] = sl < C ? ld_relaxed_gpu_u64(meta + sl) : ~0ull;
    val[sl] = (unsigned)sl;
  }
  __syncthreads();
  for (int p = tid; p < k; p += NT)
    if (pslot[p] >= 0) key[pslot[p]] = ~0ull;                   // hit this step: never a victim
  __syncthreads();
  for (int kk = 2; kk <= Cp; kk <<= 1) {                        // bitonic sort of (key, slot), ascending
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int i = tid; i < Cp; i += NT) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const bool up = (i & kk) == 0;
          const unsigned long long a = key[i], b = key[ixj];
          if ((a > b) == up) {
            key[i] = b; key[ixj] = a;
            const unsigned t = val[i]; val[i] = val[ixj]; val[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  // 3 + 4. misses in position order take the smallest keys in order
  const int per = (k + NT - 1) / NT;
  const int pa = min(k, tid * per), pb = min(k, pa + per);
  int nm = 0;
  for (int p = pa; p < pb; ++p) nm += pslot[p] < 0;
  int tot;
  int r = block_exclusive_scan<NT>(nm, tk, &tot);
  for (int p = pa; p < pb; ++p) {
    const int j = pchunk[p];
    if (pslot[p] >= 0) {                                        // hit: touched in this generation
      st_relaxed_gpu_u64(meta + pslot[p], now | (unsigned long long)(j + 1));
      continue;
    }
    const unsigned sl = val[r];
    const unsigned long long old = key[r++];                    // the victim's state (0 = empty slot)
    if (old != 0ull) st_relaxed_gpu_u64(dir + ((unsigned)old - 1u), 0ull);   // evicted chunk leaves the directory
    st_relaxed_gpu_u64(dir + j, now | sl);
    st_relaxed_gpu_u64(meta + sl, now | (unsigned long long)(j + 1));
    st_relaxed_gpu_u64(assign + p, now | sl);                   // the unit holding this miss polls it
  }
}

template <int G, bool ZSMEM>
__global__ void __cluster_dims__(kSelCL, 1, 1) __launch_bounds__(kSelThreads, 2)
k_select(Dims D, const float* __restrict__ logits, const float2* __restrict__ part, int tiles_per_head,
         float* __restrict__ zws, int32_t* __restrict__ sel,
         int32_t* __restrict__ selrest, int* __restrict__ flags, int32_t* __restrict__ sel_user, int force_fb,
         VcArgs vc) {
  TRACE_INIT;
  constexpr int NT = kSelThreads, NW = NT / 32;
  extern __shared__ __align__(16) float zdyn[];
  __shared__ TopKSmem<NT> tk;
  __shared__ float lse[G], hm[G];
  __shared__ __align__(16) int hist[256];
  __shared__ int ghist[256], below[kSelCL], info[4];
  __shared__ __align__(16) int allhist[kSelCL * 256];   // every rank's histogram (st.async pushes -> hbar)
  __shared__ __align__(8) uint64_t hbar;
  __shared__ int wdef[NW];
  __shared__ int cidx[kSelCandPush], ccnt;             // this rank's threshold-bucket candidates
  __shared__ uint32_t ckey[kSelCandPush];
  // every rank's {count, 0, 0, 0} + (index, key) pairs, pushed by st.async (completing bytes on cbar)
  __shared__ __align__(16) int4 cand_in[kSelCL][kSelCandPush / 2 + 1];
  __shared__ __align__(8) uint64_t cbar;
  // per-warp bucket histograms (z pass .. publish pass), then the gathered candidates (after #2)
  static_assert(NW * 256 == 4 * kSelCandLocal, "scratch union");
  __shared__ __align__(16) int scratch[4 * kSelCandLocal];
  int (*whist)[256] = reinterpret_cast<int (*)[256]>(scratch);
  int* aidx = scratch;
  uint32_t* akey = reinterpret_cast<uint32_t*>(scratch + kSelCandLocal);
  int* tks = scratch + 2 * kSelCandLocal;
  int* tkf = scratch + 3 * kSelCandLocal;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t crank = cluster_ctarank();
  const size_t bh = blockIdx.x / kSelCL;
  const int b = (int)(bh / D.hk), h = (int)(bh - (size_t)b * D.hk);
  const int n = D.n_c, k = D.k;
  const int n_per = (n + kSelCL - 1) / kSelCL;
  const int lo = min(n, (int)crank * n_per), len = min(n, lo + n_per) - lo;
  float* z = ZSMEM ? zdyn : zws + bh * n + lo;           // this CTA's z slice
  const float* lb = logits + ((size_t)b * D.hq + (size_t)h * G) * n + (size_t)lo * G;   // [n][G]
  int32_t* out = sel + bh * k;
  trace(1, 0);
  for (int i = tid; i < NW * 256; i += NT) (&whist[0][0])[i] = 0;
  if (tid == 0) {
    ccnt = 0; info[0] = 255; info[1] = 0;               // B = 255 unless bins 0..254 reach k
    // every rank pushes its 1 KB histogram into allhist[rank][.] of every rank with st.async, which
    // completes bytes on this barrier: no cluster barrier between the histograms and their use
    mbar_init(&hbar, 1);
    mbar_init(&cbar, 1);
    fence_mbar_init();
    mbar_expect_tx(&hbar, kSelCL * 256 * 4);
    mbar_expect_tx(&cbar, kSelCL * (kSelCandPush / 2 + 1) * 16);
  }
  cluster_arrive_relaxed();                             // #0: this CTA has started (waited on before the
                                                        //     first DSMEM store; long complete by then)
  // The sparse grid may launch now: its CTAs stage q and B_h and then poll their selection slots while
  // this grid waits for the scores and selects.  Safe before our griddepcontrol.wait: the score grid
  // triggers this grid only after ITS wait, i.e. after the previous layer's merge (which re-zeroes the
  // slots and flags) has completed, so no sparse CTA of this call can see a stale slot.
  pdl_trigger();
  pdl_wait();
  trace(1, 1);
  int* fl = flags + bh * 4;
  // the value cache's generation of this step, read before any slot is published: the merge closes it
  // once every unit of the head is done, which can precede vc_assign when all of them hit
  const unsigned long long vc_gen = (vc.dir != nullptr && crank == 0) ? ld_relaxed_gpu_u64(vc.stats + bh * 4) : 0ull;
  // score (incl. a7 window append) complete.  A relaxed store: the score grid's writes reached L2 when it
  // completed (our griddepcontrol.wait), and the readers (outlier / window units) bulk-copy from L2; a
  // release here is a membar on the critical path of the barrier below
  if (crank == 0 && tid == NT - 32) st_relaxed_gpu(&fl[0], 1);
  // ---- lse_hq from the score kernel's per-tile partials (warps < G) and the first z-pass logits: both
  //      load batches are issued before either is used (their L2 latencies overlap).  Each lane merges
  //      its tiles lane, lane+32, ... in batches of 8 (batch max, then one sum of 8 independent exps),
  //      then a fixed warp tree (max, then rescaled sum): deterministic and independent of the score grid
  constexpr int U = G >= 8 ? 1 : 4;
  float lg[U][G];
  auto load_lg = [&](int j0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT + tid;
#pragma unroll
      for (int hq = 0; hq < G; ++hq) lg[u][hq] = -INFINITY;
      if (j < len) load_row<G>(lb + (size_t)j * G, lg[u]);
    }
  };
  const float2* ph = part + ((size_t)b * D.hq + (size_t)h * G + (warp < G ? warp : 0)) * tiles_per_head;
  float2 pv[8];
  auto load_part = [&](int i0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + lane + 32 * u;
      pv[u] = i < tiles_per_head ? __ldcg(&ph[i]) : make_float2(-INFINITY, 0.f);
    }
  };
  if (warp < G) load_part(0);
  load_lg(0);
  if (warp < G) {
    if (warp == 0) trace(1, 13);
    float m = -INFINITY, e = 0.f;
    for (int i0 = 0; i0 < tiles_per_head; i0 += 32 * 8) {
      if (i0 > 0) load_part(i0);
      float mb = pv[0].x;
#pragma unroll
      for (int u = 1; u < 8; ++u) mb = fmaxf(mb, pv[u].x);
      if (mb > -INFINITY) {
        float sb = 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) sb += pv[u].y * expf(pv[u].x - mb);
        lse_merge(m, e, mb, sb);
      }
    }
    if (warp == 0) trace(1, 14);
    const float M = warp_max(m);
    const float E = warp_sum(m > -INFINITY ? e * expf(m - M) : 0.f);
    if (lane == 0) { lse[warp] = M > -INFINITY ? M + logf(E) : -INFINITY; hm[warp] = M; }
    if (warp == 0) trace(1, 15);
  }
  __syncthreads();
  // max_j z_j = max_g (max_j l_gj - lse_g): known from the partials, no extra pass
  float zmax = -INFINITY;
#pragma unroll
  for (int hq = 0; hq < G; ++hq) zmax = fmaxf(zmax, hm[hq] - lse[hq]);
  const int sq = D.sq;
  if (sq > 1) zmax += logf((float)sq);    // z = log sum_i S_i <= max_i log S_i + log s_q (an upper bound)
  trace(1, 2);
  // ---- z = max_g (l - lse) on the slice (R4, R5) + bucket histograms, one per warp: the
  //      publish pass below walks each warp's elements in the same order, so the definite chunks' slot
  //      positions follow from the per-warp counts without a block-wide scan
  int* wh = whist[warp];
  for (int j0 = 0; j0 < len; j0 += U * NT) {
    if (j0 > 0) load_lg(j0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT + tid;
      float zz;
      switch (sq) {        // compile-time s_q: the row array stays in registers
        case 1: zz = group_z<G, 1>(lg[u], lse); break;
        case 2: zz = group_z<G, 2>(lg[u], lse); break;
        case 4: zz = group_z<G, 4>(lg[u], lse); break;
        case 8: zz = group_z<G, 8>(lg[u], lse); break;
        default: zz = group_z<G, 16>(lg[u], lse); break;
      }
      if (j < len) {
        z[j] = zz;
        // the catch-all bucket 255 is never counted: if bins 0..254 hold fewer than k, B stays 255
        // and the exact radix fallback runs
        const int bk = zz > -INFINITY ? zbucket(zz, zmax) : 255;
        if (bk != 255) atomicAdd(&wh[bk], 1);
      }
    }
  }
  __syncthreads();                                                      // per-warp histograms complete
  if (tid < 256) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += whist[w][tid];
    hist[tid] = s;
  }
  trace(1, 3);
  // push this rank's histogram into allhist[crank][.] of every rank (the release-arrive of barrier #1
  // orders these remote stores), so that after the barrier all histograms are local reads
  __syncthreads();                                      // hist[] complete
  cluster_wait_acquire();                               // #0: every CTA of the cluster has started (its
                                                        //     hbar is initialised)
  if (tid < 64) {
    const int4 v = *reinterpret_cast<const int4*>(&hist[4 * tid]);
#pragma unroll
    for (int r = 0; r < kSelCL; ++r)
      st_async_v4(dsmem_addr(&allhist[crank * 256 + 4 * tid], r), v, dsmem_addr(&hbar, r));
  }
  mbar_wait(&hbar, 0);                                                  // all kSelCL histograms landed
  trace(1, 4);
  if (tid < 256) {
    int g = 0;
#pragma unroll
    for (int r = 0; r < kSelCL; ++r) g += allhist[r * 256 + tid];
    ghist[tid] = g;
  }
  __syncthreads();
  if (warp == 0) {                                      // bucket B holding the k-th largest z
    int c[8], sacc = 0;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) { c[jj] = ghist[lane * 8 + jj]; sacc += c[jj]; }
    int pre = sacc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(0xffffffffu, pre, o); if (lane >= o) pre += y; }
    pre -= sacc;
    if (pre < k && k <= pre + sacc) {
      int cum = pre;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        if (cum + c[jj] >= k) { info[0] = lane * 8 + jj; info[1] = k - cum; break; }
        cum += c[jj];
      }
    }
  }
  __syncthreads();
  trace(1, 10);
  const int B = info[0], need = info[1];
  // The selection is published into k slots (chunk id + 1; 0 = not yet) before it is complete:
  // attention is a sum over the selected set, so the chunks strictly above the threshold bucket
  // ("definite") are written to slots [0, k - need) as soon as B is known, and the `need` winners of
  // bucket B fill [k - need, k) once ranked.  Positions are deterministic: rank prefix (every rank's
  // histogram mass above B), then the warps of this rank in order, then each warp's elements in z-pass
  // order.  Each sparse-attention unit polls its own 8 slots.
  int32_t* slots = sel + bh * k;
  const bool prepub = !(B == 255 || n_per > 16384 || force_fb == 1);  // else: radix fallback publishes all k
  bool fallback = !prepub;
  // below[r]: rank r's histogram mass above B (one warp per rank), then this warp's definite count;
  // 8 independent, bank-conflict-free loads per lane
  auto mass_below = [&](const int* hrow) {
    int sacc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { const int bin = lane + 32 * i; sacc += bin < B ? hrow[bin] : 0; }
    return __reduce_add_sync(0xffffffffu, sacc);
  };
  if (warp < kSelCL) { const int sb = mass_below(&allhist[warp * 256]); if (lane == 0) below[warp] = sb; }
  if (prepub) { const int myd = mass_below(whist[warp]); if (lane == 0) wdef[warp] = myd; }
  __syncthreads();
  if (prepub) {
    int base = 0;                                       // ranks below, then warps below in this rank
    for (int r = 0; r < (int)crank; ++r) base += below[r];
    for (int w = 0; w < warp; ++w) base += wdef[w];
    // one pass over the warp's z (in z-pass order): definite -> slot, bucket B -> candidate list
    for (int j0 = 0; j0 < len; j0 += U * NT) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u * NT + tid;
        float zz = -INFINITY;
        int bk = 256;
        if (j < len) { zz = z[j]; if (zz > -INFINITY) bk = zbucket(zz, zmax); }
        const unsigned db = __ballot_sync(0xffffffffu, bk < B);
        if (bk < B) st_relaxed_gpu(&slots[base + __popc(db & ((1u << lane) - 1u))], lo + j + 1);
        base += __popc(db);
        const unsigned cb = __ballot_sync(0xffffffffu, bk == B);
        if (cb) {                                       // warp-aggregated candidate reservation
          int cbase = 0;
          if (lane == __ffs(cb) - 1) cbase = atomicAdd(&ccnt, __popc(cb));
          cbase = __shfl_sync(0xffffffffu, cbase, __ffs(cb) - 1);
          const int pos = cbase + __popc(cb & ((1u << lane) - 1u));
          if (bk == B && pos < kSelCandPush) { cidx[pos] = lo + j; ckey[pos] = f2key(zz); }
        }
      }
    }
  }
  __syncthreads();                                      // candidates and ccnt complete
  trace(1, 11);
  // Candidate exchange: this rank's count and its (index, key) pairs go to every rank by st.async,
  // completing bytes on the receiver's cbar (armed at kernel start).  No cluster barrier: its release
  // would wait until the co-resident sparse CTAs' host reads -- started by the slots just published --
  // have landed (a release on an SM waits for all of its outstanding reads, tools/probe_fence.cu).
  {
    const int mycnt = ccnt;
    if (tid <= kSelCandPush / 2) {
      int4 v = make_int4(mycnt, 0, 0, 0);
      if (tid > 0) {
        const int p0 = 2 * (tid - 1), p1 = p0 + 1;
        v = make_int4(p0 < mycnt ? cidx[p0] : 0, p0 < mycnt ? (int)ckey[p0] : 0,
                      p1 < mycnt ? cidx[p1] : 0, p1 < mycnt ? (int)ckey[p1] : 0);
      }
#pragma unroll
      for (int r = 0; r < kSelCL; ++r) st_async_v4(dsmem_addr(&cand_in[crank][tid], r), v, dsmem_addr(&cbar, r));
    }
  }
  const int per = (len + NT - 1) / NT;                  // this thread's contiguous run [ja, jb) (sel_user)
  const int ja = min(len, tid * per), jb = min(len, ja + per);
  trace(1, 5);
  mbar_wait(&cbar, 0);                                  // every rank's candidates are in cand_in
  trace(1, 6);
  int rc[kSelCL], total = 0, cmax = 0, off = 0;
#pragma unroll
  for (int r = 0; r < kSelCL; ++r) rc[r] = fallback ? 0 : cand_in[r][0].x;
#pragma unroll
  for (int r = 0; r < kSelCL; ++r) { total += rc[r]; cmax = max(cmax, rc[r]); off += r < (int)crank ? rc[r] : 0; }
  fallback = fallback || cmax > kSelCandPush || total > kSelCandLocal || force_fb == 2;
  if (!fallback) {
    // all ranks' candidates -> local smem; each CTA ranks its own (larger z first, ties -> lower
    // index, R12): rank < need is taken, and the rank is its slot offset in [k - need, k)
    for (int t = tid; t < total; t += NT) {
      int r = 0, base = 0;
#pragma unroll
      for (int rr = 0; rr < kSelCL; ++rr) { const bool past = t >= base + rc[rr] && rr == r; base += past ? rc[rr] : 0; r += past; }
      const int c = t - base;
      const int4 pr = cand_in[r][1 + (c >> 1)];
      aidx[t] = (c & 1) ? pr.z : pr.x;
      akey[t] = (uint32_t)((c & 1) ? pr.w : pr.y);
    }
    __syncthreads();
    trace(1, 8);
    for (int t = off + tid; t < off + rc[crank]; t += NT) {
      const uint32_t u = akey[t];
      const int j = aidx[t];
      int rank = 0;
#pragma unroll 8
      for (int c = 0; c < total; ++c) rank += (akey[c] > u) || (akey[c] == u && aidx[c] < j);
      if (rank < need) { st_relaxed_gpu(&slots[k - need + rank], j + 1); z[j - lo] = INFINITY; }
    }
    trace(1, 9);
    if (sel_user) {          // a3 parity output: the full selection, ascending (R12)
      __syncthreads();
      for (int t = tid; t < total; t += NT) {
        const uint32_t u = akey[t];
        const int j = aidx[t];
        int rank = 0;
        for (int c = 0; c < total; ++c) rank += (akey[c] > u) || (akey[c] == u && aidx[c] < j);
        tkf[t] = rank < need;
      }
      __syncthreads();
      for (int t = tid; t < total; t += NT) {
        if (!tkf[t]) continue;
        const int j = aidx[t];
        int ord = 0;                                     // position among the taken, by index
        for (int c = 0; c < total; ++c) ord += tkf[c] && aidx[c] < j;
        tks[ord] = j;
      }
      __syncthreads();
      int base_sel = 0;                                  // selected chunks of the ranks below
      for (int r = 0; r < (int)crank; ++r) base_sel += below[r];
      {
        int lo2 = 0, hi2 = need;                         // + taken ones with index < lo
        while (lo2 < hi2) { const int mid = (lo2 + hi2) >> 1; if (tks[mid] < lo) lo2 = mid + 1; else hi2 = mid; }
        base_sel += lo2;
      }
      int nsel = 0;
      for (int j = ja; j < jb; ++j) {
        const float zz = z[j];
        nsel += zz == INFINITY || (zz > -INFINITY && zbucket(zz, zmax) < B);
      }
      int stot;
      int pos = base_sel + block_exclusive_scan<NT>(nsel, tk, &stot);
      for (int j = ja; j < jb; ++j) {
        const float zz = z[j];
        if (zz == INFINITY || (zz > -INFINITY && zbucket(zz, zmax) < B)) sel_user[bh * k + pos++] = lo + j;
      }
    }
    trace(1, 12);
  } else {                   // pathological score distribution: exact radix select on one CTA
    float* zg = zws + bh * n;
    if (ZSMEM)
      for (int j = tid; j < len; j += NT) zg[lo + j] = z[j];
    __threadfence();
    cluster_sync_all();
    if (crank == 0) {
      int32_t* srt = selrest + bh * k;                   // scratch: the top-k, ascending
      block_topk_largest<NT>(zg, n, k, srt, tk);
      __syncthreads();
      for (int i = tid; i < k && sel_user; i += NT) sel_user[bh * k + i] = srt[i];
      if (warp == 0) {                                   // publish in ascending order (deterministic)
        int base = prepub ? k - need : 0;                // the definite ones are published already
        for (int i0 = 0; i0 < k; i0 += 32) {
          const int i = i0 + lane;
          const int j = i < k ? srt[i] : 0;
          const bool pub = i < k && (!prepub || zbucket(zg[j], zmax) >= B);
          const unsigned bal = __ballot_sync(0xffffffffu, pub);
          if (pub) st_relaxed_gpu(&slots[base + __popc(bal & ((1u << lane) - 1u))], j + 1);
          base += __popc(bal);
        }
      }
    }
  }
  trace(1, 7);
  // value cache (R26): rank 0 turns this step's selection into slot assignments
  if (vc.dir != nullptr && crank == 0) {
    __syncthreads();
    vc_assign<NT>(vc, vc_gen, sel + bh * k, bh, n, k, reinterpret_cast<uint8_t*>(zdyn), tk);
  }
}

// =============================================================================================
// a4 + a5 + a6: fused rebuild + host gather + attention over one unit of <= 64 tokens
// =============================================================================================
constexpr int kQStride = kHeadDim + 4;       // q rows (floats): conflict-free MMA A fragments
constexpr int kPStride = kUnitTok + 4;       // logit / probability rows (floats)
constexpr int kKStride = kHeadDim + 4;       // fp32 key tile rows (floats)
struct AttnSmem {      // byte offsets from the 1024-aligned base of dynamic smem
  int a, bmat, v, q, pp, p, tok, bytes;
};
// A tile: the unit's 64 gathered factor rows A[t][0:r] as UMMA K-major SWIZZLE_128B atoms (TMA boxes of
// 8 rows x 64 columns, 1 KB each; K block kb at a + kb * 8 KB, chunk c at + c * 1 KB).  The M = 128
// MMA also reads rows 64..127 (TMEM lanes 64..127, never used): the 8 KB after the last K block must be
// addressable smem (B_h follows).  Outlier / window units reuse the region for their exact K tile.
// B_h: [r][128] MN-major SWIZZLE_128B, two TMA boxes of r rows x 64 columns (LBO = r * 128 B apart).
__host__ __device__ inline AttnSmem attn_smem_layout(int r, int G) {
  AttnSmem s;
  const int nkb = (r + 63) / 64;
  int off = 0;
  s.a = off; off += nkb * 8192 > kUnitTok * kHeadDim * 2 ? nkb * 8192 : kUnitTok * kHeadDim * 2;
  s.bmat = off; off += 2 * r * 128;
  if (off < nkb * 8192 + 8192) off = nkb * 8192 + 8192;
  if (off < kUnitTok * kKStride * 4) off = kUnitTok * kKStride * 4;           // fp32 key tile (G >= 8) aliases A, B
  s.v = off; off += kUnitTok * kHeadDim * 2;                                // V tile bf16
  s.q = off; off += G * kQStride * 4;                                       // q fp32
  s.pp = off; off += 2 * G * kUnitTok * 4;                                  // logit halves (two column sets)
  s.p = off; off += G * kPStride * 4;                                       // logits / probs
  s.tok = off; off += kUnitTok * 4;
  s.bytes = off + 1024;                                                     // + base alignment slack
  return s;
}
constexpr uint32_t kIdescRebuild = umma_idesc_bf16(128, 128, false, true);   // A K-major, B_h MN-major

// a6 combine: out_hq = sum_s w_s o_s with w_s = exp(m_s - M) / sum_s' l_s' exp(m_s' - M) over the
// per-unit partials (m_s, l_s, o_s) of one q head (split-KV log-sum-exp merge, fixed order).  A grid
// of its own (one CTA per (b, hq), thread = dim), launched by PDL while the sparse grid still runs.
// It does not wait on that grid: the units write their partials as 8-byte {value, tag} pairs
// (tag = this row's epoch + 1) and the merge polls for the tags.  A grid boundary would release it
// only ~4 us after the last host read, and a per-unit release fence would stall on the SM's other
// host reads (tools/probe_fence.cu).  Afterwards it bumps the row's epoch; the first CTA of each (b, h)
// re-zeroes that head's slots and flags (every unit of the head is past them: it wrote its partials).
template <int G>
__global__ void __launch_bounds__(kHeadDim)
k_merge(Dims D, const uint2* __restrict__ o_part, const uint2* __restrict__ ml_part, int* __restrict__ epochs,
        int n_split, int32_t* __restrict__ sel, int* __restrict__ flags, uint16_t* __restrict__ out,
        int late_trigger, unsigned long long* __restrict__ vc_stats) {
  TRACE_INIT;
  extern __shared__ __align__(16) float2 mls[];          // [n_split]
  const int row = blockIdx.x, d = threadIdx.x;            // row = b * hq + hq
  if (!late_trigger) pdl_trigger();
  // (no griddepcontrol.wait: the previous merge of this row completed before this call's units read
  //  the epoch -- they start after the score grid's wait -- and this call's partials carry the tag)
  const unsigned tag = ld_volatile_u32(&epochs[row]) + 1u;
  trace(3, 0);
  const uint2* mr = ml_part + (size_t)row * n_split * 2;
  const uint2* orow = o_part + (size_t)row * n_split * kHeadDim + d;
  for (int i = d; i < n_split; i += kHeadDim) {           // (m, l) of every unit, polled with back-off
    uint2 m2, l2;
    const uint64_t t0 = globaltimer();
    for (;;) {
      m2 = ld_tagged(mr + 2 * i); l2 = ld_tagged(mr + 2 * i + 1);
      if (m2.y == tag && l2.y == tag) break;
      __nanosleep(128);
      spin_guard(t0);
    }
    mls[i] = make_float2(__uint_as_float(m2.x), __uint_as_float(l2.x));
  }
  __syncthreads();                                        // every unit's (m, l) has landed
  trace(3, 2);
  // this thread's values of the first kBatch units: loads issued now, consumed after the weights
  constexpr int kBatch = 64;
  uint2 t[kBatch];
  auto issue_o = [&](int s0) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) t[u] = s0 + u < n_split ? ld_tagged(orow + (size_t)(s0 + u) * kHeadDim) : make_uint2(0u, tag);
  };
  issue_o(0);
  trace(3, 3);
  // weights, computed once per CTA: M = max_s m_s; w_s = exp(m_s - M); L = sum_s l_s w_s
  __shared__ float red[kHeadDim / 32];
  float* w = reinterpret_cast<float*>(mls + n_split);     // [n_split]
  const int lane = d & 31, warp = d >> 5;
  float mx = -INFINITY;
  for (int s2 = d; s2 < n_split; s2 += kHeadDim) mx = fmaxf(mx, mls[s2].x);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  float M = red[0];
#pragma unroll
  for (int i = 1; i < kHeadDim / 32; ++i) M = fmaxf(M, red[i]);
  float Lp = 0.f;
  for (int s2 = d; s2 < n_split; s2 += kHeadDim) {
    const float2 ml = mls[s2];
    const float ws = ml.x > -INFINITY ? expf(ml.x - M) : 0.f;
    w[s2] = ws;
    Lp = fmaf(ml.y, ws, Lp);
  }
  Lp = warp_sum(Lp);
  __syncthreads();                                        // w[] complete; red[] reads done
  if (lane == 0) red[warp] = Lp;
  __syncthreads();
  float L = 0.f;
#pragma unroll
  for (int i = 0; i < kHeadDim / 32; ++i) L += red[i];    // fixed order: deterministic
  trace(3, 4);
  float acc = 0.f;
  for (int s0 = 0; s0 < n_split; s0 += kBatch) {
    if (s0 > 0) issue_o(s0);
    for (;;) {                                            // (a value may trail its unit's (m, l): the
      unsigned long long stale = 0ull;                    //  stale ones are re-read together)
#pragma unroll
      for (int u = 0; u < kBatch; ++u) stale |= (unsigned long long)(t[u].y != tag) << u;
      if (!stale) break;
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if ((stale >> u) & 1ull) t[u] = ld_tagged(orow + (size_t)(s0 + u) * kHeadDim);
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (s0 + u < n_split) acc = fmaf(w[s0 + u], __uint_as_float(t[u].x), acc);
  }
  if (late_trigger) pdl_trigger();                        // the next grid's prefetch after our loads
  out[(size_t)row * kHeadDim + d] = f2bf(acc / L);
  trace(3, 1);
  __syncthreads();                                        // every thread has read its partials
  if (d == 0) epochs[row] = (int)tag;                     // (the next call reads it after this grid completes)
  const int hq = row % D.hq;
  if (hq % G == 0) {                                      // one CTA per (b, h): reset for the next call
    const int bh = (row / D.hq) * D.hk + hq / G;
    int32_t* slots = sel + (size_t)bh * D.k;
    for (int i = d; i < D.k; i += kHeadDim) slots[i] = 0;
    if (d < 4) flags[(size_t)bh * 4 + d] = 0;
    if (vc_stats && d == 0) {                             // value cache: close the generation (R26)
      unsigned long long* st = vc_stats + (size_t)bh * 4;
      const unsigned long long hits = __ldcg(st + 1);
      st[1] = 0; st[2] = hits; st[3] += hits; st[0] += 1;
    }
  }
}

// tf32 operand (round to nearest) for mma.sync
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r; asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x)); return r;
}
__device__ __forceinline__ void mma_tf32(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
               "{%0, %1, %2, %3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// S[16 query rows][8 tokens of warp w] = Q . K~^T over the 128 dims (rows >= G are zero)
template <int G>
__device__ __forceinline__ void qk_tile_mma(const float* qs, const float* Ksm, int warp, int lane, float* c) {
  const int g = lane >> 2, t = lane & 3;
  c[0] = c[1] = c[2] = c[3] = 0.f;
  const float* qa = qs + g * kQStride + t;
  const float* qb = qs + (g + 8) * kQStride + t;
  const float* kr = Ksm + (8 * warp + g) * kKStride + t;
#pragma unroll 4
  for (int k0 = 0; k0 < kHeadDim; k0 += 8) {
    const uint32_t a0 = to_tf32(qa[k0]), a2 = to_tf32(qa[k0 + 4]);
    const uint32_t a1 = g + 8 < G ? to_tf32(qb[k0]) : 0u, a3 = g + 8 < G ? to_tf32(qb[k0 + 4]) : 0u;
    mma_tf32(c, a0, a1, a2, a3, to_tf32(kr[k0]), to_tf32(kr[k0 + 4]));
  }
}
// O[16 query rows][16 dims of warp w] = P . V over the unit's 64 tokens (rows past ntok contribute 0); k step
// k0 = chunk k0/8: with per_chunk, each chunk's values are waited for (barVc[chunk]) just before its step,
// otherwise all values (barVc[0]) before the first
template <int G>
__device__ __forceinline__ void pv_tile_mma(const float* P, const uint16_t* Vs, int ntok, int warp, int lane,
                                            float (*c)[4], uint64_t* barVc, bool per_chunk) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) c[nt][0] = c[nt][1] = c[nt][2] = c[nt][3] = 0.f;
  const float* pa = P + g * kPStride + t;
  const float* pb = P + (g + 8) * kPStride + t;
  if (!per_chunk) mbar_wait(&barVc[0], 0);
#pragma unroll 2
  for (int k0 = 0; k0 < kUnitTok; k0 += 8) {
    if (k0 >= ntok) break;
    if (per_chunk) mbar_wait(&barVc[k0 >> 3], 0);
    const uint32_t a0 = to_tf32(pa[k0]), a2 = to_tf32(pa[k0 + 4]);
    const uint32_t a1 = g + 8 < G ? to_tf32(pb[k0]) : 0u, a3 = g + 8 < G ? to_tf32(pb[k0 + 4]) : 0u;
    const int r0 = k0 + t, r1 = k0 + t + 4;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int dim = 16 * warp + 8 * nt + g;
      const uint32_t b0 = r0 < ntok ? to_tf32(bf2f(Vs[r0 * kHeadDim + dim])) : 0u;
      const uint32_t b1 = r1 < ntok ? to_tf32(bf2f(Vs[r1 * kHeadDim + dim])) : 0u;
      mma_tf32(c[nt], a0, a1, a2, a3, b0, b1);
    }
  }
}

template <int G>
__global__ void __launch_bounds__(256, 2)
k_sparse_attn(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmG, Dims D, Rope R, Layer Ly, const uint16_t* __restrict__ q,
              int32_t* __restrict__ sel, int* __restrict__ flags, int step,
              uint2* __restrict__ o_part, uint2* __restrict__ ml_part, const int* __restrict__ epochs, int n_sel_u,
              int n_out_u, int n_win_u,
              int n_gen_u, int n_split, float scale, uint16_t* __restrict__ dbg, int early_next) {
  TRACE_INIT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  const AttnSmem lay = attn_smem_layout(D.r, G);
  uint16_t* Vs = reinterpret_cast<uint16_t*>(smem + lay.v);
  uint8_t* As = smem + lay.a;                                  // A tile (SW128) or exact K tile [64][128]
  uint8_t* Bs = smem + lay.bmat;                               // B_h (MN-major SW128)
  float* qs = reinterpret_cast<float*>(smem + lay.q);          // [G][128]
  float* Pp = reinterpret_cast<float*>(smem + lay.pp);         // [2][G][64]
  float* P = reinterpret_cast<float*>(smem + lay.p);           // [G][64]
  int* tok = reinterpret_cast<int*>(smem + lay.tok);
  // barVc[c]: values of chunk c of a selected-chunk unit (one bulk copy each, so the PV can start on
  // the chunks that have landed); other unit kinds use barVc[0] for their single value copy
  __shared__ __align__(8) uint64_t barAB, barVc[8], barMMA;
  __shared__ uint32_t tmem_base;
  __shared__ float2 ml[G];
  __shared__ unsigned tagv[G];                                 // this call's partial tag per q row
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, sub = lane & 15;
  const int BH = D.b * D.hk;
  const int stp0 = cur_step(D, step);
  const int T_out = D.o * kChunk;
  const int nkb = (D.r + 63) >> 6;
  int T_win;                                           // this request's window incl. the s_q new tokens
  // unit kinds: 0 selected chunks, 1 outliers, 2 window (plain: context tail + generated; low-rank: tail
  // only), 3 generated tokens rebuilt from their low-rank rows (NEXT-4)
  const bool lowrank = D.lr_A != nullptr;
  int u = blockIdx.x, kind, bh, ui, split;
  if (u < BH * n_sel_u) { kind = 0; bh = u / n_sel_u; ui = u - bh * n_sel_u; split = ui; }
  else {
    u -= BH * n_sel_u;
    const int per = n_out_u + n_win_u + n_gen_u;
    bh = u / per; ui = u - bh * per;
    split = n_sel_u + ui;
    if (ui < n_out_u) kind = 1;
    else if (ui < n_out_u + n_win_u) { kind = 2; ui -= n_out_u; }
    else { kind = 3; ui -= n_out_u + n_win_u; }
  }
  const int b = bh / D.hk, h = bh - b * D.hk;
  T_win = lowrank ? req_weff(D, b) : req_weff(D, b) + stp0 + D.sq;
  const int n_gen = stp0 + D.sq;                                // generated tokens incl. this call's
  if (kind == 3 && ui * kUnitTok >= n_gen) {                    // generated unit past the live tokens
    for (int hq = tid >> 7; hq < G; hq += 2) {
      const size_t row = ((size_t)b * D.hq + (size_t)h * G + hq) * n_split + split;
      const unsigned tg = ld_volatile_u32(&epochs[(size_t)b * D.hq + (size_t)h * G + hq]) + 1u;
      st_tagged(o_part + row * kHeadDim + (tid & 127), 0.f, tg);
      if ((tid & 127) == 0) { st_tagged(ml_part + 2 * row, -INFINITY, tg); st_tagged(ml_part + 2 * row + 1, 0.f, tg); }
    }
    return;
  }
  int32_t* slots = sel + (size_t)bh * D.k;                     // k_select's unordered selection (id + 1)
  const int nch = kind == 0 ? min(8, D.k - ui * 8) : 0;        // chunks of a selected-chunk unit (>= 1)
  const bool rebuild = kind == 0 || kind == 3;
  trace(2, 0);
  if (tid == 0) {   // selected-chunk units: one arrival per chunk-issuing thread
    mbar_init(&barAB, kind == 0 ? nch : 1); mbar_init(&barMMA, 1);
    for (int c = 0; c < 8; ++c) mbar_init(&barVc[c], 1);
    fence_mbar_init();
    if (rebuild)                                          // B_h's bytes, before any arrival can complete the phase
      asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;"
                   :: "r"(smem_u32(&barAB)), "r"((uint32_t)(2 * D.r * 128)) : "memory");
  }
  if (rebuild && warp == 0) tmem_alloc<128>(&tmem_base);      // K~ accumulator: 128 lanes x 128 fp32 columns
  if (tid < G) tagv[tid] = ld_volatile_u32(&epochs[(size_t)b * D.hq + (size_t)h * G + tid]) + 1u;
  // q is a call input: stage it before waiting on the producer kernels
  for (int i = tid; i < G * kHeadDim; i += 256)
    qs[(i >> 7) * kQStride + (i & 127)] = bf2f(q[((size_t)b * D.hq + (size_t)h * G) * kHeadDim + i]);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  int ntok;
  int vc_id = -1;                              // value cache: this thread's chunk and the call's generation
  unsigned long long vc_gen = 0;
  bool vc_hit = false;                         // (a hit stays in its slot; a miss is written to the slot
                                               //  the selector assigns, k_select's vc_assign)
  const int tx = tid & 15, ty = tid >> 4;      // exact-key tile ownership: tokens ty + 16 i (i < 4), dims tx*8..+8
  float acc[4][8];
  if (rebuild) {
    // B_h does not depend on the selection: two TMA boxes (64 columns x r rows) issued at once by a thread
    // of warp 1, so the chunk threads of warp 0 never queue behind them
    if (tid == 32) {
      prefetch_tensormap(&tmB);
      tma_load_2d(Bs, &tmB, 0, bh * D.r, &barAB);
      tma_load_2d(Bs + D.r * 128, &tmB, 64, bh * D.r, &barAB);
    }
    if (kind == 3) {  // generated tokens g0 .. g0+ntok-1: low-rank rows + values, positions s_b + g (R16)
      const int g0 = ui * kUnitTok, nt = min(kUnitTok, n_gen - g0);
      cta_wait_flag(&flags[(size_t)bh * 4]);                    // (score's a7 projection is visible)
      if (tid == 0) {
        const int nblk = (nt + 7) >> 3;
        mbar_expect_tx(&barAB, nblk * nkb * 1024);
        for (int blk = 0; blk < nblk; ++blk)
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d(As + kb * 8192 + blk * 1024, &tmG, kb * 64, b * D.wcap + g0 + blk * 8, &barAB);
        mbar_expect_tx(&barVc[0], nt * kHeadDim * 2);
        bulk_g2s(Vs, Ly.V_win + ((size_t)bh * D.wcap + req_weff(D, b) + g0) * kHeadDim, nt * kHeadDim * 2, &barVc[0]);
      }
      if (tid < kUnitTok) tok[tid] = tid < nt ? req_s(D, b) + g0 + tid : 0;
    }
    // thread c < nch waits for its slot, then issues its chunk's copies at once: the value fetch of each
    // chunk starts the moment k_select publishes it
    if (kind == 0 && tid < nch) {                        // (generated units set their positions above)
      const int* sp = slots + ui * 8 + tid;
      int v;
      const uint64_t t0 = globaltimer();
      while ((v = ld_relaxed_gpu(sp)) == 0) { __nanosleep(32); spin_guard(t0); }
      const int id = v - 1;
      vc_id = id;
#pragma unroll
      for (int e = 0; e < kChunk; ++e) tok[tid * kChunk + e] = id * kChunk + e;
      // a4 operands (HBM): the chunk's 8 factor rows A[t][0:r] as nkb SWIZZLE_128B boxes (TMA tensor copies)
      mbar_expect_tx(&barAB, nkb * 1024);
      for (int kb = 0; kb < nkb; ++kb)
        tma_load_2d(As + kb * 8192 + tid * 1024, &tmA, kb * 64, b * D.s + id * kChunk, &barAB);
      // a5: the value chunk straight from pinned host memory over PCIe (zero-copy bulk copy) -- or,
      // with the value cache, from HBM when the chunk was selected in the previous step ("index
      // scan to detect the missed chunks": one directory probe per selected chunk, R26)
      const uint16_t* vsrc = Ly.V_host + ((size_t)bh * D.s + (size_t)id * kChunk) * kHeadDim;
      if (Ly.vc_dir) {
        (void)ld_acquire_gpu(sp);            // order the probes after the publication (which follows
                                             // the previous call's generation bump)
        vc_gen = ld_relaxed_gpu_u64(Ly.vc_stats + (size_t)bh * 4);
        const unsigned long long e = ld_relaxed_gpu_u64(Ly.vc_dir + (size_t)bh * D.n_c + id);
        const unsigned tag = (unsigned)(e >> 32);         // inserting generation + 1; 0 = not cached
        if (tag != 0u && tag <= (unsigned)vc_gen) {        // cached by an earlier step and still resident
          vsrc = Ly.vc_values + ((size_t)bh * Ly.vc_cap + (unsigned)e) * (kChunk * kHeadDim);
          vc_hit = true;
          atomicAdd(Ly.vc_stats + (size_t)bh * 4 + 1, 1ull);
        }
      }
      mbar_expect_tx(&barVc[tid], kChunk * kHeadDim * 2);
      bulk_g2s(Vs + tid * kChunk * kHeadDim, vsrc, kChunk * kHeadDim * 2, &barVc[tid]);
    } else if (kind == 0 && tid < kUnitTok && tid >= nch * kChunk) {
      tok[tid] = 0;                                      // padded rows (masked below)
    }
    ntok = kind == 0 ? nch * kChunk : min(kUnitTok, n_gen - ui * kUnitTok);
    if (early_next) pdl_trigger();                       // next layer's score may become resident
    trace(2, 2);
    if (D.serial)                                        // SKV_SERIALIZE: values first, then the rebuild
      for (int c = 0; c < (kind == 0 ? nch : 1); ++c) mbar_wait(&barVc[c], 0);
    // ---- K~ = A_rows . B_h on the 5th-generation tensor cores (Alg 2 "MatMul(Gather(A, I), B)"):
    //      one thread issues r/16 tcgen05.mma (M = 128 rows of which 64 are the unit's tokens, N = 128, K = 16
    //      each) into an fp32 TMEM accumulator; completion is committed to barMMA
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
      mbar_wait(&barAB, 0);
      tc_fence_after();
      trace(2, 3);
      const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs), lbo = (uint32_t)D.r * 128u;
      for (int ks = 0; ks < (D.r >> 4); ++ks)
        umma_f16(tmem, umma_desc_sw128(a0 + (ks >> 2) * 8192 + (ks & 3) * 32), umma_desc_sw128_mn(b0 + ks * 2048, lbo),
                 kIdescRebuild, ks > 0);
      umma_commit(&barMMA);
    }
    __syncwarp();
    // ---- epilogue: warps 0, 1, 4, 5 read TMEM lanes 0..63 (one token row per thread, lane quadrant =
    //      warp % 4); the two warps of a row split its 128 columns into RoPE-closed sets (rope_row)
    float x0[32], x1[32];
    const int erow = 32 * (warp & 1) + lane, eset = warp >> 2;
    int c0, c1;
    rope_col_sets(R, eset, &c0, &c1);
    const bool epi = (warp & 2) == 0;
    if (epi) {
      mbar_wait(&barMMA, 0);
      tc_fence_after();
      const uint32_t tr = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
      tmem_ld32(tr + c0, x0);
      tmem_ld32(tr + c1, x1);
      rope_row(x0, x1, c0, c1, tok[erow], R);          // RoPE at the token's absolute position (R15, R16)
    }
    if (dbg && kind == 0) {   // a4 parity hook: bf16 of the fp32 keys at the chunk's rank in the ascending selection
      mbar_wait(&barMMA, 0);                             // the MMA has consumed the A tile: reuse it for the ids
      __syncthreads();
      int* ids = reinterpret_cast<int*>(As);
      for (int i = tid; i < D.k; i += 256) {
        int v;
        const uint64_t t0 = globaltimer();
        while ((v = ld_relaxed_gpu(slots + i)) == 0) { __nanosleep(32); spin_guard(t0); }
        ids[i] = v - 1;
      }
      __syncthreads();
      if (epi && erow < ntok) {
        const int cid = tok[erow] >> 3;
        int pos = 0;
        for (int c = 0; c < D.k; ++c) pos += ids[c] < cid;
        uint16_t* drow = dbg + (((size_t)bh * D.k + pos) * kChunk + (erow & 7)) * kHeadDim;
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          *reinterpret_cast<uint4*>(drow + c0 + e) = make_uint4(pack_bf2(x0[e], x0[e + 1]), pack_bf2(x0[e + 2], x0[e + 3]),
                                                                pack_bf2(x0[e + 4], x0[e + 5]), pack_bf2(x0[e + 6], x0[e + 7]));
          *reinterpret_cast<uint4*>(drow + c1 + e) = make_uint4(pack_bf2(x1[e], x1[e + 1]), pack_bf2(x1[e + 2], x1[e + 3]),
                                                                pack_bf2(x1[e + 4], x1[e + 5]), pack_bf2(x1[e + 6], x1[e + 7]));
        }
      }
    }
    if constexpr (G >= 8) {
      // ---- logits on the tensor cores (G >= 8 query rows fill an m16 tile): the fp32 post-RoPE keys go
      //      through smem (over the consumed A / B_h tiles) and S[16][64] = Q[16][128] . K~^T runs as
      //      mma.sync m16n8k8 TF32 (q is bf16: exact; keys rounded to TF32, 2^-11 relative)
      float* Ksm = reinterpret_cast<float*>(As);
      mbar_wait(&barMMA, 0);                             // (every warp: the MMA has read A and B_h)
      __syncthreads();
      if (epi) {
        float* kr = Ksm + erow * kKStride;
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          *reinterpret_cast<float4*>(kr + c0 + e) = make_float4(x0[e], x0[e + 1], x0[e + 2], x0[e + 3]);
          *reinterpret_cast<float4*>(kr + c1 + e) = make_float4(x1[e], x1[e + 1], x1[e + 2], x1[e + 3]);
        }
      }
      __syncthreads();
      float c[4];
      qk_tile_mma<G>(qs, Ksm, warp, lane, c);
      const int g = lane >> 2, t = lane & 3, col = 8 * warp + 2 * t;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int hq = g + 8 * (x >> 1), row = col + (x & 1);
        if (hq < G) {
          const bool vis = row < ntok && (kind == 0 || ui * kUnitTok + row < stp0 + 1 + hq % D.sq);
          P[hq * kPStride + row] = vis ? c[x] * scale : -INFINITY;
        }
      }
    } else {
      // ---- logits q . k~ (fp32 keys), half a row per thread, combined below in a fixed order
      if (epi) {
  #pragma unroll 4
        for (int hq = 0; hq < G; ++hq) {
          const float* qh = qs + hq * kQStride;
          float a = 0.f, bsum = 0.f;
  #pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 qa = *reinterpret_cast<const float4*>(qh + c0 + e);
            const float4 qb = *reinterpret_cast<const float4*>(qh + c1 + e);
            a = fmaf(x0[e], qa.x, a); a = fmaf(x0[e + 1], qa.y, a); a = fmaf(x0[e + 2], qa.z, a); a = fmaf(x0[e + 3], qa.w, a);
            bsum = fmaf(x1[e], qb.x, bsum); bsum = fmaf(x1[e + 1], qb.y, bsum);
            bsum = fmaf(x1[e + 2], qb.z, bsum); bsum = fmaf(x1[e + 3], qb.w, bsum);
          }
          Pp[(eset * G + hq) * kUnitTok + erow] = a + bsum;
        }
      }
      __syncthreads();
      for (int idx = tid; idx < G * kUnitTok; idx += 256) {
        const int hq = idx / kUnitTok, row = idx - hq * kUnitTok;
        // generated low-rank unit: token g = ui*64 + row is seen by query row hq (token i = hq % s_q) iff
        // g <= step + i (causal, R28)
        const bool vis = row < ntok && (kind == 0 || ui * kUnitTok + row < stp0 + 1 + hq % D.sq);
        P[hq * kPStride + row] = vis ? (Pp[hq * kUnitTok + row] + Pp[(G + hq) * kUnitTok + row]) * scale : -INFINITY;
      }
    }
  } else {
    // ---- outlier or window (R8, R18) unit: exact keys and values from HBM
    if (early_next) pdl_trigger();
    cta_wait_flag(&flags[(size_t)bh * 4]);              // (score's window append is visible)
    const uint16_t *Ksrc, *Vsrc;
    uint16_t* Ks = reinterpret_cast<uint16_t*>(As);
    if (kind == 1) {
      ntok = min(kUnitTok, T_out - ui * kUnitTok);
      Ksrc = Ly.K_out + ((size_t)bh * T_out + ui * kUnitTok) * kHeadDim;
      Vsrc = Ly.V_out + ((size_t)bh * T_out + ui * kUnitTok) * kHeadDim;
    } else {
      ntok = min(kUnitTok, T_win - ui * kUnitTok);
      Ksrc = Ly.K_win + ((size_t)bh * D.wcap + ui * kUnitTok) * kHeadDim;
      Vsrc = Ly.V_win + ((size_t)bh * D.wcap + ui * kUnitTok) * kHeadDim;
    }
    if (ntok <= 0) {                 // window unit past the live window (grid sized for max_step)
      for (int hq = tid >> 7; hq < G; hq += 2) {
        const size_t row = ((size_t)b * D.hq + (size_t)h * G + hq) * n_split + split;
        const unsigned tg = tagv[hq];
        st_tagged(o_part + row * kHeadDim + (tid & 127), 0.f, tg);
        if ((tid & 127) == 0) { st_tagged(ml_part + 2 * row, -INFINITY, tg); st_tagged(ml_part + 2 * row + 1, 0.f, tg); }
      }
      return;
    }
    if (tid == 0) {
      mbar_expect_tx(&barAB, ntok * kHeadDim * 2);
      bulk_g2s(Ks, Ksrc, ntok * kHeadDim * 2, &barAB);
      mbar_expect_tx(&barVc[0], ntok * kHeadDim * 2);
      bulk_g2s(Vs, Vsrc, ntok * kHeadDim * 2, &barVc[0]);
    }
    mbar_wait(&barAB, 0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = ty + 16 * i;
      if (row < ntok) unpack8(*reinterpret_cast<const uint4*>(Ks + row * kHeadDim + tx * 8), acc[i]);
      else {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[i][e] = 0.f;
      }
    }
    // ---- logits q . k for G heads: 4 tokens x (<= 4 heads) per lane per pass, reduced over 16 lanes
    constexpr int HC = G < 4 ? G : 4;
#pragma unroll
    for (int h0 = 0; h0 < G; h0 += HC) {
      float pv[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) pv[x] = 0.f;
#pragma unroll
      for (int hh = 0; hh < HC; ++hh) {
        const float4* qp = reinterpret_cast<const float4*>(qs + (h0 + hh) * kQStride + tx * 8);
        const float4 q0 = qp[0], q1 = qp[1];
        const float qv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float a = 0.f;
#pragma unroll
          for (int e = 0; e < 8; ++e) a = fmaf(qv[e], acc[i][e], a);
          pv[i * HC + hh] = a;
        }
      }
      reduce_scatter16<16>(pv, sub);
      if (sub < 4 * HC) {
        const int i = sub / HC, hq = h0 + sub % HC, row = ty + 16 * i;
        // window unit: query row hq (token i = hq % s_q) sees new tokens 0..i only (causal, R28)
        const bool vis = row < ntok && (kind == 1 || (kind == 2 && lowrank) ||
                                        ui * kUnitTok + row < T_win - D.sq + 1 + hq % D.sq);
        P[hq * kPStride + row] = vis ? pv[0] * scale : -INFINITY;
      }
    }
  }
  __syncthreads();
  // ---- softmax statistics of this unit (per q head)
  for (int hq = warp; hq < G; hq += 8) {
    float x0 = P[hq * kPStride + lane], x1 = P[hq * kPStride + lane + 32];
    const float m = warp_max(fmaxf(x0, x1));
    // (a row can be fully masked: a window unit past this query token's causal limit)
    const float e0 = x0 > -INFINITY ? expf(x0 - m) : 0.f, e1 = x1 > -INFINITY ? expf(x1 - m) : 0.f;
    P[hq * kPStride + lane] = e0;
    P[hq * kPStride + lane + 32] = e1;
    const float l = warp_sum(e0 + e1);
    if (lane == 0) ml[hq] = make_float2(m, l);
  }
  trace(2, 4);
  __syncthreads();                                       // probabilities P and ml[] complete
  // a5 -> a6: the values of a selected-chunk unit land chunk by chunk (barVc[c]); the PV consumes them
  // as they arrive, so only the last chunk's 8 tokens remain once the host link delivers it.  The
  // result does not depend on the arrival order: per-chunk partial sums, combined in chunk order.
  const int nvb = kind == 0 ? nch : 1;                   // value barriers of this unit
  auto vc_write_back = [&]() {                           // a missed chunk enters the cache (R26)
    if (vc_hit) return;
    const int pos = ui * 8 + tid;                        // its position in the published selection
    const unsigned long long* as = Ly.vc_slots + (size_t)bh * (Ly.vc_cap + D.k) + Ly.vc_cap + pos;
    const uint64_t t0 = globaltimer();
    unsigned long long a;
    while ((unsigned)((a = ld_relaxed_gpu_u64(as)) >> 32) != (unsigned)(vc_gen + 1)) { __nanosleep(32); spin_guard(t0); }
    fence_proxy_async();
    bulk_s2g(Ly.vc_values + ((size_t)bh * Ly.vc_cap + (unsigned)a) * (kChunk * kHeadDim), Vs + tid * kChunk * kHeadDim,
             kChunk * kHeadDim * 2);
  };
  if constexpr (G >= 8) {
    // ---- PV on the tensor cores: O[16][128] = P[16][64] . V[64][128], mma.sync m16n8k8 TF32 (values bf16:
    //      exact; probabilities rounded to TF32); warp w owns dims 16w..16w+15; k step c = chunk c, taken
    //      in chunk order as each chunk lands
    float c[2][4];
    pv_tile_mma<G>(P, Vs, ntok, warp, lane, c, barVc, kind == 0);
    trace(2, 5);
    if (vc_id >= 0 && Ly.vc_dir) vc_write_back();
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int dim = 16 * warp + 8 * nt + 2 * t;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int hq = g + 8 * hh;
        if (hq < G) {
          const size_t row = ((size_t)b * D.hq + (size_t)h * G + hq) * n_split + split;
          st_tagged(o_part + row * kHeadDim + dim, c[nt][2 * hh], tagv[hq]);
          st_tagged(o_part + row * kHeadDim + dim + 1, c[nt][2 * hh + 1], tagv[hq]);
        }
      }
    }
  } else {
    // ---- PV: thread = (dim pair dp, q row hq < G <= 4): bf16x2 value loads, float4 probability loads
    const int dp = tid & 63, hq = tid >> 6;
    if (hq < G) {
      const float* ph = P + hq * kPStride;
      float2 acc = make_float2(0.f, 0.f);
      if (kind == 0) {
        float2 pc[8];                                    // per-chunk partial sums
        unsigned pending = (1u << nvb) - 1u;
        const uint64_t t0 = globaltimer();
        while (pending) {
          spin_guard(t0);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (((pending >> c) & 1u) && mbar_test(&barVc[c], 0)) {
              pending &= ~(1u << c);
              const float4 p0 = *reinterpret_cast<const float4*>(ph + 8 * c);
              const float4 p1 = *reinterpret_cast<const float4*>(ph + 8 * c + 4);
              const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
              float2 a = make_float2(0.f, 0.f);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint32_t v2 = *reinterpret_cast<const uint32_t*>(Vs + (8 * c + e) * kHeadDim + 2 * dp);
                a.x = fmaf(pp[e], bf_lo(v2), a.x);
                a.y = fmaf(pp[e], bf_hi(v2), a.y);
              }
              pc[c] = a;
              if (tid == c && vc_id >= 0 && Ly.vc_dir) vc_write_back();
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < nvb) { acc.x += pc[c].x; acc.y += pc[c].y; }
      } else {
        mbar_wait(&barVc[0], 0);
        const int ntok4 = (ntok + 3) & ~3;               // P is 0 past ntok; stale V rows are skipped
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
        for (int t = 0; t < ntok4; t += 4) {
          const float4 p4 = *reinterpret_cast<const float4*>(ph + t);
          const float pp[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t v2 = t + e < ntok ? *reinterpret_cast<const uint32_t*>(Vs + (t + e) * kHeadDim + 2 * dp) : 0u;
            float2& a = (e & 1) ? a1 : a0;
            a.x = fmaf(pp[e], bf_lo(v2), a.x);
            a.y = fmaf(pp[e], bf_hi(v2), a.y);
          }
        }
        acc = make_float2(a0.x + a1.x, a0.y + a1.y);
      }
      const size_t row = ((size_t)b * D.hq + (size_t)h * G + hq) * n_split + split;
      st_tagged(o_part + row * kHeadDim + 2 * dp, acc.x, tagv[hq]);
      st_tagged(o_part + row * kHeadDim + 2 * dp + 1, acc.y, tagv[hq]);
    }
    trace(2, 5);
  }
  // (m, l) last, once every thread has stored its values (and the value-cache write-back has completed:
  // the merge then closes the generation): the merge polls (m, l) first
  if (vc_id >= 0 && Ly.vc_dir) bulk_wait_all();
  __syncthreads();
  if (tid < G) {
    const size_t row = ((size_t)b * D.hq + (size_t)h * G + tid) * n_split + split;
    st_tagged(ml_part + 2 * row, ml[tid].x, tagv[tid]);
    st_tagged(ml_part + 2 * row + 1, ml[tid].y, tagv[tid]);
  }
  if (rebuild) {                                         // every TMEM read finished (tcgen05.ld waited)
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem_base);
  }
  trace(2, 8);
}

// Diagnostic (shadowkv_rope_sincos): the sine / cosine of the RoPE angle phi = fl32(fl32(t) *
// inv_freq[i]) exactly as the decode kernels compute it, for n positions x rot/2 frequencies.
__global__ void k_rope_probe(const int32_t* __restrict__ pos, int n, const float* __restrict__ inv_freq, int nf,
                             float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * nf) return;
  float s, c;
  rope_sincos(pos[i / nf], inv_freq[i % nf], &s, &c);
  out[2 * (size_t)i] = s;
  out[2 * (size_t)i + 1] = c;
}
cudaError_t launch_rope_probe(const int32_t* pos, int n, const float* inv_freq, int nf, float* out, cudaStream_t st) {
  const int total = n * nf;
  if (total > 0) k_rope_probe<<<(total + 255) / 256, 256, 0, st>>>(pos, n, inv_freq, nf, out);
  return cudaGetLastError();
}

// =============================================================================================
// host side
// =============================================================================================
static int tiles_per_head(const Dims& D) { return (D.n_c + kSTile - 1) / kSTile; }
static bool z_fits_smem(const Dims& D, int) {          // z slice in smem
  return (size_t)(((D.n_c + kSelCL - 1) / kSelCL + 3) & ~3) * 4 <= kSelectSmemMax;
}

size_t decode_ws_bytes(const Dims& D, DecodeWs* ws, char* base) {
  size_t off = ws_header_bytes(D);                  // zero-initialised per-(b,h) counters live first
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return base + o; };
  const int tph = tiles_per_head(D);
  const int n_sel_u = (D.k + 7) / 8, n_out_u = (D.o * kChunk + kUnitTok - 1) / kUnitTok;
  const int n_win_max = (D.wcap + kUnitTok - 1) / kUnitTok + 1;   // (+1: tail and generated units split, NEXT-4)
  const int n_split = n_sel_u + n_out_u + n_win_max;
  const size_t BHq = (size_t)D.b * D.hq, BHk = (size_t)D.b * D.hk;
  char* p_log = carve(BHq * D.n_c * 4);
  char* p_part = carve(BHq * tph * 8);              // per-(tile, query row) softmax partials
  char* p_z = carve(BHk * D.n_c * 4);                // select fallback / large-n_c slices
  char* p_sel = carve(BHk * D.k * 4);                // definite selections (and the radix fallback)
  char* p_rest = carve(BHk * D.k * 4);               // threshold-bucket selections
  char* p_op = carve(BHq * n_split * kHeadDim * 8);  // {value, tag} pairs
  char* p_ml = carve(BHq * n_split * 16);
  if (ws) {
    ws->logits = reinterpret_cast<float*>(p_log);
    ws->part = reinterpret_cast<float2*>(p_part);
    ws->z = reinterpret_cast<float*>(p_z);
    ws->sel = reinterpret_cast<int32_t*>(p_sel);
    ws->o_part = reinterpret_cast<uint2*>(p_op);
    ws->ml_part = reinterpret_cast<uint2*>(p_ml);
    ws->flags = reinterpret_cast<int*>(base);
    ws->epochs = reinterpret_cast<int*>(base) + (size_t)D.b * D.hk * 4;
    ws->selrest = reinterpret_cast<int32_t*>(p_rest);
    ws->n_sblk = tph;
    ws->n_split = n_split;
  }
  return off;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr; cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// tuning switches (process environment, read once); the test hooks SKV_NO_TC and
// SKV_SELECT_FALLBACK are read per call because tests toggle them inside one process
struct Tuning {
  int early_next, merge_late;
};
static const Tuning& tuning() {
  static const Tuning t = [] {
    auto is = [](const char* name, char c) { const char* v = getenv(name); return v && v[0] == c; };
    return Tuning{is("SKV_SPARSE_TRIGGER", '0') ? 0 : 1, is("SKV_MERGE_TRIGGER", 'l') ? 1 : 0};
  }();
  return t;
}

// kernel attributes of every decode instantiation, set once per device by shadowkv_init
template <int G>
static cudaError_t set_decode_attrs_g() {
  cudaError_t e;
  int optin = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  // CUDA-core scorer (test hook SKV_NO_TC): its outlier bitmap grows with n_c, so allow the device maximum
  if ((e = cudaFuncGetAttributes(&fa, k_score<G>))) return e;
  if ((e = cudaFuncSetAttribute(k_score<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes))) return e;
  if ((e = cudaFuncSetAttribute(k_select<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelectSmemMax))) return e;
  if ((e = cudaFuncSetAttribute(k_select<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelectSmemMax))) return e;
  if ((e = cudaFuncSetAttribute(k_sparse_attn<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)attn_smem_layout(256, G).bytes))) return e;
  return cudaSuccess;
}
cudaError_t init_decode_attrs() {
  cudaError_t e;
  if ((e = set_decode_attrs_g<1>()) || (e = set_decode_attrs_g<2>()) || (e = set_decode_attrs_g<4>()) ||
      (e = set_decode_attrs_g<8>()) || (e = set_decode_attrs_g<16>())) return e;
  return cudaSuccess;
}

// 2D bf16 tensor map [outer][inner] (row pitch inner * 2 bytes), box {box_inner, box_outer}, SWIZZLE_128B
static bool encode_bf16_2d(const DevCtx& ctx, CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                           uint32_t box_inner, uint32_t box_outer) {
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
  if (!enc) return false;
  const cuuint64_t gdim[2] = {inner, outer};
  const cuuint64_t gstride[1] = {inner * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int G>
static cudaError_t launch_decode_g(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                                   const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                                   int32_t* sel_ids, uint16_t* dbg_keys, const DecodeWs& ws,
                                   cudaStream_t st, int* launches, Profiler* prof, cudaEvent_t ev_sel,
                                   const DevCtx& ctx) {
  const float scale = (float)(1.0 / 11.313708498984761);    // 1/sqrt(d), d = 128 (R6)
  const AttnSmem lay = attn_smem_layout(D.r, G);
  cudaError_t e;
  const int tph = ws.n_sblk;
  const int total_tiles = D.b * D.hk * tph;
  // a1: the tcgen05 scorer (TMA + TMEM).  The CUDA-core k_score is a test hook only (SKV_NO_TC=1):
  // a failing tensor-map encode or an unplannable grid is an error, not a silent second backend.
  const char* nt = getenv("SKV_NO_TC");
  if (prof) profile_mark(prof, kScore, false, st);
  nvtxRangePushA("skv::score");
  if (nt && nt[0] == '1') {
    const int grid_s = total_tiles < 2 * ctx.n_sm ? total_tiles : 2 * ctx.n_sm;
    const size_t score_smem = (size_t)kSStages * kSTile * kHeadDim * 2 + 2 * G * kSTile * 4 +
                              (size_t)((D.n_c + 31) / 32) * 4;
    k_score<G><<<grid_s, 256, score_smem, st>>>(D, Ly.L, Ly.outlier_ids, q, ws.logits, ws.part, tph, scale, k_new,
                                                v_new, Ly.K_win, Ly.V_win, step);
    e = cudaGetLastError();
  } else {
    ScorePlan pl;
    if (!score_tc_plan(D, tph, ctx.n_sm, &pl)) return cudaErrorNotSupported;
    e = launch_score_tc<G>(D, Ly.L, Ly.outlier_ids, q, ws.logits, ws.part, tph, scale, k_new, v_new, Ly.K_win,
                           Ly.V_win, step, ctx, st);
  }
  nvtxRangePop();
  if (e) return e;
  if (prof) { profile_mark(prof, kScore, true, st); profile_mark(prof, kSelect, false, st); }
  {
    const char* fb = getenv("SKV_SELECT_FALLBACK");       // test hook: 1 / 2 force the radix fallback
    const int force_fb = fb ? atoi(fb) : 0;               // before / after the definite chunks publish
    nvtxRangePushA("skv::select");
    const bool zsm = z_fits_smem(D, G);
    size_t sel_smem = zsm ? (size_t)(((D.n_c + kSelCL - 1) / kSelCL + 3) & ~3) * 4 : 0;
    VcArgs vc{Ly.vc_dir, Ly.vc_stats, Ly.vc_slots, Ly.vc_cap, 1};
    if (Ly.vc_dir) {                                      // the value cache's slot assignment (R26)
      while (vc.Cp < vc.C) vc.Cp <<= 1;
      const size_t vb = vc_assign_smem_bytes(D.k, vc.Cp);
      if (vb > kSelectSmemMax) return cudaErrorInvalidValue;
      if (vb > sel_smem) sel_smem = vb;
    }
    if (zsm) e = launch_pdl(!D.serial, k_select<G, true>, dim3(D.b * D.hk * kSelCL), dim3(kSelThreads), sel_smem, st, D,
                            (const float*)ws.logits, (const float2*)ws.part, tph, ws.z,
                            ws.sel, ws.selrest, ws.flags, sel_ids, force_fb, vc);
    else e = launch_pdl(!D.serial, k_select<G, false>, dim3(D.b * D.hk * kSelCL), dim3(kSelThreads), sel_smem, st, D,
                        (const float*)ws.logits, (const float2*)ws.part, tph, ws.z,
                        ws.sel, ws.selrest, ws.flags, sel_ids, force_fb, vc);
    nvtxRangePop();
    if (e) return e;
    if (prof) { profile_mark(prof, kSelect, true, st); profile_mark(prof, kSparseAttn, false, st); }
    if (ev_sel && (e = cudaEventRecord(ev_sel, st))) return e;   // sub-batch pipelining: next chain may start
  }
  const int n_sel_u = (D.k + 7) / 8, n_out_u = (D.o * kChunk + kUnitTok - 1) / kUnitTok;
  const int n_live = (D.step_dev ? D.max_step : step) + D.sq;   // generated tokens the grid is sized for
  // plain window: one run of units over tail + generated; low-rank generated keys (NEXT-4): tail units
  // (exact keys) + generated units (keys rebuilt from their rank-r rows)
  const int n_win_u = D.lr_A ? (D.w_eff + kUnitTok - 1) / kUnitTok : (D.w_eff + n_live + kUnitTok - 1) / kUnitTok;
  const int n_gen_u = D.lr_A ? (n_live + kUnitTok - 1) / kUnitTok : 0;
  const int n_split = n_sel_u + n_out_u + n_win_u + n_gen_u;
  const int units = D.b * D.hk * n_split;
  // tuning hook: SKV_SPARSE_TRIGGER=0 keeps the implicit trigger at CTA exit (the next layer's score
  // grid then launches only when this grid drains)
  const int early_next = tuning().early_next;
  // TMA tensor maps of the rebuild's operands: A [b*s][r] and A_gen [b*wcap][r] in 8-row x 64-column
  // SWIZZLE_128B boxes (one chunk's K block), B [b*h_kv*r][128] in r-row x 64-column boxes (MN-major)
  CUtensorMap tmA, tmB, tmG;
  if (!encode_bf16_2d(ctx, &tmA, Ly.A, D.r, (uint64_t)D.b * D.s, 64, 8) ||
      !encode_bf16_2d(ctx, &tmB, Ly.B, kHeadDim, (uint64_t)D.b * D.hk * D.r, 64, D.r) ||
      !encode_bf16_2d(ctx, &tmG, D.lr_A ? D.lr_A : Ly.A, D.r, D.lr_A ? (uint64_t)D.b * D.wcap : (uint64_t)D.b * D.s, 64, 8))
    return cudaErrorInvalidValue;
  nvtxRangePushA("skv::sparse_attn");
  e = launch_pdl(!D.serial, k_sparse_attn<G>, dim3(units), dim3(256), (size_t)lay.bytes, st, tmA, tmB, tmG, D, R, Ly, q,
                      ws.sel, ws.flags, step, ws.o_part, ws.ml_part, (const int*)ws.epochs,
                      n_sel_u, n_out_u, n_win_u, n_gen_u, n_split, scale, dbg_keys, early_next);
  nvtxRangePop();
  if (e) return e;
  if (prof) profile_mark(prof, kSparseAttn, true, st);
  const int merge_late = tuning().merge_late;            // SKV_MERGE_TRIGGER=late: after the loads
  if (prof) profile_mark(prof, kCombine, false, st);
  nvtxRangePushA("skv::merge");
  e = launch_pdl(!D.serial, k_merge<G>, dim3(D.b * D.hq), dim3(kHeadDim), (size_t)n_split * (sizeof(float2) + sizeof(float)), st, D,
                      (const uint2*)ws.o_part, (const uint2*)ws.ml_part, ws.epochs, n_split, ws.sel, ws.flags, out,
                      merge_late, Ly.vc_stats);
  nvtxRangePop();
  if (e) return e;
  if (prof) profile_mark(prof, kCombine, true, st);
  *launches += 4;


  return cudaGetLastError();
}

static cudaError_t launch_decode_one(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                                     const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                                     int32_t* sel_ids, uint16_t* dbg_keys, const DecodeWs& ws, cudaStream_t st,
                                     int* launches, Profiler* prof, cudaEvent_t ev_sel, const DevCtx& ctx) {
  switch (D.g) {
    case 1: return launch_decode_g<1>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches, prof, ev_sel, ctx);
    case 2: return launch_decode_g<2>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches, prof, ev_sel, ctx);
    case 4: return launch_decode_g<4>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches, prof, ev_sel, ctx);
    case 8: return launch_decode_g<8>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches, prof, ev_sel, ctx);
    case 16: return launch_decode_g<16>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches, prof, ev_sel, ctx);
  }
  return cudaErrorInvalidValue;
}

// ---- request sub-batch pipelining ------------------------------------------------------------
// Requests are independent, so a large batch is cut into S sub-batches whose score -> select ->
// sparse -> merge chains run on S streams: chain s + 1 starts (event) once chain s has its
// selection, on a high-priority internal stream, so its HBM-bound scoring and its selection run
// while chain s streams its values over the host link (which would otherwise idle through them).
// The caller's stream joins every chain before returning.  Each chain has its own workspace region.
// Measured gain is small (c3, 64 requests, 4 chains: +2 %; c5, 12 requests: none): the chains'
// sparse grids hold the SMs, so a later chain's scoring only gets slots as earlier CTAs retire.
static int split_count(const Dims& D) {
  static const int env = [] { const char* v = getenv("SKV_SPLIT"); return v ? atoi(v) : 0; }();
  const int n = env > 0 ? env : (D.b >= 32 ? 4 : 1);   // measured: +2 % at c3 (64), none at c5 (12)
  return n < 1 ? 1 : (n > D.b ? D.b : (n > kMaxSplit ? kMaxSplit : n));
}
static Dims sub_dims(const Dims& D, int nb) { Dims s = D; s.b = nb; return s; }
static size_t split_ws_bytes(const Dims& D, int n, size_t* offs) {
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int r0 = D.b * i / n, r1 = D.b * (i + 1) / n;
    if (offs) offs[i] = off;
    off += (decode_ws_bytes(sub_dims(D, r1 - r0), nullptr, nullptr) + 255) & ~(size_t)255;
  }
  return off;
}
// The zero-between-calls state (counters, flags, slots) of one layout must never be scribbled on by
// another, so the profiler's single-chain layout (per-kernel events need one stream) gets a block
// of its own after the split layout.
size_t decode_ws_total_bytes(const Dims& D) {
  const int n = split_count(D);
  return split_ws_bytes(D, n, nullptr) + (n > 1 ? split_ws_bytes(D, 1, nullptr) : 0);
}

cudaError_t launch_decode(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                          const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                          int32_t* sel_ids, uint16_t* dbg_keys, char* ws_base, cudaStream_t st,
                          int* launches, Profiler* prof, const DevCtx& ctx) {
  const int nd = split_count(D);
  const int n = prof ? 1 : nd;
  if (n == 1) {
    DecodeWs ws;
    decode_ws_bytes(D, &ws, ws_base + (nd > 1 ? split_ws_bytes(D, nd, nullptr) : 0));
    return launch_decode_one(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches, prof, nullptr,
                             ctx);
  }
  // the chains' streams and events belong to the device context (created by shadowkv_init)
  const cudaStream_t* side = ctx.side;
  const cudaEvent_t* ev_sel = ctx.ev_sel;
  const cudaEvent_t* ev_done = ctx.ev_done;
  std::lock_guard<std::mutex> lk(chain_mutex(ctx.device));   // one call's fork/join at a time per device
  cudaError_t e;
  size_t offs[kMaxSplit];
  split_ws_bytes(D, n, offs);
  const size_t s = D.s, hk = D.hk, hq = D.hq, d = kHeadDim;
  for (int i = 0; i < n; ++i) {
    const int r0 = D.b * i / n, nb = D.b * (i + 1) / n - r0;
    Dims Ds = sub_dims(D, nb);
    if (D.lens) Ds.lens = D.lens + r0;
    Layer L = Ly;
    L.A = Ly.A + (size_t)r0 * s * D.r;
    L.B = Ly.B + (size_t)r0 * hk * D.r * d;
    L.L = Ly.L + (size_t)r0 * hk * D.n_c * d;
    L.outlier_ids = Ly.outlier_ids ? Ly.outlier_ids + (size_t)r0 * hk * D.o : nullptr;
    L.K_out = Ly.K_out ? Ly.K_out + (size_t)r0 * hk * D.o * kChunk * d : nullptr;
    L.V_out = Ly.V_out ? Ly.V_out + (size_t)r0 * hk * D.o * kChunk * d : nullptr;
    L.K_win = Ly.K_win + (size_t)r0 * hk * D.wcap * d;
    L.V_win = Ly.V_win + (size_t)r0 * hk * D.wcap * d;
    L.V_host = Ly.V_host + (size_t)r0 * hk * s * d;
    if (D.lr_A) { Ds.lr_A = D.lr_A + (size_t)r0 * D.wcap * D.r; Ds.lr_B = L.B; }
    if (Ly.vc_dir) {
      L.vc_values = Ly.vc_values + (size_t)r0 * hk * Ly.vc_cap * kChunk * d;
      L.vc_dir = Ly.vc_dir + (size_t)r0 * hk * D.n_c;
      L.vc_stats = Ly.vc_stats + (size_t)r0 * hk * 4;
      L.vc_slots = Ly.vc_slots + (size_t)r0 * hk * (Ly.vc_cap + D.k);
    }
    DecodeWs ws;
    decode_ws_bytes(Ds, &ws, ws_base + offs[i]);
    cudaStream_t si = i == 0 ? st : side[i - 1];
    if (i > 0 && (e = cudaStreamWaitEvent(si, ev_sel[i - 1], 0))) return e;
    e = launch_decode_one(Ds, R, L, q + (size_t)r0 * hq * d, k_new + (size_t)r0 * hk * D.sq * d,
                          v_new + (size_t)r0 * hk * D.sq * d,
                          step, out + (size_t)r0 * hq * d, sel_ids ? sel_ids + (size_t)r0 * hk * D.k : nullptr,
                          dbg_keys ? dbg_keys + (size_t)r0 * hk * D.k * kChunk * d : nullptr, ws, si, launches,
                          nullptr, i + 1 < n ? ev_sel[i] : nullptr, ctx);
    if (e) return e;
  }
  for (int i = 1; i < n; ++i) {                          // the caller's stream joins every chain
    if ((e = cudaEventRecord(ev_done[i - 1], side[i - 1]))) return e;
    if ((e = cudaStreamWaitEvent(st, ev_done[i - 1], 0))) return e;
  }
  return cudaSuccess;
}

}  // namespace skv
