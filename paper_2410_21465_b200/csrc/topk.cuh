// Block-wide exact top-k with deterministic ties (product path).
//
// Implements "ArgTopK(S2, k)" of Alg 2 and "ArgTopK(-Min(S), o)" of Alg 1:
// the k largest values of v[0..n), ties broken toward the LOWER index (R12), written in
// ascending index order.  MSB-first radix select over order-preserving 32-bit keys
// (4 passes x 8 bits, shared-memory histograms) finds the exact k-th largest key T;
// then every element with key > T plus the first (k - #{key > T}) elements with key == T
// are emitted through two block-wide exclusive scans over contiguous per-thread segments.
#pragma once
#include "common.cuh"

namespace skv {

template <int NT>
struct TopKSmem {
  int hist[256];
  int warp_tot[NT / 32];
  int bcast[4];
};

template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int x, TopKSmem<NT>& sm, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) sm.warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NT / 32 ? sm.warp_tot[lane] : 0;
    int s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) sm.warp_tot[lane] = s - w;   // exclusive warp offsets
    if (lane == 31) sm.bcast[3] = s;
  }
  __syncthreads();
  int res = sm.warp_tot[warp] + v - x;
  *total = sm.bcast[3];
  __syncthreads();
  return res;
}

// v: n floats (global/L2), out: k ids ascending.  All NT threads of the block must call.
template <int NT>
__device__ __forceinline__ void block_topk_largest(const float* __restrict__ v, int n, int k, int* __restrict__ out,
                                   TopKSmem<NT>& sm) {
  const int tid = threadIdx.x;
  uint32_t prefix = 0, mask = 0;
  int kr = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += NT) sm.hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      uint32_t u = f2key(v[i]);
      if ((u & mask) == prefix) atomicAdd(&sm.hist[(u >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns digits 255-8l .. 248-8l (descending)
      int cnt[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { cnt[j] = sm.hist[255 - 8 * tid - j]; s += cnt[j]; }
      int pre = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, pre, o);
        if (tid >= o) pre += y;
      }
      pre -= s;                                   // count of elements with larger digits
      if (pre < kr && kr <= pre + s) {
        int cum = pre;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + cnt[j] >= kr) { sm.bcast[0] = 255 - 8 * tid - j; sm.bcast[1] = kr - cum; break; }
          cum += cnt[j];
        }
      }
    }
    __syncthreads();
    prefix |= ((uint32_t)sm.bcast[0]) << shift;
    mask |= 255u << shift;
    kr = sm.bcast[1];
    __syncthreads();
  }
  // prefix = T (k-th largest key); kr = how many keys == T to take (lowest indices first)
  const uint32_t T = prefix;
  const int per = (n + NT - 1) / NT;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int gt = 0, eq = 0;
  for (int i = lo; i < hi; ++i) {
    uint32_t u = f2key(v[i]);
    gt += u > T;
    eq += u == T;
  }
  int tot;
  int eq_before = block_exclusive_scan<NT>(eq, sm, &tot);
  int take = min(max(kr - eq_before, 0), eq);
  int pos = block_exclusive_scan<NT>(gt + take, sm, &tot);
  for (int i = lo; i < hi; ++i) {
    uint32_t u = f2key(v[i]);
    bool sel = u > T;
    if (!sel && u == T && take > 0) { sel = true; --take; }
    if (sel) out[pos++] = i;
  }
}

}  // namespace skv
