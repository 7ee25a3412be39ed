// a7: the current call's K, V join the window (Alg 2 input K, V; R18), shared by both scorers.
//
// Plain window: k_new (post-RoPE) -> K_win, v_new -> V_win at slots w_eff(b) + step + i.
// Low-rank generated keys (NEXT-4, P:196 footnote; Dims::lr_A non-null): k_new is PRE-RoPE and is
// stored as one rank-r row a = sum_h k'_h B_h^T  (K' Psi with Psi[(h, j), rho] = B_h[rho][j], R14) in
// lr_A[b][step + i][:] (bf16); K_win is not written.  The attention rebuilds RoPE_t(a B_h).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace skv {

// called by every thread of the grid: thread_id / n_threads = grid-wide index / size
__device__ __forceinline__ void window_append(const Dims& D, const uint16_t* __restrict__ k_new,
                                             const uint16_t* __restrict__ v_new, uint16_t* K_win, uint16_t* V_win,
                                             int stp, int thread_id, int n_threads) {
  const bool lowrank = D.lr_A != nullptr;
  for (int idx = thread_id; idx < D.b * D.hk * D.sq * 32; idx += n_threads) {
    const int bhi = idx >> 5, arr = (idx >> 4) & 1, p = idx & 15;    // (b, h, new token i)
    if (lowrank && !arr) continue;
    const int bh = bhi / D.sq, i = bhi - bh * D.sq;
    const size_t dst = ((size_t)bh * D.wcap + req_weff(D, bh / D.hk) + stp + i) * kHeadDim + p * 8;
    const uint16_t* src = (arr ? v_new : k_new) + (size_t)bhi * kHeadDim + p * 8;
    *reinterpret_cast<uint4*>((arr ? V_win : K_win) + dst) = *reinterpret_cast<const uint4*>(src);
  }
  if (!lowrank) return;
  // one warp per (b, i, rho): a[rho] = sum_{h, j} k'[b][h][i][j] * B[b][h][rho][j]
  const int lane = thread_id & 31, wid = thread_id >> 5, nw = n_threads >> 5;
  for (int item = wid; item < D.b * D.sq * D.r; item += nw) {
    const int rho = item % D.r, bi = item / D.r, b = bi / D.sq, i = bi - b * D.sq;
    float acc = 0.f;
    for (int h = 0; h < D.hk; ++h) {
      const uint2 kv = *reinterpret_cast<const uint2*>(k_new + (((size_t)b * D.hk + h) * D.sq + i) * kHeadDim + lane * 4);
      const uint2 bv = *reinterpret_cast<const uint2*>(D.lr_B + (((size_t)b * D.hk + h) * D.r + rho) * kHeadDim + lane * 4);
      acc = fmaf(bf_lo(kv.x), bf_lo(bv.x), acc); acc = fmaf(bf_hi(kv.x), bf_hi(bv.x), acc);
      acc = fmaf(bf_lo(kv.y), bf_lo(bv.y), acc); acc = fmaf(bf_hi(kv.y), bf_hi(bv.y), acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) D.lr_A[((size_t)b * D.wcap + stp + i) * D.r + rho] = f2bf(acc);
  }
}

}  // namespace skv
