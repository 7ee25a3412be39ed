// RoPE of a rebuilt key row held in registers after a tcgen05.ld (decode's key rebuild, the build's
// key tiles).  R15: angle fl32(fl32(t) * inv_freq), rope_sincos.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace skv {

// RoPE (R15) of one token row held as two 32-column blocks x0 = cols [c0, c0+32), x1 = cols [c1, c1+32)
// of the rebuilt key.  The column sets are chosen so that every rotation pair lies in one thread:
// halves layout with rot = 128 (Llama): set s holds cols [32s, 32s+32) and their partners +64;
// rot <= 64 (halves, rot/2 in {8, 16, 32}) or interleaved: set s holds [64s, 64s+64).
// the two 32-column blocks thread set `set` (0 / 1) holds for rope_row
__device__ __forceinline__ void rope_col_sets(const Rope& R, int set, int* c0, int* c1) {
  const bool hl = !R.interleaved && R.rot > 64;
  *c0 = hl ? 32 * set : 64 * set;
  *c1 = hl ? 64 + 32 * set : 64 * set + 32;
}

__device__ __forceinline__ void rope_row(float* x0, float* x1, int c0, int c1, int t, const Rope& R) {
  if (R.interleaved) {
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      float* x = blk ? x1 : x0;
      const int cb = blk ? c1 : c0;
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        if (cb + e < R.rot) {
          float sn, cs;
          rope_sincos(t, __ldg(R.inv_freq + ((cb + e) >> 1)), &sn, &cs);
          const float a = x[e], b = x[e + 1];
          x[e] = a * cs - b * sn;
          x[e + 1] = b * cs + a * sn;
        }
      }
    }
    return;
  }
  const int half = R.rot >> 1;
  auto rot2 = [&](float& a, float& b, int i) {
    float sn, cs;
    rope_sincos(t, __ldg(R.inv_freq + i), &sn, &cs);
    const float x = a, y = b;
    a = x * cs - y * sn;
    b = y * cs + x * sn;
  };
  if (half == 64) {                                     // pairs (c0 + e, c0 + 64 + e) = (x0[e], x1[e])
#pragma unroll
    for (int e = 0; e < 32; ++e) rot2(x0[e], x1[e], c0 + e);
  } else if (c0 == 0) {                                 // set 0 holds every rotary dim (rot <= 64)
    if (half == 32) {
#pragma unroll
      for (int e = 0; e < 32; ++e) rot2(x0[e], x1[e], e);
    } else if (half == 16) {
#pragma unroll
      for (int e = 0; e < 16; ++e) rot2(x0[e], x0[e + 16], e);
    } else if (half == 8) {
#pragma unroll
      for (int e = 0; e < 8; ++e) rot2(x0[e], x0[e + 8], e);
    }
  }
}

}  // namespace skv
