// Key-tile producer: post-RoPE keys for up to 128 tokens of one (request, KV head).
//
//   k_t = RoPE_t( A[t, :r] . B_h[:r, :] )        (Alg 2 "K^sparse <- MatMul(Gather(A, I), B)",
//                                                  "RoPE(K^sparse)"; Alg 1 keys)
// or, when the caller supplied post-RoPE keys, k_t = K_rope[t] (Alg 1 input K^RoPE).
//
// CUDA-core fp32 version (v1): A rows and B_h staged in shared memory, 256 threads, each
// thread accumulates 8 tokens x 8 dims; RoPE applied in place on the fp32 tile
// (angle fl32(fl32(t) * inv_freq), reduced mod 2 pi in fp64, hardware sincos on |r| <= pi -- R15, rope_sincos).  Result: fp32 [128][128] in smem.
#pragma once
#include "common.cuh"

namespace skv {

constexpr int kTileTok = 128;
constexpr int kTileThreads = 256;

__host__ __device__ constexpr size_t keytile_smem_bytes(int r) {
  size_t ab = (size_t)kTileTok * r * 2 + (size_t)r * kHeadDim * 2;
  size_t kt = (size_t)kTileTok * kHeadDim * 4;
  return (ab > kt ? ab : kt) + kTileTok * sizeof(int);
}

struct RopeArgs {
  const float* inv_freq;
  int rot;
  int interleaved;
};

// tok[i] (smem, i < ntok) = absolute token positions. Tokens >= ntok produce zeros.
// A_b = A + b*s*r, B_bh = B + (b*h_kv + h)*r*d, Kr_bh = K_rope + (b*h_kv + h)*s*d (or nullptr).
static __device__ void produce_key_tile(const uint16_t* __restrict__ A_b, const uint16_t* __restrict__ B_bh,
                                 const uint16_t* __restrict__ Kr_bh, int r, const int* tok, int ntok,
                                 RopeArgs rope, uint8_t* smem, float* Ks /* aliases smem */) {
  const int tid = threadIdx.x;
  if (Kr_bh != nullptr) {
    // given post-RoPE keys: just widen
    __syncthreads();
    for (int idx = tid; idx < kTileTok * 16; idx += kTileThreads) {
      int i = idx >> 4, p = idx & 15;
      float f[8];
      if (i < ntok) {
        uint4 v = *reinterpret_cast<const uint4*>(Kr_bh + (size_t)tok[i] * kHeadDim + p * 8);
        unpack8(v, f);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = 0.f;
      }
      float4* dst = reinterpret_cast<float4*>(Ks + i * kHeadDim + p * 8);
      dst[0] = make_float4(f[0], f[1], f[2], f[3]);
      dst[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    __syncthreads();
    return;
  }
  uint16_t* As = reinterpret_cast<uint16_t*>(smem);                 // [128][r]
  uint16_t* Bs = As + kTileTok * r;                                 // [r][128]
  const int rv = r >> 3;                                            // 16 B pieces per A row
  for (int idx = tid; idx < kTileTok * rv; idx += kTileThreads) {
    int i = idx / rv, p = idx - i * rv;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < ntok) v = *reinterpret_cast<const uint4*>(A_b + (size_t)tok[i] * r + p * 8);
    *reinterpret_cast<uint4*>(As + i * r + p * 8) = v;
  }
  for (int idx = tid; idx < r * 16; idx += kTileThreads)
    reinterpret_cast<uint4*>(Bs)[idx] = reinterpret_cast<const uint4*>(B_bh)[idx];
  __syncthreads();

  const int tx = tid & 15, ty = tid >> 4;   // dims tx*8..+8 ; tokens ty + 16*i
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[i][e] = 0.f;
  for (int rho = 0; rho < r; ++rho) {
    float b[8];
    unpack8(*reinterpret_cast<const uint4*>(Bs + rho * kHeadDim + tx * 8), b);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float a = bf2f(As[(ty + 16 * i) * r + rho]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[i][e] = fmaf(a, b[e], acc[i][e]);
    }
  }
  __syncthreads();                     // As/Bs dead; Ks aliases them
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float4* dst = reinterpret_cast<float4*>(Ks + (ty + 16 * i) * kHeadDim + tx * 8);
    dst[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    dst[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
  }
  __syncthreads();
  // RoPE in place: one thread per (token, pair)
  const int half = rope.rot >> 1;
  for (int idx = tid; idx < kTileTok * half; idx += kTileThreads) {
    int i = idx / half, p = idx - i * half;
    if (i >= ntok) continue;
    float sn, cs;
    rope_sincos(tok[i], rope.inv_freq[p], &sn, &cs);
    int d0 = rope.interleaved ? 2 * p : p;
    int d1 = rope.interleaved ? 2 * p + 1 : p + half;
    float x0 = Ks[i * kHeadDim + d0], x1 = Ks[i * kHeadDim + d1];
    Ks[i * kHeadDim + d0] = x0 * cs - x1 * sn;
    Ks[i * kHeadDim + d1] = x1 * cs + x0 * sn;
  }
  __syncthreads();
}

}  // namespace skv
