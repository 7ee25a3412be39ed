// Algorithm 1 "ShadowKV Pre-filling" on sm_100a -- setup path (a0, untimed).
//
//   k_build_chunks          keys of 16 chunks per block -> landmark C_j and the
//                           chunk's min cosine similarity m_j (R10, R11)
//   k_build_select_outliers ArgTopK(-m, o) per (b, h): exact radix select, ties -> lower j (R12)
//   k_build_outliers_window post-RoPE keys (bf16) + values (zero-copy from host) of the outlier
//                           chunks and of the window tail (R8)
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.h"
#include "keytile.cuh"
#include "rope.cuh"
#include "topk.cuh"
#include "umma.cuh"

namespace skv {

static __device__ __forceinline__ int* tile_tok_ptr(uint8_t* smem, int r) {
  size_t ab = (size_t)kTileTok * r * 2 + (size_t)r * kHeadDim * 2;
  size_t kt = (size_t)kTileTok * kHeadDim * 4;
  return reinterpret_cast<int*>(smem + (ab > kt ? ab : kt));
}

// Key tile of the build on the 5th-generation tensor cores: K~[128 tokens][128] = A[t0.., :r] . B_h
// (the keys the factors represent, Alg 1 / Alg 2 "MatMul(A, B)") with one tcgen05.mma
// chain (M = 128 tokens, N = 128, K = r) into TMEM; RoPE in registers after tcgen05.ld (rope_row);
// the fp32 post-RoPE keys go to smem [128][kKsStride] for the chunk statistics.
// smem (1024-aligned): A tile [128 rows] K-major SWIZZLE_128B (TMA boxes of 128 rows x 64 columns, K
// block kb at kb * 16 KB) | B_h MN-major SWIZZLE_128B (two boxes of r rows x 64 columns); the fp32 key
// tile aliases both once the MMAs have completed.
constexpr int kKsStride = kHeadDim + 4;               // floats: 528-byte rows, conflict-free 16 B stores
constexpr int kChunksPerTile = kTileTok / kChunk;    // 16
__host__ __device__ constexpr size_t build_tc_smem_bytes(int r) {
  const size_t ab = (size_t)((r + 63) / 64) * 16384 + (size_t)2 * r * 128;
  const size_t ks = (size_t)kTileTok * kKsStride * 4;
  return (ab > ks ? ab : ks) + kTileTok * sizeof(int) + (size_t)kChunksPerTile * (kKsStride + 1) * 4 + 1024;
}
constexpr uint32_t kIdescBuild = umma_idesc_bf16(128, 128, false, true);

__device__ __forceinline__ void build_key_tile_tc(const CUtensorMap* tmA, const CUtensorMap* tmB, int row0, int brow0,
                                                  int r, const Rope& R, const int* tok, uint8_t* smem, float* Ks,
                                                  uint64_t* bar_ab, uint64_t* bar_mma, uint32_t* tmem_slot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nkb = (r + 63) >> 6;
  uint8_t* As = smem;
  uint8_t* Bs = smem + nkb * 16384;
  if (tid == 0) {
    mbar_init(bar_ab, 1); mbar_init(bar_mma, 1); fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) {
    mbar_expect_tx(bar_ab, nkb * 16384 + 2 * r * 128);
    for (int kb = 0; kb < nkb; ++kb) tma_load_2d(As + kb * 16384, tmA, kb * 64, row0, bar_ab);
    tma_load_2d(Bs, tmB, 0, brow0, bar_ab);
    tma_load_2d(Bs + r * 128, tmB, 64, brow0, bar_ab);
    mbar_wait(bar_ab, 0);
    tc_fence_after();
    const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs), lbo = (uint32_t)r * 128u;
    for (int ks = 0; ks < (r >> 4); ++ks)
      umma_f16(tmem, umma_desc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32), umma_desc_sw128_mn(b0 + ks * 2048, lbo),
               kIdescBuild, ks > 0);
    umma_commit(bar_mma);
  }
  __syncwarp();
  mbar_wait(bar_mma, 0);                                // (all threads: Ks below aliases the operands)
  tc_fence_after();
  const int row = 32 * (warp & 3) + lane, set = warp >> 2;
  int c0, c1;
  rope_col_sets(R, set, &c0, &c1);
  float x0[32], x1[32];
  const uint32_t tr = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  tmem_ld32(tr + c0, x0);
  tmem_ld32(tr + c1, x1);
  rope_row(x0, x1, c0, c1, tok[row], R);
  __syncthreads();                                      // every warp has read TMEM; operands are dead
  float* kr = Ks + row * kKsStride;
#pragma unroll
  for (int e = 0; e < 32; e += 4) {
    *reinterpret_cast<float4*>(kr + c0 + e) = make_float4(x0[e], x0[e + 1], x0[e + 2], x0[e + 3]);
    *reinterpret_cast<float4*>(kr + c1 + e) = make_float4(x1[e], x1[e + 1], x1[e + 2], x1[e + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

__global__ void __launch_bounds__(kTileThreads)
k_build_chunks(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Dims D, Rope R,
               Layer Ly, const uint16_t* __restrict__ K_rope, float* __restrict__ mincos, float* __restrict__ negm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  __shared__ __align__(8) uint64_t bar_ab, bar_mma;
  __shared__ uint32_t tmem_slot;
  const int tile = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t bh = (size_t)b * D.hk + h;
  float* Ks = reinterpret_cast<float*>(smem);
  const size_t ab = (size_t)((D.r + 63) / 64) * 16384 + (size_t)2 * D.r * 128;
  const size_t ksb = (size_t)kTileTok * kKsStride * 4;
  int* tok = reinterpret_cast<int*>(smem + (ab > ksb ? ab : ksb));
  const int j0 = tile * 16;
  const int ncb = req_nc(D, b);                         // this request's grid (ragged batch)
  const int ntok = max(0, min(kTileTok, (ncb - j0) * kChunk));
  if (tid < kTileTok) tok[tid] = j0 * kChunk + tid;
  if (K_rope) {                                         // given post-RoPE keys: widened copy (CUDA cores)
    __syncthreads();
    for (int idx = tid; idx < kTileTok * 16; idx += kTileThreads) {
      const int i = idx >> 4, p = idx & 15;
      float f[8];
      if (i < ntok) unpack8(*reinterpret_cast<const uint4*>(K_rope + (bh * D.s + tok[i]) * kHeadDim + p * 8), f);
      else {
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = 0.f;
      }
      float4* dst = reinterpret_cast<float4*>(Ks + i * kKsStride + p * 8);
      dst[0] = make_float4(f[0], f[1], f[2], f[3]);
      dst[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    __syncthreads();
  } else {
    build_key_tile_tc(&tmA, &tmB, b * D.s + j0 * kChunk, (int)bh * D.r, D.r, R, tok, smem, Ks, &bar_ab, &bar_mma,
                      &tmem_slot);
  }
  // chunk statistics from the fp32 key tile.  (A) thread (chunk c, dims 8q..8q+8):
  // C_j = (1/c) sum of the chunk's keys -> landmark row (bf16) and |C_j|^2 (16-lane reduction);
  // (B) thread (token t, half of the dims): <C_j, k_t> and |k_t|^2 (pair reduction), cos (zero norm
  // -> -1), m_j = min over the chunk's 8 tokens (16-lane reduction).  No per-row warp sums.
  float* Cs = reinterpret_cast<float*>(tok + kTileTok);          // [16][kKsStride] chunk means
  float* Cn = Cs + kChunksPerTile * kKsStride;                   // [16] |C_j|
  {
    const int c = tid >> 4, q = tid & 15, j = j0 + c;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      const float4* kr = reinterpret_cast<const float4*>(Ks + (c * kChunk + u) * kKsStride + q * 8);
      const float4 x = kr[0], y = kr[1];
      acc[0] += x.x; acc[1] += x.y; acc[2] += x.z; acc[3] += x.w;
      acc[4] += y.x; acc[5] += y.y; acc[6] += y.z; acc[7] += y.w;
    }
    float c2 = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) { acc[e] *= 0.125f; c2 = fmaf(acc[e], acc[e], c2); }   // (1/c) sum, c = 8
    float4* cr = reinterpret_cast<float4*>(Cs + c * kKsStride + q * 8);
    cr[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    cr[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    if (q == 0) Cn[c] = sqrtf(c2);
    if (j < D.n_c) {
      const size_t row = bh * D.n_c + j;
      uint4 pk = make_uint4(0u, 0u, 0u, 0u);               // padding past a shorter request's grid: zero row
      if (j < ncb) pk = make_uint4(pack_bf2(acc[0], acc[1]), pack_bf2(acc[2], acc[3]), pack_bf2(acc[4], acc[5]),
                                   pack_bf2(acc[6], acc[7]));
      *reinterpret_cast<uint4*>(Ly.L + row * kHeadDim + q * 8) = pk;
    }
  }
  __syncthreads();
  {
    const int t = tid >> 1, hf = tid & 1, c = t >> 3, j = j0 + c;
    const float4* kr = reinterpret_cast<const float4*>(Ks + t * kKsStride + hf * 64);
    const float4* cr = reinterpret_cast<const float4*>(Cs + c * kKsStride + hf * 64);
    float dot = 0.f, k2 = 0.f;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float4 x = kr[e], y = cr[e];
      dot = fmaf(x.x, y.x, dot); dot = fmaf(x.y, y.y, dot); dot = fmaf(x.z, y.z, dot); dot = fmaf(x.w, y.w, dot);
      k2 = fmaf(x.x, x.x, k2); k2 = fmaf(x.y, x.y, k2); k2 = fmaf(x.z, x.z, k2); k2 = fmaf(x.w, x.w, k2);
    }
    dot += __shfl_xor_sync(0xffffffffu, dot, 1);
    k2 += __shfl_xor_sync(0xffffffffu, k2, 1);
    const float den = Cn[c] * sqrtf(k2);
    float m = den > 0.f ? dot / den : -1.f;                  // zero norm -> -1
#pragma unroll
    for (int o = 2; o < 16; o <<= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((tid & 15) == 0 && j < D.n_c) {
      const size_t row = bh * D.n_c + j;
      if (j < ncb) { mincos[row] = m; negm[row] = -m; }
      else { mincos[row] = INFINITY; negm[row] = -INFINITY; } // padding: never an outlier
    }
  }
}

__global__ void __launch_bounds__(1024)
k_build_select_outliers(Dims D, const float* __restrict__ negm, int32_t* __restrict__ oids) {
  __shared__ TopKSmem<1024> sm;
  const size_t bh = (size_t)blockIdx.y * D.hk + blockIdx.x;
  block_topk_largest<1024>(negm + bh * D.n_c, D.n_c, D.o, oids + bh * D.o, sm);
}

__global__ void __launch_bounds__(kTileThreads)
k_build_outliers_window(Dims D, Rope R, Layer Ly, const uint16_t* __restrict__ K_rope) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tile = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x;
  const size_t bh = (size_t)b * D.hk + h;
  float* Ks = reinterpret_cast<float*>(smem);
  int* tok = tile_tok_ptr(smem, D.r);
  const int n_out = D.o * kChunk, total = n_out + req_weff(D, b);   // this request's window tail
  const int i0 = tile * kTileTok;
  const int ntok = min(kTileTok, total - i0);
  if (ntok <= 0) return;                                // (block-uniform) a shorter request's tail
  if (tid < kTileTok) {
    int i = i0 + tid, t = 0;
    if (i < n_out) t = Ly.outlier_ids[bh * D.o + (i >> 3)] * kChunk + (i & 7);
    else if (i < total) t = req_nc(D, b) * kChunk + (i - n_out);
    tok[tid] = t;
  }
  __syncthreads();
  produce_key_tile(Ly.A + (size_t)b * D.s * D.r, Ly.B + bh * D.r * kHeadDim,
                   K_rope ? K_rope + bh * D.s * kHeadDim : nullptr, D.r, tok, ntok,
                   RopeArgs{R.inv_freq, R.rot, R.interleaved}, smem, Ks);
  for (int idx = tid; idx < ntok * 16; idx += kTileThreads) {
    const int il = idx >> 4, p = idx & 15, i = i0 + il;
    const float* k = Ks + il * kHeadDim + p * 8;
    uint4 kb = make_uint4(pack_bf2(k[0], k[1]), pack_bf2(k[2], k[3]), pack_bf2(k[4], k[5]), pack_bf2(k[6], k[7]));
    uint4 vb = ld_stream(Ly.V_host + (bh * D.s + tok[il]) * kHeadDim + p * 8);   // zero-copy
    size_t dst = (i < n_out) ? (bh * n_out + i) * kHeadDim : (bh * D.wcap + (i - n_out)) * kHeadDim;
    uint16_t* Kd = (i < n_out) ? Ly.K_out : Ly.K_win;
    uint16_t* Vd = (i < n_out) ? Ly.V_out : Ly.V_win;
    *reinterpret_cast<uint4*>(Kd + dst + p * 8) = kb;
    *reinterpret_cast<uint4*>(Vd + dst + p * 8) = vb;
  }
}

size_t build_ws_bytes(const Dims& D, BuildWs* ws, char* base) {
  // after every decode region (all sub-batch splits): decode's counters, flags and selection slots
  // must stay zero between calls, so the build scratch never overlaps them
  size_t off = (decode_ws_total_bytes(D) + 255) & ~(size_t)255;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return base + o; };
  size_t n = (size_t)D.b * D.hk * D.n_c;
  char* p1 = carve(n * 4);
  char* p2 = carve(n * 4);
  if (ws) { ws->mincos = reinterpret_cast<float*>(p1); ws->negm = reinterpret_cast<float*>(p2); }
  return off;
}

cudaError_t init_build_attrs() {
  const int sm = (int)keytile_smem_bytes(256);          // the largest rank the ABI accepts
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_build_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)build_tc_smem_bytes(256)))) return e;
  return cudaFuncSetAttribute(k_build_outliers_window, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}

// Last kernel of every build: writes nothing.  decode's scorer is launched with PDL and reads the
// layer state (landmarks, outlier ids) before its griddepcontrol.wait; PDL only orders the
// preceding grid's writes after that wait, so the grid right before a decode must not write them.
__global__ void k_build_done() {}

static bool encode_map(const DevCtx& ctx, CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                       uint32_t box_inner, uint32_t box_outer) {
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
  const cuuint64_t gdim[2] = {inner, outer};
  const cuuint64_t gstride[1] = {inner * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc && enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_build(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* K_rope,
                         const BuildWs& ws, cudaStream_t st, int* launches, const DevCtx& ctx) {
  const size_t sm = keytile_smem_bytes(D.r);
  CUtensorMap tmA, tmB;
  if (!encode_map(ctx, &tmA, Ly.A, D.r, (uint64_t)D.b * D.s, 64, kTileTok) ||
      !encode_map(ctx, &tmB, Ly.B, kHeadDim, (uint64_t)D.b * D.hk * D.r, 64, D.r))
    return cudaErrorInvalidValue;
  dim3 g1((D.n_c + 15) / 16, D.hk, D.b);
  k_build_chunks<<<g1, kTileThreads, build_tc_smem_bytes(D.r), st>>>(tmA, tmB, D, R, Ly, K_rope, ws.mincos, ws.negm);
  ++*launches;
  if (D.o > 0) {
    k_build_select_outliers<<<dim3(D.hk, D.b), 1024, 0, st>>>(D, ws.negm, Ly.outlier_ids);
    ++*launches;
  }
  const int total = D.o * kChunk + D.w_eff;
  if (total > 0) {
    dim3 g3((total + kTileTok - 1) / kTileTok, D.hk, D.b);
    k_build_outliers_window<<<g3, kTileThreads, sm, st>>>(D, R, Ly, K_rope);
    ++*launches;
  }
  k_build_done<<<1, 32, 0, st>>>();
  ++*launches;
  return cudaGetLastError();
}

}  // namespace skv
