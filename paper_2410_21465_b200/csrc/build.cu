// Algorithm 1 "ShadowKV Pre-filling" on sm_100a -- setup path (a0, untimed).
//
//   k_build_chunks          keys of 16 chunks per block -> landmark C_j and the
//                           chunk's min cosine similarity m_j (R10, R11)
//   k_build_select_outliers ArgTopK(-m, o) per (b, h): exact radix select, ties -> lower j (R12)
//   k_build_outliers_window post-RoPE keys (bf16) + values (zero-copy from host) of the outlier
//                           chunks and of the window tail (R8)
#include "kernels.h"
#include "keytile.cuh"
#include "topk.cuh"

namespace skv {

static __device__ __forceinline__ int* tile_tok_ptr(uint8_t* smem, int r) {
  size_t ab = (size_t)kTileTok * r * 2 + (size_t)r * kHeadDim * 2;
  size_t kt = (size_t)kTileTok * kHeadDim * 4;
  return reinterpret_cast<int*>(smem + (ab > kt ? ab : kt));
}

__global__ void __launch_bounds__(kTileThreads)
k_build_chunks(Dims D, Rope R, Layer Ly, const uint16_t* __restrict__ K_rope, float* __restrict__ mincos,
               float* __restrict__ negm) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tile = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t bh = (size_t)b * D.hk + h;
  float* Ks = reinterpret_cast<float*>(smem);
  int* tok = tile_tok_ptr(smem, D.r);
  const int j0 = tile * 16;
  const int ncb = req_nc(D, b);                         // this request's grid (ragged batch)
  const int ntok = max(0, min(kTileTok, (ncb - j0) * kChunk));
  if (tid < kTileTok) tok[tid] = j0 * kChunk + tid;
  __syncthreads();
  produce_key_tile(Ly.A + (size_t)b * D.s * D.r, Ly.B + bh * D.r * kHeadDim,
                   K_rope ? K_rope + bh * D.s * kHeadDim : nullptr, D.r, tok, ntok,
                   RopeArgs{R.inv_freq, R.rot, R.interleaved}, smem, Ks);
  // warp w: chunks 2w, 2w+1 of the tile; lane: dims 4*lane..+4
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int jl = warp * 2 + cc, j = j0 + jl;
    if (j >= D.n_c) break;
    if (j >= ncb) {                                     // padding past a shorter request's grid: never
      const size_t row = bh * D.n_c + j;                // an outlier (-m = -inf), landmark row zero
      if (lane == 0) { mincos[row] = INFINITY; negm[row] = -INFINITY; }
      *reinterpret_cast<uint2*>(Ly.L + row * kHeadDim + lane * 4) = make_uint2(0u, 0u);
      continue;
    }
    float4 kv[kChunk];
    float4 C = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      kv[u] = *reinterpret_cast<const float4*>(Ks + (jl * kChunk + u) * kHeadDim + lane * 4);
      C.x += kv[u].x; C.y += kv[u].y; C.z += kv[u].z; C.w += kv[u].w;
    }
    C.x *= 0.125f; C.y *= 0.125f; C.z *= 0.125f; C.w *= 0.125f;       // (1/c) sum, c = 8
    const float cn = sqrtf(warp_sum(C.x * C.x + C.y * C.y + C.z * C.z + C.w * C.w));
    float m = INFINITY;
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      float dot = warp_sum(C.x * kv[u].x + C.y * kv[u].y + C.z * kv[u].z + C.w * kv[u].w);
      float kn = sqrtf(warp_sum(kv[u].x * kv[u].x + kv[u].y * kv[u].y + kv[u].z * kv[u].z + kv[u].w * kv[u].w));
      float den = cn * kn;
      float cosv = den > 0.f ? dot / den : -1.f;                        // zero norm -> -1
      m = fminf(m, cosv);
    }
    const size_t row = bh * D.n_c + j;
    if (lane == 0) { mincos[row] = m; negm[row] = -m; }
    uint2 pk = make_uint2(pack_bf2(C.x, C.y), pack_bf2(C.z, C.w));
    *reinterpret_cast<uint2*>(Ly.L + row * kHeadDim + lane * 4) = pk;
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
  if ((e = cudaFuncSetAttribute(k_build_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  return cudaFuncSetAttribute(k_build_outliers_window, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}

// Last kernel of every build: writes nothing.  decode's scorer is launched with PDL and reads the
// layer state (landmarks, outlier ids) before its griddepcontrol.wait; PDL only orders the
// preceding grid's writes after that wait, so the grid right before a decode must not write them.
__global__ void k_build_done() {}

cudaError_t launch_build(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* K_rope,
                         const BuildWs& ws, cudaStream_t st, int* launches) {
  const size_t sm = keytile_smem_bytes(D.r);
  dim3 g1((D.n_c + 15) / 16, D.hk, D.b);
  k_build_chunks<<<g1, kTileThreads, sm, st>>>(D, R, Ly, K_rope, ws.mincos, ws.negm);
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
