// Algorithm 2 "ShadowKV Decoding" + sparse attention, sm_100a (v1 kernels).
//
//   k_score<G>          a7 window append; a1 landmark logits l = <q, L_j>/sqrt(d) streamed from
//                       HBM (16 B/lane, half-warp per landmark row, butterfly reduce), per-block
//                       softmax partials (max, sum exp) over landmarks only (R3)
//   k_select<G>         a2 lse + z_j = max_group(l - lse); a3 exact top-k
//   k_rebuild_gather    a4 K~ = RoPE(A[sel] . B_h) on rebuild blocks, while gather
//                       blocks pull the selected 2 KB value chunks zero-copy over PCIe;
//                       the two roles share one launch so the key rebuild hides under the fetch
//                       (the paper's multi-stream overlap, P:40 / P:460, done inside one grid)
//   k_attn<G>           a6 split-KV attention over [outliers; K~/V~; window]
//   k_combine           merge of the split partials (log-sum-exp), bf16 output
#include "kernels.h"
#include "keytile.cuh"
#include "topk.cuh"

namespace skv {

// ---------------------------------------------------------------------------------------------
// half-warp transpose-reduce: 16 lanes each hold 16 partial sums v[0..16); afterwards lane `sub`
// holds the full 16-lane sum of element `sub`.
// ---------------------------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void bstage(float* v, int sub) {
  constexpr int H = N / 2;
  const bool up = sub & H;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    float send = up ? v[i] : v[i + H];
    float keep = up ? v[i + H] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, H);
  }
}
__device__ __forceinline__ float butterfly16(float* v, int sub) {
  bstage<16>(v, sub); bstage<8>(v, sub); bstage<4>(v, sub); bstage<2>(v, sub);
  return v[0];
}

// rows [row0, row0+R) of a 128-dim bf16 matrix (one row per 16 lanes, 8 dims per lane) dotted
// with G query heads held in registers; returns the dot of row (sub / G) with head (sub % G).
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
  return butterfly16(acc, sub);
}

template <int G>
__device__ __forceinline__ void load_q_regs(const uint16_t* qrow0, int sub, float (&qr)[G][8]) {
#pragma unroll
  for (int hq = 0; hq < G; ++hq) unpack8(*reinterpret_cast<const uint4*>(qrow0 + hq * kHeadDim + sub * 8), qr[hq]);
}

// ---------------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(256)
k_score(Dims D, const uint16_t* __restrict__ L, const int32_t* __restrict__ oids, const uint16_t* __restrict__ q,
        float* __restrict__ logits, float2* __restrict__ part, int n_sblk, float scale,
        const uint16_t* __restrict__ k_new, const uint16_t* __restrict__ v_new, uint16_t* K_win,
        uint16_t* V_win, int step) {
  constexpr int R = 16 / G;
  __shared__ uint32_t omask[kScoreTile / 32];
  __shared__ float2 wpart[8][G];
  const int blk = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, sub = lane & 15;
  const size_t bh = (size_t)b * D.hk + h;
  const int j0 = blk * kScoreTile;
  if (tid < kScoreTile / 32) omask[tid] = 0u;
  if (blk == 0 && tid < 2 * kHeadDim / 8) {           // a7: append the current token (R18)
    const int arr = tid >> 4, p = tid & 15;
    const size_t dst = (bh * D.wcap + D.w_eff + step) * kHeadDim + p * 8;
    const uint16_t* src = (arr ? v_new : k_new) + bh * kHeadDim + p * 8;
    *reinterpret_cast<uint4*>((arr ? V_win : K_win) + dst) = *reinterpret_cast<const uint4*>(src);
  }
  __syncthreads();
  for (int i = tid; i < D.o; i += 256) {
    int j = oids[bh * D.o + i] - j0;
    if (j >= 0 && j < kScoreTile) atomicOr(&omask[j >> 5], 1u << (j & 31));
  }
  float qr[G][8];
  load_q_regs<G>(q + ((size_t)b * D.hq + (size_t)h * G) * kHeadDim, sub, qr);
  __syncthreads();
  const uint16_t* Lbh = L + bh * D.n_c * kHeadDim;
  float* lg_base = logits + ((size_t)b * D.hq + (size_t)h * G) * D.n_c;
  float m_run = -INFINITY, s_run = 0.f;
  const int my_i = sub / G, my_hq = sub % G;
#pragma unroll 1
  for (int rb = 0; rb < kScoreTile / 8; rb += 2 * R) {
    const int rbase = j0 + warp * (kScoreTile / 8) + rb + half * R;
    uint4 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      int row = rbase + i;
      v[i] = row < D.n_c ? ld_stream(Lbh + (size_t)row * kHeadDim + sub * 8) : make_uint4(0, 0, 0, 0);
    }
    const float dot = rows_dot_q<G>(v, qr, sub);
    const int row = rbase + my_i;
    if (row < D.n_c) {
      const int jl = row - j0;
      const bool is_out = (omask[jl >> 5] >> (jl & 31)) & 1u;
      const float l = is_out ? -INFINITY : dot * scale;
      lg_base[(size_t)my_hq * D.n_c + row] = l;
      if (!is_out) lse_merge(m_run, s_run, l, 1.f);
    }
  }
#pragma unroll
  for (int msk = G; msk < 32; msk <<= 1) {
    float m2 = __shfl_xor_sync(0xffffffffu, m_run, msk), s2 = __shfl_xor_sync(0xffffffffu, s_run, msk);
    lse_merge(m_run, s_run, m2, s2);
  }
  if (lane < G) wpart[warp][lane] = make_float2(m_run, s_run);
  __syncthreads();
  if (tid < G) {
    float m = -INFINITY, s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) lse_merge(m, s, wpart[w][tid].x, wpart[w][tid].y);
    part[((size_t)b * D.hq + (size_t)h * G + tid) * n_sblk + blk] = make_float2(m, s);
  }
}

// ---------------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(1024)
k_select(Dims D, const float* __restrict__ logits, const float2* __restrict__ part, int n_sblk,
         float* __restrict__ z, int32_t* __restrict__ sel, int32_t* __restrict__ sel_user) {
  __shared__ TopKSmem<1024> sm;
  __shared__ float lse[G];
  const int h = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t bh = (size_t)b * D.hk + h;
  if (warp < G) {
    const float2* p = part + ((size_t)b * D.hq + (size_t)h * G + warp) * n_sblk;
    float m = -INFINITY, s = 0.f;
    for (int i = lane; i < n_sblk; i += 32) lse_merge(m, s, p[i].x, p[i].y);
#pragma unroll
    for (int msk = 16; msk > 0; msk >>= 1) {
      float m2 = __shfl_xor_sync(0xffffffffu, m, msk), s2 = __shfl_xor_sync(0xffffffffu, s, msk);
      lse_merge(m, s, m2, s2);
    }
    if (lane == 0) lse[warp] = m + logf(s);
  }
  __syncthreads();
  float* zb = z + bh * D.n_c;
  const float* lb = logits + ((size_t)b * D.hq + (size_t)h * G) * D.n_c;
  for (int j = tid; j < D.n_c; j += 1024) {
    float zz = -INFINITY;
#pragma unroll
    for (int hq = 0; hq < G; ++hq) zz = fmaxf(zz, lb[(size_t)hq * D.n_c + j] - lse[hq]);
    zb[j] = zz;
  }
  __syncthreads();
  int32_t* out = sel + bh * D.k;
  block_topk_largest<1024>(zb, D.n_c, D.k, out, sm);
  if (sel_user) {
    __syncthreads();
    for (int i = tid; i < D.k; i += 1024) sel_user[bh * D.k + i] = out[i];
  }
}

// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTileThreads)
k_rebuild_gather(Dims D, Rope R, Layer Ly, const int32_t* __restrict__ sel, uint16_t* __restrict__ Kt,
                 uint16_t* __restrict__ Vt, uint16_t* __restrict__ dbg, int n_gather_blocks) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if ((int)blockIdx.x < n_gather_blocks) {
    // ---- value gather (a5): 2 KB chunk = 8 tokens x 128 dims, 4 x 16 B per lane, 2 chunks in flight
    const int total = D.b * D.hk * D.k;
    const int gw = blockIdx.x * (kTileThreads / 32) + warp, nw = n_gather_blocks * (kTileThreads / 32);
    for (int c0 = gw * 2; c0 < total; c0 += nw * 2) {
      uint4 v[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ci = c0 + u;
        if (ci < total) {
          const int bhi = ci / D.k;
          const uint16_t* src = Ly.V_host + ((size_t)bhi * D.s + (size_t)sel[ci] * kChunk) * kHeadDim;
#pragma unroll
          for (int x = 0; x < 4; ++x) v[u][x] = ld_stream(reinterpret_cast<const uint4*>(src) + lane + 32 * x);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ci = c0 + u;
        if (ci < total) {
          uint4* dst = reinterpret_cast<uint4*>(Vt + (size_t)ci * kChunk * kHeadDim);
#pragma unroll
          for (int x = 0; x < 4; ++x) dst[lane + 32 * x] = v[u][x];
        }
      }
    }
    return;
  }
  // ---- key rebuild (a4): 16 selected chunks = 128 tokens per block
  const int rb = blockIdx.x - n_gather_blocks;
  const int tiles = (D.k + 15) / 16;
  const int tile = rb % tiles;
  const size_t bh = rb / tiles;
  const int b = (int)(bh / D.hk);
  float* Ks = reinterpret_cast<float*>(smem);
  size_t ab = (size_t)kTileTok * D.r * 2 + (size_t)D.r * kHeadDim * 2, kt = (size_t)kTileTok * kHeadDim * 4;
  int* tok = reinterpret_cast<int*>(smem + (ab > kt ? ab : kt));
  const int ntok = min(kTileTok, (D.k - tile * 16) * kChunk);
  if (tid < kTileTok) {
    int ci = tile * 16 + (tid >> 3);
    tok[tid] = ci < D.k ? sel[bh * D.k + ci] * kChunk + (tid & 7) : 0;
  }
  __syncthreads();
  produce_key_tile(Ly.A + (size_t)b * D.s * D.r, Ly.B + bh * D.r * kHeadDim, nullptr, D.r, tok, ntok,
                   RopeArgs{R.inv_freq, R.rot, R.interleaved}, smem, Ks);
  for (int idx = tid; idx < ntok * 16; idx += kTileThreads) {
    const int il = idx >> 4, p = idx & 15;
    const float* k = Ks + il * kHeadDim + p * 8;
    uint4 kb = make_uint4(pack_bf2(k[0], k[1]), pack_bf2(k[2], k[3]), pack_bf2(k[4], k[5]), pack_bf2(k[6], k[7]));
    const size_t dst = (bh * D.k * kChunk + (size_t)tile * kTileTok + il) * kHeadDim + p * 8;
    *reinterpret_cast<uint4*>(Kt + dst) = kb;
    if (dbg) *reinterpret_cast<uint4*>(dbg + dst) = kb;
  }
}

// ---------------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(128)
k_attn(Dims D, Layer Ly, const uint16_t* __restrict__ q, const uint16_t* __restrict__ Kt,
       const uint16_t* __restrict__ Vt, int step, float* __restrict__ o_part, float2* __restrict__ ml_part,
       int n_split, float scale) {
  constexpr int R = 16 / G;
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* Ksm = reinterpret_cast<uint16_t*>(smem);                    // [128][128]
  uint16_t* Vsm = Ksm + kAttnTile * kHeadDim;                           // [128][128]
  float* P = reinterpret_cast<float*>(Vsm + kAttnTile * kHeadDim);       // [G][128]
  __shared__ float2 ml[G];
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, sub = lane & 15;
  const size_t bh = (size_t)b * D.hk + h;
  const int T_out = D.o * kChunk, T_sel = D.k * kChunk, T_win = D.w_eff + step + 1;
  const int T = T_out + T_sel + T_win;
  const int t0 = split * kAttnTile, nt = min(kAttnTile, T - t0);
  for (int idx = tid; idx < kAttnTile * 16; idx += 128) {
    const int i = idx >> 4, p = idx & 15, t = t0 + i;
    uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
    if (i < nt) {
      size_t off;
      const uint16_t *Ks, *Vs;
      if (t < T_out) { off = (bh * T_out + t) * kHeadDim; Ks = Ly.K_out; Vs = Ly.V_out; }
      else if (t < T_out + T_sel) { off = (bh * T_sel + (t - T_out)) * kHeadDim; Ks = Kt; Vs = Vt; }
      else { off = (bh * D.wcap + (t - T_out - T_sel)) * kHeadDim; Ks = Ly.K_win; Vs = Ly.V_win; }
      kv = *reinterpret_cast<const uint4*>(Ks + off + p * 8);
      vv = *reinterpret_cast<const uint4*>(Vs + off + p * 8);
    }
    reinterpret_cast<uint4*>(Ksm)[idx] = kv;
    reinterpret_cast<uint4*>(Vsm)[idx] = vv;
  }
  float qr[G][8];
  load_q_regs<G>(q + ((size_t)b * D.hq + (size_t)h * G) * kHeadDim, sub, qr);
  __syncthreads();
  // logits: 8 half-warps x 16 rows each
  const int hw = warp * 2 + half;
#pragma unroll 1
  for (int rb = 0; rb < 16; rb += R) {
    const int r0 = hw * 16 + rb;
    uint4 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = reinterpret_cast<const uint4*>(Ksm + (r0 + i) * kHeadDim)[sub];
    const float dot = rows_dot_q<G>(v, qr, sub);
    const int row = r0 + sub / G;
    P[(sub % G) * kAttnTile + row] = row < nt ? dot * scale : -INFINITY;
  }
  __syncthreads();
  // per-head max / exp / sum (warp w handles heads w, w+4, ...)
  for (int hq = warp; hq < G; hq += 4) {
    float x[4], m = -INFINITY;
#pragma unroll
    for (int u = 0; u < 4; ++u) { x[u] = P[hq * kAttnTile + lane + 32 * u]; m = fmaxf(m, x[u]); }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) { float e = expf(x[u] - m); P[hq * kAttnTile + lane + 32 * u] = e; s += e; }
    s = warp_sum(s);
    if (lane == 0) ml[hq] = make_float2(m, s);
  }
  __syncthreads();
  // PV: thread = output dim
  float acc[G];
#pragma unroll
  for (int hq = 0; hq < G; ++hq) acc[hq] = 0.f;
  for (int t = 0; t < nt; ++t) {
    const float v = bf2f(Vsm[t * kHeadDim + tid]);
#pragma unroll
    for (int hq = 0; hq < G; ++hq) acc[hq] = fmaf(P[hq * kAttnTile + t], v, acc[hq]);
  }
#pragma unroll
  for (int hq = 0; hq < G; ++hq) {
    const size_t row = ((size_t)b * D.hq + (size_t)h * G + hq) * n_split + split;
    o_part[row * kHeadDim + tid] = acc[hq];
    if (tid == 0) ml_part[row] = ml[hq];
  }
}

__global__ void __launch_bounds__(128)
k_combine(Dims D, const float* __restrict__ o_part, const float2* __restrict__ ml_part, int n_split,
          uint16_t* __restrict__ out) {
  const size_t row = (size_t)blockIdx.y * D.hq + blockIdx.x;
  const float2* ml = ml_part + row * n_split;
  float M = -INFINITY;
  for (int i = 0; i < n_split; ++i) M = fmaxf(M, ml[i].x);
  float Ls = 0.f, acc = 0.f;
  for (int i = 0; i < n_split; ++i) {
    const float w = expf(ml[i].x - M);
    Ls = fmaf(ml[i].y, w, Ls);
    acc = fmaf(o_part[(row * n_split + i) * kHeadDim + threadIdx.x], w, acc);
  }
  out[row * kHeadDim + threadIdx.x] = f2bf(acc / Ls);
}

// ---------------------------------------------------------------------------------------------
size_t decode_ws_bytes(const Dims& D, DecodeWs* ws, char* base) {
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return base + o; };
  const int n_sblk = (D.n_c + kScoreTile - 1) / kScoreTile;
  const int T_max = D.o * kChunk + D.k * kChunk + D.wcap;
  const int n_split = (T_max + kAttnTile - 1) / kAttnTile;
  const size_t BHq = (size_t)D.b * D.hq, BHk = (size_t)D.b * D.hk;
  char* p_log = carve(BHq * D.n_c * 4);
  char* p_part = carve(BHq * n_sblk * 8);
  char* p_z = carve(BHk * D.n_c * 4);
  char* p_sel = carve(BHk * D.k * 4);
  char* p_kt = carve(BHk * D.k * kChunk * kHeadDim * 2);
  char* p_vt = carve(BHk * D.k * kChunk * kHeadDim * 2);
  char* p_op = carve(BHq * n_split * kHeadDim * 4);
  char* p_ml = carve(BHq * n_split * 8);
  if (ws) {
    ws->logits = reinterpret_cast<float*>(p_log);
    ws->part = reinterpret_cast<float2*>(p_part);
    ws->z = reinterpret_cast<float*>(p_z);
    ws->sel = reinterpret_cast<int32_t*>(p_sel);
    ws->Kt = reinterpret_cast<uint16_t*>(p_kt);
    ws->Vt = reinterpret_cast<uint16_t*>(p_vt);
    ws->o_part = reinterpret_cast<float*>(p_op);
    ws->ml_part = reinterpret_cast<float2*>(p_ml);
    ws->n_sblk = n_sblk;
    ws->n_split = n_split;
  }
  return off;
}

template <int G>
static cudaError_t launch_decode_g(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                                   const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                                   int32_t* sel_ids, uint16_t* dbg_keys, const DecodeWs& ws,
                                   cudaStream_t st, int* launches) {
  const float scale = (float)(1.0 / 11.313708498984761);    // 1/sqrt(d), d = 128 (R6)
  k_score<G><<<dim3(ws.n_sblk, D.hk, D.b), 256, 0, st>>>(D, Ly.L, Ly.outlier_ids, q, ws.logits, ws.part,
                                                         ws.n_sblk, scale, k_new, v_new, Ly.K_win, Ly.V_win, step);
  k_select<G><<<dim3(D.hk, D.b), 1024, 0, st>>>(D, ws.logits, ws.part, ws.n_sblk, ws.z, ws.sel, sel_ids);
  const size_t sm = keytile_smem_bytes(D.r);
  cudaError_t e = cudaFuncSetAttribute(k_rebuild_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int n_rebuild = D.b * D.hk * ((D.k + 15) / 16);
  k_rebuild_gather<<<n_sm + n_rebuild, kTileThreads, sm, st>>>(D, R, Ly, ws.sel, ws.Kt, ws.Vt, dbg_keys, n_sm);
  const int T = D.o * kChunk + D.k * kChunk + D.w_eff + step + 1;
  const int n_split_used = (T + kAttnTile - 1) / kAttnTile;
  const size_t asm_bytes = 2 * kAttnTile * kHeadDim * 2 + G * kAttnTile * 4;
  e = cudaFuncSetAttribute(k_attn<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asm_bytes);
  if (e != cudaSuccess) return e;
  k_attn<G><<<dim3(n_split_used, D.hk, D.b), 128, asm_bytes, st>>>(D, Ly, q, ws.Kt, ws.Vt, step, ws.o_part,
                                                                   ws.ml_part, n_split_used, scale);
  k_combine<<<dim3(D.hq, D.b), 128, 0, st>>>(D, ws.o_part, ws.ml_part, n_split_used, out);
  *launches += 5;
  return cudaGetLastError();
}

cudaError_t launch_decode(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                          const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                          int32_t* sel_ids, uint16_t* dbg_keys, const DecodeWs& ws, cudaStream_t st,
                          int* launches) {
  switch (D.g) {
    case 1: return launch_decode_g<1>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches);
    case 2: return launch_decode_g<2>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches);
    case 4: return launch_decode_g<4>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches);
    case 8: return launch_decode_g<8>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches);
    case 16: return launch_decode_g<16>(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, ws, st, launches);
  }
  return cudaErrorInvalidValue;
}

}  // namespace skv
