// Alg 1 "A in R^{b x s x r}, B in R^{b x h_kv x r x d} <- SVD(K)" on the GPU.
//
// Per request, the pre-RoPE keys of all KV heads form X[t, h*d + j] = K[h][t][j] (R14), an
// s x D matrix with D = h_kv * d <= 4096 and s >> D.  Its truncated SVD is taken through the D x D
// Gram matrix, which is where s enters (2 s D^2 flops, tensor cores):
//   1. G = X^T X                      k_gram_tc: our tcgen05 kernel, one 128 x 128 block (h, h' >= h)
//                                     per CTA, split over token ranges; both operands are the keys
//                                     as stored ([t][j] rows = MN-major SWIZZLE_128B TMA boxes), fp32
//                                     accumulation in TMEM, partial blocks to a workspace
//   2. G -> fp64, symmetrised         k_gram_reduce: sums the token-range partials in a fixed order
//   3. G = V diag(lambda) V^T         cuSOLVER dsyevdx, only the top r eigenpairs (fp64; the D x D
//                                     eigenproblem is independent of s; SKV_FACT_EIG=full: dsyevd)
//   4. W = top-r eigenvectors (sigma_i = sqrt(lambda_i), descending), B_h = W[h*d:(h+1)*d, :]^T
//                                     k_take_top; W^T also as two bf16 planes hi + lo (hi = bf16(W),
//                                     lo = bf16(W - hi): ~16 significant bits for the projection)
//   5. A = X W  (= U_r Sigma_r)       k_project_tc: tcgen05, M = 128 tokens, N = r, K = D in 64-wide
//                                     blocks, X . W_hi + X . W_lo accumulated in TMEM, bf16 out
// The Gram route squares the condition number; it only matters below the truncation (sigma_i with
// i > r), where bf16 storage noise of K already sits.  Prefill, not the decode hot path: this runs
// once per context and is timed against prefill attention in tools/svd_overhead.py (Fig 1c).
#include <cusolverDn.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace skv {

// ---------------------------------------------------------------------------------------------
// 1. Gram blocks on the tensor cores
// ---------------------------------------------------------------------------------------------
constexpr int kGTok = 64;                        // tokens per pipeline stage (K of 4 MMAs)
constexpr int kGStages = 6;
constexpr uint32_t kGBox = kGTok * 128;          // one 64-token x 64-column box: 8 KB
constexpr uint32_t kGStage = 4 * kGBox;          // A and B, two column halves each
constexpr uint32_t kIdescGram = umma_idesc_bf16(128, 128, true, true);   // both operands MN-major
size_t gram_smem_bytes() { return 1024 + (size_t)kGStages * kGStage; }

// upper-triangle block pair p -> (h, h2), h <= h2
__device__ __forceinline__ void gram_pair(int p, int hk, int* h, int* h2) {
  int hh = 0;
  while (p >= hk - hh) { p -= hk - hh; ++hh; }
  *h = hh; *h2 = hh + p;
}

// Gp[split][D][D] (row-major fp32): block rows h*128.., cols h2*128.. = sum over the split's tokens of
// K_h[t]^T K_h2[t]  (D = A^T B with A[m = j][k = t] = K_h[t][j], B[n = j'][k = t] = K_h2[t][j'])
__global__ void __launch_bounds__(128, 1)
k_gram_tc(const __grid_constant__ CUtensorMap tmK, int head0, int hk, int s, int n_split, float* __restrict__ Gp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  __shared__ __align__(8) uint64_t full[kGStages], empty[kGStages], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int h, h2;
  gram_pair(blockIdx.x, hk, &h, &h2);
  const bool diag = h == h2;
  const int D = hk * 128, split = blockIdx.y;
  const int nst_all = (s + kGTok - 1) / kGTok;
  const int st0 = (int)((long long)nst_all * split / n_split), st1 = (int)((long long)nst_all * (split + 1) / n_split);
  const int nst = st1 - st0;
  if (tid == 0) {
    for (int i = 0; i < kGStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
    prefetch_tensormap(&tmK);
  }
  if (warp == 0) tmem_alloc<128>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {                                       // TMA producer
    for (int i = 0; i < nst; ++i) {
      const int stg = i % kGStages;
      if (i >= kGStages) mbar_wait(&empty[stg], ((i / kGStages) - 1) & 1);
      uint8_t* base = smem + stg * kGStage;
      const int t = (st0 + i) * kGTok;
      mbar_expect_tx(&full[stg], diag ? 2 * kGBox : 4 * kGBox);
      tma_load_3d(base, &tmK, 0, t, head0 + h, &full[stg]);
      tma_load_3d(base + kGBox, &tmK, 64, t, head0 + h, &full[stg]);
      if (!diag) {
        tma_load_3d(base + 2 * kGBox, &tmK, 0, t, head0 + h2, &full[stg]);
        tma_load_3d(base + 3 * kGBox, &tmK, 64, t, head0 + h2, &full[stg]);
      }
    }
  } else if (tid == 32) {                               // MMA issuer
    for (int i = 0; i < nst; ++i) {
      const int stg = i % kGStages;
      mbar_wait(&full[stg], (i / kGStages) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(smem + stg * kGStage), b0 = diag ? a0 : a0 + 2 * kGBox;
#pragma unroll
      for (int ks = 0; ks < kGTok / 16; ++ks)
        umma_f16(tmem, umma_desc_sw128_mn(a0 + ks * 2048, kGBox), umma_desc_sw128_mn(b0 + ks * 2048, kGBox),
                 kIdescGram, (i > 0 || ks > 0) ? 1u : 0u);
      umma_commit(&empty[stg]);
    }
    umma_commit(&done);                                 // (arrives immediately when nothing was issued)
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  const int j = 32 * warp + lane;                       // TMEM lane = row j of block (h, h2)
  float* row = Gp + ((size_t)split * D + (size_t)h * 128 + j) * D + (size_t)h2 * 128;
#pragma unroll 1
  for (int c = 0; c < 128; c += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
#pragma unroll
    for (int e = 0; e < 32; e += 4)
      *reinterpret_cast<float4*>(row + c + e) = nst > 0 ? make_float4(v[e], v[e + 1], v[e + 2], v[e + 3])
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

// 2. Gd (column-major fp64, cuSOLVER) = sum of the split partials in split order, symmetrised: the
//    upper-triangle blocks are read as computed, the lower ones transposed, diagonal blocks averaged
__global__ void k_gram_reduce(const float* __restrict__ Gp, int n_split, int D, double* __restrict__ Gd) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;   // column-major element (row i, col j)
  if (idx >= D * D) return;
  const int i = idx % D, j = idx / D;
  const int bi = i >> 7, bj = j >> 7;
  double a = 0.0, b = 0.0;
  for (int sp = 0; sp < n_split; ++sp) {
    const float* G = Gp + (size_t)sp * D * D;
    if (bi <= bj) a += (double)G[(size_t)i * D + j];
    if (bi >= bj) b += (double)G[(size_t)j * D + i];
  }
  Gd[idx] = bi < bj ? a : (bi > bj ? b : 0.5 * (a + b));
}

// W^T planes: WT[rho][i] = bf16(w), WT[r + rho][i] = bf16(w - bf16(w)), w = eigenvector D-1-rho
// (dsyevd: ascending eigenvalues, vectors in columns); sign fixed so the largest-|.| component is
// positive (deterministic factors; A.B is sign-free).  col0: the column of the largest eigenpair
// (D - 1 for the full solve, r - 1 for the top-r range solve).
__global__ void k_take_top(const double* __restrict__ V, const double* __restrict__ lam, int D, int r, int hk,
                           int col0, uint16_t* __restrict__ WT, uint16_t* __restrict__ B, float* __restrict__ sigma) {
  const int rho = blockIdx.x;
  const double* v = V + (size_t)(col0 - rho) * D;
  __shared__ double best_abs[32];
  __shared__ double best_val[32];
  double ba = -1.0, bv = 0.0;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const double x = v[i];
    if (fabs(x) > ba) { ba = fabs(x); bv = x; }
  }
  for (int o = 16; o; o >>= 1) {
    const double oa = __shfl_xor_sync(0xffffffffu, ba, o), ov = __shfl_xor_sync(0xffffffffu, bv, o);
    if (oa > ba || (oa == ba && ov > bv)) { ba = oa; bv = ov; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { best_abs[warp] = ba; best_val[warp] = bv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (best_abs[w] > ba || (best_abs[w] == ba && best_val[w] > bv)) { ba = best_abs[w]; bv = best_val[w]; }
    best_val[0] = bv;
    if (sigma) sigma[rho] = (float)sqrt(fmax(lam[col0 - rho], 0.0));
  }
  __syncthreads();
  const double sg = best_val[0] < 0.0 ? -1.0 : 1.0;
  const int d = D / hk;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float w = (float)(sg * v[i]);
    const uint16_t hi = f2bf(w);
    WT[(size_t)rho * D + i] = hi;
    WT[(size_t)(r + rho) * D + i] = f2bf(w - bf2f(hi));
    const int h = i / d, j = i - h * d;
    B[((size_t)h * r + rho) * d + j] = hi;
  }
}

// ---------------------------------------------------------------------------------------------
// 5. A = X . W on the tensor cores: CTA = 128 tokens x r columns, K = D in 64-wide blocks (one head
//    half each); stage = X box (128 tokens x 64, K-major) + W^T hi and lo boxes (r rows x 64, K-major)
// ---------------------------------------------------------------------------------------------
constexpr int kPStages = 3;                      // ring depth (fewer at large r: shared memory)
__host__ __device__ constexpr uint32_t proj_stage_bytes(int r) { return 16384u + 2u * (uint32_t)r * 128u; }
static int proj_stages(int r) { return (1024 + 3 * (size_t)proj_stage_bytes(r) <= 227 * 1024) ? 3 : 2; }
size_t project_smem_bytes(int r) { return 1024 + (size_t)proj_stages(r) * proj_stage_bytes(r); }

__global__ void __launch_bounds__(128, 1)
k_project_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int head0, int hk,
             int s, int r, int nstage, uint16_t* __restrict__ A) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  __shared__ __align__(8) uint64_t full[kPStages], empty[kPStages], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = blockIdx.x * 128, nkb = 2 * hk;
  const uint32_t stage = proj_stage_bytes(r);
  const uint32_t idesc = umma_idesc_bf16(128, r, false, false);
  if (tid == 0) {
    for (int i = 0; i < nstage; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
    prefetch_tensormap(&tmX);
    prefetch_tensormap(&tmW);
  }
  if (warp == 0) tmem_alloc<256>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {                                       // TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int stg = kb % nstage;
      if (kb >= nstage) mbar_wait(&empty[stg], ((kb / nstage) - 1) & 1);
      uint8_t* base = smem + stg * stage;
      mbar_expect_tx(&full[stg], stage);
      tma_load_3d(base, &tmX, (kb & 1) * 64, t0, head0 + (kb >> 1), &full[stg]);
      tma_load_2d(base + 16384, &tmW, kb * 64, 0, &full[stg]);
      tma_load_2d(base + 16384 + r * 128, &tmW, kb * 64, r, &full[stg]);
    }
  } else if (tid == 32) {                               // MMA issuer
    for (int kb = 0; kb < nkb; ++kb) {
      const int stg = kb % nstage;
      mbar_wait(&full[stg], (kb / nstage) & 1);
      tc_fence_after();
      const uint32_t x0 = smem_u32(smem + stg * stage), w0 = x0 + 16384, w1 = w0 + r * 128;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        umma_f16(tmem, umma_desc_sw128(x0 + ks * 32), umma_desc_sw128(w0 + ks * 32), idesc, (kb > 0 || ks > 0) ? 1u : 0u);
        umma_f16(tmem, umma_desc_sw128(x0 + ks * 32), umma_desc_sw128(w1 + ks * 32), idesc, 1u);
      }
      umma_commit(&empty[stg]);
    }
    umma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  const int t = t0 + 32 * warp + lane;
  uint16_t* arow = A + (size_t)t * r;
  for (int c = 0; c < r; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
    if (t < s) {
      uint4* dst = reinterpret_cast<uint4*>(arow + c);
      dst[0] = make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]), pack_bf2(v[4], v[5]), pack_bf2(v[6], v[7]));
      dst[1] = make_uint4(pack_bf2(v[8], v[9]), pack_bf2(v[10], v[11]), pack_bf2(v[12], v[13]), pack_bf2(v[14], v[15]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

cudaError_t init_factorize_attrs() {
  cudaError_t e;
  size_t proj = 0;
  for (int r = 16; r <= 256; r += 16) proj = project_smem_bytes(r) > proj ? project_smem_bytes(r) : proj;
  if ((e = cudaFuncSetAttribute(k_gram_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem_bytes()))) return e;
  return cudaFuncSetAttribute(k_project_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)proj);
}

namespace {
struct Handles {
  cusolverDnHandle_t solver = nullptr;
  int device = -1;
};
Handles g_h;

cudaError_t handles(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_h.device != dev) {                  // one handle per process (re-created if the device changes)
    if (g_h.solver) cusolverDnDestroy(g_h.solver);
    g_h = Handles{};
    if (cusolverDnCreate(&g_h.solver) != CUSOLVER_STATUS_SUCCESS) return cudaErrorUnknown;
    g_h.device = dev;
  }
  if (cusolverDnSetStream(g_h.solver, st) != CUSOLVER_STATUS_SUCCESS) return cudaErrorUnknown;
  return cudaSuccess;
}
}  // namespace

// token-range splits of the Gram blocks: about one CTA per SM of a 148-SM B200 over the P upper-triangle
// blocks (a fixed count, so the fp32 summation order -- and the factors -- do not depend on the device)
static int gram_splits(int hk, int s) {
  const int P = hk * (hk + 1) / 2;
  int n = 148 / P;
  if (n > 64) n = 64;
  const int steps = (s + kGTok - 1) / kGTok;
  if (n > steps) n = steps;
  return n < 1 ? 1 : n;
}

// workspace (one request at a time): Gram partials fp32, Gd fp64, lambda fp64, W^T hi/lo bf16, info,
// dsyevd work
size_t factorize_ws_bytes(int D, int r, FactorizeWs* ws, char* base) {
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return base + o; };
  const int hk = D / 128;
  const int nsp = gram_splits(hk, 1 << 30);
  char* g = carve((size_t)nsp * D * D * 4);
  char* gd = carve((size_t)D * D * 8);
  char* lam = carve((size_t)D * 8);
  char* w = carve((size_t)2 * r * D * 2);
  char* info = carve(256);
  const size_t lwork = (size_t)4 * D * D + 64 * D + (1 << 20);     // >= cuSOLVER's dsyevd query (doubles)
  char* work = carve(lwork * 8);
  if (ws) {
    ws->Gp = reinterpret_cast<float*>(g);
    ws->Gd = reinterpret_cast<double*>(gd);
    ws->lam = reinterpret_cast<double*>(lam);
    ws->WT = reinterpret_cast<uint16_t*>(w);
    ws->info = reinterpret_cast<int*>(info);
    ws->work = reinterpret_cast<double*>(work);
    ws->lwork = lwork;
  }
  return off;
}

static bool encode(const DevCtx& ctx, CUtensorMap* map, int rank, const void* base, const cuuint64_t* dims,
                   const cuuint64_t* strides, const cuuint32_t* box) {
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc && enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

FactorizeResult launch_factorize(int b, int hk, int d, int s, int r, const uint16_t* K, uint16_t* A, uint16_t* B,
                                 float* sigma, const FactorizeWs& ws, cudaStream_t st, int* launches,
                                 const DevCtx& ctx) {
  FactorizeResult res{cudaSuccess, 0, nullptr};
  const int D = hk * d;
  if ((res.err = handles(st)) != cudaSuccess) { res.what = "cuSOLVER handle"; return res; }
  int lwork = 0, meig = 0;
  const char* ev = getenv("SKV_FACT_EIG");
  const bool full = ev && ev[0] == 'f';                 // tuning / cross-check: the full eigensolve
  const cusolverStatus_t qs = full
      ? cusolverDnDsyevd_bufferSize(g_h.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, ws.Gd, D, ws.lam,
                                    &lwork)
      : cusolverDnDsyevdx_bufferSize(g_h.solver, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER,
                                     D, ws.Gd, D, 0.0, 0.0, D - r + 1, D, &meig, ws.lam, &lwork);
  if (qs != CUSOLVER_STATUS_SUCCESS) { res.err = cudaErrorUnknown; res.what = "eigensolver bufferSize"; return res; }
  if ((size_t)lwork > ws.lwork) {
    res.err = cudaErrorInvalidValue; res.unused = lwork; res.what = "dsyevd needs more workspace"; return res;
  }
  // the keys of all requests and heads as a 3D tensor {128 dims, s tokens, b*h_kv heads}: boxes never
  // cross a head (tokens past s read as zeros)
  CUtensorMap tmK, tmX, tmW;
  const cuuint64_t kd[3] = {(cuuint64_t)d, (cuuint64_t)s, (cuuint64_t)b * hk};
  const cuuint64_t ks[2] = {(cuuint64_t)d * 2, (cuuint64_t)s * d * 2};
  const cuuint32_t gbox[3] = {64, kGTok, 1}, pbox[3] = {64, 128, 1};
  const cuuint64_t wd[2] = {(cuuint64_t)D, (cuuint64_t)2 * r};
  const cuuint64_t wsd[1] = {(cuuint64_t)D * 2};
  const cuuint32_t wbox[2] = {64, (cuuint32_t)r};
  if (!encode(ctx, &tmK, 3, K, kd, ks, gbox) || !encode(ctx, &tmX, 3, K, kd, ks, pbox) ||
      !encode(ctx, &tmW, 2, ws.WT, wd, wsd, wbox)) {
    res.err = cudaErrorInvalidValue; res.what = "tensor map"; return res;
  }
  const int nsp = gram_splits(hk, s), P = hk * (hk + 1) / 2;
  for (int bi = 0; bi < b; ++bi) {
    // 1. Gram blocks (h, h2 >= h), token-range partials
    k_gram_tc<<<dim3(P, nsp), 128, gram_smem_bytes(), st>>>(tmK, bi * hk, hk, s, nsp, ws.Gp);
    // 2. fp64, symmetrised, partials summed in order
    k_gram_reduce<<<(D * D + 255) / 256, 256, 0, st>>>(ws.Gp, nsp, D, ws.Gd);
    // 3. eigen-decomposition
    const cusolverStatus_t es = full
        ? cusolverDnDsyevd(g_h.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, ws.Gd, D, ws.lam, ws.work,
                           (int)ws.lwork, ws.info)
        : cusolverDnDsyevdx(g_h.solver, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D,
                            ws.Gd, D, 0.0, 0.0, D - r + 1, D, &meig, ws.lam, ws.work, (int)ws.lwork, ws.info);
    if (es != CUSOLVER_STATUS_SUCCESS) { res.err = cudaErrorUnknown; res.what = "eigensolver"; return res; }
    // 4. top-r eigenvectors -> W^T (hi, lo), B_h, sigma
    k_take_top<<<r, 256, 0, st>>>(ws.Gd, ws.lam, D, r, hk, full ? D - 1 : r - 1, ws.WT, B + (size_t)bi * hk * r * d,
                                  sigma ? sigma + (size_t)bi * r : nullptr);
    // 5. A = X W on the tensor cores
    k_project_tc<<<(s + 127) / 128, 128, project_smem_bytes(r), st>>>(tmX, tmW, bi * hk, hk, s, r,
                                                                      proj_stages(r), A + (size_t)bi * s * r);
    *launches += 4;
    if ((res.err = cudaGetLastError()) != cudaSuccess) { res.what = "kernel launch"; return res; }
  }
  return res;
}

}  // namespace skv
