// Alg 1 "A in R^{b x s x r}, B in R^{b x h_kv x r x d} <- SVD(K)" on the GPU.
//
// Per request, the pre-RoPE keys of all KV heads form X[t, h*d + j] = K[h][t][j] (R14), an
// s x D matrix with D = h_kv * d <= 4096 and s >> D.  Its truncated SVD is taken through the D x D
// Gram matrix, which is where s enters (2 s D^2 flops, tensor cores):
//   1. G = X^T X                      cuBLAS bf16 x bf16 -> fp32 GEMMs on tensor cores, one d x d
//                                     block per (h, h') pair (X is h-blocked, not one strided matrix)
//   2. G -> fp64, symmetrised         k_gram_to_f64
//   3. G = V diag(lambda) V^T         cuSOLVER dsyevdx, only the top r eigenpairs (fp64; the D x D
//                                     eigenproblem is independent of s; SKV_FACT_EIG=full: dsyevd)
//   4. W = top-r eigenvectors (sigma_i = sqrt(lambda_i), descending), B_h = W[h*d:(h+1)*d, :]^T
//                                     k_take_top
//   5. A = X W  (= U_r Sigma_r)       k_project: fp32 CUDA-core contraction of the bf16 keys with the
//                                     fp32 W (s x D x r, 43 GFLOP at 128K), bf16 out
// The Gram route squares the condition number; it only matters below the truncation (sigma_i with
// i > r), where bf16 storage noise of K already sits.  Prefill, not the decode hot path: this runs
// once per context and is timed against prefill attention in tools/svd_overhead.py (Fig 1c).
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace skv {

__global__ void k_gram_to_f64(const float* __restrict__ G, double* __restrict__ Gd, int D) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;        // column-major element (row, col)
  if (i >= D * D) return;
  const int row = i % D, col = i / D;
  Gd[i] = 0.5 * ((double)G[i] + (double)G[(size_t)row * D + col]);
}

// W[(h,j)][rho] = eigenvector D-1-rho (dsyevd: ascending eigenvalues, vectors in columns);
// sign fixed so the largest-|.| component is positive (deterministic factors; A.B is sign-free).
// col0: the column of the largest eigenpair (eigenvalues ascend: D - 1 for the full solve, r - 1 for the
// top-r range solve)
__global__ void k_take_top(const double* __restrict__ V, const double* __restrict__ lam, int D, int r, int hk,
                           int col0, float* __restrict__ W, uint16_t* __restrict__ B, float* __restrict__ sigma) {
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
    W[(size_t)i * r + rho] = w;
    const int h = i / d, j = i - h * d;
    B[((size_t)h * r + rho) * d + j] = f2bf(w);
  }
}

// A[t][rho] = sum_{h,j} K[h][t][j] W[(h,j)][rho]: CTA = 64 tokens x all r (r <= 256, r % 16 == 0);
// thread = 4 tokens x r/16 columns; K and W staged through smem 32 dims at a time.
constexpr int kPT = 64, kPK = 32;
__global__ void __launch_bounds__(256) k_project(const uint16_t* __restrict__ K, const float* __restrict__ W,
                                                 uint16_t* __restrict__ A, int s, int hk, int d, int r) {
  __shared__ float Ks[kPK][kPT + 1];
  __shared__ float Ws[kPK][256];
  const int t0 = blockIdx.x * kPT, tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;            // tokens ty + 16 i; columns tx + 16 c
  const int ncol = r >> 4;
  float acc[4][16];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[i][c] = 0.f;
  const int D = hk * d;
  for (int k0 = 0; k0 < D; k0 += kPK) {
    const int h = k0 / d, j0 = k0 - h * d;
    const uint16_t* Kh = K + (size_t)h * s * d;
    for (int e = tid; e < kPT * kPK; e += 256) {     // 32 consecutive dims of 64 tokens (64 B rows)
      const int tt = e / kPK, jj = e - tt * kPK;
      const int t = t0 + tt;
      Ks[jj][tt] = t < s ? bf2f(Kh[(size_t)t * d + j0 + jj]) : 0.f;
    }
    for (int e = tid; e < kPK * r; e += 256) {
      const int kk = e / r, c = e - kk * r;
      Ws[kk][c] = W[(size_t)(k0 + kk) * r + c];
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kPK; ++kk) {
      float kv[4], wv[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) kv[i] = Ks[kk][ty + 16 * i];
#pragma unroll
      for (int c = 0; c < 16; ++c) wv[c] = c < ncol ? Ws[kk][tx + 16 * c] : 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[i][c] = fmaf(kv[i], wv[c], acc[i][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty + 16 * i;
    if (t >= s) continue;
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < ncol) A[(size_t)t * r + tx + 16 * c] = f2bf(acc[i][c]);
  }
}

namespace {
struct Handles {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  int device = -1;
};
Handles g_h;

cudaError_t handles(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_h.device != dev) {                  // one pair per process (re-created if the device changes)
    if (g_h.blas) cublasDestroy(g_h.blas);
    if (g_h.solver) cusolverDnDestroy(g_h.solver);
    g_h = Handles{};
    if (cublasCreate(&g_h.blas) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    if (cusolverDnCreate(&g_h.solver) != CUSOLVER_STATUS_SUCCESS) return cudaErrorUnknown;
    g_h.device = dev;
  }
  if (cublasSetStream(g_h.blas, st) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  if (cusolverDnSetStream(g_h.solver, st) != CUSOLVER_STATUS_SUCCESS) return cudaErrorUnknown;
  return cudaSuccess;
}
}  // namespace

// workspace (one request at a time): G fp32, Gd fp64, lambda fp64, W fp32, info, cuBLAS and dsyevd work
size_t factorize_ws_bytes(int D, int r, FactorizeWs* ws, char* base) {
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return base + o; };
  char* g = carve((size_t)D * D * 4);
  char* gd = carve((size_t)D * D * 8);
  char* lam = carve((size_t)D * 8);
  char* w = carve((size_t)D * r * 4);
  char* info = carve(256);
  char* blas = carve(kFactorizeBlasWs);
  const size_t lwork = (size_t)4 * D * D + 64 * D + (1 << 20);     // >= cuSOLVER's dsyevd query (doubles)
  char* work = carve(lwork * 8);
  if (ws) {
    ws->G = reinterpret_cast<float*>(g);
    ws->Gd = reinterpret_cast<double*>(gd);
    ws->lam = reinterpret_cast<double*>(lam);
    ws->W = reinterpret_cast<float*>(w);
    ws->info = reinterpret_cast<int*>(info);
    ws->blas_ws = blas;
    ws->work = reinterpret_cast<double*>(work);
    ws->lwork = lwork;
  }
  return off;
}

FactorizeResult launch_factorize(int b, int hk, int d, int s, int r, const uint16_t* K, uint16_t* A, uint16_t* B,
                                 float* sigma, const FactorizeWs& ws, cudaStream_t st, int* launches) {
  FactorizeResult res{cudaSuccess, 0, nullptr};
  const int D = hk * d;
  if ((res.err = handles(st)) != cudaSuccess) { res.what = "cuBLAS/cuSOLVER handle"; return res; }
  if (cublasSetWorkspace(g_h.blas, ws.blas_ws, kFactorizeBlasWs) != CUBLAS_STATUS_SUCCESS) {
    res.err = cudaErrorUnknown; res.what = "cublasSetWorkspace"; return res;
  }
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
  const float one = 1.f, zero = 0.f;
  for (int bi = 0; bi < b; ++bi) {
    const uint16_t* Kb = K + (size_t)bi * hk * s * d;
    // 1. G_{h,h'} = K_h^T K_h' (column-major d x s operands, fp32 accumulate on tensor cores)
    for (int h = 0; h < hk; ++h) {
      if (cublasGemmStridedBatchedEx(g_h.blas, CUBLAS_OP_N, CUBLAS_OP_T, d, d, s, &one,
                                     Kb + (size_t)h * s * d, CUDA_R_16BF, d, 0,
                                     Kb, CUDA_R_16BF, d, (long long)s * d, &zero,
                                     ws.G + (size_t)h * d, CUDA_R_32F, D, (long long)d * D, hk,
                                     CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS) {
        res.err = cudaErrorUnknown; res.what = "cublasGemmStridedBatchedEx (Gram)"; return res;
      }
    }
    // 2. fp64, symmetrised
    k_gram_to_f64<<<(D * D + 255) / 256, 256, 0, st>>>(ws.G, ws.Gd, D);
    // 3. eigen-decomposition
    const cusolverStatus_t es = full
        ? cusolverDnDsyevd(g_h.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, ws.Gd, D, ws.lam, ws.work,
                           (int)ws.lwork, ws.info)
        : cusolverDnDsyevdx(g_h.solver, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D,
                            ws.Gd, D, 0.0, 0.0, D - r + 1, D, &meig, ws.lam, ws.work, (int)ws.lwork, ws.info);
    if (es != CUSOLVER_STATUS_SUCCESS) { res.err = cudaErrorUnknown; res.what = "eigensolver"; return res; }
    // 4. top-r eigenvectors -> W, B_h, sigma
    k_take_top<<<r, 256, 0, st>>>(ws.Gd, ws.lam, D, r, hk, full ? D - 1 : r - 1, ws.W, B + (size_t)bi * hk * r * d,
                                  sigma ? sigma + (size_t)bi * r : nullptr);
    // 5. A = X W
    k_project<<<(s + kPT - 1) / kPT, 256, 0, st>>>(Kb, ws.W, A + (size_t)bi * s * r, s, hk, d, r);
    *launches += 3;
    if ((res.err = cudaGetLastError()) != cudaSuccess) { res.what = "kernel launch"; return res; }
  }
  return res;
}

}  // namespace skv
