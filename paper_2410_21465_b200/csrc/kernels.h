// Host-side launchers for the ShadowKV kernels (internal to libshadowkv.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <mutex>

namespace skv {

struct Dims {          // validated, derived sizes
  int b, hq, hk, g, d, s, r, c, o, k, w, wcap;   // hq, g: query ROWS (q heads x s_q query tokens)
  int n_c, w_eff;
  int trace_slot;      // tuning only: which [4][4096][16] block of the trace buffer this call stamps
  const int* step_dev; // graph-replayable decode: step read on the device (nullable), clamped to
  int max_step;        // [0, max_step]; the grid is sized for max_step
  int sq;              // s_q query tokens per call (rows of one q head are consecutive: hq*s_q + i)
  const int* lens;     // ragged batch: device int32 [b] per-request context lengths (nullable = all s);
                       // then s, n_c are the padded layout sizes and w_eff is the largest per-request w_eff
  // low-rank generated keys (NEXT-4; nullable = plain window): the layer's B and its A_gen rows
  const uint16_t* lr_B;
  uint16_t* lr_A;      // [b][wcap][r]: row g = generated token g (decode step index)
  int serial;          // SKV_SERIALIZE: no PDL overlap, values before rebuild (bit-identical check)
};
#ifdef __CUDACC__
// per-request sizes of a ragged batch (R8 applied to each request's own length)
__device__ __forceinline__ int req_s(const Dims& D, int b) { return D.lens ? __ldg(D.lens + b) : D.s; }
__device__ __forceinline__ int req_nc(const Dims& D, int b) { return D.lens ? (__ldg(D.lens + b) - D.w) / D.c : D.n_c; }
__device__ __forceinline__ int req_weff(const Dims& D, int b) {
  return D.lens ? __ldg(D.lens + b) - req_nc(D, b) * D.c : D.w_eff;
}
#endif
constexpr size_t kTraceSlot = (size_t)4 * 4096 * 16;

struct Rope {
  const float* inv_freq;
  int rot, interleaved;
};

struct Layer {
  const uint16_t* A;
  const uint16_t* B;
  uint16_t* L;
  int32_t* outlier_ids;
  uint16_t *K_out, *V_out, *K_win, *V_win;
  const uint16_t* V_host;
  uint16_t* A_gen;                    // optional low-rank generated keys [b][wcap][r] (NEXT-4)
  // optional value-chunk cache (R26): least-recently-selected, capacity vc_cap slots; all null = off
  uint16_t* vc_values;                // [b][hk][C][c][d]
  unsigned long long* vc_dir;         // [b][hk][n_c]  (tag << 32) | slot; tag = inserting generation + 1
  unsigned long long* vc_stats;       // [b][hk][4]    {generation, step hits (scratch), last hits, total hits}
  unsigned long long* vc_slots;       // [b][hk][C + k] per slot ((last generation + 1) << 32) | (chunk + 1);
                                      //                then the step's miss -> slot assignments {slot, gen + 1}
  int vc_cap;                         // C >= k
};

// workspace carving (256-B aligned regions)
struct BuildWs {
  float* mincos;     // [b][hk][n_c]
  float* negm;       // [b][hk][n_c]  (-m, keys for the outlier top-o)
};
struct DecodeWs {
  int* flags;        // [b][hk][4] {score_done, -, -, -}; zeroed again by each call's merger
  int* epochs;       // [b][hq] calls merged so far per query row (zero-initialised once): the sparse units
                     // tag this call's partials with epoch + 1, the merge waits for that tag, then bumps
  int32_t* selrest;  // [b][hk][k] radix-fallback scratch (top-k, ascending)
  float* logits;     // [b][hk][n_c][G]: landmark-major, the G rows of a landmark contiguous (one vector
                     // store in the score epilogue, one vector load per landmark in k_select)
  float2* part;      // [b][hq][tiles_per_head] per-tile softmax partials (max, sumexp) of each query row
  float* z;          // [b][hk][n_c]     (only when n_c does not fit the select kernel's smem)
  int32_t* sel;      // [b][hk][k] published selection, unordered, chunk id + 1 (0 = not yet); re-zeroed
  uint2* o_part;     // [b][hq][n_split][d]  {fp32 bits, tag}: 8-byte value + flag pairs
  uint2* ml_part;    // [b][hq][n_split][2]  {m bits, tag}, {l bits, tag}
  int n_sblk, n_split;
};

constexpr int kSTile = 128;                       // landmark rows per score tile (32 KB)
constexpr int kSStages = 3;                       // score smem ring depth (2 CTAs / SM)
constexpr int kUnitTok = 64;                      // tokens per attention unit (8 chunks)
constexpr size_t kSelectSmemMax = 160 * 1024;     // per-CTA z slice + its logits kept in smem
constexpr int kSelCL = 8;                         // select: CTAs per (request, KV head) cluster
constexpr int kSelThreads = 512;
constexpr int kMaxVcCapacity = 4096;              // value-cache slots per (request, KV head)
constexpr int kSelCandLocal = 1024;               // threshold-bucket candidates of a cluster (all ranks)
constexpr int kSelCandPush = 128;                 // threshold-bucket candidates per CTA (more: radix fallback)

// header (zero-filled once by the caller): 4 flags per (b, h_kv), then one partial epoch per query row
inline size_t ws_header_bytes(const Dims& D) {
  return (((size_t)D.b * D.hk * 4 + (size_t)D.b * D.hq) * 4 + 255) & ~(size_t)255;
}
size_t build_ws_bytes(const Dims& D, BuildWs* ws, char* base);
size_t decode_ws_bytes(const Dims& D, DecodeWs* ws, char* base);

// Optional per-kernel CUDA-event timing (shadowkv_profile_*): kernel ids below.
enum KernelId { kScore = 0, kSelect = 1, kSparseAttn = 2, kReserved = 3, kCombine = 4, kNumKernelIds = 5 };
struct Profiler;                                            // defined in abi.cu
void profile_mark(Profiler* p, int kernel, bool end, cudaStream_t st);

cudaError_t set_trace_buffer(void* dev_ptr);      // decode.cu: nullptr disables
cudaError_t set_trace_buffer_tc(void* dev_ptr);   // score_tc.cu (kernel slot 0)

// ---- per-device runtime context (shadowkv_init): everything a decode / build call would otherwise
// create or configure on first use -- kernel smem attributes, the sub-batch side streams and events,
// the SM count, the driver's tensor-map encoder -- is set up once per device, under a lock, so the
// hot path never allocates and concurrent calls (different streams / devices) share nothing mutable.
constexpr int kMaxSplit = 8;                      // request sub-batch chains (decode.cu)
constexpr int kMaxDevices = 64;
struct DevCtx {
  int device = -1;
  int n_sm = 0;
  cudaStream_t side[kMaxSplit] = {};
  cudaEvent_t ev_sel[kMaxSplit] = {}, ev_done[kMaxSplit] = {};
  void* encode_tiled = nullptr;                   // cuTensorMapEncodeTiled (driver entry point)
};
// the calling thread's current device's context, or nullptr if shadowkv_init was not called for it
const DevCtx* current_ctx();
cudaError_t init_device(int device, const char** what);   // idempotent; thread-safe
cudaError_t init_decode_attrs();                  // decode.cu: kernel attributes (current device)
cudaError_t init_build_attrs();                   // build.cu
cudaError_t init_score_tc_attrs();                // score_tc.cu
std::mutex& chain_mutex(int device);              // serialises sub-batch chain enqueues per device

// score_tc.cu: tcgen05 landmark scoring (a1).  The plan must satisfy the kernel's static limits (tiles
// and KV heads per CTA, partial slots per head); score_tc_plan returns false (and the decode call
// SKV_EUNSUPPORTED) when no grid does, e.g. a single request of several million tokens.
struct ScorePlan {
  int grid, tiles_per_cta, heads_per_cta, ctas_per_head;
};
bool score_tc_plan(const Dims& D, int tiles_per_head, int n_sm, ScorePlan* plan);
template <int G>
cudaError_t launch_score_tc(const Dims& D, const uint16_t* L, const int32_t* oids, const uint16_t* q,
                            float* logits, float2* part, int tiles_per_head, float scale,
                            const uint16_t* k_new, const uint16_t* v_new, uint16_t* K_win, uint16_t* V_win,
                            int step, const DevCtx& ctx, cudaStream_t st);

// each returns cudaGetLastError() after its launches and adds to *launches
cudaError_t launch_build(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* K_rope,
                         const BuildWs& ws, cudaStream_t st, int* launches, const DevCtx& ctx);
cudaError_t launch_decode(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                          const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                          int32_t* sel_ids, uint16_t* dbg_keys, char* ws_base, cudaStream_t st,
                          int* launches, Profiler* prof, const DevCtx& ctx);
size_t decode_ws_total_bytes(const Dims& D);   // every sub-batch split's workspace fits
cudaError_t launch_rope_probe(const int32_t* pos, int n, const float* inv_freq, int nf, float* out, cudaStream_t st);

// factorize.cu: Alg 1 "A, B <- SVD(K)" through the D x D Gram matrix (NEXT-2)
struct FactorizeWs {
  float* Gp;         // [splits][D][D] fp32 Gram block partials (row-major, upper block triangle)
  double* Gd;        // [D][D] fp64, overwritten by the eigenvectors
  double* lam;       // [D] eigenvalues, ascending
  uint16_t* WT;      // [2][r][D] bf16: W^T hi and lo planes
  int* info;
  double* work;      // dsyevd work
  size_t lwork;      // doubles
};
struct FactorizeResult {
  cudaError_t err;
  int unused;
  const char* what;  // failing step
};
size_t factorize_ws_bytes(int D, int r, FactorizeWs* ws, char* base);
cudaError_t init_factorize_attrs();
FactorizeResult launch_factorize(int b, int hk, int d, int s, int r, const uint16_t* K, uint16_t* A, uint16_t* B,
                                 float* sigma, const FactorizeWs& ws, cudaStream_t st, int* launches,
                                 const DevCtx& ctx);

}  // namespace skv
