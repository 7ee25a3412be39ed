/*
 * shadowkv.h -- C ABI of the B200 (sm_100a) ShadowKV decode-time sparse-attention path.
 *
 * ShadowKV (arXiv 2410.21465).  Citations: "P:n" = PAPER.md line n (LaTeX source),
 * "S:n" = SPEC.md line n, "Rn" = reading n of the register in DESIGN.md.
 *
 * Two operations, both asynchronous on the caller's CUDA stream:
 *   shadowkv_build_cache  -- Algorithm 1 "ShadowKV Pre-filling" minus the SVD
 *                            (the caller supplies the rank-r factors A, B, R14).
 *   shadowkv_decode_step  -- Algorithm 2 "ShadowKV Decoding" followed by the sparse
 *                            attention over outliers + selected chunks + local window
 *                            ("accurate sparse attention computation with selected KV pairs
 *                            and static outliers").
 *
 * Conventions
 *   - All pointers are caller-owned; the library never allocates, frees or synchronises.
 *   - bf16 tensors are passed as uint16_t* holding IEEE bfloat16 bit patterns.
 *   - "device" pointers are cudaMalloc'd (or torch CUDA) memory on the current device;
 *     "host-mapped" pointers are page-locked host memory that is mapped into the device
 *     address space (cudaHostAlloc / cudaHostRegister; under UVA the host pointer itself).
 *   - All device/host buffers must be 16-byte aligned and densely packed in the stated layout.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Errors: the call validates its arguments on the host before enqueuing anything.  On a
 *     non-OK status nothing was enqueued and shadowkv_last_error() (thread-local) explains why.
 *     Faults inside kernels surface at the caller's next synchronisation -- or, with the
 *     environment variable SKV_DEBUG_SYNC=1, as SKV_ECUDA of the call itself (every enqueuing call
 *     then synchronises its stream, except while the stream is being captured into a graph).
 *   - Setup: shadowkv_init(device) once per device before any build / decode call on it.  It creates
 *     and configures everything the calls would otherwise set up on first use (kernel attributes,
 *     internal streams and events, the tensor-map encoder), so build / decode never allocate, and a
 *     device that was not initialised gives SKV_ESTATE.
 *   - Ordering: decode_step's first kernel is launched with programmatic dependent launch and reads
 *     the layer's landmarks and outlier_ids before it waits on the preceding kernel of `stream`.
 *     If you rewrite those two arrays with your own KERNEL, do not enqueue decode_step directly after
 *     it (put any other stream operation in between, e.g. an event record, or a build_cache: its last
 *     kernel writes nothing).  Copies (cudaMemcpyAsync) are fully ordered.
 *   - Debug: SKV_SERIALIZE=1 runs the decode kernels without overlap (no PDL, values before the key
 *     rebuild); outputs are bit-identical to the overlapped schedule.  NVTX ranges name each ABI call
 *     and each kernel launch (skv::score, skv::select, skv::sparse_attn, skv::merge).
 *
 * Symbols: b batch, h_q / h_kv query / KV heads (g = h_q / h_kv, q head hq uses KV head
 * floor(hq/g), R2), d = head_dim, s = ctx_len, r = rank, c = chunk, o = n_outlier, k = budget,
 * w = window_ctx; n_c = floor((s - w) / c) chunks on the grid, w_eff = s - n_c*c window tokens
 * (R8), n_L = n_c - o landmarks per KV head.
 */
#ifndef SHADOWKV_H
#define SHADOWKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHADOWKV_ABI_VERSION 7

#if defined(__GNUC__)
#define SKV_API __attribute__((visibility("default")))
#else
#define SKV_API
#endif

typedef enum {
  SKV_OK = 0,
  SKV_EINVAL = 1,        /* bad argument (null pointer, size out of range, window overflow) */
  SKV_EUNSUPPORTED = 2,  /* valid per the paper but not compiled: d != 128, c != 8, g not in {1,2,4,8,16} */
  SKV_ECUDA = 3,         /* a CUDA runtime call or kernel launch failed */
  SKV_ESTATE = 4         /* V_host is not page-locked + device-mapped; shadowkv_init not called */
} skv_status;

typedef struct {
  int32_t batch;        /* b >= 1 requests (uniform ctx_len across the batch)                   */
  int32_t n_q_heads;    /* h_q                                                                  */
  int32_t n_kv_heads;   /* h_kv; h_q % h_kv == 0                                                */
  int32_t head_dim;     /* d; must be 128                                                       */
  int32_t ctx_len;      /* s; context tokens at absolute positions 0..s-1 (R16)                 */
  int32_t rank;         /* r; multiple of 16, 16 <= r <= 256 ("SVD rank r")               */
  int32_t chunk;        /* c; must be 8 ("chunks of eight tokens")                 */
  int32_t n_outlier;    /* o; 0 <= o < n_c                                              */
  int32_t budget;       /* k selected chunks per KV head; 1 <= k <= n_L           */
  int32_t window_ctx;   /* w; context tail kept exact on the GPU (R8)                           */
  int32_t window_cap;   /* ring capacity in tokens per KV head; >= w_eff + (tokens you will decode) */
  int32_t q_len;        /* s_q query tokens per decode call (Alg 2's Q in R^{b x h_q x s_q x d},
                           P:164; e.g. speculative verification); 0 or 1 = one token.  The s_q
                           tokens share one selection (S1 = sum over s_q of the softmax)
                           and attend causally among themselves (R28).  Needs g * s_q in
                           {1, 2, 4, 8, 16} (else SKV_EUNSUPPORTED).                          */
  /* Ragged batch: per-request context lengths s_b <= ctx_len.  Both NULL = every
   * request has ctx_len tokens.  Otherwise ctx_len is the PADDED length every [..][s][..] layout
   * (A, V_host, K_rope) and the landmark grid [..][n_c][..] (n_c of ctx_len) are strided by, and
   * request b uses its own grid n_c(b) = floor((s_b - w)/c), window tail w_eff(b) = s_b - n_c(b)*c
   * (R8 per request), decode positions s_b + step + i.  Each s_b must leave o + k chunks on its
   * grid: s_b >= w + c*(o + k) (SKV_EINVAL otherwise).  window_cap must hold the largest w_eff(b). */
  const int32_t *ctx_lens;      /* host int32 [b] (validated on every call)                       */
  const int32_t *ctx_lens_dev;  /* device int32 [b], the same values (read by the kernels)        */
} skv_dims;

typedef struct {
  int32_t rotary_dim;     /* even, 2 <= rotary_dim <= d; dims >= rotary_dim pass through (R15);
                             halves layout additionally needs rotary_dim in {16, 32, 64, 128}
                             (else SKV_EUNSUPPORTED)                                            */
  int32_t interleaved;    /* 0: halves layout (x_i, x_{i+rot/2}) [Llama]; 1: pairs (2i, 2i+1) [GLM] */
  const float *inv_freq;  /* device, rotary_dim/2 fp32; angle = fl32(fl32(t) * inv_freq[i])      */
} skv_rope;

typedef struct {
  /* rank-r pre-RoPE key factors: K_pre[b][h][t][:] ~= A[b][t][:] . B[b][h][:][:] */
  const uint16_t *A;        /* device bf16 [b][s][r]                                           */
  const uint16_t *B;        /* device bf16 [b][h_kv][r][d]                                     */
  /* GPU-resident state written by build_cache, read by decode_step */
  uint16_t *landmarks;      /* device bf16 [b][h_kv][n_c][d]: chunk means of post-RoPE keys on
                               the full grid; rows of outlier chunks are never scored   */
  int32_t *outlier_ids;     /* device int32 [b][h_kv][o], ascending                     */
  uint16_t *K_out;          /* device bf16 [b][h_kv][o*c][d] post-RoPE outlier keys     */
  uint16_t *V_out;          /* device bf16 [b][h_kv][o*c][d] outlier values                     */
  uint16_t *K_win;          /* device bf16 [b][h_kv][window_cap][d]: slots [0,w_eff) = context
                               tail, slot w_eff+step = token generated at decode step `step`    */
  uint16_t *V_win;          /* device bf16 [b][h_kv][window_cap][d]                             */
  /* offloaded values V^CPU: all s positions kept; outlier/window rows are never read */
  const uint16_t *V_host;   /* host-mapped bf16 [b][h_kv][s][d], read zero-copy over PCIe        */
  /* Optional GPU-resident value-chunk cache ("considering the temporal locality of the KV
   * cache, a cache policy can be leveraged"; "we conduct an index scan to detect the missed
   * chunks"; policy per SPEC S:139-146, DESIGN R26): least-recently-SELECTED replacement at chunk
   * granularity, capacity C = vc_capacity chunks per (request, KV head), C >= k (0 = k).  A selected chunk
   * whose directory entry is valid is a HIT: its values are copied from its HBM slot instead of the host
   * link.  Each MISS takes a slot: an empty one, else the least recently selected cached chunk that this
   * step did not select (ties -> the lower chunk id is evicted first); its values are written there once
   * they arrive.  Values are bit copies either way, so outputs do not depend on the cache state.  All four
   * pointers NULL = no cache; all four or none.  build_cache zero-fills vc_dir, vc_stats and vc_slots (a
   * new prefill starts cold); a caller may also reset the cache by zero-filling those three.  Not shared
   * between layers. */
  uint16_t *vc_values;      /* device bf16 [b][h_kv][C][c][d]: C value slots per KV head            */
  uint64_t *vc_dir;         /* device [b][h_kv][n_c]: (tag << 32) | slot; tag = generation + 1 of
                               the step that inserted the chunk; zero = not cached              */
  uint64_t *vc_stats;       /* device [b][h_kv][4]: {generation (decode steps run), scratch,
                               hits in the last step, hits in total}; read them after a sync    */
  /* Optional low-rank storage of generated keys (P:196 footnote "new pre-RoPE keys K' can be stored
   * as K' Psi and projected back with Psi^T").  NULL = plain window.  Non-NULL: decode's
   * k_new is PRE-RoPE; each generated token g (= step + i) is stored as one rank-r row
   * A_gen[b][g][:] = bf16(sum_h k'_h B_h^T) (Psi[(h, j), rho] = B_h[rho][j], R14) -- r values per token
   * for all heads instead of h_kv*d -- and attended with the key RoPE_{s_b+g}(A_gen[b][g] . B_h);
   * K_win slots >= w_eff are then neither written nor read (values still go to V_win).  Exact when
   * k' lies in the span of the B rows (e.g. B from shadowkv_factorize). */
  uint16_t *A_gen;          /* device bf16 [b][window_cap][r]                                    */
  /* value cache (continued, ABI 7): per-slot state and the capacity */
  uint64_t *vc_slots;       /* device [b][h_kv][C + k]: slot s < C holds ((generation of its last
                               selection + 1) << 32) | (chunk id + 1), 0 = empty; entries C.. are
                               the step's miss -> slot assignments (scratch)                     */
  int32_t vc_capacity;      /* C: value slots per (request, KV head); 0 = k; k <= C <= n_c       */
  int32_t reserved0;
} skv_layer;

/* One-time setup for `device` (idempotent, thread-safe): kernel shared-memory attributes for every
 * compiled GQA group, the SM count, 8 high-priority internal streams + 16 events for the sub-batch
 * chains of large batches, and the driver's cuTensorMapEncodeTiled.  Required before build / decode
 * on that device (SKV_ESTATE otherwise); SKV_ECUDA if any of it fails.  Leaves the current device
 * unchanged. */
SKV_API skv_status shadowkv_init(int32_t device);

/* Launch plan of the tcgen05 landmark scorer (a1) for these dims on a GPU with n_sm SMs, pure host
 * arithmetic: plan[0] grid (CTAs), plan[1] tiles (128 landmarks) per CTA, plan[2] KV heads a CTA's
 * tile range may touch, plan[3] CTAs per KV head (softmax partial slots used by the selector).
 * SKV_EUNSUPPORTED when no grid satisfies the kernel's limits (<= 256 tiles and <= 4 KV heads per
 * CTA, <= 64 partial slots per KV head), e.g. one request of ~8M tokens with 8 KV heads; decode_step
 * returns the same status for such dims. */
SKV_API skv_status shadowkv_score_plan(const skv_dims *dims, int32_t n_sm, int32_t *plan);

/* Diagnostic: sin / cos of the RoPE angle phi = fl32(fl32(pos[p]) * inv_freq[i]) exactly as the
 * decode kernels compute them (R15: fp64 reduction mod 2 pi, then the hardware sincos on |r| <= pi),
 * for p < n, i < rotary_dim/2.  pos: device int32 [n]; sincos: device fp32 [n][rotary_dim/2][2]
 * (sin, cos).  Asynchronous on `stream`. */
SKV_API skv_status shadowkv_rope_sincos(const skv_rope *rope, const int32_t *pos, int32_t n, float *sincos,
                                        void *stream);

/* Bytes of scratch `workspace` (device, 256-byte aligned) that build_cache and decode_step need
 * for these dims.  Returns 0 on invalid dims (see shadowkv_last_error). Pure host arithmetic.
 * The workspace must be ZERO-FILLED once before its first use (it holds per-(request, KV head)
 * completion counters that every call leaves at zero); one workspace may serve many layers but
 * only one stream at a time. */
SKV_API size_t shadowkv_workspace_bytes(const skv_dims *dims);

/* Algorithm 1 for every request and KV head, on `stream`:
 *   keys    = K_rope if non-NULL (device bf16 [b][h_kv][s][d], post-RoPE),
 *             else RoPE_t(A[t] . B_h) at absolute positions t (the keys the factors represent);
 *   C_j     = mean of the c keys of chunk j;   landmarks <- bf16(C)
 *   m_j     = min_t cos(C_j, k_t) (R10, R11; zero norm -> -1)
 *   outlier_ids <- the o chunks with smallest m (ties -> lower j, R12), ascending
 *   K_out, V_out <- keys / values of those chunks; values read zero-copy from V_host
 *   K_win, V_win slots [0, w_eff) <- the context tail (R8)
 * With a value cache (vc_*), zero-fills vc_dir, vc_stats and vc_slots (cold cache for the new context).
 * Requires V_host page-locked and mapped (checked once here; SKV_ESTATE otherwise). */
SKV_API skv_status shadowkv_build_cache(const skv_dims *dims, const skv_rope *rope, const skv_layer *layer,
                                const uint16_t *K_rope, void *workspace, void *stream);

/* One decode step of Algorithm 2 for the whole batch, on `stream`:
 *   a7  K_win/V_win slot w_eff+step <- k_new, v_new (Alg 2 input K, V; R18)
 *   a1  l_{hq,j} = <q_hq, L_{h,j}> / sqrt(d) over landmarks j (R6)
 *   a2  z_{h,j} = max_{hq in group h} log sum_{i < s_q} softmax_j(l_{hq,i,.})_j  (= log S2, P:169-172,
 *       R4, R5; for s_q = 1: max_hq (l_{hq,j} - logsumexp_j l_{hq,.}))
 *   a3  I_h = ArgTopK(z_h, k), ties -> lower chunk id, ascending (R12)
 *   a4  K~ = RoPE_t(A[t] . B_h) for the k*c tokens of I_h at their absolute positions
 *   a5  V~ = V_host rows of those tokens, gathered zero-copy over the host link; with a
 *       value cache, chunks selected in the previous step are copied from vc_values instead, and
 *       every selected chunk is written to this step's slot buffer (R26)
 *   a6  out_{hq,i} = softmax attention of query token i over outlier tokens + K~/V~ + window slots
 *       [0, w_eff+step+i] (R17; causal among the new tokens, R28)
 * Ragged batches (dims.ctx_lens): s, w_eff, positions and the chunk grid are per request (R29).
 * Low-rank generated keys (layer.A_gen): generated tokens are attended with RoPE_t(A_gen[g] . B_h) (R30).
 * q      device bf16 [b][h_q][s_q][d], token i post-RoPE at position s+step+i (R16)
 * k_new  device bf16 [b][h_kv][s_q][d] post-RoPE (pre-RoPE with layer.A_gen);  v_new [b][h_kv][s_q][d]
 *        (written to window slots w_eff+step .. w_eff+step+s_q-1; the next call's step is step+s_q)
 * out    device bf16 [b][h_q][s_q][d]
 * sel_ids   nullable device int32 [b][h_kv][k]  -- parity hook for a3
 * dbg_keys  nullable device bf16 [b][h_kv][k*c][d] -- parity hook for a4 (rebuilt, post-RoPE)
 * Requires window_cap >= w_eff + step + s_q (SKV_EINVAL otherwise); SKV_EUNSUPPORTED when the
 * scorer has no launch plan for the dims (shadowkv_score_plan).
 * Streams: all work is ordered after earlier work on `stream`, and later work on `stream` is
 * ordered after all of it.  For batches of >= 32 requests the call pipelines request sub-batches:
 * it forks part of the work onto the device's internal high-priority streams (event fork/join,
 * capture-safe) and joins them back into `stream` before returning (SKV_SPLIT=n overrides the
 * sub-batch count).  Calls from several host threads are safe (the fork/join enqueue is serialised
 * per device); each concurrent call needs its own workspace. */
SKV_API skv_status shadowkv_decode_step(const skv_dims *dims, const skv_rope *rope, const skv_layer *layer,
                                const uint16_t *q, const uint16_t *k_new, const uint16_t *v_new,
                                int32_t step, uint16_t *out, int32_t *sel_ids, uint16_t *dbg_keys,
                                void *workspace, void *stream);

/* Graph-replayable variant of shadowkv_decode_step: identical computation, but the step index is
 * read on the device from *step_dev (int32, 4-byte aligned, device memory, written by work ordered
 * before this call on `stream`, e.g. an increment captured in the same CUDA graph), so one captured
 * graph serves every decode step.  Values are clamped to [0, max_step]; the launch is sized for
 * max_step (window units past the live window contribute nothing).  Requires window_cap >= w_eff +
 * max_step + 1.  Same buffers, streams and errors as shadowkv_decode_step. */
SKV_API skv_status shadowkv_decode_step_dev(const skv_dims *dims, const skv_rope *rope, const skv_layer *layer,
                                    const uint16_t *q, const uint16_t *k_new, const uint16_t *v_new,
                                    const int32_t *step_dev, int32_t max_step, uint16_t *out, int32_t *sel_ids,
                                    uint16_t *dbg_keys, void *workspace, void *stream);

/* Bytes of scratch `workspace` (device, 256-byte aligned) shadowkv_factorize needs for these dims
 * (independent of batch and ctx_len: requests are factorised one after another).  0 on invalid dims. */
SKV_API size_t shadowkv_factorize_workspace_bytes(const skv_dims *dims);

/* Algorithm 1's "A, B <- SVD(K)" on the GPU, for every request, on `stream`: the rank-r
 * truncated SVD of the pre-RoPE keys with all KV heads concatenated per token (X[t][h*d + j] =
 * K_pre[b][h][t][j], R14), X = U S V^T, split as A = U_r S_r (shared by the heads) and
 * B_h = (V_r^T)[:, h*d:(h+1)*d] -- exactly the factors shadowkv_build_cache / decode_step take.
 * Computed through the D x D Gram matrix (D = h_kv*d): G = X^T X (our tcgen05 kernel: 128 x 128
 * blocks, bf16 in, fp32 TMEM accumulation, split over token ranges, partials summed in a fixed order),
 * eigen-decomposition in fp64 (cuSOLVER dsyevdx, top r), A = X V_r (our tcgen05 kernel; V_r as bf16 hi +
 * lo planes).  Each singular vector's largest-magnitude component is made positive (deterministic
 * factors).  Dims used: batch, n_kv_heads, head_dim (must be 128), ctx_len, rank (multiple of 16,
 * 16 <= r <= min(256, s, h_kv*d)); h_kv*d <= 4096.  Prefill-time ("linear cost"), not the
 * decode hot path; creates one cuSOLVER handle per process on first use; needs shadowkv_init.
 * K_pre  device bf16 [b][h_kv][s][d]  (Alg 1 input K)
 * A      device bf16 [b][s][r]        (out)
 * B      device bf16 [b][h_kv][r][d]  (out)
 * sigma  nullable device fp32 [b][r]  (out) singular values sigma_1 >= ... >= sigma_r */
SKV_API skv_status shadowkv_factorize(const skv_dims *dims, const uint16_t *K_pre, uint16_t *A, uint16_t *B,
                              float *sigma, void *workspace, void *stream);

/* Thread-local description of the last non-OK status ("" if none). */
SKV_API const char *shadowkv_last_error(void);

/* SHADOWKV_ABI_VERSION of the loaded library. */
SKV_API int32_t shadowkv_abi_version(void);

/* Number of kernel launches the last successful decode_step / build_cache enqueued
 * (evidence for bench.py's gpu_launches count). */
SKV_API int32_t shadowkv_last_launch_count(void);

/* Optional kernel timing for benchmarks (not needed for correctness).  begin() creates
 * 2*capacity CUDA events; while active, every decode_step records an event pair on its stream
 * around each kernel whose id bit is set in kernel_mask (ids: 0 score, 1 select,
 * 2 fused rebuild+gather+attention, 3 reserved, 4 combine).  end() synchronises on the recorded events, writes
 * the summed milliseconds and launch counts per id into total_ms[5] / counts[5] (nullable) and
 * destroys the events.  Not thread-safe; one profiling session per process. */
SKV_API skv_status shadowkv_profile_begin(int32_t capacity, int32_t kernel_mask);
/* Tuning aid: when dev_buf (device, >= 4*4096*16 uint64) is non-NULL, decode kernels write
 * %globaltimer stamps [0 score | 1 select | 2 sparse-attn | 3 merge][CTA < 4096][event < 16] into it.
 * NULL (the default) disables the stamps. */
SKV_API skv_status shadowkv_trace_buffer(void *dev_buf);
SKV_API skv_status shadowkv_profile_end(double *total_ms, int32_t *counts);

#ifdef __cplusplus
}
#endif
#endif /* SHADOWKV_H */
