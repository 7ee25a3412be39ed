// C ABI of libshadowkv.so (see include/shadowkv.h): argument validation, workspace carving
// and kernel orchestration.  Host-side only; kernels live in build.cu / decode.cu.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdarg>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "shadowkv.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
bool g_trace_on = false;       // tuning: trace buffer installed
int g_trace_calls = 0;

skv_status fail(skv_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

// SKV_DEBUG_SYNC=1 (SURVEY §5 failure detection): after every enqueuing ABI call, synchronise the
// stream and turn an asynchronous kernel fault into this call's SKV_ECUDA.  Skipped while the stream
// is being captured into a CUDA graph (a sync there would invalidate the capture).
skv_status debug_sync(void* stream, const char* call) {
  static const bool on = [] { const char* v = getenv("SKV_DEBUG_SYNC"); return v && v[0] == '1'; }();
  if (!on) return SKV_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) cudaGetLastError();
  if (cs != cudaStreamCaptureStatusNone) return SKV_OK;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SKV_ECUDA, "%s: kernel fault (SKV_DEBUG_SYNC): %s", call, cudaGetErrorString(e));
  return SKV_OK;
}

// The device context shadowkv_init set up for the calling thread's current device.
const skv::DevCtx* need_ctx() {
  const skv::DevCtx* c = skv::current_ctx();
  if (!c) {
    int dev = -1;
    cudaGetDevice(&dev);
    cudaGetLastError();
    fail(SKV_ESTATE, "shadowkv_init(%d) was not called for the current device", dev);
  }
  return c;
}

struct NvtxRange {             // an NVTX range around each ABI call (visible in nsys / ncu --nvtx)
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Validate dims (S:46, S:189, S:245 error classes) and derive n_c, w_eff (R8).
skv_status check_dims(const skv_dims* d, skv::Dims* D) {
  if (!d) return fail(SKV_EINVAL, "dims is NULL");
  if (d->batch < 1) return fail(SKV_EINVAL, "batch must be >= 1 (got %d)", d->batch);
  if (d->n_q_heads < 1 || d->n_kv_heads < 1) return fail(SKV_EINVAL, "head counts must be >= 1");
  if (d->n_q_heads % d->n_kv_heads) return fail(SKV_EINVAL, "n_q_heads %% n_kv_heads != 0 (GQA)");
  const int sq = d->q_len <= 0 ? 1 : d->q_len;
  const int g = d->n_q_heads / d->n_kv_heads * sq;       // query rows per KV head
  if (d->head_dim != 128) return fail(SKV_EUNSUPPORTED, "head_dim must be 128 (got %d)", d->head_dim);
  if (d->chunk != 8) return fail(SKV_EUNSUPPORTED, "chunk must be 8 (got %d)", d->chunk);
  if (g != 1 && g != 2 && g != 4 && g != 8 && g != 16)
    return fail(SKV_EUNSUPPORTED, "GQA group x q_len = %d not in {1,2,4,8,16}", g);
  if (d->rank < 16 || d->rank > 256) return fail(SKV_EINVAL, "rank %d out of range [16, 256]", d->rank);
  if (d->rank % 16) return fail(SKV_EUNSUPPORTED, "rank %d not a multiple of 16", d->rank);
  if (d->window_ctx < 0) return fail(SKV_EINVAL, "window_ctx must be >= 0");
  if (d->ctx_len < d->window_ctx + d->chunk)
    return fail(SKV_EINVAL, "ctx_len %d leaves no chunk outside the window (w=%d, c=%d)", d->ctx_len,
                d->window_ctx, d->chunk);
  if (d->ctx_len >= (1 << 24) - 65536) return fail(SKV_EINVAL, "ctx_len must be < 2^24 - 65536 (fp32 positions)");
  const int n_c = (d->ctx_len - d->window_ctx) / d->chunk;
  const int w_eff = d->ctx_len - n_c * d->chunk;
  if (d->n_outlier < 0 || d->n_outlier >= n_c)
    return fail(SKV_EINVAL, "n_outlier %d must satisfy 0 <= o < n_c = %d", d->n_outlier, n_c);
  if (d->budget < 1 || d->budget > n_c - d->n_outlier)
    return fail(SKV_EINVAL, "budget %d must satisfy 1 <= k <= n_L = %d", d->budget, n_c - d->n_outlier);
  int w_eff_max = w_eff;
  if ((d->ctx_lens == nullptr) != (d->ctx_lens_dev == nullptr))
    return fail(SKV_EINVAL, "ctx_lens and ctx_lens_dev: give both or neither");
  if (d->ctx_lens) {                                     // ragged batch: every request's own grid (R8)
    if (reinterpret_cast<uintptr_t>(d->ctx_lens_dev) & 3u) return fail(SKV_EINVAL, "ctx_lens_dev must be 4-byte aligned");
    w_eff_max = 0;
    const long long need = (long long)d->window_ctx + (long long)d->chunk * (d->n_outlier + d->budget);
    for (int b = 0; b < d->batch; ++b) {
      const int sb = d->ctx_lens[b];
      if (sb > d->ctx_len || sb < need)
        return fail(SKV_EINVAL, "ctx_lens[%d] = %d outside [w + c*(o + k) = %lld, ctx_len = %d]", b, sb, need,
                    d->ctx_len);
      const int ncb = (sb - d->window_ctx) / d->chunk;
      w_eff_max = w_eff_max > sb - ncb * d->chunk ? w_eff_max : sb - ncb * d->chunk;
    }
  }
  if (d->window_cap < w_eff_max || d->window_cap < 1)
    return fail(SKV_EINVAL, "window_cap %d < w_eff %d", d->window_cap, w_eff_max);
  *D = skv::Dims{d->batch, d->n_q_heads * sq, d->n_kv_heads, g, d->head_dim, d->ctx_len, d->rank, d->chunk,
                 d->n_outlier, d->budget, d->window_ctx, d->window_cap, n_c, w_eff_max, 0, nullptr, 0, sq,
                 d->ctx_lens_dev};
  return SKV_OK;
}

skv_status check_rope(const skv_rope* r, int head_dim, skv::Rope* R) {
  if (!r) return fail(SKV_EINVAL, "rope is NULL");
  if (r->rotary_dim < 2 || r->rotary_dim > head_dim || (r->rotary_dim & 1))
    return fail(SKV_EINVAL, "rotary_dim %d must be even and in [2, %d]", r->rotary_dim, head_dim);
  if (!r->inv_freq) return fail(SKV_EINVAL, "rope.inv_freq is NULL");
  if (!r->interleaved && r->rotary_dim != 16 && r->rotary_dim != 32 && r->rotary_dim != 64 && r->rotary_dim != 128)
    return fail(SKV_EUNSUPPORTED, "halves-layout rotary_dim %d: must be 16, 32, 64 or 128 (rotation pairs of a key "
                "row must fall in one thread's column set after the tcgen05 rebuild)", r->rotary_dim);
  *R = skv::Rope{r->inv_freq, r->rotary_dim, r->interleaved ? 1 : 0};
  return SKV_OK;
}

skv_status check_layer(const skv_layer* l, const skv::Dims& D, skv::Layer* Ly) {
  if (!l) return fail(SKV_EINVAL, "layer is NULL");
  struct { const void* p; const char* n; bool need; } ptrs[] = {
      {l->A, "A", true}, {l->B, "B", true}, {l->landmarks, "landmarks", true},
      {l->outlier_ids, "outlier_ids", D.o > 0}, {l->K_out, "K_out", D.o > 0}, {l->V_out, "V_out", D.o > 0},
      {l->K_win, "K_win", true}, {l->V_win, "V_win", true}, {l->V_host, "V_host", true}};
  for (auto& p : ptrs) {
    if (p.need && !p.p) return fail(SKV_EINVAL, "layer.%s is NULL", p.n);
    if (p.p && !aligned16(p.p)) return fail(SKV_EINVAL, "layer.%s is not 16-byte aligned", p.n);
  }
  const int n_vc = (l->vc_values != nullptr) + (l->vc_dir != nullptr) + (l->vc_stats != nullptr) +
                   (l->vc_slots != nullptr);
  if (n_vc != 0 && n_vc != 4)
    return fail(SKV_EINVAL, "layer.vc_values / vc_dir / vc_stats / vc_slots: give all four or none");
  if (n_vc && (!aligned16(l->vc_values) || !aligned16(l->vc_dir) || !aligned16(l->vc_stats) || !aligned16(l->vc_slots)))
    return fail(SKV_EINVAL, "layer.vc_* must be 16-byte aligned");
  const int vc_cap = l->vc_capacity == 0 ? D.k : l->vc_capacity;
  if (n_vc && (vc_cap < D.k || vc_cap > D.n_c || vc_cap > skv::kMaxVcCapacity))
    return fail(SKV_EINVAL, "layer.vc_capacity %d: need budget %d <= C <= min(n_c %d, %d)", (int)l->vc_capacity, D.k,
                D.n_c, skv::kMaxVcCapacity);
  if (l->A_gen && (reinterpret_cast<uintptr_t>(l->A_gen) & 15u)) return fail(SKV_EINVAL, "layer.A_gen must be 16-byte aligned");
  *Ly = skv::Layer{l->A, l->B, l->landmarks, l->outlier_ids, l->K_out, l->V_out, l->K_win, l->V_win, l->V_host,
                   l->A_gen, l->vc_values, reinterpret_cast<unsigned long long*>(l->vc_dir),
                   reinterpret_cast<unsigned long long*>(l->vc_stats),
                   reinterpret_cast<unsigned long long*>(l->vc_slots), n_vc ? vc_cap : 0};
  return SKV_OK;
}

// SKV_SERIALIZE=1 (SURVEY §5 race detection): no programmatic dependent launch between the decode
// kernels, and every sparse-attention unit waits for its values before rebuilding its keys, i.e. the
// overlapped schedule run serially.  Outputs must be bit-identical to the overlapped run (tested).
int serial_mode() {
  const char* v = getenv("SKV_SERIALIZE");
  return v && v[0] == '1';
}

size_t ws_bytes(const skv::Dims& D) {
  return skv::build_ws_bytes(D, nullptr, nullptr);   // build scratch sits after every decode region
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Optional CUDA-event timing of individual kernels inside decode_step (bench.py's roofline).
// Events are created in shadowkv_profile_begin (outside any timed region); decode_step only
// records them on its own stream.
namespace skv {
struct Profiler {
  int capacity = 0, mask = 0;            // mask: bit i -> time kernel id i
  int used = 0;
  cudaEvent_t* ev = nullptr;             // [capacity][2]
  int* kid = nullptr;
  int open_slot[kNumKernelIds];
};
void profile_mark(Profiler* p, int kernel, bool end, cudaStream_t st) {
  if (!(p->mask & (1 << kernel))) return;
  if (!end) {
    if (p->used >= p->capacity) { p->open_slot[kernel] = -1; return; }
    int i = p->used++;
    p->kid[i] = kernel;
    p->open_slot[kernel] = i;
    cudaEventRecord(p->ev[2 * i], st);
  } else if (p->open_slot[kernel] >= 0) {
    cudaEventRecord(p->ev[2 * p->open_slot[kernel] + 1], st);
  }
}
}  // namespace skv

namespace {
skv::Profiler* g_prof = nullptr;
}

extern "C" {

skv_status shadowkv_init(int32_t device) {
  const char* what = "";
  cudaError_t e = skv::init_device(device, &what);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(SKV_ECUDA, "shadowkv_init(%d): %s: %s", device, what, cudaGetErrorString(e)); }
  g_err.clear();
  return SKV_OK;
}

skv_status shadowkv_score_plan(const skv_dims* dims, int32_t n_sm, int32_t* plan) {
  skv::Dims D;
  skv_status st;
  if ((st = check_dims(dims, &D)) != SKV_OK) return st;
  if (n_sm < 1 || !plan) return fail(SKV_EINVAL, "n_sm must be >= 1 and plan non-NULL");
  skv::ScorePlan p{};
  const bool ok = skv::score_tc_plan(D, (D.n_c + skv::kSTile - 1) / skv::kSTile, n_sm, &p);
  plan[0] = p.grid; plan[1] = p.tiles_per_cta; plan[2] = p.heads_per_cta; plan[3] = p.ctas_per_head;
  if (!ok) return fail(SKV_EUNSUPPORTED, "no score grid for these dims: %d tiles / %d KV heads per CTA exceed the "
                       "scorer's limits (a single request of this length needs more KV heads or a shorter context)",
                       p.tiles_per_cta, p.heads_per_cta);
  return SKV_OK;
}

skv_status shadowkv_rope_sincos(const skv_rope* rope, const int32_t* pos, int32_t n, float* sincos, void* stream) {
  skv::Rope R;
  skv_status st;
  if ((st = check_rope(rope, 128, &R)) != SKV_OK) return st;
  if (n < 0 || (n > 0 && (!pos || !sincos))) return fail(SKV_EINVAL, "n >= 0 and non-NULL pos / sincos required");
  cudaError_t e = skv::launch_rope_probe(pos, n, R.inv_freq, R.rot / 2, sincos, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(SKV_ECUDA, "rope probe: %s", cudaGetErrorString(e));
  g_err.clear();
  return SKV_OK;
}

skv_status shadowkv_profile_begin(int32_t capacity, int32_t kernel_mask) {
  if (g_prof) return fail(SKV_ESTATE, "profiling already active");
  if (capacity < 1 || kernel_mask <= 0) return fail(SKV_EINVAL, "capacity and kernel_mask must be positive");
  auto* p = new skv::Profiler();
  p->capacity = capacity; p->mask = kernel_mask;
  p->ev = new cudaEvent_t[2 * (size_t)capacity];
  p->kid = new int[capacity];
  for (int i = 0; i < 2 * capacity; ++i) {
    cudaError_t e = cudaEventCreate(&p->ev[i]);
    if (e != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaEventDestroy(p->ev[j]);
      delete[] p->ev; delete[] p->kid; delete p;
      return fail(SKV_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
    }
  }
  g_prof = p;
  return SKV_OK;
}

skv_status shadowkv_profile_end(double* total_ms, int32_t* counts) {
  if (!g_prof) return fail(SKV_ESTATE, "profiling not active");
  skv::Profiler* p = g_prof;
  g_prof = nullptr;
  for (int k = 0; k < skv::kNumKernelIds; ++k) { if (total_ms) total_ms[k] = 0.0; if (counts) counts[k] = 0; }
  skv_status st = SKV_OK;
  for (int i = 0; i < p->used; ++i) {
    if (cudaEventSynchronize(p->ev[2 * i + 1]) != cudaSuccess) { st = fail(SKV_ECUDA, "event sync failed"); break; }
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p->ev[2 * i], p->ev[2 * i + 1]) == cudaSuccess) {
      if (total_ms) total_ms[p->kid[i]] += ms;
      if (counts) counts[p->kid[i]] += 1;
    }
  }
  for (int i = 0; i < 2 * p->capacity; ++i) cudaEventDestroy(p->ev[i]);
  delete[] p->ev; delete[] p->kid; delete p;
  return st;
}


skv_status shadowkv_trace_buffer(void* dev_buf) {
  g_trace_on = dev_buf != nullptr;
  g_trace_calls = 0;
  cudaError_t e = skv::set_trace_buffer(dev_buf);
  if (e == cudaSuccess) e = skv::set_trace_buffer_tc(dev_buf);
  if (e != cudaSuccess) return fail(SKV_ECUDA, "trace buffer: %s", cudaGetErrorString(e));
  return SKV_OK;
}

const char* shadowkv_last_error(void) { return g_err.c_str(); }
int32_t shadowkv_abi_version(void) { return SHADOWKV_ABI_VERSION; }
int32_t shadowkv_last_launch_count(void) { return g_launches; }

size_t shadowkv_workspace_bytes(const skv_dims* dims) {
  skv::Dims D;
  if (check_dims(dims, &D) != SKV_OK) return 0;
  return ws_bytes(D);
}

skv_status shadowkv_build_cache(const skv_dims* dims, const skv_rope* rope, const skv_layer* layer,
                                const uint16_t* K_rope, void* workspace, void* stream) {
  NvtxRange nv("shadowkv_build_cache");
  skv::Dims D; skv::Rope R; skv::Layer Ly;
  skv_status st;
  if ((st = check_dims(dims, &D)) != SKV_OK) return st;
  if ((st = check_rope(rope, D.d, &R)) != SKV_OK) return st;
  if ((st = check_layer(layer, D, &Ly)) != SKV_OK) return st;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(SKV_EINVAL, "workspace must be non-NULL and 256-byte aligned");
  if (K_rope && !aligned16(K_rope)) return fail(SKV_EINVAL, "K_rope is not 16-byte aligned");
  const skv::DevCtx* ctx = need_ctx();
  if (!ctx) return SKV_ESTATE;
  // V_host must be page-locked and device-mapped at the same address (UVA), P:136 V^CPU
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, Ly.V_host);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(SKV_ECUDA, "cudaPointerGetAttributes(V_host): %s", cudaGetErrorString(e)); }
  if (attr.type != cudaMemoryTypeHost || attr.devicePointer != (void*)Ly.V_host)
    return fail(SKV_ESTATE, "V_host must be page-locked host memory mapped at the same device address");
  skv::BuildWs ws;
  skv::build_ws_bytes(D, &ws, static_cast<char*>(workspace));
  int launches = 0;
  if (Ly.vc_dir) {     // a new context starts with a cold value cache (R26)
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((e = cudaMemsetAsync(Ly.vc_dir, 0, (size_t)D.b * D.hk * D.n_c * 8, s)) != cudaSuccess ||
        (e = cudaMemsetAsync(Ly.vc_stats, 0, (size_t)D.b * D.hk * 4 * 8, s)) != cudaSuccess ||
        (e = cudaMemsetAsync(Ly.vc_slots, 0, (size_t)D.b * D.hk * (Ly.vc_cap + D.k) * 8, s)) != cudaSuccess)
      return fail(SKV_ECUDA, "value-cache reset: %s", cudaGetErrorString(e));
  }
  e = skv::launch_build(D, R, Ly, K_rope, ws, static_cast<cudaStream_t>(stream), &launches, *ctx);
  if (e != cudaSuccess) return fail(SKV_ECUDA, "build launch failed: %s", cudaGetErrorString(e));
  g_launches = launches;
  g_err.clear();
  return debug_sync(stream, "shadowkv_build_cache");
}

// Alg 1 "A, B <- SVD(K)": dims used are batch, n_kv_heads, head_dim, ctx_len, rank.
static skv_status check_factorize_dims(const skv_dims* d, int* D) {
  if (!d) return fail(SKV_EINVAL, "dims is NULL");
  if (d->batch < 1 || d->n_kv_heads < 1 || d->head_dim < 1 || d->ctx_len < 1)
    return fail(SKV_EINVAL, "batch, n_kv_heads, head_dim and ctx_len must be >= 1");
  if (d->head_dim != 128) return fail(SKV_EUNSUPPORTED, "head_dim must be 128 (got %d)", d->head_dim);
  const long long Dl = (long long)d->n_kv_heads * d->head_dim;
  if (Dl > 4096) return fail(SKV_EUNSUPPORTED, "n_kv_heads * head_dim = %lld > 4096", Dl);
  if (d->rank < 16 || d->rank > 256 || d->rank % 16)
    return fail(SKV_EINVAL, "rank %d must be a multiple of 16 in [16, 256]", d->rank);
  if (d->rank > Dl || d->rank > d->ctx_len)
    return fail(SKV_EINVAL, "rank %d exceeds min(ctx_len, n_kv_heads * head_dim)", d->rank);
  *D = (int)Dl;
  return SKV_OK;
}

size_t shadowkv_factorize_workspace_bytes(const skv_dims* dims) {
  int D = 0;
  if (check_factorize_dims(dims, &D) != SKV_OK) return 0;
  return skv::factorize_ws_bytes(D, dims->rank, nullptr, nullptr);
}

skv_status shadowkv_factorize(const skv_dims* dims, const uint16_t* K_pre, uint16_t* A, uint16_t* B, float* sigma,
                              void* workspace, void* stream) {
  int D = 0;
  skv_status st;
  if ((st = check_factorize_dims(dims, &D)) != SKV_OK) return st;
  if (!K_pre || !A || !B) return fail(SKV_EINVAL, "K_pre, A and B must be non-NULL");
  if (!aligned16(K_pre) || !aligned16(A) || !aligned16(B) || (sigma && !aligned16(sigma)))
    return fail(SKV_EINVAL, "K_pre/A/B/sigma must be 16-byte aligned");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(SKV_EINVAL, "workspace must be non-NULL and 256-byte aligned");
  NvtxRange nv("shadowkv_factorize");
  const skv::DevCtx* ctx = need_ctx();
  if (!ctx) return SKV_ESTATE;
  skv::FactorizeWs ws;
  skv::factorize_ws_bytes(D, dims->rank, &ws, static_cast<char*>(workspace));
  int launches = 0;
  skv::FactorizeResult r = skv::launch_factorize(dims->batch, dims->n_kv_heads, dims->head_dim, dims->ctx_len,
                                                 dims->rank, K_pre, A, B, sigma, ws,
                                                 static_cast<cudaStream_t>(stream), &launches, *ctx);
  if (r.err != cudaSuccess)
    return fail(SKV_ECUDA, "factorize (%s%s%d): %s", r.what ? r.what : "?", r.unused ? ", lwork " : "", r.unused,
                cudaGetErrorString(r.err));
  g_launches = launches;
  g_err.clear();
  return debug_sync(stream, "shadowkv_factorize");
}

static skv_status decode_impl(const skv_dims* dims, const skv_rope* rope, const skv_layer* layer,
                              const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                              int32_t step, const int32_t* step_dev, uint16_t* out, int32_t* sel_ids,
                              uint16_t* dbg_keys, void* workspace, void* stream) {
  NvtxRange nv(step_dev ? "shadowkv_decode_step_dev" : "shadowkv_decode_step");
  skv::Dims D; skv::Rope R; skv::Layer Ly;
  skv_status st;
  if ((st = check_dims(dims, &D)) != SKV_OK) return st;
  if (step_dev) {
    if (reinterpret_cast<uintptr_t>(step_dev) & 3u) return fail(SKV_EINVAL, "step_dev must be 4-byte aligned");
    D.step_dev = step_dev;
    D.max_step = step;                                   // step carries max_step for the device variant
  }
  if ((st = check_rope(rope, D.d, &R)) != SKV_OK) return st;
  if ((st = check_layer(layer, D, &Ly)) != SKV_OK) return st;
  if (step < 0) return fail(SKV_EINVAL, "step must be >= 0");
  D.lr_A = Ly.A_gen;                                     // low-rank generated keys (NEXT-4)
  D.lr_B = Ly.A_gen ? Ly.B : nullptr;
  if (D.w_eff + step + D.sq > D.wcap)
    return fail(SKV_EINVAL, "window overflow: w_eff %d + step %d + q_len %d > window_cap %d", D.w_eff, step, D.sq,
                D.wcap);
  if (!q || !k_new || !v_new || !out) return fail(SKV_EINVAL, "q, k_new, v_new and out must be non-NULL");
  if (!aligned16(q) || !aligned16(k_new) || !aligned16(v_new) || !aligned16(out) ||
      (sel_ids && !aligned16(sel_ids)) || (dbg_keys && !aligned16(dbg_keys)))
    return fail(SKV_EINVAL, "q/k_new/v_new/out/sel_ids/dbg_keys must be 16-byte aligned");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(SKV_EINVAL, "workspace must be non-NULL and 256-byte aligned");
  if (g_trace_on) {          // consecutive calls stamp consecutive trace blocks (SKV_TRACE_SLOTS, default 1)
    const char* ns = getenv("SKV_TRACE_SLOTS");
    const int n = ns ? atoi(ns) : 1;
    D.trace_slot = n > 1 ? g_trace_calls++ % n : 0;
  }
  const skv::DevCtx* ctx = need_ctx();
  if (!ctx) return SKV_ESTATE;
  D.serial = serial_mode();
  int launches = 0;
  cudaError_t e = skv::launch_decode(D, R, Ly, q, k_new, v_new, step, out, sel_ids, dbg_keys, static_cast<char*>(workspace),
                                     static_cast<cudaStream_t>(stream), &launches, g_prof, *ctx);
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return fail(SKV_EUNSUPPORTED, "no tcgen05 score grid for these dims (see shadowkv_score_plan)");
  }
  if (e != cudaSuccess) return fail(SKV_ECUDA, "decode launch failed: %s", cudaGetErrorString(e));
  g_launches = launches;
  g_err.clear();
  return debug_sync(stream, step_dev ? "shadowkv_decode_step_dev" : "shadowkv_decode_step");
}

skv_status shadowkv_decode_step(const skv_dims* dims, const skv_rope* rope, const skv_layer* layer,
                                const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                                int32_t step, uint16_t* out, int32_t* sel_ids, uint16_t* dbg_keys,
                                void* workspace, void* stream) {
  return decode_impl(dims, rope, layer, q, k_new, v_new, step, nullptr, out, sel_ids, dbg_keys, workspace, stream);
}

skv_status shadowkv_decode_step_dev(const skv_dims* dims, const skv_rope* rope, const skv_layer* layer,
                                    const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                                    const int32_t* step_dev, int32_t max_step, uint16_t* out, int32_t* sel_ids,
                                    uint16_t* dbg_keys, void* workspace, void* stream) {
  if (!step_dev) return fail(SKV_EINVAL, "step_dev must be non-NULL");
  return decode_impl(dims, rope, layer, q, k_new, v_new, max_step, step_dev, out, sel_ids, dbg_keys, workspace,
                     stream);
}

}  // extern "C"
