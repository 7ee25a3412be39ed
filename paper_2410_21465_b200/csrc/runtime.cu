// Per-device runtime context of libshadowkv.so (host side).
//
// Everything the decode / build calls would otherwise create or configure lazily -- the large-smem
// kernel attributes of every template instantiation, the SM count, the sub-batch chains' side
// streams and events, the driver's tensor-map encoder -- is set up once per device by
// shadowkv_init (under a lock; idempotent).  The hot path then only reads this context: it never
// allocates, and a device it was not initialised for is an error (SKV_ESTATE), not a silent
// first-use setup on the wrong device.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

#include "kernels.h"

namespace skv {

namespace {
DevCtx g_ctx[kMaxDevices];
std::atomic<bool> g_ready[kMaxDevices];
std::mutex g_init_mu;
}  // namespace

const DevCtx* current_ctx() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) { cudaGetLastError(); return nullptr; }
  return g_ready[dev].load(std::memory_order_acquire) ? &g_ctx[dev] : nullptr;
}

cudaError_t init_device(int device, const char** what) {
  *what = "";
  if (device < 0 || device >= kMaxDevices) { *what = "device index"; return cudaErrorInvalidDevice; }
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (g_ready[device].load(std::memory_order_acquire)) return cudaSuccess;
  int prev = 0;
  cudaError_t e = cudaGetDevice(&prev);
  if (e) { *what = "cudaGetDevice"; return e; }
  if ((e = cudaSetDevice(device))) { *what = "cudaSetDevice"; return e; }
  DevCtx c;
  c.device = device;
  auto done = [&](cudaError_t err, const char* w) { *what = w; cudaSetDevice(prev); return err; };
  if ((e = cudaDeviceGetAttribute(&c.n_sm, cudaDevAttrMultiProcessorCount, device))) return done(e, "SM count");
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);           // hi = greatest priority (numerically lowest)
  for (int i = 0; i < kMaxSplit; ++i) {
    if ((e = cudaStreamCreateWithPriority(&c.side[i], cudaStreamNonBlocking, hi))) return done(e, "side stream");
    if ((e = cudaEventCreateWithFlags(&c.ev_sel[i], cudaEventDisableTiming))) return done(e, "event");
    if ((e = cudaEventCreateWithFlags(&c.ev_done[i], cudaEventDisableTiming))) return done(e, "event");
  }
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if ((e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q)) || q != cudaDriverEntryPointSuccess)
    return done(e ? e : cudaErrorNotSupported, "cuTensorMapEncodeTiled entry point");
  c.encode_tiled = p;
  if ((e = init_decode_attrs())) return done(e, "decode kernel attributes");
  if ((e = init_score_tc_attrs())) return done(e, "score kernel attributes");
  if ((e = init_build_attrs())) return done(e, "build kernel attributes");
  if ((e = init_factorize_attrs())) return done(e, "factorize kernel attributes");
  g_ctx[device] = c;
  g_ready[device].store(true, std::memory_order_release);
  return done(cudaSuccess, "");
}

// serialises the enqueue of sub-batch chains (they share the device's side streams and events)
std::mutex& chain_mutex(int device) {
  static std::mutex mu[kMaxDevices];
  return mu[device];
}

}  // namespace skv
