// Host-side launchers for the ShadowKV kernels (internal to libshadowkv.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace skv {

struct Dims {          // validated, derived sizes
  int b, hq, hk, g, d, s, r, c, o, k, w, wcap;
  int n_c, w_eff;
};

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
};

// workspace carving (256-B aligned regions)
struct BuildWs {
  float* mincos;     // [b][hk][n_c]
  float* negm;       // [b][hk][n_c]  (-m, keys for the outlier top-o)
};
struct DecodeWs {
  float* logits;     // [b][hq][n_c]
  float2* part;      // [b][hq][n_sblk]  softmax partials (max, sumexp)
  float* z;          // [b][hk][n_c]
  int32_t* sel;      // [b][hk][k]
  uint16_t* Kt;      // [b][hk][k*c][d]
  uint16_t* Vt;      // [b][hk][k*c][d]
  float* o_part;     // [b][hq][n_split][d]
  float2* ml_part;   // [b][hq][n_split]
  int n_sblk, n_split;
};

constexpr int kScoreTile = 256;   // chunks per score block
constexpr int kAttnTile = 128;    // tokens per attention split

size_t build_ws_bytes(const Dims& D, BuildWs* ws, char* base);
size_t decode_ws_bytes(const Dims& D, DecodeWs* ws, char* base);

// each returns cudaGetLastError() after its launches and adds to *launches
cudaError_t launch_build(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* K_rope,
                         const BuildWs& ws, cudaStream_t st, int* launches);
cudaError_t launch_decode(const Dims& D, const Rope& R, const Layer& Ly, const uint16_t* q,
                          const uint16_t* k_new, const uint16_t* v_new, int step, uint16_t* out,
                          int32_t* sel_ids, uint16_t* dbg_keys, const DecodeWs& ws, cudaStream_t st,
                          int* launches);

}  // namespace skv
