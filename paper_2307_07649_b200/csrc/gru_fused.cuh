// Fused GRU freshen on tcgen05 (freshen_memory + gru_update, trainer.hpp:111-124,
// gru.hpp:32-67): one kernel replaces GEMM -> sigmoid -> GEMM -> tanh/blend.
#pragma once

#include <cuda.h>

#include "gemm_tma.cuh"

namespace tgb {

struct GruFusedParams {
  CUtensorMap xg_hi, xg_lo;    // GRU input [U x (gin + 1)]: [mail2 | phi | e | s | 1]
  CUtensorMap wzr_hi, wzr_lo;  // [Wz | bz ; Wr | br]       [2d x (gin + 1)], 64-row boxes (r)
  CUtensorMap wz_hi, wz_lo;    // the same matrix, 32-row boxes (the slice's z rows)
  CUtensorMap whm_hi, whm_lo;  // Wh, mail columns          [d x md], 32-row boxes
  CUtensorMap whs_hi, whs_lo;  // [Wh_s | bh]               [d x (d + 1)], 32-row boxes
  const int* U_dev = nullptr;  // runtime support count
  int cap_U = 0, d = 0, ds = 0, gin = 0, nclu = 1;  // nclu: 32-unit slices per tile (set by the launcher)
  const int32_t* supports = nullptr;
  const float* mem = nullptr;       // read view memory rows [U x d] (s)
  const int32_t* mail_ev = nullptr; // cached mail event per view row (-1: none)
  const float* stat = nullptr;      // static table [N x ds]
  float* gates = nullptr;           // [U x 3d]: a_z, a_r, a_h (pre-activations), for the backward
  float* s_hat = nullptr;           // [U x d]
  BfMat rs, nf;                     // [r * s | 1] and [s_hat | static | 1] operands
  int* flag = nullptr;
};

// The fused kernel serves d + 1 <= 128 (every CTA recomputes all r columns of
// its 128-row tile: 128 TMEM columns).
inline bool gru_fused_supported(int64_t d) { return d >= 1 && d + 1 <= 128; }

// Debug timeline: host == nullptr arms a [cap_ctas x 16] globaltimer buffer;
// otherwise synchronises, copies it out and disarms.
void gru_debug_trace(unsigned long long* host, int cap_ctas, int* n_ctas);

// Tensor maps are built here (cached); the caller fills the rest of p.
void gru_fused_launch(GruFusedParams p, const BfMat& xg, const BfMat& wzr, const BfMat& whm, const BfMat& whs,
                      int64_t md, cudaStream_t s);

}  // namespace tgb
