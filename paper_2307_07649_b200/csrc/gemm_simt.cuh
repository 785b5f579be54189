// Grouped fp32 SIMT GEMM with K-segmented, arbitrarily strided operands.
//
// This is the exact-fp32 path used for parity with the f64 reference
// (tolerance 1e-4 relative): each output element is an in-order fp32 FMA
// chain over k (deterministic), and long reductions (weight gradients, whose
// K is the number of gathered rows) use a fixed split-K partition followed by
// an in-order reduction of the partials, so results are bitwise reproducible.
//
// C[M x N] = alpha * A[M x K] . B[K x N] + beta * C + bias[n]
// A(m, k) = a.seg[s].p[m * rs + (k - kb[s]) * cs] for the segment s holding k.
#pragma once

#include "common.cuh"

namespace tgb {

struct Seg {
  const float* p = nullptr;
  int64_t rs = 0, cs = 0;
};

struct Operand {
  Seg seg[4];
  int kb[5] = {0, 0, 0, 0, 0};  // segment s covers [kb[s], kb[s+1])
  int nseg = 0;
};

struct GemmProblem {
  int M = 0, N = 0, K = 0;
  const int* M_dev = nullptr;  // runtime row count (<= M), device-resident
  const int* K_dev = nullptr;  // runtime reduction length (<= K), device-resident
  Operand a, b;
  float* C = nullptr;
  int64_t ldc = 0;
  float alpha = 1.0f, beta = 0.0f;
  const float* bias = nullptr;
  int splits = 1;
  float* ws = nullptr;  // splits > 1: partials [splits][M][N]
};

constexpr int kMaxGroup = 8;

struct GemmGroup {
  GemmProblem p[kMaxGroup];
  int count = 0;
};

// Builders ---------------------------------------------------------------
inline Operand op_dense(const float* p, int64_t rs, int64_t cs, int K) {
  Operand o;
  o.seg[0] = {p, rs, cs};
  o.kb[0] = 0;
  o.kb[1] = K;
  o.nseg = 1;
  return o;
}

// Appends a K-segment of length len.
inline void op_append(Operand& o, const float* p, int64_t rs, int64_t cs, int len) {
  const int s = o.nseg;
  o.seg[s] = {p, rs, cs};
  o.kb[s + 1] = o.kb[s] + len;
  o.nseg = s + 1;
}

// A row-major [M x K] (lda), i.e. "x" in y = x W^T.
inline Operand A_rows(const float* p, int64_t lda, int K) { return op_dense(p, lda, 1, K); }
// A = Y^T where Y is row-major [K x M] (ldy): A(m, k) = Y[k, m].
inline Operand A_trans(const float* p, int64_t ldy, int K) { return op_dense(p, 1, ldy, K); }
// B = W^T where W is row-major [N x K] (ldw): B(k, n) = W[n, k].
inline Operand B_wT(const float* p, int64_t ldw, int K) { return op_dense(p, 1, ldw, K); }
// B = W where W is row-major [K x N] (ldw).
inline Operand B_w(const float* p, int64_t ldw, int K) { return op_dense(p, ldw, 1, K); }

// Process-wide GEMM engine for the training step:
//  kGemmTma (default): tcgen05 bf16x3 fed by TMA from pre-split bf16 operands
//                      (gemm_tma.cu) -- fp32-class accuracy;
//  kGemmSimt:          fp32 FMA on CUDA cores (gemm_simt.cu) -- exact fp32 path;
//  kGemmGather:        tcgen05 bf16x3 that gathers + splits fp32 operands inside
//                      the GEMM (gemm_tc.cu) -- no pre-split operands needed.
enum GemmImpl { kGemmSimt = 0, kGemmTma = 1, kGemmGather = 2 };
constexpr int kGemmTensor = kGemmGather;  // debug-hook name of the gather engine
void set_gemm_impl(int impl);
int gemm_impl();
void gemm_group_launch(const GemmGroup& g, cudaStream_t s);
void gemm_group_launch_simt(const GemmGroup& g, cudaStream_t s);
void gemm_group_launch_tc(const GemmGroup& g, cudaStream_t s);
void splitk_reduce_launch(const GemmGroup& g, cudaStream_t s);
void gemm_tc_prepare();
void tc_gemm_prepare();
// One-time kernel attributes (call before any stream capture).
inline void gemm_kernels_prepare() {
  gemm_tc_prepare();
  tc_gemm_prepare();
}

}  // namespace tgb
