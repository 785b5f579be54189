// TMA-fed, warp-specialized tcgen05 GEMM over pre-split bf16 operands.
//
// Producers of GEMM operands (assemble / activation / backward kernels and the
// per-step weight pack) write every fp32 value x as a bf16 pair
// (hi = bf16(x), lo = bf16(x - hi)) into a BfMat. A GEMM operand is a view of a
// BfMat (column block [col0, col0 + cols) x capacity rows) described by TMA
// tensor maps with EXACT logical dims, so TMA zero-fills every K / N pad; rows
// past a runtime count are zeroed by the producers up to the next multiple of
// 64 (the K-chunk), so split-K reductions never read stale rows.
// The kernel computes D = A_hi B_hi + A_hi B_lo + A_lo B_hi (fp32 in TMEM).
#pragma once

#include <vector>

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace tgb {

struct BfMat {
  __nv_bfloat16* hi = nullptr;
  __nv_bfloat16* lo = nullptr;
  int64_t rows = 0;  // capacity rows
  int64_t ld = 0;    // elements per row (multiple of 8)
  bool valid() const { return hi != nullptr; }
};

BfMat bf_alloc(int64_t rows, int64_t cols);
void bf_free(BfMat& m);
// Splits a row-major fp32 matrix into an existing BfMat (rows x cols).
void bf_from_f32(const BfMat& m, const float* src, int64_t rows, int64_t cols, int64_t ld_src, cudaStream_t s);

// Device-side writer (kernels receive BfMat by value; hi == nullptr => skip).
__device__ __forceinline__ void bf_put(const BfMat& m, int64_t r, int64_t c, float v) {
  if (m.hi == nullptr) return;
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  m.hi[r * m.ld + c] = h;
  m.lo[r * m.ld + c] = __float2bfloat16_rn(v - __bfloat162float(h));
}

struct TmaOp {
  CUtensorMap hi;
  CUtensorMap lo;
  int kmajor = 1;  // 1: contiguous along K (rows = M or N), 0: contiguous along M/N (rows = K)
  int box_rows = 0;
};

struct TcProblem {
  TmaOp a, b;
  int M = 0, N = 0, K = 0;     // capacities; N includes a bias column when C2 is set
  const int* M_dev = nullptr;  // runtime M (A K-major rows)
  const int* K_dev = nullptr;  // runtime K (MN-major reductions over rows)
  float* C = nullptr;
  int64_t ldc = 0;
  float* C2 = nullptr;         // when set, output column N-1 goes to C2[m]
  float alpha = 1.0f, beta = 0.0f;
  int splits = 1;
  float* ws = nullptr;         // split-K partials [splits][M][ldw]
  int ldw = 0;                 // partial row stride (0: N); a multiple of 4 enables bulk stores
  int ntile = 0;               // UMMA N per tile (multiple of 16, <= 256)
  // set by tc_group_launch: output tensor map (fp32 [splits][rows][cols], 32 x 32
  // boxes, 128 B swizzle) and the epilogue mode (0 per-lane stores, 1 TMA
  // store, 2 TMA reduce-add for beta = 1)
  CUtensorMap cmap;
  int c_mode = 0;
};

constexpr int kMaxTc = 8;
struct TcGroup {
  TcProblem p[kMaxTc];
  int count = 0;
  // every M_dev / K_dev is final before the launch (written by a kernel at
  // least two launches back in stream order, or across a full dependency):
  // the GEMM reads them before griddepcontrol.wait
  bool sizes_ready = false;
};

// Operand views. A K-major: matrix [M rows x K cols]; MN-major: stored
// [K rows x M cols]. B K-major: stored [N rows x K cols]; MN-major: [K x N].
// (col0 % 8 == 0 so the view base is 16-byte aligned.)
TmaOp tma_view(const BfMat& m, int64_t col0, int64_t cols, int64_t rows, bool kmajor, int box_rows);
// UMMA N per tile: the fewest tiles of width <= cap, balanced (a 272-wide
// problem runs as 2 x 144, not 256 + 16, so no CTA streams a full A tile for
// a sliver of outputs).
inline int tc_ntile(int N, int cap = 256) {
  const int tiles = (N + cap - 1) / cap;
  const int w = (N + tiles - 1) / tiles;
  return static_cast<int>(std::min<int64_t>(cap, (w + 15) / 16 * 16));
}

// GEMM launch trace (bench.py's kernel roofline): while a trace is active on
// the calling thread, every tc_group_launch brackets its tcgen05 kernel with
// CUDA events and records the group's problem shapes (capacities plus the
// device pointers of the runtime row counts).
struct TcTraceEntry {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int count = 0;
  int M[kMaxTc] = {}, N[kMaxTc] = {}, K[kMaxTc] = {}, splits[kMaxTc] = {};
  const int* M_dev[kMaxTc] = {};
  const int* K_dev[kMaxTc] = {};
};
void tc_trace_begin();
std::vector<TcTraceEntry> tc_trace_end();  // caller destroys the events

extern int g_tc_bulk_store;  // 0: per-lane epilogue stores only (A/B switch)

// reduce_stream / ev (optional): the split-K reduction of the group's split
// problems runs on reduce_stream after ev (recorded on s past the GEMM).
void tc_group_launch(const TcGroup& g, cudaStream_t s, cudaStream_t reduce_stream = nullptr,
                     cudaEvent_t ev = nullptr);
// Debug: average microseconds of one launch of an M x N x K K-major problem
// and (optionally) a per-CTA globaltimer trace [2*148 x 8].
void tc_debug_bench(int M, int N, int K, int ntile, int iters, double* us, unsigned long long* trace_out,
                    int* grid_out);

}  // namespace tgb
