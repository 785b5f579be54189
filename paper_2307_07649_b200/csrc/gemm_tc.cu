// Grouped GEMM on the 5th-generation tensor cores (tcgen05 / UMMA, sm_100a).
//
// Same problem interface as gemm_simt.cu (GemmProblem: strided, K-segmented
// fp32 operands, device-side row counts, split-K). Each CTA computes a
// 128 x N_tile (N_tile <= 256) output tile:
//   * all 8 warps gather the fp32 A / B tiles from global (coalesced along the
//     operand's unit-stride direction), split every value into a bf16 pair
//     hi = bf16(x), lo = bf16(x - hi), and store them into shared memory in the
//     canonical K-major SWIZZLE_128B layout (8-row x 128 B swizzle atoms);
//   * one thread issues tcgen05.mma.kind::f16 (bf16 x bf16 -> fp32 in TMEM):
//     D += Ahi*Bhi + Ahi*Blo + Alo*Bhi per 16-deep k-step ("bf16x3": ~2^-17
//     relative per product, i.e. fp32-class accuracy for the 1e-4 parity bound);
//   * two shared-memory stages: the MMAs of stage s run while the warps fill
//     stage s^1; tcgen05.commit -> mbarrier releases a stage;
//   * epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32(w%4).. = rows),
//     alpha/beta/bias, or a split-K partial for the in-order reduction.
#include <mutex>
#include <cuda_bf16.h>

#include "gemm_simt.cuh"

namespace tgb {

namespace {

constexpr int TBM = 128;         // UMMA_M (cta_group::1)
constexpr int TBK = 64;          // k per stage = one 128 B swizzle row of bf16
constexpr int TBN_MAX = 256;     // UMMA_N max
constexpr int TNT = 128;         // epilogue threads (4 warps x 32 TMEM lanes)
constexpr int TNT2 = 256;        // threads per CTA (all produce; warps w, w+4 share lanes)
constexpr int kStages = 2;
constexpr int kATile = TBM * TBK * 2;         // 16 KB per bf16 tile
constexpr int kBTile = TBN_MAX * TBK * 2;     // 32 KB per bf16 tile
constexpr int kStageBytes = 2 * kATile + 2 * kBTile;  // hi + lo for A and B
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 64;

struct TcParams {
  GemmProblem p[kMaxGroup];
  int tiles_m[kMaxGroup], tiles_n[kMaxGroup];
  int count;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Canonical K-major SW128 offset of element (row, k) in a [rows x 64] bf16 tile.
__device__ __forceinline__ uint32_t sw128_off(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ int seg_of(const Operand& o, int k) {
  int s = 0;
#pragma unroll
  for (int x = 1; x < 4; ++x)
    if (x < o.nseg && k >= o.kb[x]) s = x;
  return s;
}

// A(m, k) and B(k, n) through the operand descriptors (see gemm_simt.cuh).
__device__ __forceinline__ float ld_a(const Operand& o, int64_t m, int k) {
  const int s = seg_of(o, k);
  const Seg& sg = o.seg[s];
  return sg.p[m * sg.rs + static_cast<int64_t>(k - o.kb[s]) * sg.cs];
}
__device__ __forceinline__ float ld_b(const Operand& o, int k, int64_t n) {
  const int s = seg_of(o, k);
  const Seg& sg = o.seg[s];
  return sg.p[static_cast<int64_t>(k - o.kb[s]) * sg.rs + n * sg.cs];
}

__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(v[2 * q]);
    const __nv_bfloat16 h1 = __float2bfloat16_rn(v[2 * q + 1]);
    const __nv_bfloat16 l0 = __float2bfloat16_rn(v[2 * q] - __bfloat162float(h0));
    const __nv_bfloat16 l1 = __float2bfloat16_rn(v[2 * q + 1] - __bfloat162float(h1));
    h[q] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) |
           (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
    l[q] = static_cast<uint32_t>(__bfloat16_as_ushort(l0)) |
           (static_cast<uint32_t>(__bfloat16_as_ushort(l1)) << 16);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Fills one operand's [rows_tile x 64] hi/lo tiles. Work unit = (row, 8-k
// chunk) -> one 16-byte swizzled store per tile. All loads of a thread's units
// are issued before any conversion (memory-level parallelism).
//  k_fast (unit stride along k): 8 consecutive lanes cover one row's 64 k
//    (two 128-bit loads per unit when the operand is aligned, single-segment);
//  row-fast (unit stride along rows): consecutive lanes take consecutive rows.
template <bool IS_A, int MAXU>
__device__ __forceinline__ void fill_tile(const Operand& o, int r0, int rows_valid, int rows_tile,
                                          int k0, int K, uint8_t* hi_tile, uint8_t* lo_tile) {
  const Seg& s0 = o.seg[0];
  const int64_t kstride = IS_A ? s0.cs : s0.rs;
  const int64_t rstride = IS_A ? s0.rs : s0.cs;
  const bool k_fast = kstride == 1;
  const int units = rows_tile * 8;
  float v[MAXU][8];
  if (k_fast) {
    const bool vec = o.nseg == 1 && (rstride & 3) == 0 && ((reinterpret_cast<uintptr_t>(s0.p) & 15) == 0);
#pragma unroll
    for (int i = 0; i < MAXU; ++i) {
      const int u = threadIdx.x + i * TNT2;
      const int r = u >> 3, c = u & 7;
      const int kb = k0 + c * 8;
      const bool rok = u < units && r < rows_valid;
      if (vec && rok && kb + 8 <= K) {
        const float4* src = reinterpret_cast<const float4*>(s0.p + static_cast<int64_t>(r0 + r) * rstride + kb);
        const float4 x0 = __ldg(src), x1 = __ldg(src + 1);
        v[i][0] = x0.x; v[i][1] = x0.y; v[i][2] = x0.z; v[i][3] = x0.w;
        v[i][4] = x1.x; v[i][5] = x1.y; v[i][6] = x1.z; v[i][7] = x1.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int k = kb + q;
          v[i][q] = (rok && k < K) ? (IS_A ? ld_a(o, r0 + r, k) : ld_b(o, k, r0 + r)) : 0.0f;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < MAXU; ++i) {
      const int u = threadIdx.x + i * TNT2;
      if (u < units) {
        uint4 h, l;
        split8(v[i], h, l);
        const uint32_t off = sw128_off(u >> 3, u & 7);
        *reinterpret_cast<uint4*>(hi_tile + off) = h;
        *reinterpret_cast<uint4*>(lo_tile + off) = l;
      }
    }
  } else {
    const bool single = o.nseg == 1;
#pragma unroll
    for (int i = 0; i < MAXU; ++i) {
      const int u = threadIdx.x + i * TNT2;
      const int r = u % rows_tile, c = u / rows_tile;
      const int kb = k0 + c * 8;
      const bool rok = u < units && r < rows_valid;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = kb + q;
        if (single)
          v[i][q] = (rok && k < K) ? s0.p[static_cast<int64_t>(r0 + r) * rstride + static_cast<int64_t>(k) * kstride] : 0.0f;
        else
          v[i][q] = (rok && k < K) ? (IS_A ? ld_a(o, r0 + r, k) : ld_b(o, k, r0 + r)) : 0.0f;
      }
    }
#pragma unroll
    for (int i = 0; i < MAXU; ++i) {
      const int u = threadIdx.x + i * TNT2;
      if (u < units) {
        uint4 h, l;
        split8(v[i], h, l);
        const uint32_t off = sw128_off(u % rows_tile, u / rows_tile);
        *reinterpret_cast<uint4*>(hi_tile + off) = h;
        *reinterpret_cast<uint4*>(lo_tile + off) = l;
      }
    }
  }
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B (8-row
// group stride), LBO = 1 (unused for swizzled K-major), version 1 (sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor: bf16 x bf16 -> f32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t make_idesc(int n) {
  uint32_t d = 0;
  d |= 1u << 4;                                  // c_format F32
  d |= 1u << 7;                                  // a_format BF16
  d |= 1u << 10;                                 // b_format BF16
  d |= static_cast<uint32_t>(n >> 3) << 17;      // N >> 3
  d |= static_cast<uint32_t>(TBM >> 4) << 24;    // M >> 4
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(TNT2, 1) gemm_tc_kernel(const __grid_constant__ TcParams gp) {
  const int pi = blockIdx.y;
  if (pi >= gp.count) return;
  const GemmProblem& P = gp.p[pi];
  const int tm = gp.tiles_m[pi], tn = gp.tiles_n[pi];
  const int tile = blockIdx.x;
  if (tile >= tm * tn * P.splits) return;
  const int split = tile / (tm * tn);
  const int t2 = tile % (tm * tn);
  const int m0 = (t2 / tn) * TBM;
  const int n0 = (t2 % tn) * TBN_MAX;
  const int M = P.M_dev ? min(P.M, *P.M_dev) : P.M;
  if (m0 >= M && P.splits == 1) return;
  const int N = P.N;
  const int Kcap = P.K;
  const int K = P.K_dev ? min(Kcap, *P.K_dev) : Kcap;
  const int kper = ((Kcap + P.splits - 1) / P.splits + TBK - 1) / TBK * TBK;
  const int kbeg = split * kper;
  const int kend = min(K, kbeg + kper);
  const int nvalid = min(TBN_MAX, N - n0);
  const int ntile = (nvalid + 15) / 16 * 16;
  const int mvalid = min(TBM, M - m0);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TBN_MAX));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int nk = (kend > kbeg && m0 < M) ? (kend - kbeg + TBK - 1) / TBK : 0;
  const uint32_t idesc = make_idesc(ntile);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    if (kc >= kStages) mbar_wait(bars + s, ((kc >> 1) - 1) & 1);
    uint8_t* st = smem + s * kStageBytes;
    uint8_t* a_hi = st;
    uint8_t* a_lo = st + kATile;
    uint8_t* b_hi = st + 2 * kATile;
    uint8_t* b_lo = st + 2 * kATile + kBTile;
    const int k0 = kbeg + kc * TBK;
    fill_tile<true, TBM * 8 / TNT2>(P.a, m0, mvalid, TBM, k0, kend, a_hi, a_lo);
    fill_tile<false, TBN_MAX * 8 / TNT2>(P.b, n0, nvalid, ntile, k0, kend, b_hi, b_lo);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo);
      const uint32_t sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
#pragma unroll
      for (int ks = 0; ks < TBK / 16; ++ks) {
        const uint32_t adv = ks * 32;  // 16 bf16 = 32 B along k inside the swizzle row
        const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
        mma_bf16(tmem, make_desc(sa_hi + adv), make_desc(sb_hi + adv), idesc, acc0);
        mma_bf16(tmem, make_desc(sa_hi + adv), make_desc(sb_lo + adv), idesc, 1u);
        mma_bf16(tmem, make_desc(sa_lo + adv), make_desc(sb_hi + adv), idesc, 1u);
      }
      mma_commit(bars + s);
    }
  }
  if (nk > 0) mbar_wait(bars + ((nk - 1) & 1), ((nk - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // Epilogue: warp w reads TMEM lanes [32 (w % 4), +32) = tile rows; warps w
  // and w + 4 take alternating 16-column chunks.
  const int quarter = warp & 3;
  const int row = quarter * 32 + lane;
  const int m = m0 + row;
  for (int c0 = (warp >> 2) * 16; c0 < ntile; c0 += 32) {
    uint32_t v[16];
    if (nk > 0) {
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0u;
    }
    if (P.splits > 1) {
      if (m < P.M) {
        float* ws = P.ws + static_cast<int64_t>(split) * P.M * P.N + static_cast<int64_t>(m) * N;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int n = n0 + c0 + q;
          if (c0 + q < nvalid) ws[n] = (m < M) ? __uint_as_float(v[q]) : 0.0f;
        }
      }
    } else if (m < M) {
      float* crow = P.C + static_cast<int64_t>(m) * P.ldc;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int n = n0 + c0 + q;
        if (c0 + q < nvalid) {
          float val = P.alpha * __uint_as_float(v[q]);
          if (P.beta != 0.0f) val += P.beta * crow[n];
          if (P.bias) val += P.bias[n];
          crow[n] = val;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TBN_MAX));
}

}  // namespace

void splitk_reduce_launch(const GemmGroup& g, cudaStream_t s);

void gemm_tc_prepare() {
  // the attribute is per device: set it once on every device this process uses
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  TGB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!(done >> dev & 1ull)) {
    TGB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    done |= 1ull << dev;
  }
}

void gemm_group_launch_tc(const GemmGroup& g, cudaStream_t s) {
  if (g.count == 0) return;
  gemm_tc_prepare();
  TcParams gp{};
  gp.count = g.count;
  int max_tiles = 0;
  bool any_split = false;
  for (int i = 0; i < g.count; ++i) {
    gp.p[i] = g.p[i];
    gp.tiles_m[i] = static_cast<int>(ceil_div(g.p[i].M, TBM));
    gp.tiles_n[i] = static_cast<int>(ceil_div(g.p[i].N, TBN_MAX));
    const int t = gp.tiles_m[i] * gp.tiles_n[i] * g.p[i].splits;
    max_tiles = t > max_tiles ? t : max_tiles;
    any_split |= g.p[i].splits > 1;
  }
  if (max_tiles == 0) return;
  gemm_tc_kernel<<<dim3(max_tiles, g.count), TNT2, kSmemBytes, s>>>(gp);
  TGB_CUDA(cudaGetLastError());
  if (any_split) splitk_reduce_launch(g, s);
}

}  // namespace tgb
