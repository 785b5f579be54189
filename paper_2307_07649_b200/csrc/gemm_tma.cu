// TMA-fed, warp-specialized, persistent tcgen05 GEMM (see gemm_tma.cuh).
//
// CTA = 10 warps: warp 0 issues TMA loads (one elected lane), warp 1 owns the
// TMEM allocation and issues tcgen05.mma (one elected lane), warps 2-9 run the
// epilogue (warp w reads TMEM lanes 32 (w % 4) .. +32, alternate 32-column chunks). Each CTA walks the
// flattened tiles of all problems of the group round-robin. Two shared-memory
// stages of {A_hi, A_lo, B_hi, B_lo} (128 B swizzled, K-major or MN-major per
// operand) form a full/empty mbarrier ring that runs across tile boundaries;
// two TMEM accumulators (tfull/tempty barriers) let the epilogue of tile t
// overlap the MMAs of tile t+1.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>

#include "gemm_tma.cuh"
#include "tc_ptx.cuh"

namespace tgb {

namespace {

constexpr int kBM = 128, kBK = 64, kStMax = 6;
constexpr int kEpiWarps = 8;                      // two warps per TMEM lane quarter
constexpr int kThreads = 64 + 32 * kEpiWarps;     // producer, MMA, epilogue
constexpr int kATileB = kBM * kBK * 2;   // 16 KB (one of hi / lo)
constexpr int kEpiStageB = kEpiWarps * 32 * 32 * 4;  // static epilogue staging tiles
constexpr int kSmemMax = 232448 - kEpiStageB - 1024;  // opt-in dynamic maximum per CTA (static tile is 1 KB aligned)

// Shared-memory / TMEM geometry is sized by the group's widest N tile, so
// narrow-tile groups fit several CTAs per SM.
struct TcParams {
  TcProblem p[kMaxTc];
  int tiles_m[kMaxTc], tiles_n[kMaxTc];
  int tile_base[kMaxTc + 1];  // flattened tile index of each problem's first tile
  int count;
  int b_tile_bytes;  // per hi / lo B tile: roundup64(max ntile) * 128
  int stage_bytes;
  int tmem_cols;     // power of two >= max(32, max ntile)
  int stages;        // shared-memory ring depth (2..kStMax), as deep as the CTA budget allows
  int sizes_early;   // runtime sizes final before launch: read them before griddepcontrol.wait
};

// Optional per-CTA timeline (debug benchmark only): 8 globaltimer stamps per CTA.
__device__ unsigned long long* g_tc_trace = nullptr;
__device__ int g_tc_epi_mode = 0;  // debug: 1 skips global stores, 2 skips TMEM loads
__device__ __forceinline__ void trace(int slot) {
  unsigned long long* t = g_tc_trace;
  if (t) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    t[blockIdx.x * 16 + slot] = v;
  }
}

// Tile geometry of flattened tile index t (identical in every role).
struct TileInfo {
  int pi, m0, n0, split, kbeg, nk, M;
};

// rt_m / rt_k: each problem's runtime M / K (shared memory, read once per CTA)
__device__ __forceinline__ bool tile_info(const TcParams& gp, const int* rt_m, const int* rt_k, int t, TileInfo& ti) {
  int pi = 0;
  while (pi + 1 < gp.count && t >= gp.tile_base[pi + 1]) ++pi;
  const TcProblem& P = gp.p[pi];
  const int local = t - gp.tile_base[pi];
  const int tm = gp.tiles_m[pi], tn = gp.tiles_n[pi];
  ti.pi = pi;
  ti.split = local / (tm * tn);
  const int t2 = local % (tm * tn);
  ti.m0 = (t2 / tn) * kBM;
  ti.n0 = (t2 % tn) * P.ntile;
  ti.M = rt_m[pi];
  if (ti.m0 >= ti.M && P.splits == 1) return false;  // beyond the runtime rows: no work, no output
  const int Kcap = P.K;
  const int K = rt_k[pi];
  // split-K partition of the RUNTIME reduction length (64-row chunks): the
  // splits stay balanced however loose the capacity is; still a fixed
  // function of the data, so the reduction order is deterministic.
  const int kper = ((K + P.splits - 1) / P.splits + kBK - 1) / kBK * kBK;
  ti.kbeg = ti.split * kper;
  const int kend = min(K, ti.kbeg + kper);
  ti.nk = (kend > ti.kbeg && ti.m0 < ti.M) ? (kend - ti.kbeg + kBK - 1) / kBK : 0;
  return true;
}

// Persistent CTA: static round-robin over the flattened tiles of the group.
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const __grid_constant__ TcParams gp) {
  if (threadIdx.x == 0) trace(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kStageB = gp.stage_bytes, kBTileB = gp.b_tile_bytes;
  const uint32_t kSt = static_cast<uint32_t>(gp.stages);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kStageB);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;   // [2] accumulator ready for the epilogue
  uint64_t* tempty = tfull + 2;    // [2] accumulator drained by the epilogue
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ __align__(1024) float epi_stage[kEpiWarps * 32 * 32];  // epilogue staging (128 B swizzle)
  __shared__ int rt_m[kMaxTc], rt_k[kMaxTc];  // runtime M / K per problem
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = gp.tile_base[gp.count];
  auto load_sizes = [&]() {
    if (threadIdx.x < gp.count) {
      const TcProblem& Q = gp.p[threadIdx.x];
      rt_m[threadIdx.x] = Q.M_dev ? min(Q.M, *Q.M_dev) : Q.M;
      rt_k[threadIdx.x] = Q.K_dev ? min(Q.K, *Q.K_dev) : Q.K;
    }
  };
  // sizes produced well before this launch (the plan's counts) are read
  // before griddepcontrol.wait: their load latency overlaps the predecessor
  if (gp.sizes_early) load_sizes();

  // Prologue independent of the predecessor's output (it overlaps its tail
  // under programmatic dependent launch): descriptor prefetch, barriers, TMEM.
  if (warp == 0 && lane < gp.count) {
    const TcProblem& Q = gp.p[lane];
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&Q.a.hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&Q.a.lo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&Q.b.hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&Q.b.lo)) : "memory");
  }
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kSt; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, kEpiWarps);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(gp.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int acc_cols = gp.tmem_cols / 2;
  pdl_wait();  // operands (and, unless sizes_early, runtime sizes) come from the predecessor
  pdl_trigger();
  if (!gp.sizes_early) {
    load_sizes();
    __syncthreads();
  }
  if (threadIdx.x == 0) trace(1);

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        TileInfo ti;
        if (!tile_info(gp, rt_m, rt_k, t, ti)) continue;
        const TcProblem& P = gp.p[ti.pi];
        const bool a_k = P.a.kmajor != 0, b_k = P.b.kmajor != 0;
        const int b_boxes = b_k ? 1 : (P.ntile + 63) / 64;
        const uint32_t a_bytes = a_k ? static_cast<uint32_t>(P.a.box_rows) * 128u : 8192u * 2u;
        const uint32_t b_bytes = b_k ? static_cast<uint32_t>(P.b.box_rows) * 128u : 8192u * static_cast<uint32_t>(b_boxes);
        const uint32_t stage_tx = 2u * (a_bytes + b_bytes);
        for (int kc = 0; kc < ti.nk; ++kc, ++it) {
          const uint32_t s = it % kSt;
          if (it >= kSt) mbar_wait(empty + s, ((it / kSt) - 1) & 1);
          uint8_t* st = smem + s * kStageB;
          if (it == 0) trace(7);
          mbar_expect_tx(full + s, stage_tx);
          const int k0 = ti.kbeg + kc * kBK;
          for (int h = 0; h < 2; ++h) {
            const CUtensorMap* am = h ? &P.a.lo : &P.a.hi;
            const CUtensorMap* bm = h ? &P.b.lo : &P.b.hi;
            uint8_t* ad = st + h * kATileB;
            uint8_t* bd = st + 2 * kATileB + h * kBTileB;
            if (a_k) {
              tma_2d(ad, am, k0, ti.m0, full + s);
            } else {
              tma_2d(ad, am, ti.m0, k0, full + s);
              tma_2d(ad + 8192, am, ti.m0 + 64, k0, full + s);
            }
            if (b_k) {
              tma_2d(bd, bm, k0, ti.n0, full + s);
            } else {
              for (int j = 0; j < b_boxes; ++j) tma_2d(bd + j * 8192, bm, ti.n0 + 64 * j, k0, full + s);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        TileInfo ti;
        if (!tile_info(gp, rt_m, rt_k, t, ti)) continue;
        const TcProblem& P = gp.p[ti.pi];
        const bool a_k = P.a.kmajor != 0, b_k = P.b.kmajor != 0;
        const uint32_t acc = lt & 1;
        if (lt >= 2) mbar_wait(tempty + acc, ((lt >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dtm = tmem + acc * static_cast<uint32_t>(acc_cols);
        const uint32_t id = idesc(P.ntile, a_k, b_k);
        for (int kc = 0; kc < ti.nk; ++kc, ++it) {
          const uint32_t s = it % kSt;
          mbar_wait(full + s, (it / kSt) & 1);
          if (it == 0) trace(2);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint8_t* st = smem + s * kStageB;
          const uint32_t ahi = su32(st), alo = su32(st + kATileB);
          const uint32_t bhi = su32(st + 2 * kATileB), blo = su32(st + 2 * kATileB + kBTileB);
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {
            const uint32_t aoff = a_k ? ks * 32u : ks * 2048u;
            const uint32_t boff = b_k ? ks * 32u : ks * 2048u;
            const uint32_t accf = (kc > 0 || ks > 0) ? 1u : 0u;
            umma(dtm, sdesc(ahi + aoff, a_k), sdesc(bhi + boff, b_k), id, accf);
            umma(dtm, sdesc(ahi + aoff, a_k), sdesc(blo + boff, b_k), id, 1u);
            umma(dtm, sdesc(alo + aoff, a_k), sdesc(bhi + boff, b_k), id, 1u);
          }
          umma_commit(empty + s);
        }
        if (ti.nk > 0)
          umma_commit(tfull + acc);
        else
          mbar_arrive(tfull + acc);
        trace(3);
        ++lt;
      }
    }
  } else {
    // epilogue warps 2..9: warp w reads TMEM lanes 32 (w % 4) .. + 32
    const int quarter = warp & 3;
    const int ehalf = (warp - 2) >> 2;  // the two warps of a quarter take alternate 32-column chunks
    const int epi_mode = g_tc_epi_mode;
    float* stg = epi_stage + (warp - 2) * (32 * 32);
    const uint32_t stg_s = su32(stg);
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      TileInfo ti;
      if (!tile_info(gp, rt_m, rt_k, t, ti)) continue;
      const TcProblem& P = gp.p[ti.pi];
      const uint32_t acc = lt & 1;
      mbar_wait(tfull + acc, (lt >> 1) & 1);
      if (warp == 2 && lane == 0) trace(4);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // problem fields in registers (P lives in parameter space, indexed)
      const int N = P.N;
      const int ntile = P.ntile;
      const int nvalid = min(ntile, N - ti.n0);
      const int n0 = ti.n0;
      const int splits = P.splits;
      const int PM = P.M;
      const float alpha = P.alpha, beta = P.beta;
      float* const Cp = P.C;
      float* const C2p = P.C2;
      float* const wsp = P.ws;
      const int64_t ldcp = P.ldc;
      const int ldw = P.ldw > 0 ? P.ldw : N;
      const int cmode = epi_mode == 0 ? P.c_mode : 0;
      const CUtensorMap* cmap = &P.cmap;
      // TMEM -> registers (thread = row) -> 128 B-swizzled shared tile (alpha
      // applied, rows past the runtime count zeroed) -> one TMA tensor store
      // (or reduce-add for beta = 1) per 32 x 32 chunk; a per-lane store path
      // remains for unaligned outputs and partial row quarters.
      const int mb = ti.m0 + quarter * 32;  // first row of this warp
      const int row = mb + lane;
      const bool live = row < ti.M;
      const int npart = splits > 1 ? ldw : static_cast<int>(ldcp);
      float* const vbase = splits > 1 ? wsp + static_cast<int64_t>(ti.split) * PM * ldw : Cp;
      const int rmax = splits > 1 ? PM : ti.M;  // rows to write (zeros past ti.M for partials)
      const int ncols = (C2p && splits == 1) ? N - 1 : N;  // columns of C (map extent)
      const bool rows_tma = mb + 32 <= ti.M || ti.M >= PM;  // else partial quarter: per-lane path
      const bool vec_ok = epi_mode != 1 && (npart & 3) == 0 && (reinterpret_cast<uintptr_t>(vbase) & 15) == 0 &&
                          beta == 0.0f;
      for (int c0 = 32 * ehalf; c0 < ntile; c0 += 64) {
        const int halves = min(2, (ntile - c0) / 16);
        uint32_t v[32];
        if (ti.nk > 0 && epi_mode != 2) {
          const uint32_t ta = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                              acc * static_cast<uint32_t>(acc_cols) + static_cast<uint32_t>(c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                "=r"(v[14]), "=r"(v[15])
              : "r"(ta));
          if (halves == 2) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
                  "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(ta + 16u));
          } else {
#pragma unroll
            for (int q = 16; q < 32; ++q) v[q] = 0u;
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = 0u;
        }
        // the previous chunk's bulk store must have read the staging tile
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o;
          o.x = live ? alpha * __uint_as_float(v[4 * j + 0]) : 0.0f;
          o.y = live ? alpha * __uint_as_float(v[4 * j + 1]) : 0.0f;
          o.z = live ? alpha * __uint_as_float(v[4 * j + 2]) : 0.0f;
          o.w = live ? alpha * __uint_as_float(v[4 * j + 3]) : 0.0f;
          *reinterpret_cast<float4*>(stg + lane * 32 + ((j ^ (lane & 7)) << 2)) = o;
        }
        __syncwarp();
        if (warp == 2 && lane == 0 && c0 < 96) trace(8 + 2 * (c0 / 32));
        // a 16-wide last chunk may only use the bulk store if nothing of a
        // neighbouring tile lies in its upper 16 columns (the map clips at ncols)
        if (cmode != 0 && rows_tma && (halves == 2 || n0 + c0 + 16 >= ncols)) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int cx = n0 + c0, cy = mb, cz = splits > 1 ? ti.split : 0;
            if (cmode == 2)
              asm volatile(
                  "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(cmap)),
                  "r"(stg_s), "r"(cx), "r"(cy), "r"(cz)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(cmap)),
                  "r"(stg_s), "r"(cx), "r"(cy), "r"(cz)
                  : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          if (C2p && splits == 1 && n0 + c0 <= N - 1 && N - 1 < n0 + c0 + 16 * halves && live) {
            const int cc = N - 1 - n0 - c0;  // the bias column goes to C2 (beta == 0 here)
            C2p[row] = stg[lane * 32 + (((cc >> 2) ^ (lane & 7)) << 2) + (cc & 3)];
          }
          if (warp == 2 && lane == 0 && c0 < 96) trace(9 + 2 * (c0 / 32));
          continue;
        }
        if (vec_ok && halves == 2 && c0 + 32 <= nvalid && ((n0 + c0) & 3) == 0 && !(C2p && n0 + c0 + 32 > N - 1)) {
          const int rr = lane >> 3, ch = lane & 7, cc = ch * 4;
          float* dst0 = vbase + static_cast<int64_t>(mb + rr) * npart + n0 + c0 + cc;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int r = 4 * k + rr;
            const float4 o = *reinterpret_cast<const float4*>(stg + r * 32 + ((ch ^ (r & 7)) << 2));
            if (mb + r < rmax) *reinterpret_cast<float4*>(dst0 + static_cast<int64_t>(4 * k) * npart) = o;
          }
          if (warp == 2 && lane == 0 && c0 < 96) trace(9 + 2 * (c0 / 32));
          __syncwarp();
          continue;
        }
        const int col = c0 + lane;                 // this lane's column in the tile
        const bool col_ok = lane < 16 * halves && col < nvalid && epi_mode != 1;
        const int n = n0 + col;
        const int sw = lane >> 2, sl = lane & 3;   // swizzled column read: conflict-free per row
        if (splits > 1) {
          const int rows = min(32, PM - mb);
          float* wrow = wsp + (static_cast<int64_t>(ti.split) * PM + mb) * ldw + n;
          for (int r0 = 0; r0 < rows; r0 += 8) {
            float val[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int r = r0 + k;
              val[k] = stg[r * 32 + ((sw ^ (r & 7)) << 2) + sl];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (r0 + k < rows && col_ok) wrow[static_cast<int64_t>(r0 + k) * ldw] = val[k];
          }
        } else {
          const bool to_c2 = C2p && n == N - 1;
          const int rows = min(32, ti.M - mb);
          const int64_t ldc = ldcp;
          float* crow = Cp + static_cast<int64_t>(mb) * ldc + n;
          for (int r0 = 0; r0 < rows; r0 += 8) {
            float val[8], prev[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int r = r0 + k;
              val[k] = stg[r * 32 + ((sw ^ (r & 7)) << 2) + sl];
              prev[k] = 0.0f;
            }
            if (beta != 0.0f) {
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (r0 + k < rows && col_ok) prev[k] = to_c2 ? C2p[mb + r0 + k] : crow[(r0 + k) * ldc];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (r0 + k < rows && col_ok) {
                const float x = val[k] + beta * prev[k];
                if (to_c2) C2p[mb + r0 + k] = x;
                else crow[(r0 + k) * ldc] = x;
              }
            }
          }
        }
        if (warp == 2 && lane == 0 && c0 < 96) trace(9 + 2 * (c0 / 32));
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (warp == 2 && lane == 0) trace(5);
      ++lt;
    }
    // bulk stores must have READ shared memory before the CTA exits; their
    // global writes complete with the grid (as CUTLASS's epilogue tail)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(gp.tmem_cols));
  if (threadIdx.x == 0) trace(6);
}

__global__ void tc_splitk_reduce_kernel(const __grid_constant__ TcParams gp) {
  pdl_wait();
  pdl_trigger();
  const TcProblem& P = gp.p[blockIdx.y];
  if (P.splits <= 1) return;
  const int N = P.N, S = P.splits;
  const int64_t total = static_cast<int64_t>(P.M) * N;
  const int64_t ldw = P.ldw > 0 ? P.ldw : N, pstride = static_cast<int64_t>(P.M) * ldw;
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(x / N), n = static_cast<int>(x - static_cast<int64_t>(m) * N);
    const float* src = P.ws + static_cast<int64_t>(m) * ldw + n;
    // the partials in split order (fixed summation order), 8 loads in flight
    float s = 0.0f;
    for (int sp = 0; sp < S; sp += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = sp + k < S ? src[(sp + k) * pstride] : 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (sp + k < S) s += v[k];
    }
    const float v = P.alpha * s;
    if (P.C2 && n == P.N - 1) {
      P.C2[m] = P.beta != 0.0f ? v + P.beta * P.C2[m] : v;
    } else {
      float* c = P.C + m * P.ldc + n;
      *c = P.beta != 0.0f ? v + P.beta * *c : v;
    }
  }
}

__global__ void bf_from_f32_kernel(BfMat m, const float* __restrict__ src, int64_t rows, int64_t cols,
                                   int64_t ld_src) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = rows * cols;
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bf_put(m, x / cols, x % cols, src[(x / cols) * ld_src + x % cols]);
}

// ---------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw Error(kCuda, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap encode(void* base, int64_t inner, int64_t outer, int64_t ld_bytes, int box_inner, int box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_bytes)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

// fp32 output map [depth][rows][cols] (row stride ld_bytes, plane stride
// rows * ld_bytes), 32 x 32 x 1 boxes with 128 B swizzle (the epilogue's
// staging layout). Cached: the step's outputs are fixed buffers.
bool encode_out(float* base, int64_t cols, int64_t rows, int64_t depth, int64_t ld_bytes, CUtensorMap* out) {
  using Key = std::tuple<const void*, int64_t, int64_t, int64_t, int64_t>;
  struct H {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(std::get<0>(k)) ^ (std::get<1>(k) * 0x9e3779b97f4a7c15ull) ^
             (std::get<2>(k) * 0xbf58476d1ce4e5b9ull) ^ (std::get<3>(k) << 7) ^ (std::get<4>(k) * 31);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, H> cache;
  // every row segment must start and end on a 16-byte boundary: a clipped
  // box edge inside a 16-byte granule races with the neighbouring columns'
  // writers (measured: graph-mode runs diverged with a 2-column output)
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld_bytes & 15) != 0 || (cols & 3) != 0 || cols <= 0 ||
      rows <= 0)
    return false;
  const Key key = std::make_tuple(static_cast<const void*>(base), cols, rows, depth, ld_bytes);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(depth)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld_bytes), static_cast<cuuint64_t>(ld_bytes * rows)};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  cache.emplace(key, m);
  *out = m;
  return true;
}

using MapKey = std::tuple<const void*, const void*, int64_t, int64_t, int64_t, int, int>;

struct KeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(std::get<0>(k)) ^ (std::hash<const void*>()(std::get<1>(k)) << 1);
    h ^= std::hash<int64_t>()(std::get<2>(k)) * 0x9e3779b97f4a7c15ull;
    h ^= std::hash<int64_t>()(std::get<3>(k)) * 0xbf58476d1ce4e5b9ull;
    h ^= std::hash<int64_t>()(std::get<4>(k)) * 0x94d049bb133111ebull;
    h ^= static_cast<size_t>(std::get<5>(k) * 131 + std::get<6>(k));
    return h;
  }
};

}  // namespace

// TGNN_TC_BULK (bit mask, default 7): 1 plain stores, 2 split-K partials, 4 reduce-add;
// 0 forces the per-lane epilogue stores (A/B measurements)
int g_tc_bulk_store = env_knob("TGNN_TC_BULK", 7, 0, 7);

BfMat bf_alloc(int64_t rows, int64_t cols) {
  BfMat m;
  m.rows = rows;
  m.ld = (cols + 7) / 8 * 8;
  const size_t bytes = static_cast<size_t>(std::max<int64_t>(rows, 1)) * m.ld * sizeof(__nv_bfloat16);
  TGB_CUDA(cudaMalloc(&m.hi, bytes));
  TGB_CUDA(cudaMalloc(&m.lo, bytes));
  TGB_CUDA(cudaMemset(m.hi, 0, bytes));
  TGB_CUDA(cudaMemset(m.lo, 0, bytes));
  return m;
}

void bf_from_f32(const BfMat& m, const float* src, int64_t rows, int64_t cols, int64_t ld_src, cudaStream_t s) {
  if (rows * cols == 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(rows * cols, 256), 4 * num_sms()));
  launch_pdl(bf_from_f32_kernel, dim3(blocks), dim3(256), 0, s, m, src, rows, cols, ld_src);
  TGB_CUDA(cudaGetLastError());
}

void bf_free(BfMat& m) {
  if (m.hi) cudaFree(m.hi);
  if (m.lo) cudaFree(m.lo);
  m = BfMat{};
}

TmaOp tma_view(const BfMat& m, int64_t col0, int64_t cols, int64_t rows, bool kmajor, int box_rows) {
  TGB_REQUIRE(col0 % 8 == 0, kConfig, "tma_view: column offset must be a multiple of 8");
  TGB_REQUIRE(col0 + cols <= m.ld && rows <= m.rows && cols > 0 && rows > 0, kConfig, "tma_view: out of range");
  static std::mutex mu;
  static std::unordered_map<MapKey, TmaOp, KeyHash> cache;
  const int box_outer = kmajor ? box_rows : 64;
  const MapKey key = std::make_tuple(static_cast<const void*>(m.hi + col0), static_cast<const void*>(m.lo + col0),
                                     cols, rows, m.ld, box_outer, kmajor ? 1 : 0);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  TmaOp op;
  op.kmajor = kmajor ? 1 : 0;
  op.box_rows = box_outer;
  op.hi = encode(m.hi + col0, cols, rows, m.ld * 2, 64, box_outer);
  op.lo = encode(m.lo + col0, cols, rows, m.ld * 2, 64, box_outer);
  cache.emplace(key, op);
  return op;
}

void tc_gemm_prepare() {
  // the attribute is per device: set it once on every device this process uses
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  TGB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!(done >> dev & 1ull)) {
    TGB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
    done |= 1ull << dev;
  }
}

namespace {
thread_local std::vector<TcTraceEntry>* g_trace = nullptr;
}

void tc_trace_begin() {
  delete g_trace;
  g_trace = new std::vector<TcTraceEntry>();
}

std::vector<TcTraceEntry> tc_trace_end() {
  std::vector<TcTraceEntry> out;
  if (g_trace) out.swap(*g_trace);
  delete g_trace;
  g_trace = nullptr;
  return out;
}

void tc_group_launch(const TcGroup& g, cudaStream_t s, cudaStream_t reduce_stream, cudaEvent_t ev) {
  if (g.count == 0) return;
  tc_gemm_prepare();
  TcParams gp;
  std::memset(&gp, 0, sizeof(gp));
  gp.count = g.count;
  gp.sizes_early = g.sizes_ready ? 1 : 0;
  int max_tiles = 0, max_ntile = 16;
  bool any_split = false;
  for (int i = 0; i < g.count; ++i) {
    gp.p[i] = g.p[i];
    TcProblem& Q = gp.p[i];
    // epilogue: bulk tensor stores where the output layout allows them
    Q.c_mode = 0;
    if (g_tc_bulk_store) {
      if (Q.splits > 1) {
        const int ldw = Q.ldw > 0 ? Q.ldw : Q.N;
        if ((g_tc_bulk_store & 2) && encode_out(Q.ws, Q.N, Q.M, Q.splits, 4ll * ldw, &Q.cmap)) Q.c_mode = 1;
      } else if (((g_tc_bulk_store & 1) && Q.beta == 0.0f) || ((g_tc_bulk_store & 4) && Q.beta == 1.0f && !Q.C2)) {
        const int cols = Q.C2 ? Q.N - 1 : Q.N;
        if (encode_out(Q.C, cols, Q.M, 1, 4 * Q.ldc, &Q.cmap)) Q.c_mode = Q.beta == 0.0f ? 1 : 2;
      }
    }
    TGB_REQUIRE(g.p[i].ntile % 16 == 0 && g.p[i].ntile >= 16 && g.p[i].ntile <= 256, kConfig,
                "tc gemm: ntile must be a multiple of 16 in [16, 256]");
    gp.tiles_m[i] = static_cast<int>(ceil_div(g.p[i].M, kBM));
    gp.tiles_n[i] = static_cast<int>(ceil_div(g.p[i].N, g.p[i].ntile));
    const int t = gp.tiles_m[i] * gp.tiles_n[i] * g.p[i].splits;
    max_tiles = std::max(max_tiles, t);
    max_ntile = std::max(max_ntile, g.p[i].ntile);
    any_split |= g.p[i].splits > 1;
  }
  if (max_tiles == 0) return;
  gp.tile_base[0] = 0;
  for (int i = 0; i < g.count; ++i)
    gp.tile_base[i + 1] = gp.tile_base[i] + gp.tiles_m[i] * gp.tiles_n[i] * g.p[i].splits;
  gp.b_tile_bytes = (max_ntile + 63) / 64 * 64 * 128;
  gp.stage_bytes = 2 * kATileB + 2 * gp.b_tile_bytes;
  int cols = 32;
  while (cols < 2 * max_ntile) cols *= 2;  // two accumulator stages
  gp.tmem_cols = cols;
  // Ring depth: as many stages as fit. Groups with more tiles than SMs keep
  // two CTAs per SM (one's epilogue overlaps the other's loads) when two
  // stages each still fit; otherwise one CTA per SM with a deeper ring.
  const int total_tiles = gp.tile_base[g.count];
  const int fixed = 1024 + 256;
  int budget = kSmemMax - fixed;
  const int half = 113 * 1024 - kEpiStageB - fixed;  // two CTAs per SM
  if (total_tiles > num_sms() && half / gp.stage_bytes >= 2 && cols <= 256) budget = half;
  gp.stages = std::max(2, std::min(kStMax, budget / gp.stage_bytes));
  const int smem = gp.stages * gp.stage_bytes + fixed;
  int ctas_per_sm = (228 * 1024) / (smem + kEpiStageB + 1024);
  if (ctas_per_sm < 1) ctas_per_sm = 1;
  if (ctas_per_sm * cols > 512) ctas_per_sm = 512 / cols;
  const int grid = std::min(gp.tile_base[g.count], num_sms() * ctas_per_sm);
  TcTraceEntry* tr = nullptr;
  if (g_trace) {
    g_trace->emplace_back();
    tr = &g_trace->back();
    TGB_CUDA(cudaEventCreate(&tr->e0));
    TGB_CUDA(cudaEventCreate(&tr->e1));
    tr->count = g.count;
    for (int i = 0; i < g.count; ++i) {
      tr->M[i] = g.p[i].M;
      tr->N[i] = g.p[i].N;
      tr->K[i] = g.p[i].K;
      tr->splits[i] = g.p[i].splits;
      tr->M_dev[i] = g.p[i].M_dev;
      tr->K_dev[i] = g.p[i].K_dev;
    }
    TGB_CUDA(cudaEventRecord(tr->e0, s));
  }
  launch_pdl(tc_gemm_kernel, dim3(grid), dim3(kThreads), smem, s, gp);
  TGB_CUDA(cudaGetLastError());
  if (tr) TGB_CUDA(cudaEventRecord(tr->e1, s));
  if (any_split) {
    cudaStream_t rs = s;
    if (reduce_stream && ev) {  // the split outputs are leaves: reduce them off the critical path
      TGB_CUDA(cudaEventRecord(ev, s));
      TGB_CUDA(cudaStreamWaitEvent(reduce_stream, ev, 0));
      rs = reduce_stream;
    }
    int64_t most = 0;
    for (int i = 0; i < g.count; ++i)
      if (g.p[i].splits > 1) most = std::max<int64_t>(most, static_cast<int64_t>(g.p[i].M) * g.p[i].N);
    const int bx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((most + 255) / 256, 8 * num_sms() / g.count)));
    launch_pdl(tc_splitk_reduce_kernel, dim3(dim3(bx, g.count)), dim3(256), 0, rs, gp);
    TGB_CUDA(cudaGetLastError());
  }
}

void tc_debug_bench(int M, int N, int K, int ntile, int iters, double* us, unsigned long long* trace_out,
                    int* grid_out) {
  const int mode = iters >= 1000 ? iters / 1000 : 0;  // debug epilogue mode rides on iters
  iters = iters % 1000;
  TGB_CUDA(cudaMemcpyToSymbol(g_tc_epi_mode, &mode, sizeof(int)));
  BfMat a = bf_alloc(M, K), b = bf_alloc(N, K);
  float* c = nullptr;
  TGB_CUDA(cudaMalloc(&c, sizeof(float) * static_cast<size_t>(M) * N));
  TcGroup tg;
  TcProblem& T = tg.p[tg.count++];
  T.M = M;
  T.N = N;
  T.K = K;
  T.ntile = ntile > 0 ? ntile : tc_ntile(N);
  T.a = tma_view(a, 0, K, M, true, 128);
  T.b = tma_view(b, 0, K, N, true, T.ntile);
  T.C = c;
  T.ldc = N;
  cudaEvent_t e0, e1;
  TGB_CUDA(cudaEventCreate(&e0));
  TGB_CUDA(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) tc_group_launch(tg, nullptr);
  TGB_CUDA(cudaEventRecord(e0, nullptr));
  for (int x = 0; x < iters; ++x) tc_group_launch(tg, nullptr);
  TGB_CUDA(cudaEventRecord(e1, nullptr));
  TGB_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  TGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *us = 1e3 * ms / iters;
  const int tiles = static_cast<int>(ceil_div(M, 128) * ceil_div(N, T.ntile));
  *grid_out = std::min(tiles, num_sms() * 2);
  if (trace_out) {
    unsigned long long* d = nullptr;
    TGB_CUDA(cudaMalloc(&d, sizeof(unsigned long long) * 16 * 2 * num_sms()));
    TGB_CUDA(cudaMemset(d, 0, sizeof(unsigned long long) * 16 * 2 * num_sms()));
    TGB_CUDA(cudaMemcpyToSymbol(g_tc_trace, &d, sizeof(d)));
    tc_group_launch(tg, nullptr);
    TGB_CUDA(cudaDeviceSynchronize());
    unsigned long long* z = nullptr;
    TGB_CUDA(cudaMemcpyToSymbol(g_tc_trace, &z, sizeof(z)));
    TGB_CUDA(cudaMemcpy(trace_out, d, sizeof(unsigned long long) * 16 * 2 * num_sms(), cudaMemcpyDeviceToHost));
    cudaFree(d);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(c);
  bf_free(a);
  bf_free(b);
  const int zero = 0;
  TGB_CUDA(cudaMemcpyToSymbol(g_tc_epi_mode, &zero, sizeof(int)));
}

}  // namespace tgb
