// Fused GRU freshen (freshen_memory + gru_update, trainer.hpp:111-124,
// gru.hpp:32-67) as ONE tcgen05 kernel per (128-row tile, 32-unit slice).
//
// The unfused chain is five launches: [Xg Wzr^T | Xg Whm^T] GEMM -> sigmoid
// -> [r*s | 1] Whs^T GEMM (beta = 1) -> tanh / blend, each paying launch,
// ramp and drain on the barrier's critical path, with the gates
// round-tripping through L2. Here nq = ceil(d / 32) independent CTAs share a
// 128-row tile of the read view; CTA q owns hidden units [32 q, 32 q + 32):
//   1. GEMM1 (TMA -> 2-stage SMEM ring -> tcgen05.mma, bf16x3, fp32 in TMEM),
//      N = 192: ALL the r columns (128, as [r*s | 1] needs every unit) plus
//      this CTA's z and h_m columns, K = gin + 1 (bias via the ones column of
//      Xg); the h_m rows come from Wh's mail columns, whose tensor map ends at
//      K = md (TMA zero-fills past it). Recomputing r in every slice costs
//      tensor time but needs no cross-CTA exchange.
//   2. epilogue warps: r = sigma, [r*s | 1] -> bf16 hi / lo straight into the
//      swizzled A operand of GEMM2 in shared memory; z = sigma of the slice.
//   3. GEMM2: [r*s | 1] [Wh_s | bh]^T for the slice's units accumulated onto
//      the h_m columns in TMEM (K = 64 per swizzle atom); its B tile was loaded
//      by TMA into the freed ring stage.
//   4. epilogue: h = tanh, s_hat = (1 - z) s + z h (rows with a cached mail;
//      s otherwise), written with the pre-activations a_z, a_r, a_h (for the backward), the slice of the
//      [r*s | 1] operand of the Wh_s weight gradient, and the node operand NF
//      = [s_hat | static | 1] of the attention projections (the last slice
//      adds the static block); operand rows [U, roundup64(U)) are zeroed
//      (split-K reductions read whole 64-row chunks).
// All global traffic of the epilogue is staged through shared memory so it
// is row-contiguous; loops stay rolled (a large unrolled epilogue ran out of
// the instruction cache on the few SMs the kernel occupies).
// Warps: 0 TMA producer, 1 TMEM owner + MMA issuer, 2-17 epilogue (TMEM lane
// quarter = warp % 4, thread = row).
#include <mutex>

#include "gru_fused.cuh"
#include "tc_ptx.cuh"

namespace tgb {

namespace {

constexpr int kGfEpiWarps = 16;  // four per TMEM lane quarter
constexpr int kGfThreads = 64 + 32 * kGfEpiWarps;
constexpr int kGfStages = 2;
constexpr int kGfATile = 128 * 128;                    // 128 rows x 64 bf16 (one swizzle atom), per plane
constexpr int kGfBTile = 192 * 128;                    // [r 128 | z 32 | h_m 32] rows x 64 bf16, per plane
constexpr int kGfStage = 2 * kGfATile + 2 * kGfBTile;  // 80 KB
constexpr int kGfRS = 4 * kGfATile;                    // [hi atom 0 | hi atom 1 | lo atom 0 | lo atom 1]
constexpr int kGfSmem = kGfStages * kGfStage + kGfRS + 256 + 1024;
constexpr int kGfTmemCols = 256;
constexpr int kGfSlice = 32;  // hidden units per CTA
constexpr int kLdS = 129;     // staging row stride (floats): conflict-free row-per-thread access

// Optional per-CTA timeline (debug: tgnn_debug_gru_trace): globaltimer stamps.
__device__ unsigned long long* g_gf_trace = nullptr;
__device__ __forceinline__ void gf_stamp(int slot) {
  unsigned long long* t = g_gf_trace;
  if (t) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    t[blockIdx.x * 16 + slot] = v;
  }
}

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ void split_bf(float v, __nv_bfloat16& h, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(v);
  l = __float2bfloat16_rn(v - __bfloat162float(h));
}

// 8 consecutive values -> one 16-byte hi chunk and one lo chunk
__device__ __forceinline__ void pack8(const float (&v)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat16 h0, l0, h1, l1;
    split_bf(v[2 * q], h0, l0);
    split_bf(v[2 * q + 1], h1, l1);
    h[q] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) | (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
    l[q] = static_cast<uint32_t>(__bfloat16_as_ushort(l0)) | (static_cast<uint32_t>(__bfloat16_as_ushort(l1)) << 16);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__global__ void __launch_bounds__(kGfThreads, 1) gru_fused_kernel(const __grid_constant__ GruFusedParams p) {
  if (threadIdx.x == 0) gf_stamp(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* rs = smem + kGfStages * kGfStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(rs + kGfRS);
  uint64_t* empty = full + kGfStages;
  uint64_t* tfull = empty + kGfStages;  // GEMM1 accumulators ready
  uint64_t* t2full = tfull + 1;         // GEMM2 accumulated
  uint64_t* rsbar = t2full + 1;         // [r*s | 1] operand written
  uint64_t* wbar = rsbar + 1;           // Wh_s tile landed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = p.nclu;  // slices per tile
  const int m0 = static_cast<int>(blockIdx.x / nq) * 128;
  const int u0 = kGfSlice * static_cast<int>(blockIdx.x % nq);
  const int d = p.d;
  const int natoms = (d + 1 + 63) / 64;  // K atoms of [r*s | 1]

  if (warp == 0 && lane == 0) {
    const CUtensorMap* maps[10] = {&p.xg_hi, &p.xg_lo, &p.wzr_hi, &p.wzr_lo, &p.wz_hi,
                                   &p.wz_lo, &p.whm_hi, &p.whm_lo, &p.whs_hi, &p.whs_lo};
    for (const CUtensorMap* m : maps) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGfStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tfull, 1);
    mbar_init(t2full, 1);
    mbar_init(rsbar, kGfEpiWarps);  // one arrival per epilogue warp
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(kGfTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  pdl_wait();  // Xg / view / weights come from the predecessors
  pdl_trigger();
  if (threadIdx.x == 0) gf_stamp(1);
  const int U = min(*p.U_dev, p.cap_U);
  const bool live = m0 < U;
  const int nk = (p.gin + 1 + 63) / 64;

  if (live && warp == 0 && lane == 0) {
    // ---- producer: GEMM1 k-blocks, then Wh_s into the freed stage 0
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kGfStages;
      if (kb >= kGfStages) mbar_wait(empty + s, ((kb / kGfStages) - 1) & 1);
      mbar_expect_tx(full + s, kGfStage);
      uint8_t* st = smem + s * kGfStage;
      const int k0 = kb * 64;
      tma_2d(st, &p.xg_hi, k0, m0, full + s);
      tma_2d(st + kGfATile, &p.xg_lo, k0, m0, full + s);
      for (int h = 0; h < 2; ++h) {
        const CUtensorMap* wz = h ? &p.wzr_lo : &p.wzr_hi;
        uint8_t* bd = st + 2 * kGfATile + h * kGfBTile;
        tma_2d(bd, wz, k0, d, full + s);                                   // r rows [0, 64)
        tma_2d(bd + 64 * 128, wz, k0, d + 64, full + s);                   // r rows [64, 128)
        tma_2d(bd + 128 * 128, h ? &p.wz_lo : &p.wz_hi, k0, u0, full + s);  // z rows of the slice (32)
        tma_2d(bd + 160 * 128, h ? &p.whm_lo : &p.whm_hi, k0, u0, full + s);  // h_m rows (K < md)
      }
    }
    gf_stamp(2);
    mbar_wait(tfull, 0);  // every GEMM1 MMA has completed: the ring is free
    mbar_expect_tx(wbar, 4 * kGfSlice * 128);
    for (int a = 0; a < 2; ++a) {
      tma_2d(smem + a * 4096, &p.whs_hi, 64 * a, u0, wbar);
      tma_2d(smem + 8192 + a * 4096, &p.whs_lo, 64 * a, u0, wbar);
    }
  } else if (live && warp == 1 && lane == 0) {
    // ---- MMA issuer
    const uint32_t id1 = idesc(192, true, true);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kGfStages;
      mbar_wait(full + s, (kb / kGfStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint8_t* st = smem + s * kGfStage;
      const uint32_t ahi = su32(st), alo = su32(st + kGfATile);
      const uint32_t bhi = su32(st + 2 * kGfATile), blo = su32(st + 2 * kGfATile + kGfBTile);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t o = ks * 32u;
        umma(tmem, sdesc(ahi + o, true), sdesc(bhi + o, true), id1, (kb > 0 || ks > 0) ? 1u : 0u);
        umma(tmem, sdesc(ahi + o, true), sdesc(blo + o, true), id1, 1u);
        umma(tmem, sdesc(alo + o, true), sdesc(bhi + o, true), id1, 1u);
      }
      umma_commit(empty + s);
    }
    umma_commit(tfull);
    gf_stamp(3);
    mbar_wait(wbar, 0);
    mbar_wait(rsbar, 0);
    gf_stamp(4);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t id2 = idesc(kGfSlice, true, true);
    const uint32_t dst = tmem + 160;  // the slice's h_m columns
    for (int a = 0; a < natoms; ++a) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t o = ks * 32u;
        const uint32_t ahi = su32(rs + a * kGfATile) + o, alo = su32(rs + (2 + a) * kGfATile) + o;
        const uint32_t bhi = su32(smem + a * 4096) + o, blo = su32(smem + 8192 + a * 4096) + o;
        umma(dst, sdesc(ahi, true), sdesc(bhi, true), id2, 1u);
        umma(dst, sdesc(ahi, true), sdesc(blo, true), id2, 1u);
        umma(dst, sdesc(alo, true), sdesc(bhi, true), id2, 1u);
      }
    }
    umma_commit(t2full);
  } else if (live && warp >= 2) {
    // ---- epilogue: TMEM lane = row of the tile (quarter warp % 4); the four
    // warps of a quarter split the columns; every global access is staged
    // through shared memory in the idle second ring stage
    constexpr int kEt = 32 * kGfEpiWarps;
    const int et = threadIdx.x - 64;
    const int q = warp & 3;
    const int sl = (warp - 2) >> 2;  // 0..3: this warp's column share
    const int trow = 32 * q + lane;
    const int row = m0 + trow;
    const bool rv = row < U;
    const int tail_end = min(p.cap_U, (U + 63) / 64 * 64);  // operand rows zeroed past U
    const int rows_out = min(128, tail_end - m0);           // rows written (valid + tail)
    const int rows_v = min(128, U - m0);                    // valid rows
    const uint32_t tl = tmem + (static_cast<uint32_t>(32 * q) << 16);
    const bool last = static_cast<int>(blockIdx.x % nq) == nq - 1;
    const int nu = max(0, min(kGfSlice, d - u0));  // this CTA's hidden units
    const int ds = p.ds;
    const int64_t ld3 = 3 * static_cast<int64_t>(d);
    // stage 1 (idle after GEMM1): S [128][kLdS] = s (all units), then the
    // slice's s_hat; stage 0 past the Wh_s tile (16 KB): X [128][33] = z / r /
    // h of the slice, node ids
    float* S = reinterpret_cast<float*>(smem + kGfStage);
    float* X = reinterpret_cast<float*>(smem + 16384);
    int32_t* nodes = reinterpret_cast<int32_t*>(X + 128 * 33);
    auto epi_sync = [] { asm volatile("bar.sync 1, %0;" ::"r"(kEt) : "memory"); };
    // coalesced row-segment store of staged columns [c_lo, c_lo + nc) (tile columns)
    auto store_rows = [&](const float* src, int lds, int c_lo, int nc, float* dst, int64_t ld) {
#pragma unroll 4
      for (int idx = et; idx < rows_v * 32; idx += kEt) {
        const int r = idx >> 5, c = idx & 31;
        if (c < nc) dst[static_cast<int64_t>(m0 + r) * ld + u0 + c] = src[r * lds + c_lo + c];
      }
    };
    mbar_wait(tfull, 0);  // GEMM1 done: the ring is idle
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (et == 0) gf_stamp(5);
    // (a) s = the view's memory (all d units) of the tile's rows, node ids
#pragma unroll 1
    for (int base = et; base < 128 * 128; base += kEt * 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = base + kEt * k, r = idx >> 7, c = idx & 127;
        v[k] = (m0 + r < U && c < d) ? p.mem[static_cast<int64_t>(m0 + r) * d + c] : 0.0f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = base + kEt * k;
        S[(idx >> 7) * kLdS + (idx & 127)] = v[k];
      }
    }
    if (et < 128) nodes[et] = m0 + et < U ? p.supports[m0 + et] : 0;
    epi_sync();
    if (et == 0) gf_stamp(11);
    // (b) [r*s | 1]: 16 chunks of 8 units, four per warp; r for the slice and
    // z staged for the slice's Gates rows
    float* srow = S + trow * kLdS;
    float* xrow = X + trow * 33;
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int chunk = sl + 4 * k;  // unit chunk 0..15
      uint32_t vb[8];
      tmem_ld8(tl + 8 * chunk, vb);
      tmem_ld_wait();
      float rsv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int u = 8 * chunk + e;
        float v = 0.0f;
        if (u < d) v = sigm(__uint_as_float(vb[e])) * srow[u];
        else if (u == d) v = 1.0f;  // the bias column
        rsv[e] = rv ? v : 0.0f;     // rows past U: zeros (operand tail, inert MMA rows)
      }
      uint4 hi, lo;
      pack8(rsv, hi, lo);
      const int atom = chunk >> 3, ch = chunk & 7;
      const int off = trow * 128 + ((ch ^ (trow & 7)) << 4);
      *reinterpret_cast<uint4*>(rs + atom * kGfATile + off) = hi;
      *reinterpret_cast<uint4*>(rs + (2 + atom) * kGfATile + off) = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy (UMMA reads it)
    __syncwarp();
    if (lane == 0) mbar_arrive(rsbar);
    {  // z of the slice: chunk sl of the z columns
      uint32_t va[8];
      tmem_ld8(tl + 128 + 8 * sl, va);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) xrow[8 * sl + e] = __uint_as_float(va[e]);
    }
    epi_sync();
    if (et == 0) gf_stamp(12);
    store_rows(X, 33, 0, nu, p.gates, ld3);  // a_z (pre-activation, for the backward)
    // the slice of the [r*s | 1] operand in global memory (Wh_s weight
    // gradient): four 16-byte chunks per row, from the swizzled shared copy
#pragma unroll 1
    for (int idx = et; idx < rows_out * 4; idx += kEt) {
      const int r = idx >> 2, cc = idx & 3;
      const int col = u0 + 8 * cc;
      if (col + 8 > p.rs.ld || !(col < u0 + nu || (last && col <= d))) continue;
      const int atom = col >> 6, ch = (col >> 3) & 7;
      const int off = r * 128 + ((ch ^ (r & 7)) << 4);
      const int64_t g = static_cast<int64_t>(m0 + r) * p.rs.ld + col;
      *reinterpret_cast<uint4*>(p.rs.hi + g) = *reinterpret_cast<const uint4*>(rs + atom * kGfATile + off);
      *reinterpret_cast<uint4*>(p.rs.lo + g) = *reinterpret_cast<const uint4*>(rs + (2 + atom) * kGfATile + off);
    }
    epi_sync();
    {  // r of the slice (the r columns u0 .. u0 + 31 of the accumulator)
      uint32_t vb[8];
      tmem_ld8(tl + u0 + 8 * sl, vb);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) xrow[8 * sl + e] = __uint_as_float(vb[e]);
    }
    epi_sync();
    store_rows(X, 33, 0, nu, p.gates + d, ld3);  // a_r
    // (c) GEMM2 done: h = tanh (staged in X), s_hat = (1 - z) s + z h (into S)
    if (et == 0) gf_stamp(6);
    mbar_wait(t2full, 0);
    if (et == 0) gf_stamp(7);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    epi_sync();
    {
      const bool has = rv && p.mail_ev[row] >= 0;
      uint32_t va[8], vb[8];
      tmem_ld8(tl + 128 + 8 * sl, va);  // z
      tmem_ld8(tl + 160 + 8 * sl, vb);  // h
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = 8 * sl + e, u = u0 + j;
        if (j >= nu) continue;
        const float ah = __uint_as_float(vb[e]);
        const float h = tanhf(ah);
        float out = srow[u];
        if (has) {
          const float az = __uint_as_float(va[e]);
          out = sigm(-az) * out + sigm(az) * h;
          if (!isfinite(out)) atomicExch(p.flag, 1);
        }
        srow[u] = out;
        xrow[j] = ah;
      }
    }
    epi_sync();
    store_rows(X, 33, 0, nu, p.gates + 2 * d, ld3);  // a_h
    store_rows(S, kLdS, u0, nu, p.s_hat, d);         // s_hat
    // NF = [s_hat | static | 1]: the slice's unit columns; the last slice also
    // the static block and the ones column; rows [U, roundup64(U)) zero
    const int nf_end = last ? d + ds + 1 : u0 + kGfSlice;
    const int nch = (nf_end - u0 + 7) / 8;
#pragma unroll 1
    for (int base = et; base < rows_out * nch; base += kEt * 4) {
      float o8[4][8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // four chunks' loads in flight
        const int idx = base + kEt * k;
        const int r = idx / nch, col = u0 + 8 * (idx % nch);
        const bool valid = idx < rows_out * nch && m0 + r < U;
        const int64_t so = static_cast<int64_t>(nodes[valid ? r : 0]) * ds - d;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = col + e;
          float v = 0.0f;
          if (valid) {
            if (c < d) v = S[r * kLdS + c];
            else if (c < d + ds) v = p.stat[so + c];
            else if (c == d + ds) v = 1.0f;
          }
          o8[k][e] = v;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int idx = base + kEt * k;
        const int r = idx / nch, col = u0 + 8 * (idx % nch);
        if (idx >= rows_out * nch || col + 8 > p.nf.ld) continue;
        uint4 hi, lo;
        pack8(o8[k], hi, lo);
        const int64_t g = static_cast<int64_t>(m0 + r) * p.nf.ld + col;
        *reinterpret_cast<uint4*>(p.nf.hi + g) = hi;
        *reinterpret_cast<uint4*>(p.nf.lo + g) = lo;
      }
    }
  }
  if (threadIdx.x == 64) gf_stamp(8);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) gf_stamp(9);
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kGfTmemCols));
  if (threadIdx.x == 0) gf_stamp(10);
}

}  // namespace

void gru_debug_trace(unsigned long long* host, int cap_ctas, int* n_ctas) {
  static unsigned long long* buf = nullptr;
  static int cap = 0;
  if (!host) {  // arm: (re)allocate and zero the device buffer
    if (cap < cap_ctas) {
      if (buf) cudaFree(buf);
      TGB_CUDA(cudaMalloc(&buf, sizeof(unsigned long long) * 16 * cap_ctas));
      cap = cap_ctas;
    }
    TGB_CUDA(cudaMemset(buf, 0, sizeof(unsigned long long) * 16 * cap));
    TGB_CUDA(cudaMemcpyToSymbol(g_gf_trace, &buf, sizeof(buf)));
    return;
  }
  TGB_CUDA(cudaDeviceSynchronize());
  TGB_CUDA(cudaMemcpy(host, buf, sizeof(unsigned long long) * 16 * std::min(cap, cap_ctas), cudaMemcpyDeviceToHost));
  unsigned long long* z = nullptr;
  TGB_CUDA(cudaMemcpyToSymbol(g_gf_trace, &z, sizeof(z)));
  *n_ctas = cap;
}

void gru_fused_launch(GruFusedParams p, const BfMat& xg, const BfMat& wzr, const BfMat& whm, const BfMat& whs,
                      int64_t md, cudaStream_t s) {
  TGB_REQUIRE(gru_fused_supported(p.d), kConfig, "fused GRU: d_mem + 1 must be <= 128");
  static_assert(16384 + 128 * 33 * 4 + 128 * 4 <= kGfStage && 128 * kLdS * 4 <= kGfStage, "epilogue staging");
  TGB_REQUIRE(p.nf.ld % 8 == 0 && p.rs.ld % 8 == 0, kConfig, "fused GRU: operand rows must be 16-byte aligned");
  const TmaOp a = tma_view(xg, 0, p.gin + 1, p.cap_U, true, 128);
  const TmaOp bz = tma_view(wzr, 0, p.gin + 1, 2 * p.d, true, 64);
  const TmaOp bz32 = tma_view(wzr, 0, p.gin + 1, 2 * p.d, true, kGfSlice);
  const TmaOp bh = tma_view(whm, 0, md, p.d, true, kGfSlice);
  const TmaOp b2 = tma_view(whs, 0, p.d + 1, p.d, true, kGfSlice);
  p.xg_hi = a.hi;
  p.xg_lo = a.lo;
  p.wzr_hi = bz.hi;
  p.wzr_lo = bz.lo;
  p.wz_hi = bz32.hi;
  p.wz_lo = bz32.lo;
  p.whm_hi = bh.hi;
  p.whm_lo = bh.lo;
  p.whs_hi = b2.hi;
  p.whs_lo = b2.lo;
  p.nclu = static_cast<int>((p.d + kGfSlice - 1) / kGfSlice);  // slices per 128-row tile
  {
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    TGB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!(done >> dev & 1ull)) {
      TGB_CUDA(cudaFuncSetAttribute(gru_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGfSmem));
      done |= 1ull << dev;
    }
  }
  const int tiles = static_cast<int>((p.cap_U + 127) / 128);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(tiles * p.nclu));
  cfg.blockDim = dim3(kGfThreads);
  cfg.dynamicSmemBytes = kGfSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = prio;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  TGB_CUDA(cudaLaunchKernelEx(&cfg, gru_fused_kernel, p));
}

}  // namespace tgb
