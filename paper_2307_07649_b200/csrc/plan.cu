// Temporal sampler, negative sampler and sub-batch planning on device.
//
//  K2 negatives      sample_negatives      temporal_graph.hpp:355-370
//  K1 sampler        sample_recent_neighbors temporal_graph.hpp:296-318
//  K3 support dedup  plan_sub_batch        trainer.hpp:76-106
//
// All three are integer/f64-compare work bounded by HBM/L2 latency; results are
// bit-identical to the reference (no floating-point arithmetic except t - t_e,
// which is the same IEEE f64 subtraction).
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "plan.cuh"

namespace tgb {

namespace {

// Block-wide exclusive scan of one int per thread (blockDim.x == 1024).
__device__ int block_excl_scan(int v, int* smem_warp, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = smem_warp[lane];
    int s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    smem_warp[lane] = s - w;  // exclusive warp offsets
    if (lane == 31) smem_warp[32] = s;
  }
  __syncthreads();
  const int out = smem_warp[wid] + x - v;
  total = smem_warp[32];
  __syncthreads();
  return out;
}

// Negatives for the slice: event e draws index (e - batch_begin) of the
// global-batch stream (trainer.hpp:539-544).
__global__ void negatives_kernel(const PlanArgs* __restrict__ args, int64_t N, int64_t boundary,
                                 int32_t* __restrict__ negs) {
  pdl_wait();
  pdl_trigger();
  const PlanArgs a = *args;
  if (!a.valid || a.neg_mode != 1) return;
  const int64_t B = a.end - a.begin;
  const int64_t lo = boundary >= 0 ? boundary : 0;
  const uint64_t span = static_cast<uint64_t>(N - lo);
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < B; x += gridDim.x * blockDim.x) {
    const uint64_t i = static_cast<uint64_t>(a.begin + x - a.batch_begin);
    const uint64_t h = hash64_5(a.seed, kTagNegatives, static_cast<uint64_t>(a.batch_index),
                                static_cast<uint64_t>(a.group), i);
    negs[x] = static_cast<int32_t>(lo + static_cast<int64_t>(rng_first_u64(h) % span));
  }
}

// evaluate_mrr distractors (trainer.hpp:413-423): candidate s of event e draws
// lo + Rng(hash64(seed, "eval", e, s)).next_below(span) until it differs from
// the event's destination.
__global__ void eval_negatives_kernel(const PlanArgs* __restrict__ args, DGraph g, int per_event,
                                      int32_t* __restrict__ negs) {
  pdl_wait();
  pdl_trigger();
  const PlanArgs a = *args;
  if (!a.valid || a.neg_mode != 2 || per_event <= 0) return;
  const int64_t total = (a.end - a.begin) * per_event;
  const int64_t lo = g.boundary >= 0 ? g.boundary : 0;
  const uint64_t span = static_cast<uint64_t>(g.N - lo);
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int64_t e = a.begin + x / per_event;
    const uint64_t s = static_cast<uint64_t>(x % per_event);
    const int32_t dst = g.dst[e];
    const uint64_t h =
        splitmix64(hash_fold(hash_fold(hash_fold(a.seed, kTagEval), static_cast<uint64_t>(e)), s));
    uint64_t st = splitmix64(h ^ 0xa02bdbf7bb3c0a7ull);  // Rng(h)
    int64_t v;
    do {
      st = splitmix64(st);
      v = lo + static_cast<int64_t>(st % span);
    } while (v == dst);
    negs[x] = static_cast<int32_t>(v);
  }
}

// Warp-cooperative lower_bound over inc_t[lo, hi) for the first entry >= t.
__device__ __forceinline__ int64_t warp_lower_bound(const double* __restrict__ inc_t, int64_t lo,
                                                    int64_t hi, double t) {
  const int lane = threadIdx.x & 31;
  // invariant: all idx < lo have inc_t < t, all idx >= hi have inc_t >= t
  while (hi - lo > 32) {
    const int64_t len = hi - lo;
    const int64_t p = lo + (static_cast<int64_t>(lane) * len) / 32;
    const bool pred = inc_t[p] < t;
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    const int c = __popc(bal);
    if (c == 0) return lo;
    const int64_t plast = lo + (static_cast<int64_t>(c - 1) * len) / 32;
    const int64_t pnext = c < 32 ? lo + (static_cast<int64_t>(c) * len) / 32 : hi;
    lo = plast + 1;
    hi = pnext;
  }
  const int64_t idx = lo + lane;
  const bool pred = idx < hi && inc_t[idx] < t;
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

// One warp per root: roots are event-major (src, dst, negatives...). Neighbours are
// the min(n, have) most recent incidence entries strictly before t, newest first.
__global__ void sample_kernel(const PlanArgs* __restrict__ args, DGraph g, DPlan pl,
                              uint32_t* __restrict__ bitmap) {
  pdl_wait();
  pdl_trigger();
  const PlanArgs a = *args;
  if (!a.valid) return;
  const int64_t B = a.end - a.begin;
  const int rpe = pl.rpe;
  const int64_t R = rpe * B;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int n = pl.n;
  for (int64_t r = warp; r < R; r += nwarps) {
    const int64_t e = a.begin + r / rpe;
    const int side = static_cast<int>(r % rpe);
    const int32_t v = side == 0 ? g.src[e]
                    : (side == 1 ? g.dst[e] : pl.negs[(r / rpe) * (rpe - 2) + side - 2]);
    const double t = g.t[e];
    const int64_t base = g.inc_ptr[v];
    const int64_t end = g.inc_ptr[v + 1];
    const int64_t lb = warp_lower_bound(g.inc_t, base, end, t);
    const int64_t have = lb - base;
    const int take = static_cast<int>(have < n ? have : n);
    if (lane < take) {
      const int64_t idx = lb - 1 - lane;
      const int32_t w = g.inc_nbr[idx];
      pl.slot_node[r * n + lane] = w;
      pl.slot_event[r * n + lane] = g.inc_eid[idx];
      pl.slot_dt[r * n + lane] = t - g.inc_t[idx];
      atomicOr(&bitmap[w >> 5], 1u << (w & 31));
    }
    if (lane == 0) {
      pl.root_node[r] = v;
      pl.root_t[r] = t;
      pl.nbr_cnt[r] = take;
      atomicOr(&bitmap[v >> 5], 1u << (v & 31));
    }
  }
}

// Single CTA: pair offsets (scan of neighbour counts) and the sorted unique
// support list (scan of the node bitmap == sort + unique, trainer.hpp:102-104).
// Clears the bitmap for the next plan.
__global__ void __launch_bounds__(1024) plan_finalize_kernel(const PlanArgs* __restrict__ args,
                                                             int64_t N, DPlan pl,
                                                             uint32_t* __restrict__ bitmap) {
  pdl_wait();
  pdl_trigger();
  __shared__ int sw[33];
  const PlanArgs a = *args;
  const int B = a.valid ? static_cast<int>(a.end - a.begin) : 0;
  const int R = pl.rpe * B;
  int carry = 0, total = 0;
  for (int base = 0; base < R; base += 1024) {
    const int r = base + threadIdx.x;
    const int c = r < R ? pl.nbr_cnt[r] : 0;
    const int ex = block_excl_scan(c, sw, total);
    if (r < R) pl.pair_ptr[r] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) pl.pair_ptr[R] = carry;
  const int P = carry;
  const int64_t words = (N + 31) / 32;
  int ucarry = 0;
  for (int64_t base = 0; base < words; base += 1024) {
    const int64_t w = base + threadIdx.x;
    uint32_t bits = w < words ? bitmap[w] : 0u;
    const int cnt = __popc(bits);
    const int ex = block_excl_scan(cnt, sw, total);
    int pos = ucarry + ex;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int32_t node = static_cast<int32_t>(w * 32 + b);
      pl.supports[pos] = node;
      pl.sup_row[node] = pos;
      ++pos;
    }
    if (w < words) bitmap[w] = 0u;
    ucarry += total;
  }
  if (threadIdx.x == 0) {
    pl.sizes[kSzB] = B;
    pl.sizes[kSzR] = R;
    pl.sizes[kSzP] = P;
    pl.sizes[kSzU] = ucarry;
    pl.sizes[kSzItems] = R + P;
    pl.sizes[kSz2B] = 2 * B;
  }
}

// Compacts pairs (root-major), resolves support rows, and emits the routing
// items (roots then pairs) keyed by support row.
__global__ void pairs_kernel(DPlan pl) {
  pdl_wait();
  pdl_trigger();
  const int R = pl.sizes[kSzR];
  const int n = pl.n;
  const int cap_items = pl.cap_R + pl.cap_P;
  const int R_cap = pl.cap_R;
  const int nn = n > 0 ? n : 1;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < R_cap * nn; x += gridDim.x * blockDim.x) {
    const int r = x / nn, m = x % nn;
    if (r < R && m < pl.nbr_cnt[r]) {
      const int p = pl.pair_ptr[r] + m;
      const int32_t w = pl.slot_node[r * n + m];
      const int su = pl.sup_row[w];
      pl.pair_node[p] = w;
      pl.pair_event[p] = pl.slot_event[r * n + m];
      pl.pair_dt[p] = pl.slot_dt[r * n + m];
      pl.pair_root[p] = r;
      pl.pair_sup[p] = su;
      pl.item_key[R + p] = su;
      pl.item_val[R + p] = R + p;
    }
    if (m == 0) {
      if (r < R) {
        const int su = pl.sup_row[pl.root_node[r]];
        pl.root_sup[r] = su;
        pl.item_key[r] = su;
        pl.item_val[r] = r;
      }
    }
  }
  // pad the unused item tail with the sentinel key (sorts last)
  const int items = R + pl.sizes[kSzP];
  for (int x = items + blockIdx.x * blockDim.x + threadIdx.x; x < cap_items;
       x += gridDim.x * blockDim.x) {
    pl.item_key[x] = pl.cap_U;
    pl.item_val[x] = x;
  }
}

__global__ void routing_ptr_kernel(DPlan pl) {
  pdl_wait();
  pdl_trigger();
  const int items = pl.sizes[kSzItems];
  const int U = pl.sizes[kSzU];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gridDim.x * blockDim.x) {
    const int k = pl.item_key_s[i];
    if (i == 0 || pl.item_key_s[i - 1] != k) pl.sup_item_ptr[k] = i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) pl.sup_item_ptr[U] = items;
}

// ReadView gather (DirectMemoryClient::read, shared_buffers.hpp:138-153 +
// pack_mail_row, memory_store.hpp:73-80): one warp per support row, 128-bit
// vectorised when d % 4 == 0.
__global__ void gather_view_kernel(DPlan pl, DMem st, DView vw) {
  pdl_wait();
  pdl_trigger();
  const int U = pl.sizes[kSzU];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t d = st.d;
  for (int64_t u = warp; u < U; u += nwarps) {
    const int64_t v = pl.supports[u];
    if ((d & 3) == 0) {
      const float4* sm = reinterpret_cast<const float4*>(st.memory + v * d);
      float4* dm = reinterpret_cast<float4*>(vw.mem + u * d);
      for (int64_t x = lane; x < d / 4; x += 32) dm[x] = sm[x];
      const float4* sl = reinterpret_cast<const float4*>(st.mail_mem + v * 2 * d);
      float4* dl = reinterpret_cast<float4*>(vw.mail_mem + u * 2 * d);
      for (int64_t x = lane; x < d / 2; x += 32) dl[x] = sl[x];
    } else {
      for (int64_t x = lane; x < d; x += 32) vw.mem[u * d + x] = st.memory[v * d + x];
      for (int64_t x = lane; x < 2 * d; x += 32) vw.mail_mem[u * 2 * d + x] = st.mail_mem[v * 2 * d + x];
    }
    if (lane == 0) {
      vw.mail_t[u] = st.mail_t[v];
      vw.mail_dt[u] = st.mail_dt[v];
      vw.mail_ev[u] = st.mail_ev[v];
    }
  }
}

__global__ void set_args_kernel(PlanArgs* dst, PlanArgs a) {
  pdl_wait();
  pdl_trigger(); *dst = a; }

__global__ void select_args_kernel(const BarrierDesc* __restrict__ desc, const int* __restrict__ ctr,
                                   int offset, PlanArgs* dst) {
  pdl_wait();
  pdl_trigger();
  *dst = desc[*ctr + offset].args;
}

__global__ void sample_queries_kernel(DGraph g, const int32_t* __restrict__ nodes,
                                      const double* __restrict__ times, int count, int n,
                                      int32_t* __restrict__ nbr_node, int32_t* __restrict__ nbr_event,
                                      double* __restrict__ nbr_dt, int32_t* __restrict__ nbr_count) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = warp; q < count; q += nwarps) {
    const int32_t v = nodes[q];
    const double t = times[q];
    const int64_t base = g.inc_ptr[v];
    const int64_t lb = warp_lower_bound(g.inc_t, base, g.inc_ptr[v + 1], t);
    const int64_t have = lb - base;
    const int take = static_cast<int>(have < n ? have : n);
    if (lane < take) {
      const int64_t idx = lb - 1 - lane;
      nbr_node[q * n + lane] = g.inc_nbr[idx];
      nbr_event[q * n + lane] = g.inc_eid[idx];
      nbr_dt[q * n + lane] = t - g.inc_t[idx];
    }
    if (lane == 0) nbr_count[q] = take;
  }
}

}  // namespace

void select_plan_args_launch(PlanArgs* dst, const BarrierDesc* desc, const int* ctr, cudaStream_t s,
                             int offset) {
  launch_pdl(select_args_kernel, dim3(1), dim3(1), 0, s, desc, ctr, offset, dst);
  TGB_CUDA(cudaGetLastError());
}

void set_plan_args_launch(PlanArgs* dst, const PlanArgs& a, cudaStream_t s) {
  launch_pdl(set_args_kernel, dim3(1), dim3(1), 0, s, dst, a);
  TGB_CUDA(cudaGetLastError());
}

void sample_queries_launch(const DGraph& g, const int32_t* nodes, const double* times, int count,
                           int n, int32_t* nbr_node, int32_t* nbr_event, double* nbr_dt,
                           int32_t* nbr_count, cudaStream_t s) {
  if (count <= 0) return;
  int blocks = static_cast<int>(ceil_div(count, 8));
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  launch_pdl(sample_queries_kernel, dim3(blocks), dim3(256), 0, s, g, nodes, times, count, n, nbr_node, nbr_event,
                                               nbr_dt, nbr_count);
  TGB_CUDA(cudaGetLastError());
}

void negatives_only_launch(const DGraph& g, const PlanArgs* args, int count, int32_t* negs,
                           cudaStream_t s) {
  launch_pdl(negatives_kernel, dim3(static_cast<int>(ceil_div(count, 256))), dim3(256), 0, s, args, g.N, g.boundary, negs);
  TGB_CUDA(cudaGetLastError());
}

size_t plan_sort_tmp_bytes(int cap_items, int bits) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr),
                                  static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), cap_items, 0, bits);
  return bytes;
}

void plan_launch(const DGraph& g, DPlan& pl, cudaStream_t s, cudaStream_t side) {
  uint32_t* bitmap = pl.bitmap;
  const int B = pl.cap_B;
  if (!pl.eval_negs && pl.rpe == 3) {
    launch_pdl(negatives_kernel, dim3(static_cast<int>(ceil_div(B, 256))), dim3(256), 0, s, pl.args, g.N, g.boundary,
                                                                        pl.negs);
  } else if (pl.eval_negs && pl.rpe > 2) {
    const int64_t total = static_cast<int64_t>(B) * (pl.rpe - 2);
    launch_pdl(eval_negatives_kernel, dim3(static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 8 * num_sms()))), dim3(256), 0, s, 
        pl.args, g, pl.rpe - 2, pl.negs);
  }
  TGB_CUDA(cudaGetLastError());
  const int R = pl.cap_R;
  const int warps_per_block = 8;
  int blocks = static_cast<int>(ceil_div(R, warps_per_block));
  if (blocks > 4 * num_sms() * 8) blocks = 4 * num_sms() * 8;
  launch_pdl(sample_kernel, dim3(blocks), dim3(32 * warps_per_block), 0, s, pl.args, g, pl, bitmap);
  TGB_CUDA(cudaGetLastError());
  launch_pdl(plan_finalize_kernel, dim3(1), dim3(1024), 0, s, pl.args, g.N, pl, bitmap);
  TGB_CUDA(cudaGetLastError());
  const int slots = pl.cap_R * (pl.n > 0 ? pl.n : 1);
  launch_pdl(pairs_kernel, dim3(static_cast<int>(ceil_div(slots, 256))), dim3(256), 0, s, pl);
  TGB_CUDA(cudaGetLastError());
  if (!pl.routing) return;
  const int cap_items = pl.cap_R + pl.cap_P;
  cudaStream_t ss = s;
  if (side && pl.ev_pairs) {
    TGB_CUDA(cudaEventRecord(pl.ev_pairs, s));
    TGB_CUDA(cudaStreamWaitEvent(side, pl.ev_pairs, 0));
    ss = side;
  }
  size_t bytes = pl.sort_tmp_bytes;
  TGB_CUDA(cub::DeviceRadixSort::SortPairs(pl.sort_tmp, bytes, pl.item_key, pl.item_key_s,
                                           pl.item_val, pl.item_val_s, cap_items, 0,
                                           pl.sort_bits, ss));
  launch_pdl(routing_ptr_kernel, dim3(static_cast<int>(ceil_div(cap_items, 256))), dim3(256), 0, ss, pl);
  TGB_CUDA(cudaGetLastError());
  if (pl.ev_sorted) TGB_CUDA(cudaEventRecord(pl.ev_sorted, ss));
}

void gather_view_launch(const DPlan& pl, const DMem& st, DView& vw, cudaStream_t s) {
  int blocks = static_cast<int>(ceil_div(pl.cap_U, 8));
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  launch_pdl(gather_view_kernel, dim3(blocks), dim3(256), 0, s, pl, st, vw);
  TGB_CUDA(cudaGetLastError());
}

}  // namespace tgb
