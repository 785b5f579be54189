// C ABI (include/tgnn_b200.h): host runtime of the B200 DistTGL training step.
//
// Host C++ owns contexts, the device T-CSR, node-memory replicas, the trainer
// core (parameters, gradients, Adam state, workspaces) and the i x j x k
// schedule; every compute step is a CUDA kernel on the context stream and
// every exchange is an NCCL collective on the same stream (NVLink/NVSwitch).

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tgnn_b200.h"
#include "common.cuh"
#include "device_types.cuh"
#include "host/checkpoint.hpp"
#include "host/dataset.hpp"
#include "host/schedule.hpp"
#include "host/synth.hpp"
#include "nccl_dyn.hpp"
#include "graph.cuh"
#include "plan.cuh"
#include "step.cuh"
#include "gemm_tma.cuh"
#include "gru_fused.cuh"

using namespace tgb;

namespace {

thread_local std::string g_err;

#define NCCL_CHECK(x)                                                                 \
  do {                                                                                \
    ncclResult_t r__ = (x);                                                           \
    if (r__ != ncclSuccess)                                                           \
      throw ::tgb::Error(::tgb::kNccl, std::string(#x) + ": " + nccl::api().GetErrorString(r__)); \
  } while (0)

#define API_BEGIN try {
#define API_END                                  \
  }                                              \
  catch (const tgb::Error& e) {                  \
    g_err = e.what();                            \
    return e.code;                               \
  }                                              \
  catch (const std::bad_alloc& e) {              \
    g_err = std::string("host allocation: ") + e.what(); \
    return kCuda;                                \
  }                                              \
  catch (const std::exception& e) {              \
    g_err = e.what();                            \
    return 8;                                    \
  }                                              \
  return 0;

template <typename T>
T* dalloc(size_t n) {
  T* p = nullptr;
  TGB_CUDA(cudaMalloc(&p, (n > 0 ? n : 1) * sizeof(T)));
  return p;
}

template <typename T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) TGB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <typename T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) TGB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

ModelDims dims_of(const tgnn_model_config* c) {
  ModelDims m;
  m.d_mem = c->d_mem;
  m.d_time = c->d_time;
  m.d_static = c->d_static;
  m.d_attn = c->d_attn;
  m.d_hidden = c->d_hidden;
  m.d_e = c->d_e;
  m.n_neighbors = c->n_neighbors;
  m.num_nodes = c->num_nodes;
  m.max_t = c->max_t;
  return m;
}

host::TrainCfg train_of(const tgnn_train_config* c) {
  host::TrainCfg t;
  t.i = c->i;
  t.j = c->j;
  t.k = c->k;
  t.p = c->p;
  t.q = c->q;
  t.epochs = c->epochs;
  t.local_batch = c->local_batch;
  t.lr_base = c->lr_base;
  t.seed = c->seed;
  t.local_batch_ref = c->local_batch_ref;
  t.neg_groups = c->neg_groups;
  return t;
}

void validate_dims(const ModelDims& m) {
  TGB_REQUIRE(m.d_mem >= 1 && m.d_attn >= 1 && m.d_time >= 0 && m.d_static >= 0 && m.d_e >= 0,
              kConfig, "model: dimensions must be positive");
  TGB_REQUIRE(m.d_attn <= 256, kConfig, "model: d_attn above 256 is not supported on device");
  TGB_REQUIRE(m.n_neighbors >= 0 && m.n_neighbors <= 32, kConfig,
              "model: n_neighbors must lie in [0, 32] on device");
  TGB_REQUIRE(m.num_nodes > 0, kConfig, "model: num_nodes must be positive");
}

// init_params (ref model.hpp:122-141): U(+-1/sqrt(cols)) for every rank-2
// tensor except omega and the static table, streams keyed by the 1-based
// tensor slot; omega log-spaced over [1e-5, 1] / max_t.
std::vector<double> host_init_params(const ModelDims& m, uint64_t seed) {
  const ParamLayout L = ParamLayout::make(m);
  std::vector<double> flat(static_cast<size_t>(L.total), 0.0);
  for (int x = 0; x < tNumTensors; ++x) {
    const bool rank2 = !(x == tOmega || x == tBz || x == tBr || x == tBh || x == tBq || x == tBk ||
                         x == tBv || x == tB1 || x == tB2);
    if (!rank2 || x == tStatic) continue;
    host::Stream st(host::hash64_3(seed, 0x696e6974ull, static_cast<uint64_t>(x + 1)));
    const double bound = 1.0 / std::sqrt(static_cast<double>(L.cols[x]));
    double* p = flat.data() + L.off[x];
    const int64_t n = L.rows[x] * L.cols[x];
    for (int64_t q = 0; q < n; ++q) p[q] = -bound + (bound - (-bound)) * st.unit();
  }
  const int64_t dt = m.d_time;
  for (int64_t i = 0; i < dt; ++i) {
    const double frac = dt == 1 ? 1.0 : static_cast<double>(i) / static_cast<double>(dt - 1);
    flat[static_cast<size_t>(L.off[tOmega] + i)] =
        std::pow(10.0, -5.0 * (1.0 - frac)) / std::max(m.max_t, 1e-12);
  }
  return flat;
}

}  // namespace

// ----------------------------------------------------------------- handles
constexpr int kFlagIngest = 2;  // d_flag bit: an ingested event differed from the indexed one

__global__ void ingest_verify_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                     const double* __restrict__ t, const int32_t* __restrict__ g_src,
                                     const int32_t* __restrict__ g_dst, const double* __restrict__ g_t,
                                     int64_t count, int* flag) {
  bool bad = false;
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < count;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= src[x] != g_src[x] || dst[x] != g_dst[x] || __double_as_longlong(t[x]) != __double_as_longlong(g_t[x]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, kFlagIngest);
}

struct tgnn_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // plan-only work overlapped with the step
  cudaStream_t comm = nullptr;  // gradient all-reduce buckets overlapped with the GRU backward
  cudaStream_t aux = nullptr;   // next barrier's plan / read, overlapped with this barrier's step
  cudaStream_t br = nullptr;    // leaves of the step (gradient zeroing, root writes, loss)
  cudaStream_t edge = nullptr;  // per-pair edge projection, overlapped with the GRU
  cudaStream_t h2d = nullptr;   // event ingestion (copy engine), overlapped with earlier work
  cudaEvent_t ev_h2d = nullptr;
  cudaStream_t xch = nullptr;   // i-axis write exchange (broadcast + apply), off the critical path
  cudaStream_t hd = nullptr;    // the head gradient bucket's all-reduce + Adam (its own communicator)
  cudaStream_t d2h = nullptr;   // asynchronous result reads, off the compute stream
  cudaEvent_t ev_d2h = nullptr;
  int* d_flag = nullptr;

  void check_numeric() {
    int f = 0;
    TGB_CUDA(cudaMemcpyAsync(&f, d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
    TGB_CUDA(cudaStreamSynchronize(stream));
    if (f) {
      TGB_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), stream));
      if (f & kFlagIngest)
        throw Error(kProtocol, "ingest: events differ from the finalized graph (src, dst and t must match "
                               "the indexed stream; only edge features may be rewritten)");
      throw Error(kNumeric, "non-finite value in the training step");
    }
  }
  void use() const { TGB_CUDA(cudaSetDevice(device)); }
};

struct tgnn_graph {
  tgnn_ctx* ctx = nullptr;
  DGraph d;
  // tgnn_graph_ingest staging: incoming src / dst / t are verified against
  // the finalized (indexed) events instead of overwriting them
  int32_t* st_src = nullptr;
  int32_t* st_dst = nullptr;
  double* st_t = nullptr;
  int64_t st_cap = 0;
  ~tgnn_graph() {
    void* ptrs[] = {d.src, d.dst, d.t, d.inc_ptr, d.inc_t, d.inc_eid, d.inc_nbr, d.efeat, st_src, st_dst, st_t};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

struct tgnn_memstore {
  tgnn_ctx* ctx = nullptr;
  DMem d;
  int32_t* win = nullptr;
  ~tgnn_memstore() {
    void* ptrs[] = {d.memory, d.mail_mem, d.last_update, d.mail_t, d.mail_dt, d.mail_ev, win};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

namespace {

void plan_alloc(DPlan& pl, int cap_B, int n, int cap_U, int64_t N, int rpe = 3, int routing = 1,
                int eval_negs = 0) {
  pl.cap_B = cap_B;
  pl.n = n;
  pl.rpe = rpe;
  pl.routing = routing;
  pl.eval_negs = eval_negs;
  pl.cap_R = rpe * cap_B;
  pl.cap_P = pl.cap_R * (n > 0 ? n : 1);
  pl.cap_U = cap_U;
  pl.args = dalloc<PlanArgs>(1);
  pl.sizes = dalloc<int32_t>(kSzCount);
  TGB_CUDA(cudaMemset(pl.sizes, 0, sizeof(int32_t) * kSzCount));
  pl.negs = dalloc<int32_t>(static_cast<size_t>(cap_B) * std::max(rpe - 2, 1));
  pl.root_node = dalloc<int32_t>(pl.cap_R);
  pl.root_t = dalloc<double>(pl.cap_R);
  pl.nbr_cnt = dalloc<int32_t>(pl.cap_R);
  const size_t slots = static_cast<size_t>(pl.cap_R) * (n > 0 ? n : 1);
  pl.slot_node = dalloc<int32_t>(slots);
  pl.slot_event = dalloc<int32_t>(slots);
  pl.slot_dt = dalloc<double>(slots);
  pl.pair_ptr = dalloc<int32_t>(pl.cap_R + 1);
  pl.pair_node = dalloc<int32_t>(pl.cap_P);
  pl.pair_event = dalloc<int32_t>(pl.cap_P);
  pl.pair_root = dalloc<int32_t>(pl.cap_P);
  pl.pair_sup = dalloc<int32_t>(pl.cap_P);
  pl.pair_dt = dalloc<double>(pl.cap_P);
  pl.root_sup = dalloc<int32_t>(pl.cap_R);
  pl.supports = dalloc<int32_t>(cap_U);
  pl.sup_row = dalloc<int32_t>(static_cast<size_t>(N));
  const int items = pl.cap_R + pl.cap_P;
  pl.item_key = dalloc<int32_t>(items);
  pl.item_val = dalloc<int32_t>(items);
  pl.item_key_s = dalloc<int32_t>(items);
  pl.item_val_s = dalloc<int32_t>(items);
  pl.sup_item_ptr = dalloc<int32_t>(cap_U + 1);
  int bits = 1;
  while ((1ll << bits) <= cap_U) ++bits;
  pl.sort_bits = bits;
  pl.sort_tmp_bytes = plan_sort_tmp_bytes(items, bits);
  TGB_CUDA(cudaMalloc(&pl.sort_tmp, pl.sort_tmp_bytes > 0 ? pl.sort_tmp_bytes : 1));
  TGB_CUDA(cudaEventCreateWithFlags(&pl.ev_pairs, cudaEventDisableTiming));
  TGB_CUDA(cudaEventCreateWithFlags(&pl.ev_sorted, cudaEventDisableTiming));
  pl.bitmap = dalloc<uint32_t>(static_cast<size_t>((N + 31) / 32));
  TGB_CUDA(cudaMemset(pl.bitmap, 0, sizeof(uint32_t) * ((N + 31) / 32)));
}

void plan_free(DPlan& pl) {
  void* ptrs[] = {pl.args, pl.sizes, pl.negs, pl.root_node, pl.root_t, pl.nbr_cnt, pl.slot_node,
                  pl.slot_event, pl.slot_dt, pl.pair_ptr, pl.pair_node, pl.pair_event, pl.pair_root,
                  pl.pair_sup, pl.pair_dt, pl.root_sup, pl.supports, pl.sup_row, pl.item_key,
                  pl.item_val, pl.item_key_s, pl.item_val_s, pl.sup_item_ptr, pl.sort_tmp,
                  pl.bitmap};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (pl.ev_pairs) cudaEventDestroy(pl.ev_pairs);
  if (pl.ev_sorted) cudaEventDestroy(pl.ev_sorted);
  pl = DPlan{};
}

void view_alloc(DView& v, int cap_U, int64_t d) {
  v.cap_U = cap_U;
  v.mem = dalloc<float>(static_cast<size_t>(cap_U) * d);
  v.mail_mem = dalloc<float>(static_cast<size_t>(cap_U) * 2 * d);
  v.mail_t = dalloc<double>(cap_U);
  v.mail_dt = dalloc<double>(cap_U);
  v.mail_ev = dalloc<int32_t>(cap_U);
}

void view_free(DView& v) {
  void* ptrs[] = {v.mem, v.mail_mem, v.mail_t, v.mail_dt, v.mail_ev};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  v = DView{};
}

int cap_U_for(int64_t N, int cap_B, int64_t n) {
  const int64_t c = std::min<int64_t>(N, 3ll * cap_B * (n + 1));
  return static_cast<int>(std::max<int64_t>(c, 1));
}

}  // namespace

struct tgnn_trainer {
  tgnn_ctx* ctx = nullptr;
  tgnn_graph* g = nullptr;
  ModelDims m;
  ParamLayout L;
  uint64_t seed = 1;
  float *params = nullptr, *grads = nullptr, *am = nullptr, *av = nullptr;
  int64_t adam_t = 0;
  StepWork w;
  std::vector<DPlan> plans;
  std::vector<DView> views;
  double* d_loss = nullptr;
  int cap_B = 0, cap_U = 0;
  int last_U = -1;

  StepCtx sc() {
    StepCtx c;
    c.m = m;
    c.L = L;
    c.g = &g->d;
    c.params = params;
    c.grads = grads;
    c.w = &w;
    c.d_numeric_flag = ctx->d_flag;
    return c;
  }

  void init(tgnn_ctx* cx, tgnn_graph* gr, const ModelDims& md, int64_t max_local_batch, uint64_t sd,
            int subs) {
    ctx = cx;
    g = gr;
    m = md;
    if (m.num_nodes <= 0) m.num_nodes = gr->d.N;
    TGB_REQUIRE(m.num_nodes == gr->d.N, kConfig, "model num_nodes does not match the dataset");
    TGB_REQUIRE(m.d_e == gr->d.d_e, kConfig, "model edge feature width does not match the dataset");
    validate_dims(m);
    TGB_REQUIRE(max_local_batch >= 1 && max_local_batch <= (1 << 24), kConfig,
                "trainer: local batch out of range");
    L = ParamLayout::make(m);
    seed = sd;
    cap_B = static_cast<int>(max_local_batch);
    cap_U = cap_U_for(m.num_nodes, cap_B, m.n_neighbors);
    params = dalloc<float>(L.total);
    grads = dalloc<float>(L.total);
    am = dalloc<float>(L.total);
    av = dalloc<float>(L.total);
    TGB_CUDA(cudaMemset(grads, 0, sizeof(float) * L.total));
    TGB_CUDA(cudaMemset(am, 0, sizeof(float) * L.total));
    TGB_CUDA(cudaMemset(av, 0, sizeof(float) * L.total));
    set_params(host_init_params(m, seed).data());
    step_alloc(w, m, cap_B, cap_U, m.num_nodes);
    // >= 2 slots: the graph-mode pipeline plans barrier b + 1 into the other slot
    subs = std::max(subs, 2);
    plans.resize(static_cast<size_t>(subs));
    views.resize(static_cast<size_t>(subs));
    for (int s = 0; s < subs; ++s) {
      plan_alloc(plans[static_cast<size_t>(s)], cap_B, static_cast<int>(m.n_neighbors), cap_U, m.num_nodes);
      view_alloc(views[static_cast<size_t>(s)], cap_U, m.d_mem);
    }
    d_loss = dalloc<double>(1);
  }

  void set_params(const double* flat) {
    std::vector<float> f(static_cast<size_t>(L.total));
    for (int64_t x = 0; x < L.total; ++x) f[static_cast<size_t>(x)] = static_cast<float>(flat[x]);
    TGB_CUDA(cudaMemcpy(params, f.data(), sizeof(float) * f.size(), cudaMemcpyHostToDevice));
  }
  void get_flat(const float* src, double* out) {
    std::vector<float> f(static_cast<size_t>(L.total));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    TGB_CUDA(cudaMemcpy(f.data(), src, sizeof(float) * f.size(), cudaMemcpyDeviceToHost));
    for (int64_t x = 0; x < L.total; ++x) out[x] = f[static_cast<size_t>(x)];
  }

  void adam(double lr, float grad_scale) {
    ++adam_t;
    const double c1 = 1.0 - std::pow(0.9, static_cast<double>(adam_t));
    const double c2 = 1.0 - std::pow(0.999, static_cast<double>(adam_t));
    adam_launch(params, grads, am, av, L.total, static_cast<float>(lr), static_cast<float>(c1),
                static_cast<float>(c2), grad_scale, ctx->stream);
  }

  ~tgnn_trainer() {
    step_free(w);
    for (auto& p : plans) plan_free(p);
    for (auto& v : views) view_free(v);
    void* ptrs[] = {params, grads, am, av, d_loss};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

// j > 1 graph mode: the stint-start barrier's per-sub plan args of this rank
// and, per team in pair order, whether the group's copy resets before its read.
constexpr int kMaxStintJ = 8;
struct StintDesc {
  PlanArgs args[kMaxStintJ];
  int32_t reset[kMaxStintJ];
};

// evaluate_mrr / replay_batch (trainer.hpp:336-468) on device: a private
// memory copy rebuilt by replaying the prefix, forward-only workspaces sized
// for 2 + n_negatives roots per event, and per-event rank counts that the host
// folds in event order (acc += 1 / (1 + worse_or_equal), as the reference).
struct tgnn_evaluator {
  tgnn_ctx* ctx = nullptr;
  tgnn_graph* g = nullptr;
  ModelDims m;
  ParamLayout L;
  int cap_B = 0, n_neg = 0;
  float* params = nullptr;
  StepWork w;
  DPlan pe, pr;  // evaluation plan (candidates + neighbours), replay plan (src, dst only)
  DView vw;
  std::unique_ptr<tgnn_memstore> st;
  int32_t* d_cnt = nullptr;
  int64_t cnt_cap = 0;

  StepCtx sc() {
    StepCtx c;
    c.m = m;
    c.L = L;
    c.g = &g->d;
    c.params = params;
    c.grads = nullptr;
    c.w = &w;
    c.d_numeric_flag = ctx->d_flag;
    return c;
  }

  void init(tgnn_ctx* cx, tgnn_graph* gr, const ModelDims& md, int64_t batch, int negatives);

  void set_params(const double* flat) {
    std::vector<float> f(static_cast<size_t>(L.total));
    for (int64_t x = 0; x < L.total; ++x) f[static_cast<size_t>(x)] = static_cast<float>(flat[x]);
    TGB_CUDA(cudaMemcpyAsync(params, f.data(), sizeof(float) * f.size(), cudaMemcpyHostToDevice, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  }

  // replay_batch over [begin, end) in slices of at most cap_B events.
  void replay(DMem& state, int64_t begin, int64_t end, int64_t batch) {
    cudaStream_t s = ctx->stream;
    StepCtx c = sc();
    for (int64_t b = begin; b < end; b += batch) {
      PlanArgs a;
      a.begin = b;
      a.end = std::min(end, b + batch);
      a.batch_begin = b;
      a.neg_mode = 0;
      a.valid = 1;
      set_plan_args_launch(pr.args, a, s);
      plan_launch(g->d, pr, s);
      gather_view_launch(pr, state, vw, s);
      substep_gru_launch(c, pr, vw, s);
      root_writes_launch(c, pr, vw, s, &state);
    }
  }

  double evaluate(int64_t eval_begin, int64_t eval_end, uint64_t seed, int64_t* queries) {
    const DGraph& G = g->d;
    TGB_REQUIRE(eval_begin >= 0 && eval_end <= G.E && eval_begin <= eval_end, kConfig,
                "evaluate_mrr: event range out of bounds");
    const int64_t lo = G.boundary >= 0 ? G.boundary : 0;
    TGB_REQUIRE(n_neg == 0 || G.N - lo >= 2, kConfig,
                "evaluate_mrr: destination partition too small to sample distractors");
    cudaStream_t s = ctx->stream;
    const int64_t Q = eval_end - eval_begin;
    if (Q > cnt_cap) {
      if (d_cnt) cudaFree(d_cnt);
      d_cnt = dalloc<int32_t>(static_cast<size_t>(Q));
      cnt_cap = Q;
    }
    reset_state_launch(st->d, s);
    replay(st->d, 0, eval_begin, cap_B);
    StepCtx c = sc();
    for (int64_t b = eval_begin; b < eval_end; b += cap_B) {
      PlanArgs a;
      a.begin = b;
      a.end = std::min(eval_end, b + cap_B);
      a.batch_begin = b;
      a.seed = seed;
      a.neg_mode = 2;
      a.valid = 1;
      set_plan_args_launch(pe.args, a, s);
      plan_launch(G, pe, s);
      gather_view_launch(pe, st->d, vw, s);
      substep_gru_launch(c, pe, vw, s);
      attn_forward_launch(c, pe, s);
      eval_rank_launch(c, pe, d_cnt, eval_begin, s);
      // the batch's replay: its roots' s_hat are the ones just computed
      root_writes_launch(c, pe, vw, s, &st->d);
    }
    std::vector<int32_t> cnt(static_cast<size_t>(Q));
    d2h(cnt.data(), d_cnt, static_cast<size_t>(Q), s);
    ctx->check_numeric();
    double acc = 0.0;
    for (int64_t q = 0; q < Q; ++q) acc += 1.0 / static_cast<double>(1 + cnt[static_cast<size_t>(q)]);
    *queries = Q;
    return Q > 0 ? acc / static_cast<double>(Q) : 0.0;
  }

  ~tgnn_evaluator() {
    step_free(w);
    plan_free(pe);
    plan_free(pr);
    view_free(vw);
    if (params) cudaFree(params);
    if (d_cnt) cudaFree(d_cnt);
  }
};

// In-process communicator (include/tgnn_b200.h, tgnn_local_hub): the ranks of
// a job are host threads of ONE process -- the reference's own threading model
// (trainer threads sharing host arrays, trainer.hpp:671-674) -- on one device
// or several. A collective is a host rendezvous at enqueue time plus cross-
// stream CUDA events: every rank publishes its buffer and a ready event, waits
// for the others' events, reduces ALL ranks' buffers in ascending rank order
// into private scratch (so every replica computes the identical sum, the
// reference's average_active_grads order, trainer.hpp:473-483), then, after a
// second rendezvous (nobody still reads its input), copies the result back.
// Nothing spins on the device; a rank that never arrives times out the others.
constexpr int kLocalMax = 16;
struct tgnn_local_hub {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<tgnn_run*> runs;
  std::vector<const void*> src;

  void rendezvous() {
    static const int secs = [] {
      const char* e = std::getenv("TGNN_LOCAL_TIMEOUT_S");
      const int v = e ? std::atoi(e) : 0;
      return v > 0 ? v : 300;
    }();
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw Error(kProtocol, "local hub: another rank failed");
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(secs), [&] { return gen != g || broken; });
    if (!ok) {
      broken = true;
      cv.notify_all();
      throw Error(kProtocol, "local hub: rendezvous timed out (a rank stopped issuing collectives)");
    }
    if (gen == g) throw Error(kProtocol, "local hub: another rank failed");
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

struct tgnn_run {
  tgnn_ctx* ctx = nullptr;
  tgnn_graph* g = nullptr;
  std::unique_ptr<tgnn_trainer> tr;
  std::unique_ptr<tgnn_memstore> mem;
  host::Schedule sched;
  host::TrainCfg tc;
  int rank = 0, nranks = 1;
  int group = 0, team = 0, member = 0, group_size = 1;
  ncclComm_t comm = nullptr, gcomm = nullptr;
  ncclComm_t hcomm = nullptr;  // duplicate of comm for the head bucket (its own stream, no FIFO behind the tail)
  // graph capture of consecutive barriers: the tail range's update (all-reduce
  // + Adam of attention / static / decoder, 88 % of the parameters) may finish
  // under the NEXT barrier's GRU forward; its first reader waits for it
  bool defer_tail = false, tail_pending = false;
  bool comm_ready = false;
  // in-process exchange (tgnn_run_local_init) instead of NCCL
  tgnn_local_hub* hub = nullptr;
  cudaEvent_t ev_lready = nullptr, ev_ldone = nullptr;
  void* lscratch = nullptr;
  size_t lscratch_bytes = 0;
  double* d_losses = nullptr;
  void* gathered = nullptr;  // [i, wpack_bytes]
  int64_t next_barrier = 0;
  int64_t launches = -1;
  PhaseMarks marks;
  bool marks_ready = false;
  // CUDA-graph mode (j == 1): per-barrier descriptors + a device counter make
  // every barrier the same graph, captured once and relaunched.
  bool use_graphs = false;
  BarrierDesc* d_desc = nullptr;
  int* d_ctr = nullptr;
  // the tail-range Adam's own barrier counter: deferred inside a multi-barrier
  // graph it may run after the main stream advanced d_ctr, so it keeps its own
  // (advanced on the tail chain's stream right after the update)
  int* d_ctr_tail = nullptr;
  cudaGraph_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // barrier b runs exec[b % 2]
  // kMultiBarrier consecutive barriers (from an even b) captured as one graph:
  // fewer graph launches, so the device starts each barrier's first kernel sooner
  cudaGraph_t mgraph = nullptr;
  cudaGraphExec_t mexec = nullptr;
  // j > 1: one graph per sub-iteration position s = b % j (a whole stint is
  // j consecutive launches); per-stint plan args and team resets in d_stint
  // (j > 1: 2 j of them -- [plan set][position]; a stint's j plans live in
  // set (stint start / j) % 2, and the previous stint's last position plans
  // the next stint into the other set on the aux stream)
  std::vector<cudaGraph_t> sgraph;
  std::vector<cudaGraphExec_t> sexec;
  StintDesc* d_stint = nullptr;
  std::vector<StintDesc> h_stint;  // host copy (eager planning of a stint)
  int64_t stint_planned = -1;      // stint start whose plans the graphs prepared ahead
  int64_t prepared = -1;  // barrier whose plan + read view are ready in plans/views[b % 2]
  cudaEvent_t ev_fork = nullptr, ev_written = nullptr, ev_next = nullptr;
  cudaEvent_t ev_gru = nullptr, ev_gzero = nullptr, ev_dec = nullptr, ev_brjoin = nullptr, ev_edge = nullptr;
  cudaEvent_t ev_red = nullptr, ev_artail = nullptr, ev_upd = nullptr, ev_mid = nullptr;
  cudaEvent_t ev_tail = nullptr, ev_head = nullptr, ev_comm = nullptr;
  // segment snapshots (DaemonOp::Snapshot): slot per snapshot pair of this
  // rank's memory copy, memory + last_update copied after the pair's writes
  bool snaps = false;
  std::vector<int64_t> snap_slot;            // per pair of the group (-1: none)
  std::vector<std::array<int64_t, 2>> snap_meta;  // sweep, segment per slot
  int64_t snap_taken = 0;
  float* d_snap_mem = nullptr;
  double* d_snap_lu = nullptr;
  // daemon op-log records [barriers x 4] (R first, R len, W first, W len)
  bool oplog = false;
  int64_t* d_oplog = nullptr;
  // validation / metrics rows (run_training, trainer.hpp:725-743)
  int64_t val_begin = 0, val_end = 0, eval_batch = 0;
  int eval_negatives = 49;
  std::unique_ptr<tgnn_evaluator> ev;
  size_t eval_cursor = 0;
  cudaEvent_t ev_t0 = nullptr;
  struct Row {
    int64_t barrier = 0;
    double val_mrr = 0;
    cudaEvent_t done = nullptr;
  };
  std::vector<Row> rows;

  ~tgnn_run() {
    if (d_oplog) cudaFree(d_oplog);
    if (d_snap_mem) cudaFree(d_snap_mem);
    if (d_snap_lu) cudaFree(d_snap_lu);
    for (Row& row : rows)
      if (row.done) cudaEventDestroy(row.done);
    if (ev_t0) cudaEventDestroy(ev_t0);
    if (ev_tail) cudaEventDestroy(ev_tail);
    if (ev_head) cudaEventDestroy(ev_head);
    if (ev_comm) cudaEventDestroy(ev_comm);
    for (int p = 0; p < 2; ++p) {
      if (exec[p]) cudaGraphExecDestroy(exec[p]);
      if (graph[p]) cudaGraphDestroy(graph[p]);
    }
    if (mexec) cudaGraphExecDestroy(mexec);
    if (mgraph) cudaGraphDestroy(mgraph);
    for (auto e : sexec)
      if (e) cudaGraphExecDestroy(e);
    for (auto g : sgraph)
      if (g) cudaGraphDestroy(g);
    if (d_stint) cudaFree(d_stint);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_written) cudaEventDestroy(ev_written);
    if (ev_next) cudaEventDestroy(ev_next);
    cudaEvent_t more[] = {ev_gru, ev_gzero, ev_dec, ev_brjoin, ev_edge, ev_red, ev_artail, ev_upd, ev_mid};
    for (cudaEvent_t e : more)
      if (e) cudaEventDestroy(e);
    if (d_desc) cudaFree(d_desc);
    if (d_ctr) cudaFree(d_ctr);
    if (d_ctr_tail) cudaFree(d_ctr_tail);
    if (ev_lready) cudaEventDestroy(ev_lready);
    if (ev_ldone) cudaEventDestroy(ev_ldone);
    if (lscratch) cudaFree(lscratch);
    if (hcomm) nccl::api().CommDestroy(hcomm);
    if (gcomm) nccl::api().CommDestroy(gcomm);
    if (comm) nccl::api().CommDestroy(comm);
    if (d_losses) cudaFree(d_losses);
    if (gathered) cudaFree(gathered);
  }
};

// ----------------------------------------------------------------- runtime pieces
namespace {

// ----------------------------------------------------------------- exchange
// Every collective of a run goes through comm_allreduce / comm_bcast_packs:
// NCCL over NVLink (one process per GPU, tgnn_run_comm_init) or the in-process
// hub (tgnn_run_local_init). Both backends see the same call sequence on
// every rank, so the op-log, the schedule and the replicas are unchanged.
enum class RedTy { F32, F64, U64 };
enum class RedOp { Sum, Min, Max };

struct LocalSrcs {
  const void* p[kLocalMax];
  int n;
};

template <typename T, int OP>
__global__ void local_reduce_kernel(LocalSrcs src, int64_t count, T* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < count; x += stride) {
    T acc = static_cast<const T*>(src.p[0])[x];
    for (int q = 1; q < src.n; ++q) {  // ascending rank order
      const T v = static_cast<const T*>(src.p[q])[x];
      acc = OP == 0 ? acc + v : OP == 1 ? (v < acc ? v : acc) : (v > acc ? v : acc);
    }
    out[x] = acc;
  }
}

size_t red_size(RedTy t) { return t == RedTy::F32 ? 4 : 8; }

template <typename T>
void local_reduce_typed(RedOp op, const LocalSrcs& src, int64_t count, void* out, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>((count + 255) / 256, 4 * num_sms()));
  if (count <= 0) return;
  if (op == RedOp::Sum) local_reduce_kernel<T, 0><<<grid, 256, 0, s>>>(src, count, static_cast<T*>(out));
  else if (op == RedOp::Min) local_reduce_kernel<T, 1><<<grid, 256, 0, s>>>(src, count, static_cast<T*>(out));
  else local_reduce_kernel<T, 2><<<grid, 256, 0, s>>>(src, count, static_cast<T*>(out));
  TGB_CUDA(cudaGetLastError());
}

// Marks the hub broken when a collective-issuing call fails on one rank, so
// the other ranks fail at their next rendezvous instead of timing out.
struct HubGuard {
  tgnn_run* r;
  bool armed = true;
  explicit HubGuard(tgnn_run* run) : r(run) {}
  ~HubGuard() {
    if (armed && r->hub) r->hub->fail();
  }
  void ok() { armed = false; }
};

void local_wait_all(tgnn_run* r, bool done, cudaStream_t s) {
  tgnn_local_hub* h = r->hub;
  for (int q = 0; q < h->n; ++q)
    if (q != r->rank) TGB_CUDA(cudaStreamWaitEvent(s, done ? h->runs[q]->ev_ldone : h->runs[q]->ev_lready, 0));
}

void comm_allreduce(tgnn_run* r, void* buf, size_t count, RedTy ty, RedOp op, cudaStream_t s,
                    ncclComm_t nc = nullptr) {
  if (r->nranks == 1 || count == 0) return;
  if (r->hub) {
    tgnn_local_hub* h = r->hub;
    const size_t bytes = count * red_size(ty);
    if (r->lscratch_bytes < bytes) {
      if (r->lscratch) {
        TGB_CUDA(cudaStreamSynchronize(s));
        cudaFree(r->lscratch);
      }
      r->lscratch = dalloc<char>(bytes);
      r->lscratch_bytes = bytes;
    }
    h->src[static_cast<size_t>(r->rank)] = buf;
    TGB_CUDA(cudaEventRecord(r->ev_lready, s));
    h->rendezvous();
    local_wait_all(r, false, s);
    LocalSrcs src{};
    src.n = h->n;
    for (int q = 0; q < h->n; ++q) src.p[q] = h->src[static_cast<size_t>(q)];
    if (ty == RedTy::F32) local_reduce_typed<float>(op, src, static_cast<int64_t>(count), r->lscratch, s);
    else if (ty == RedTy::F64) local_reduce_typed<double>(op, src, static_cast<int64_t>(count), r->lscratch, s);
    else local_reduce_typed<unsigned long long>(op, src, static_cast<int64_t>(count), r->lscratch, s);
    TGB_CUDA(cudaEventRecord(r->ev_ldone, s));
    h->rendezvous();  // every rank has enqueued its reads of every input
    local_wait_all(r, true, s);
    TGB_CUDA(cudaMemcpyAsync(buf, r->lscratch, bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  const ncclDataType_t dt = ty == RedTy::F32 ? ncclFloat : ty == RedTy::F64 ? ncclDouble : ncclUint64;
  const ncclRedOp_t o = op == RedOp::Sum ? ncclSum : op == RedOp::Min ? ncclMin : ncclMax;
  NCCL_CHECK(nccl::api().AllReduce(buf, buf, count, dt, o, nc ? nc : r->comm, s));
}

// The flat gradient in the two buckets of the graph pipeline's split-phase
// update (update_split): tail [split, end) on the global communicator, head
// [0, split) on its duplicate -- the same NCCL calls, so the direct path
// reproduces the graph path's sums bitwise at any rank count.
int64_t grad_split(const tgnn_trainer* tr) { return (tr->L.off[tWq] + 3) / 4 * 4; }

void comm_allreduce_grads(tgnn_run* r, cudaStream_t s) {
  tgnn_trainer* tr = r->tr.get();
  const int64_t split = grad_split(tr);
  comm_allreduce(r, tr->grads + split, static_cast<size_t>(tr->L.total - split), RedTy::F32, RedOp::Sum, s);
  comm_allreduce(r, tr->grads, static_cast<size_t>(split), RedTy::F32, RedOp::Sum, s, r->hcomm);
}

// The write packs of team `team`'s i members into r->gathered[member]
// (memory group exchange of the i-axis): grouped NCCL broadcasts
// over the group communicator, or device copies from the members' packs.
void comm_bcast_packs(tgnn_run* r, int team, cudaStream_t s) {
  tgnn_trainer* tr = r->tr.get();
  const size_t pb = tr->w.wpack_bytes;
  const int i = r->tc.i;
  char* dst = static_cast<char*>(r->gathered);
  if (r->hub) {
    tgnn_local_hub* h = r->hub;
    h->src[static_cast<size_t>(r->rank)] = tr->w.wpack;
    TGB_CUDA(cudaEventRecord(r->ev_lready, s));
    h->rendezvous();
    const int base = r->group * i * r->tc.j + team * i;
    for (int mm = 0; mm < i; ++mm) {
      const int q = base + mm;
      if (q != r->rank) TGB_CUDA(cudaStreamWaitEvent(s, h->runs[static_cast<size_t>(q)]->ev_lready, 0));
      TGB_CUDA(cudaMemcpyAsync(dst + static_cast<size_t>(mm) * pb, h->src[static_cast<size_t>(q)], pb,
                               cudaMemcpyDefault, s));
    }
    TGB_CUDA(cudaEventRecord(r->ev_ldone, s));
    h->rendezvous();  // every reader has enqueued its copy of every pack
    local_wait_all(r, true, s);
    return;
  }
  NCCL_CHECK(nccl::api().GroupStart());
  for (int mm = 0; mm < i; ++mm)
    NCCL_CHECK(nccl::api().Broadcast(tr->w.wpack, dst + static_cast<size_t>(mm) * pb, pb, ncclChar, team * i + mm,
                                     r->gcomm, s));
  NCCL_CHECK(nccl::api().GroupEnd());
}

// Applies the gathered packs in ascending member order (later members win on
// equal nodes: memory_daemon.hpp:35-38).
void apply_gathered(tgnn_run* r, cudaStream_t s) {
  tgnn_trainer* tr = r->tr.get();
  const size_t pb = tr->w.wpack_bytes;
  std::vector<WriteSet> sets;
  for (int mm = 0; mm < r->tc.i; ++mm)
    sets.push_back(pack_view(static_cast<char*>(r->gathered) + static_cast<size_t>(mm) * pb, 2 * tr->cap_B,
                             tr->m.d_mem));
  apply_writes_launch(sets, r->mem->d, r->mem->win, s);
}


tgnn_memstore* memstore_new(tgnn_ctx* ctx, int64_t N, int64_t d) {
  TGB_REQUIRE(N > 0 && d > 0, kConfig, "memstore: invalid shape");
  auto* m = new tgnn_memstore();
  m->ctx = ctx;
  m->d.N = N;
  m->d.d = d;
  m->d.memory = dalloc<float>(static_cast<size_t>(N * d));
  m->d.mail_mem = dalloc<float>(static_cast<size_t>(N * 2 * d));
  m->d.last_update = dalloc<double>(N);
  m->d.mail_t = dalloc<double>(N);
  m->d.mail_dt = dalloc<double>(N);
  m->d.mail_ev = dalloc<int32_t>(N);
  m->win = dalloc<int32_t>(N);
  TGB_CUDA(cudaMemset(m->win, 0, sizeof(int32_t) * N));
  reset_state_launch(m->d, ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  return m;
}

void upload_view(tgnn_trainer* tr, DView& v, int U, const double* view_mem, const double* view_mail) {
  const int64_t d = tr->m.d_mem, mw = 2 * d + 3;
  std::vector<float> mem(static_cast<size_t>(U * d)), mail(static_cast<size_t>(U * 2 * d));
  std::vector<double> mt(U), mdt(U);
  std::vector<int32_t> mev(U);
  for (int64_t u = 0; u < U; ++u) {
    for (int64_t x = 0; x < d; ++x) mem[u * d + x] = static_cast<float>(view_mem[u * d + x]);
    for (int64_t x = 0; x < 2 * d; ++x) mail[u * 2 * d + x] = static_cast<float>(view_mail[u * mw + x]);
    mt[u] = view_mail[u * mw + 2 * d];
    mdt[u] = view_mail[u * mw + 2 * d + 1];
    mev[u] = static_cast<int32_t>(view_mail[u * mw + 2 * d + 2]);
  }
  TGB_CUDA(cudaMemcpy(v.mem, mem.data(), sizeof(float) * mem.size(), cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(v.mail_mem, mail.data(), sizeof(float) * mail.size(), cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(v.mail_t, mt.data(), sizeof(double) * U, cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(v.mail_dt, mdt.data(), sizeof(double) * U, cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(v.mail_ev, mev.data(), sizeof(int32_t) * U, cudaMemcpyHostToDevice));
}

int plan_size(tgnn_ctx* ctx, const DPlan& pl, SizeIdx which) {
  int32_t sz[kSzCount];
  TGB_CUDA(cudaMemcpyAsync(sz, pl.sizes, sizeof(sz), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  return sz[which];
}

// Plan with explicit negatives (parity path) on plans[slot].
void plan_explicit(tgnn_trainer* tr, int slot, int64_t begin, int64_t end, const int64_t* negatives) {
  tgnn_ctx* ctx = tr->ctx;
  const DGraph& g = tr->g->d;
  TGB_REQUIRE(begin >= 0 && end <= g.E && begin <= end, kConfig,
              "plan_sub_batch: event range out of bounds");
  TGB_REQUIRE(end - begin <= tr->cap_B, kConfig, "plan_sub_batch: slice exceeds the trainer capacity");
  DPlan& pl = tr->plans[static_cast<size_t>(slot)];
  const int64_t B = end - begin;
  std::vector<int32_t> negs(static_cast<size_t>(B));
  for (int64_t x = 0; x < B; ++x) {
    TGB_REQUIRE(negatives[x] >= 0 && negatives[x] < g.N, kConfig, "plan_sub_batch: negative out of range");
    negs[static_cast<size_t>(x)] = static_cast<int32_t>(negatives[x]);
  }
  TGB_CUDA(cudaMemcpyAsync(pl.negs, negs.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, ctx->stream));
  PlanArgs a;
  a.begin = begin;
  a.end = end;
  a.batch_begin = begin;
  a.seed = tr->seed;
  a.neg_mode = 0;
  a.valid = 1;
  set_plan_args_launch(pl.args, a, ctx->stream);
  plan_launch(g, pl, ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
}

// DaemonOp::Snapshot (memory_daemon.hpp:94-105): the replica's memory and
// last_update after the write bracket of `pair`, when the pair closes its
// segment (parallel.hpp:288-290).
void take_snapshot(tgnn_run* r, int64_t pair, cudaStream_t s) {
  if (pair < 0 || pair >= static_cast<int64_t>(r->snap_slot.size())) return;
  const int64_t slot = r->snap_slot[static_cast<size_t>(pair)];
  if (slot < 0) return;
  const DMem& st = r->mem->d;
  TGB_CUDA(cudaMemcpyAsync(r->d_snap_mem + slot * st.N * st.d, st.memory, sizeof(float) * st.N * st.d,
                           cudaMemcpyDeviceToDevice, s));
  TGB_CUDA(cudaMemcpyAsync(r->d_snap_lu + slot * st.N, st.last_update, sizeof(double) * st.N,
                           cudaMemcpyDeviceToDevice, s));
  r->snap_taken = std::max(r->snap_taken, slot + 1);
}

// One barrier of a run on this rank (TrainerCore::iterate + the daemon's
// read/write brackets + average_active_grads + Adam::step).
void run_barrier(tgnn_run* r, int64_t b) {
  r->prepared = -1;  // the direct path reuses slot 0
  tgnn_ctx* ctx = r->ctx;
  tgnn_trainer* tr = r->tr.get();
  cudaStream_t s = ctx->stream;
  const host::TrainCfg& c = r->tc;
  const host::Task t = r->sched.task(r->rank, b);
  StepCtx sc = tr->sc();
  sc.marks = r->marks.on ? &r->marks : nullptr;
  sc.mark(phPlan, s);
  double* loss_slot = r->d_losses + b;
  const int i = c.i, j = c.j;
  // j > 1: the stint's plan set (shared with the stint graphs, so the two
  // paths can alternate mid-stint)
  const size_t base = j > 1 ? static_cast<size_t>(((b / j) % 2) * j) : 0;
  std::vector<DPlan>& plans = tr->plans;
  std::vector<DView>& views = tr->views;
  if (b % j == 0) {
    // Stint start: the group's teams read and write in pair order (the
    // daemon plan's R/W brackets, parallel.hpp:278-291). A team publishes its
    // root writes right after its GRU freshen; the rows are identical to the
    // reference's post-step writes (they depend only on the read view and s_hat).
    for (int tt = 0; tt < j; ++tt) {
      const int probe = r->group * i * j + tt * i;  // member 0 of team tt
      const host::Task tk = r->sched.task(probe, b);
      if (!tk.active) continue;
      if (tk.reset_before) reset_state_launch(r->mem->d, s);
      if (tt == r->team) {
        for (int sub = 0; sub < t.subs; ++sub) {
          PlanArgs a;
          a.begin = t.slice_begin;
          a.end = t.slice_end;
          a.batch_begin = t.batch_begin;
          a.batch_index = t.batch;
          a.group = t.neg_group[static_cast<size_t>(sub)];
          a.seed = c.seed;
          a.neg_mode = 1;
          a.valid = 1;
          DPlan& pl = plans[base + static_cast<size_t>(sub)];
          set_plan_args_launch(pl.args, a, s);
          plan_launch(r->g->d, pl, s, ctx->side);
          gather_view_launch(pl, r->mem->d, views[base + static_cast<size_t>(sub)], s);
        }
        substep_gru_launch(sc, plans[base], views[base], s);
        sc.mark(phWrites, s);
        root_writes_launch(sc, plans[base], views[base], s, r->group_size > 1 ? nullptr : &r->mem->d);
        if (r->oplog) {
          OplogPlans op;
          op.n = std::min(t.subs, 8);
          for (int x = 0; x < op.n; ++x) {
            op.sizes[x] = plans[base + static_cast<size_t>(x)].sizes;
            op.supports[x] = plans[base + static_cast<size_t>(x)].supports;
          }
          oplog_record_launch(sc, op, r->d_oplog, b, s);
        }
      }
      if (r->group_size > 1) {
        comm_bcast_packs(r, tt, s);
        apply_gathered(r, s);
      }
      if (r->snaps) take_snapshot(r, (b / j) * j + tt, s);
    }
    if (t.active) {
      substep_rest_launch(sc, plans[base], views[base], loss_slot, s);
    } else {
      TGB_CUDA(cudaMemsetAsync(tr->grads, 0, sizeof(float) * tr->L.total, s));
      TGB_CUDA(cudaMemsetAsync(loss_slot, 0, sizeof(double), s));
    }
  } else {
    if (t.active) {
      substep_launch(sc, plans[base + static_cast<size_t>(t.sub)], views[base + static_cast<size_t>(t.sub)],
                     loss_slot, s);
    } else {
      TGB_CUDA(cudaMemsetAsync(tr->grads, 0, sizeof(float) * tr->L.total, s));
      TGB_CUDA(cudaMemsetAsync(loss_slot, 0, sizeof(double), s));
    }
  }
  // average_active_grads (trainer.hpp:473-483): idle ranks contribute zeros.
  sc.mark(phAllreduce, s);
  comm_allreduce_grads(r, s);
  const int64_t active = r->sched.active_trainers[static_cast<size_t>(b)];
  sc.mark(phAdam, s);
  tr->adam_t = b;  // Adam's step counter advances on every rank at every barrier
  tr->adam(c.lr_eff(), 1.0f / static_cast<float>(active > 0 ? active : 1));
  sc.mark(phCount, s);
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// average_active_grads (trainer.hpp:473-483) as two NCCL buckets on the comm
// stream: [off[tWq], end) once ev_tail fires (overlapping the GRU backward),
// then [0, off[tWq]) after the step; the compute stream waits before Adam.
// Split-phase update: the tail range [off[tWq], end) -- attention, static
// table, decoder, 88 % of the parameters -- is final once ev_tail fires
// (after gru_bwd1): it is all-reduced (N > 1) and Adam-updated on a side
// stream while the GRU backward still runs; the head range [0, off[tWq))
// follows after the step. (The omega gradient's attention part reads the old
// Wk / Wv time rows before ev_tail.)
void update_split(tgnn_run* r, const StepCtx& sc, cudaStream_t s) {
  tgnn_trainer* tr = r->tr.get();
  cudaStream_t c = r->nranks > 1 ? r->ctx->comm : r->ctx->br;
  // 16-byte aligned split: the few Wq entries below it join the head bucket
  const int64_t split = grad_split(tr);
  TGB_CUDA(cudaStreamWaitEvent(c, r->ev_tail, 0));
  if (c != r->ctx->br) TGB_CUDA(cudaStreamWaitEvent(c, r->ev_brjoin, 0));  // the branch's tail gradients
  cudaStream_t u = c;  // the tail update
  if (r->nranks > 1) {
    NCCL_CHECK(nccl::api().AllReduce(tr->grads + split, tr->grads + split, static_cast<size_t>(tr->L.total - split),
                                          ncclFloat, ncclSum, r->comm, c));
    // the tail Adam on the (idle by now) branch stream
    TGB_CUDA(cudaEventRecord(r->ev_artail, c));
    TGB_CUDA(cudaStreamWaitEvent(r->ctx->br, r->ev_artail, 0));
    u = r->ctx->br;
  }
  adam_pack_launch(sc, tr->am, tr->av, u, r->d_desc, r->d_ctr_tail, split, tr->L.total);
  incr_launch(r->d_ctr_tail, u);
  TGB_CUDA(cudaEventRecord(r->ev_upd, u));
  if (r->nranks > 1) {
    // the head bucket (omega + GRU, the next barrier's first readers) on its
    // own stream and communicator: not queued behind the tail all-reduce
    cudaStream_t h = r->ctx->hd;
    TGB_CUDA(cudaEventRecord(r->ev_head, s));
    TGB_CUDA(cudaStreamWaitEvent(h, r->ev_head, 0));
    NCCL_CHECK(nccl::api().AllReduce(tr->grads, tr->grads, static_cast<size_t>(split), ncclFloat, ncclSum, r->hcomm, h));
    adam_pack_launch(sc, tr->am, tr->av, h, r->d_desc, r->d_ctr, 0, split);
    TGB_CUDA(cudaEventRecord(r->ev_comm, h));
    TGB_CUDA(cudaStreamWaitEvent(s, r->ev_comm, 0));
  } else {
    adam_pack_launch(sc, tr->am, tr->av, s, r->d_desc, r->d_ctr, 0, split);
  }
  if (r->defer_tail) {
    r->tail_pending = true;  // the next barrier of this capture waits before its first tail read
  } else {
    TGB_CUDA(cudaStreamWaitEvent(s, r->ev_upd, 0));
    r->tail_pending = false;
  }
}

void barrier_body_slot(tgnn_run* r, int p, bool xg_split);

// Graph body (j == 1): the same launch sequence for every barrier; all
// per-barrier values come from d_desc[*d_ctr]. Barrier b runs on slot p =
// b % 2 (plan + read view prepared by the previous barrier) and prepares
// barrier b + 1 in slot 1 - p on the aux stream: its sampling / plan / routing
// sort overlaps this barrier's GRU, and its memory read (after this barrier's
// writes, and the next sweep's reset) overlaps this barrier's backward.
void barrier_body_dev(tgnn_run* r, int p) {
  tgnn_ctx* ctx = r->ctx;
  tgnn_trainer* tr = r->tr.get();
  // slot p's GRU input operand is w.bf.Xg while this body is enqueued (the
  // other slot's, w.xg_alt, is pre-assembled for the next barrier on aux)
  const bool xg_split = gemm_impl() == kGemmTma && tr->w.xg_alt.valid();
  if (xg_split && p == 1) std::swap(tr->w.bf.Xg, tr->w.xg_alt);
  try {
    barrier_body_slot(r, p, xg_split);
  } catch (...) {
    if (xg_split && p == 1) std::swap(tr->w.bf.Xg, tr->w.xg_alt);
    throw;
  }
  if (xg_split && p == 1) std::swap(tr->w.bf.Xg, tr->w.xg_alt);
}

void barrier_body_slot(tgnn_run* r, int p, bool xg_split) {
  tgnn_ctx* ctx = r->ctx;
  tgnn_trainer* tr = r->tr.get();
  cudaStream_t s = ctx->stream, aux = ctx->aux;
  StepCtx sc = tr->sc();
  sc.xg_pre = xg_split;
  sc.d_ctr = r->d_ctr;
  sc.packed = true;  // by the previous barrier's Adam (or the prologue)
  sc.marks = r->marks.on ? &r->marks : nullptr;  // profiling graph only
  sc.mark(phPlan, s);
  DPlan& pl = tr->plans[static_cast<size_t>(p)];
  DView& vw = tr->views[static_cast<size_t>(p)];
  DPlan& nx = tr->plans[static_cast<size_t>(1 - p)];
  DView& nv = tr->views[static_cast<size_t>(1 - p)];
  // fork: plan of barrier b + 1 (routing sort on the side stream)
  TGB_CUDA(cudaEventRecord(r->ev_fork, s));
  TGB_CUDA(cudaStreamWaitEvent(aux, r->ev_fork, 0));
  select_plan_args_launch(nx.args, r->d_desc, r->d_ctr, aux, 1);
  plan_launch(r->g->d, nx, aux, ctx->side);
  // branch: gradient zeroing now, the root writes after the GRU, the loss later
  cudaStream_t br = ctx->br;
  TGB_CUDA(cudaStreamWaitEvent(br, r->ev_fork, 0));
  TGB_CUDA(cudaMemsetAsync(tr->grads, 0, sizeof(float) * tr->L.total, br));
  TGB_CUDA(cudaEventRecord(r->ev_gzero, br));
  sc.br = br;
  sc.ev_g_zero = r->ev_gzero;
  sc.ev_br_dec = r->ev_dec;
  sc.ev_br_join = r->ev_brjoin;
  sc.ev_red = r->ev_red;
  // edge branch: the plan-only half of the attention projection runs beside the GRU
  static const bool no_edge = std::getenv("TGNN_NOEDGE") != nullptr;  // A/B: edge part inline
  // the previous barrier's tail update (deferred inside this capture): the
  // edge branch reads Wq / Wk / Wv edge columns, gru_out the static table
  const bool tail_wait = r->tail_pending;
  r->tail_pending = false;
  if (tail_wait) sc.ev_params_tail = r->ev_upd;
  if (gemm_impl() == kGemmTma && !no_edge) {
    TGB_CUDA(cudaStreamWaitEvent(ctx->edge, r->ev_fork, 0));
    if (tail_wait) TGB_CUDA(cudaStreamWaitEvent(ctx->edge, r->ev_upd, 0));
    StepCtx se = sc;
    se.marks = nullptr;  // phase markers live on the main stream
    const bool join = edge_join_enabled(r->tr->m.d_mem);
    attn_edge_launch(se, pl, ctx->edge, !join);
    TGB_CUDA(cudaEventRecord(r->ev_edge, ctx->edge));
    sc.ev_edge = r->ev_edge;
    sc.edge_gemm_joined = join;
  }
  // this barrier: its plan was sorted inside the previous graph
  cudaEvent_t sorted = pl.ev_sorted;
  pl.ev_sorted = nullptr;
  try {
    substep_gru_launch(sc, pl, vw, s);
    cudaStream_t ws = s;
    if (r->group_size == 1) {  // single writer: direct writes on the branch
      TGB_CUDA(cudaEventRecord(r->ev_gru, s));
      TGB_CUDA(cudaStreamWaitEvent(br, r->ev_gru, 0));
      ws = br;
    }
    root_writes_launch(sc, pl, vw, ws, r->group_size > 1 ? nullptr : &r->mem->d);
    if (r->oplog) {
      OplogPlans op;
      op.n = 1;
      op.sizes[0] = pl.sizes;
      op.supports[0] = pl.supports;
      oplog_record_launch(sc, op, r->d_oplog, 0, ws);
    }
    if (r->group_size > 1) {
      // the i-axis write exchange only feeds the NEXT barrier's read: it runs
      // on its own stream beside this barrier's attention / backward (the
      // group communicator is distinct from the gradient all-reduce's)
      TGB_CUDA(cudaEventRecord(r->ev_gru, s));
      TGB_CUDA(cudaStreamWaitEvent(ctx->xch, r->ev_gru, 0));
      comm_bcast_packs(r, 0, ctx->xch);
      apply_gathered(r, ctx->xch);
      ws = ctx->xch;
    }
    // join: the next barrier reads the memory copy once this barrier's writes landed
    TGB_CUDA(cudaEventRecord(r->ev_written, ws));
    // the next read (reset, gather, GRU-input view columns) starts after this
    // barrier's decoder, not beside its projections (TGNN_AUXMID; A/B: 1 best)
    // (0: beside the projections; 1 after the decoder, 2 after the attention
    // backward kernel -- recorded on every GEMM engine)
    static const int mid_at = env_knob("TGNN_AUXMID", 1, 0, 2);
    auto next_read = [&] {
      TGB_CUDA(cudaStreamWaitEvent(aux, r->ev_written, 0));
      if (mid_at > 0) TGB_CUDA(cudaStreamWaitEvent(aux, r->ev_mid, 0));
      reset_cond_launch(r->mem->d, r->d_desc, r->d_ctr, aux, 1);
      gather_view_launch(nx, r->mem->d, nv, aux);
      if (xg_split) assemble_gru_view_launch(sc, nx, nv, tr->w.xg_alt, aux);
      TGB_CUDA(cudaStreamWaitEvent(aux, nx.ev_sorted, 0));
      TGB_CUDA(cudaEventRecord(r->ev_next, aux));
    };
    if (mid_at == 0) next_read();
    sc.ev_tail_grads = r->ev_tail;
    sc.ev_mid = mid_at > 0 ? r->ev_mid : nullptr;
    sc.mid_at = mid_at;
    substep_rest_launch(sc, pl, vw, r->d_losses, s);
    if (mid_at > 0) next_read();
    sc.mark(phAdam, s);
    update_split(r, sc, s);
    TGB_CUDA(cudaStreamWaitEvent(s, r->ev_next, 0));
    incr_launch(r->d_ctr, s);
    sc.mark(phCount, s);
  } catch (...) {
    pl.ev_sorted = sorted;
    throw;
  }
  pl.ev_sorted = sorted;
}

__global__ void select_stint_args_kernel(const StintDesc* __restrict__ sd, const int* __restrict__ ctr, int offset,
                                         int sub, PlanArgs* dst) {
  *dst = sd[*ctr + offset].args[sub];
}

__global__ void reset_stint_kernel(DMem st, const StintDesc* __restrict__ sd, const int* __restrict__ ctr, int team) {
  if (!sd[*ctr].reset[team]) return;
  const int64_t n = st.N * st.d;
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < 3 * n; x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (x < n) st.memory[x] = 0.0f;
    else st.mail_mem[x - n] = 0.0f;
  }
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < st.N; x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    st.last_update[x] = 0.0;
    st.mail_t[x] = 0.0;
    st.mail_dt[x] = 0.0;
    st.mail_ev[x] = -1;
  }
}

// Graph body for j > 1 at stint position sidx: the direct path's launch
// sequence with every per-barrier value taken from the device tables. At the
// stint start the group's teams run the daemon's R/W chain in pair order (an
// idle team contributes an empty plan and an empty write pack, so every rank
// issues the same collectives); later positions run their pre-planned sub.
// Graph body for j > 1 at stint position sidx with the stint's plans in plan
// set `set` (slots set*j .. set*j + j - 1): the direct path's launch sequence
// with every per-barrier value taken from the device tables. The plans were
// made one stint ahead (by the previous stint's last position, on the aux
// stream), so the stint-start team chain is only the daemon's R/W brackets:
// the gathers, the GRU freshen, the root writes and their exchange per team in
// pair order (an idle team contributes an empty plan and an empty write pack,
// so every rank issues the same collectives). The rest of each position runs
// the j = 1 pipeline's branches and split-phase update.
void barrier_body_stint(tgnn_run* r, int sidx, int set) {
  tgnn_ctx* ctx = r->ctx;
  tgnn_trainer* tr = r->tr.get();
  cudaStream_t s = ctx->stream;
  StepCtx sc = tr->sc();
  sc.d_ctr = r->d_ctr;
  sc.packed = true;  // by the previous barrier's Adam (or the segment prologue)
  const int j = r->tc.j;
  const size_t base = static_cast<size_t>(set * j), nbase = static_cast<size_t>((1 - set) * j);
  std::vector<cudaEvent_t> saved(tr->plans.size());
  for (size_t x = 0; x < tr->plans.size(); ++x) saved[x] = tr->plans[x].ev_sorted;
  auto restore = [&]() {
    for (size_t x = 0; x < tr->plans.size(); ++x) tr->plans[x].ev_sorted = saved[x];
  };
  TGB_CUDA(cudaEventRecord(r->ev_fork, s));
  cudaStream_t br = ctx->br;
  TGB_CUDA(cudaStreamWaitEvent(br, r->ev_fork, 0));
  TGB_CUDA(cudaMemsetAsync(tr->grads, 0, sizeof(float) * tr->L.total, br));
  TGB_CUDA(cudaEventRecord(r->ev_gzero, br));
  sc.br = br;
  sc.ev_g_zero = r->ev_gzero;
  sc.ev_br_dec = r->ev_dec;
  sc.ev_br_join = r->ev_brjoin;
  sc.ev_red = r->ev_red;
  sc.ev_tail_grads = r->ev_tail;
  try {
    for (int sub = 0; sub < j; ++sub) tr->plans[base + static_cast<size_t>(sub)].ev_sorted = nullptr;  // sorted ahead
    DPlan& pl = tr->plans[base + static_cast<size_t>(sidx)];
    DView& vw = tr->views[base + static_cast<size_t>(sidx)];
    if (gemm_impl() == kGemmTma) {  // the plan-only half of the attention projection, from the start
      TGB_CUDA(cudaStreamWaitEvent(ctx->edge, r->ev_fork, 0));
      StepCtx se = sc;
      const bool join = edge_join_enabled(tr->m.d_mem);
      attn_edge_launch(se, pl, ctx->edge, !join);
      TGB_CUDA(cudaEventRecord(r->ev_edge, ctx->edge));
      sc.ev_edge = r->ev_edge;
      sc.edge_gemm_joined = join;
    }
    const bool plan_next = sidx == j - 1;
    if (plan_next) {  // the next stint's plans into the other set, beside this position
      cudaStream_t aux = ctx->aux;
      TGB_CUDA(cudaStreamWaitEvent(aux, r->ev_fork, 0));
      for (int sub = 0; sub < j; ++sub) {
        DPlan& nx = tr->plans[nbase + static_cast<size_t>(sub)];
        select_stint_args_kernel<<<1, 1, 0, aux>>>(r->d_stint, r->d_ctr, 1, sub, nx.args);
        TGB_CUDA(cudaGetLastError());
        plan_launch(r->g->d, nx, aux, ctx->side);
      }
      for (int sub = 0; sub < j; ++sub) {
        DPlan& nx = tr->plans[nbase + static_cast<size_t>(sub)];
        if (nx.ev_sorted) TGB_CUDA(cudaStreamWaitEvent(aux, nx.ev_sorted, 0));
      }
      TGB_CUDA(cudaEventRecord(r->ev_next, aux));
    }
    if (sidx == 0) {
      for (int tt = 0; tt < j; ++tt) {
        reset_stint_kernel<<<4 * num_sms(), 256, 0, s>>>(r->mem->d, r->d_stint, r->d_ctr, tt);
        TGB_CUDA(cudaGetLastError());
        if (tt == r->team) {
          // the read bracket: sub 0's view on the chain, the later subs' views
          // beside its GRU freshen (joined before this team's writes land)
          gather_view_launch(pl, r->mem->d, vw, s);
          TGB_CUDA(cudaEventRecord(r->ev_gru, s));
          TGB_CUDA(cudaStreamWaitEvent(ctx->aux, r->ev_gru, 0));
          for (int sub = 1; sub < j; ++sub)
            gather_view_launch(tr->plans[base + static_cast<size_t>(sub)], r->mem->d,
                               tr->views[base + static_cast<size_t>(sub)], ctx->aux);
          TGB_CUDA(cudaEventRecord(r->ev_written, ctx->aux));
          substep_gru_launch(sc, pl, vw, s);
          root_writes_launch(sc, pl, vw, s, nullptr);
          TGB_CUDA(cudaStreamWaitEvent(s, r->ev_written, 0));
          if (r->oplog) {
            OplogPlans op;
            op.n = j;
            for (int x = 0; x < j; ++x) {
              op.sizes[x] = tr->plans[base + static_cast<size_t>(x)].sizes;
              op.supports[x] = tr->plans[base + static_cast<size_t>(x)].supports;
            }
            oplog_record_launch(sc, op, r->d_oplog, 0, s);
          }
        }
        comm_bcast_packs(r, tt, s);
        apply_gathered(r, s);
      }
    } else {
      substep_gru_launch(sc, pl, vw, s);
    }
    substep_rest_launch(sc, pl, vw, r->d_losses, s);
    const bool defer = r->defer_tail;
    r->defer_tail = false;  // every position is its own graph: join the tail update
    update_split(r, sc, s);
    r->defer_tail = defer;
    if (plan_next) TGB_CUDA(cudaStreamWaitEvent(s, r->ev_next, 0));
    incr_launch(r->d_ctr, s);
  } catch (...) {
    restore();
    throw;
  }
  restore();
}

// Eager planning of stint b0 (the first stint of a run, or after the direct
// path ran the previous stint's last position) into its plan set.
void plan_stint_now(tgnn_run* r, int64_t b0) {
  tgnn_trainer* tr = r->tr.get();
  cudaStream_t s = r->ctx->stream;
  const int j = r->tc.j;
  const size_t base = static_cast<size_t>(((b0 / j) % 2) * j);
  const StintDesc& sd = r->h_stint[static_cast<size_t>(b0)];
  for (int sub = 0; sub < j; ++sub) {
    DPlan& pl = tr->plans[base + static_cast<size_t>(sub)];
    set_plan_args_launch(pl.args, sd.args[sub], s);
    plan_launch(r->g->d, pl, s, r->ctx->side);
  }
  for (int sub = 0; sub < j; ++sub) {
    DPlan& pl = tr->plans[base + static_cast<size_t>(sub)];
    if (pl.ev_sorted) TGB_CUDA(cudaStreamWaitEvent(s, pl.ev_sorted, 0));
  }
  r->stint_planned = b0;
}

void ensure_graph_events(tgnn_run* r) {
  if (r->ev_fork) return;
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_fork, cudaEventDisableTiming));
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_written, cudaEventDisableTiming));
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_next, cudaEventDisableTiming));
  cudaEvent_t* more[] = {&r->ev_gru,  &r->ev_gzero, &r->ev_dec,    &r->ev_brjoin,
                         &r->ev_edge, &r->ev_red,   &r->ev_artail, &r->ev_upd, &r->ev_mid};
  for (cudaEvent_t* e : more) TGB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  cudaEvent_t* upd[] = {&r->ev_tail, &r->ev_head, &r->ev_comm};
  for (cudaEvent_t* e : upd)
    if (!*e) TGB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void build_stint_graphs(tgnn_run* r) {
  cudaStream_t s = r->ctx->stream;
  gemm_kernels_prepare();
  ensure_graph_events(r);
  TGB_CUDA(cudaStreamSynchronize(s));
  const int j = r->tc.j;
  r->sgraph.assign(static_cast<size_t>(2 * j), nullptr);
  r->sexec.assign(static_cast<size_t>(2 * j), nullptr);
  for (int x = 0; x < 2 * j; ++x) {
    TGB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      barrier_body_stint(r, x % j, x / j);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    TGB_CUDA(cudaStreamEndCapture(s, &r->sgraph[static_cast<size_t>(x)]));
    TGB_CUDA(cudaGraphInstantiate(&r->sexec[static_cast<size_t>(x)], r->sgraph[static_cast<size_t>(x)], 0));
  }
  // the plans' routing-sort events were only recorded inside the captures:
  // record them once eagerly so a direct barrier (profiling) may wait on them
  for (auto& pl : r->tr->plans)
    if (pl.ev_sorted) TGB_CUDA(cudaEventRecord(pl.ev_sorted, r->ctx->side));
  size_t n = 0;
  TGB_CUDA(cudaGraphGetNodes(r->sgraph[0], nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  TGB_CUDA(cudaGraphGetNodes(r->sgraph[0], nodes.data(), &n));
  int64_t kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    TGB_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) ++kernels;
  }
  r->launches = kernels;
}

constexpr int kMultiBarrier = 4;

void build_graph(tgnn_run* r) {
  cudaStream_t s = r->ctx->stream;
  gemm_kernels_prepare();
  TGB_CUDA(cudaStreamSynchronize(s));
  ensure_graph_events(r);
  for (int p = 0; p < 2; ++p) {
    TGB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      barrier_body_dev(r, p);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    TGB_CUDA(cudaStreamEndCapture(s, &r->graph[p]));
    TGB_CUDA(cudaGraphInstantiate(&r->exec[p], r->graph[p], 0));
  }
  TGB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    for (int x = 0; x < kMultiBarrier; ++x) {
      r->defer_tail = x + 1 < kMultiBarrier;  // joined by the capture's last barrier
      barrier_body_dev(r, x & 1);
    }
    r->defer_tail = false;
  } catch (...) {
    r->defer_tail = false;
    r->tail_pending = false;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  TGB_CUDA(cudaStreamEndCapture(s, &r->mgraph));
  TGB_CUDA(cudaGraphInstantiate(&r->mexec, r->mgraph, 0));
  size_t n = 0;
  TGB_CUDA(cudaGraphGetNodes(r->graph[0], nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  TGB_CUDA(cudaGraphGetNodes(r->graph[0], nodes.data(), &n));
  int64_t kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    TGB_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) ++kernels;
  }
  r->launches = kernels;
}

// Graph-mode prologue: plan + read of barrier b into slot b % 2 (the reset of
// its sweep first), as barrier b - 1's graph would have left them.
void prepare_barrier(tgnn_run* r, int64_t b) {
  tgnn_ctx* ctx = r->ctx;
  tgnn_trainer* tr = r->tr.get();
  cudaStream_t s = ctx->stream;
  DPlan& pl = tr->plans[static_cast<size_t>(b & 1)];
  set_int_kernel<<<1, 1, 0, s>>>(r->d_ctr, static_cast<int>(b));
  set_int_kernel<<<1, 1, 0, s>>>(r->d_ctr_tail, static_cast<int>(b));
  TGB_CUDA(cudaGetLastError());
  reset_cond_launch(r->mem->d, r->d_desc, r->d_ctr, s, 0);
  select_plan_args_launch(pl.args, r->d_desc, r->d_ctr, s, 0);
  plan_launch(r->g->d, pl, s, ctx->side);
  gather_view_launch(pl, r->mem->d, tr->views[static_cast<size_t>(b & 1)], s);
  if (gemm_impl() == kGemmTma && tr->w.xg_alt.valid())  // the graph body assembles only the time columns
    assemble_gru_view_launch(tr->sc(), pl, tr->views[static_cast<size_t>(b & 1)],
                             (b & 1) ? tr->w.xg_alt : tr->w.bf.Xg, s);
  TGB_CUDA(cudaStreamWaitEvent(s, pl.ev_sorted, 0));
  pack_weights(tr->sc(), s);
  r->prepared = b;
}

}  // namespace

void tgnn_evaluator::init(tgnn_ctx* cx, tgnn_graph* gr, const ModelDims& md, int64_t batch, int negatives) {
  ctx = cx;
  g = gr;
  m = md;
  if (m.num_nodes <= 0) m.num_nodes = gr->d.N;
  TGB_REQUIRE(m.num_nodes == gr->d.N, kConfig, "model num_nodes does not match the dataset");
  TGB_REQUIRE(m.d_e == gr->d.d_e, kConfig, "model edge feature width does not match the dataset");
  validate_dims(m);
  TGB_REQUIRE(batch > 0, kConfig, "evaluate_mrr: batch size must be positive");
  TGB_REQUIRE(negatives >= 0, kConfig, "evaluate_mrr: negative distractor count");
  const int64_t rpe = 2 + static_cast<int64_t>(negatives);
  const int64_t nn = std::max<int64_t>(m.n_neighbors, 1);
  TGB_REQUIRE(rpe * batch * (nn + 1) < (1ll << 31), kConfig,
              "evaluate_mrr: batch x candidates x neighbours exceeds the device index range");
  L = ParamLayout::make(m);
  cap_B = static_cast<int>(batch);
  n_neg = negatives;
  const int64_t N = m.num_nodes;
  const int cap_U = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(N, rpe * batch * (m.n_neighbors + 1))));
  params = dalloc<float>(static_cast<size_t>(L.total));
  step_alloc(w, m, cap_B, cap_U, N, static_cast<int>(rpe), true);
  plan_alloc(pe, cap_B, static_cast<int>(m.n_neighbors), cap_U, N, static_cast<int>(rpe), 0, 1);
  plan_alloc(pr, cap_B, 0, static_cast<int>(std::min<int64_t>(N, 2 * batch)), N, 2, 0);
  view_alloc(vw, cap_U, m.d_mem);
  st.reset(memstore_new(ctx, N, m.d_mem));
}

namespace {

// One metrics row at eval barrier b (rank 0 evaluates with its own weights).
// Replica invariant: every rank holds bitwise the same
// parameters. Collective: the parameter fingerprint's min and max over ranks
// must agree. Returns the fingerprint.
uint64_t check_replicas(tgnn_run* r) {
  cudaStream_t s = r->ctx->stream;
  unsigned long long* d = dalloc<unsigned long long>(3);
  params_hash_launch(r->tr->params, r->tr->L.total, d, s);
  TGB_CUDA(cudaMemcpyAsync(d + 1, d, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
  TGB_CUDA(cudaMemcpyAsync(d + 2, d, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
  comm_allreduce(r, d + 1, 1, RedTy::U64, RedOp::Min, s);
  comm_allreduce(r, d + 2, 1, RedTy::U64, RedOp::Max, s);
  unsigned long long h[3];
  TGB_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  TGB_CUDA(cudaStreamSynchronize(s));
  cudaFree(d);
  if (h[1] != h[2])
    throw Error(kProtocol, "run: replica parameters diverged by barrier " + std::to_string(r->next_barrier));
  return h[0];
}

void run_eval_point(tgnn_run* r, int64_t b) {
  tgnn_run::Row row;
  row.barrier = b;
  if (r->nranks > 1) check_replicas(r);  // once per eval point (epoch-equivalent)
  if (r->rank == 0 && r->val_end > r->val_begin) {
    const int64_t batch = r->eval_batch > 0 ? r->eval_batch : r->tc.local_batch;
    if (!r->ev || r->ev->cap_B != batch || r->ev->n_neg != r->eval_negatives) {
      r->ev = std::make_unique<tgnn_evaluator>();
      r->ev->init(r->ctx, r->g, r->tr->m, batch, r->eval_negatives);
    }
    TGB_CUDA(cudaMemcpyAsync(r->ev->params, r->tr->params, sizeof(float) * r->tr->L.total,
                             cudaMemcpyDeviceToDevice, r->ctx->stream));
    int64_t q = 0;
    row.val_mrr = r->ev->evaluate(r->val_begin, r->val_end, r->tc.seed, &q);
  }
  TGB_CUDA(cudaEventCreate(&row.done));
  TGB_CUDA(cudaEventRecord(row.done, r->ctx->stream));
  r->rows.push_back(row);
}

}  // namespace


// ----------------------------------------------------------------- C ABI
extern "C" {

const char* tgnn_last_error(void) { return g_err.c_str(); }
int tgnn_version(void) { return 1; }

int tgnn_device_count(int* out) {
  API_BEGIN
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *out = n;
  API_END
}

int tgnn_ctx_create(int device, tgnn_ctx** out) {
  API_BEGIN
  TGB_CUDA(cudaSetDevice(device));
  auto* c = new tgnn_ctx();
  c->device = device;
  // the step's critical path runs at the highest stream priority (carried into
  // every launch and captured graph node by launch_pdl); branches at the lowest
  int lo_prio = 0, hi_prio = 0;
  TGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->comm, cudaStreamNonBlocking, hi_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, lo_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->br, cudaStreamNonBlocking, lo_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->edge, cudaStreamNonBlocking, lo_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->h2d, cudaStreamNonBlocking, hi_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->xch, cudaStreamNonBlocking, hi_prio));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->hd, cudaStreamNonBlocking, hi_prio));
  TGB_CUDA(cudaEventCreateWithFlags(&c->ev_h2d, cudaEventDisableTiming));
  TGB_CUDA(cudaStreamCreateWithPriority(&c->d2h, cudaStreamNonBlocking, lo_prio));
  TGB_CUDA(cudaEventCreateWithFlags(&c->ev_d2h, cudaEventDisableTiming));
  c->d_flag = dalloc<int>(1);
  TGB_CUDA(cudaMemset(c->d_flag, 0, sizeof(int)));
  *out = c;
  API_END
}

int tgnn_ctx_destroy(tgnn_ctx* ctx) {
  API_BEGIN
  if (!ctx) return 0;
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->d_flag);
  cudaStreamSynchronize(ctx->side);
  cudaStreamSynchronize(ctx->comm);
  cudaStreamSynchronize(ctx->aux);
  cudaStreamSynchronize(ctx->br);
  cudaStreamSynchronize(ctx->edge);
  cudaStreamSynchronize(ctx->h2d);
  cudaStreamSynchronize(ctx->d2h);
  cudaStreamSynchronize(ctx->xch);
  cudaStreamSynchronize(ctx->hd);
  cudaEventDestroy(ctx->ev_h2d);
  cudaEventDestroy(ctx->ev_d2h);
  cudaStreamDestroy(ctx->h2d);
  cudaStreamDestroy(ctx->d2h);
  cudaStreamDestroy(ctx->xch);
  cudaStreamDestroy(ctx->hd);
  cudaStreamDestroy(ctx->aux);
  cudaStreamDestroy(ctx->br);
  cudaStreamDestroy(ctx->edge);
  cudaStreamDestroy(ctx->side);
  cudaStreamDestroy(ctx->comm);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  API_END
}

int tgnn_ctx_synchronize(tgnn_ctx* ctx) {
  API_BEGIN
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->d2h));  // asynchronous result reads
  API_END
}

int tgnn_ctx_stream(tgnn_ctx* ctx, void** stream_out) {
  API_BEGIN
  *stream_out = reinterpret_cast<void*>(ctx->stream);
  API_END
}

int tgnn_gen_synthetic(const tgnn_synth_params* p, int64_t* src, int64_t* dst, double* t,
                       float* efeat, int64_t* bipartite_boundary) {
  API_BEGIN
  host::SynthConfig c;
  c.nodes = p->nodes;
  c.events = p->events;
  c.burst_prob = p->burst_prob;
  c.pref_prob = p->pref_prob;
  c.prefs_per_src = p->prefs_per_src;
  c.src_frac = p->src_frac;
  c.bipartite = p->bipartite != 0;
  c.d_e = p->d_e;
  c.zipf_s = p->zipf_s;
  c.seed = p->seed;
  *bipartite_boundary = host::synthesize(c, src, dst, t, efeat);
  API_END
}

namespace {

// Allocates the event arrays of an E-event graph (T-CSR built by finalize).
std::unique_ptr<tgnn_graph> graph_alloc(tgnn_ctx* ctx, int64_t num_nodes, int64_t boundary, int64_t E, int64_t d_e) {
  TGB_REQUIRE(num_nodes > 0, kConfig, "graph: num_nodes must be positive");
  TGB_REQUIRE(num_nodes < (1ll << 31) && E < (1ll << 30), kConfig, "graph: too large for int32 ids");
  if (boundary >= 0)
    TGB_REQUIRE(boundary > 0 && boundary < num_nodes, kConfig,
                "graph: bipartite boundary leaves an empty partition");
  TGB_REQUIRE(E >= 0 && d_e >= 0, kConfig, "graph: invalid sizes");
  auto g = std::make_unique<tgnn_graph>();
  g->ctx = ctx;
  DGraph& D = g->d;
  D.N = num_nodes;
  D.boundary = boundary;
  D.E = E;
  D.d_e = d_e;
  D.d_e_pad = (d_e + 3) / 4 * 4;
  D.src = dalloc<int32_t>(E);
  D.dst = dalloc<int32_t>(E);
  D.t = dalloc<double>(E);
  D.efeat = dalloc<float>(static_cast<size_t>(E * std::max<int64_t>(D.d_e_pad, 1)));
  if (D.d_e_pad > D.d_e)
    TGB_CUDA(cudaMemset(D.efeat, 0, sizeof(float) * static_cast<size_t>(E * D.d_e_pad)));
  return g;
}

int graph_create_impl(tgnn_ctx* ctx, int64_t num_nodes, int64_t boundary, int64_t E,
                      const int64_t* src, const int64_t* dst, const double* t, const float* ef32,
                      const double* ef64, int64_t d_e, tgnn_graph** out) {
  API_BEGIN
  ctx->use();
  // TemporalGraph::finalize (temporal_graph.hpp:55-91): events and feature
  // rows go up as given; sort, validation and the T-CSR run on the device.
  auto g = graph_alloc(ctx, num_nodes, boundary, E, d_e);
  DGraph& D = g->d;
  cudaStream_t s = ctx->stream;
  // ids outside [0, N) become -1 so int32 narrowing cannot hide them
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(E, (64ll << 20) / (4 * std::max<int64_t>(D.d_e_pad, 4))));
  std::vector<int32_t> s32(static_cast<size_t>(std::min(chunk, std::max<int64_t>(E, 1))));
  std::vector<int32_t> d32(s32.size());
  std::vector<float> buf(d_e > 0 ? s32.size() * static_cast<size_t>(D.d_e_pad) : 0, 0.0f);
  for (int64_t e0 = 0; e0 < E; e0 += chunk) {
    const int64_t n = std::min(chunk, E - e0);
    for (int64_t x = 0; x < n; ++x) {
      const int64_t a = src[e0 + x], b = dst[e0 + x];
      s32[static_cast<size_t>(x)] = a >= 0 && a < num_nodes ? static_cast<int32_t>(a) : -1;
      d32[static_cast<size_t>(x)] = b >= 0 && b < num_nodes ? static_cast<int32_t>(b) : -1;
    }
    TGB_CUDA(cudaMemcpyAsync(D.src + e0, s32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    TGB_CUDA(cudaMemcpyAsync(D.dst + e0, d32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    TGB_CUDA(cudaMemcpyAsync(D.t + e0, t + e0, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    if (d_e > 0) {
      for (int64_t x = 0; x < n; ++x) {
        float* row = buf.data() + x * D.d_e_pad;
        for (int64_t f = 0; f < d_e; ++f)
          row[f] = ef32 ? ef32[(e0 + x) * d_e + f] : static_cast<float>(ef64[(e0 + x) * d_e + f]);
      }
      TGB_CUDA(cudaMemcpyAsync(D.efeat + e0 * D.d_e_pad, buf.data(), sizeof(float) * n * D.d_e_pad,
                               cudaMemcpyHostToDevice, s));
    }
    TGB_CUDA(cudaStreamSynchronize(s));  // pageable staging is reused
  }
  graph_finalize_device(D, s);
  *out = g.release();
  API_END
}

}  // namespace

int tgnn_graph_create(tgnn_ctx* ctx, int64_t num_nodes, int64_t bipartite_boundary, int64_t num_events,
                      const int64_t* src, const int64_t* dst, const double* t, const float* efeat,
                      int64_t d_e, tgnn_graph** out) {
  return graph_create_impl(ctx, num_nodes, bipartite_boundary, num_events, src, dst, t, efeat, nullptr,
                           d_e, out);
}

int tgnn_graph_create_f64(tgnn_ctx* ctx, int64_t num_nodes, int64_t bipartite_boundary,
                          int64_t num_events, const int64_t* src, const int64_t* dst, const double* t,
                          const double* efeat, int64_t d_e, tgnn_graph** out) {
  return graph_create_impl(ctx, num_nodes, bipartite_boundary, num_events, src, dst, t, nullptr, efeat,
                           d_e, out);
}

int tgnn_graph_destroy(tgnn_graph* g) {
  API_BEGIN
  delete g;
  API_END
}

int tgnn_graph_info(tgnn_graph* g, int64_t* num_nodes, int64_t* boundary, int64_t* num_events,
                    int64_t* d_e) {
  API_BEGIN
  *num_nodes = g->d.N;
  *boundary = g->d.boundary;
  *num_events = g->d.E;
  *d_e = g->d.d_e;
  API_END
}

int tgnn_graph_events(tgnn_graph* g, int64_t* src, int64_t* dst, double* t) {
  API_BEGIN
  g->ctx->use();
  const int64_t E = g->d.E;
  std::vector<int32_t> a(static_cast<size_t>(E)), b(static_cast<size_t>(E));
  cudaStream_t s = g->ctx->stream;
  d2h(a.data(), g->d.src, static_cast<size_t>(E), s);
  d2h(b.data(), g->d.dst, static_cast<size_t>(E), s);
  d2h(t, g->d.t, static_cast<size_t>(E), s);
  TGB_CUDA(cudaStreamSynchronize(s));
  for (int64_t e = 0; e < E; ++e) {
    src[e] = a[static_cast<size_t>(e)];
    dst[e] = b[static_cast<size_t>(e)];
  }
  API_END
}

int tgnn_sample_recent_neighbors(tgnn_graph* g, const int64_t* nodes, const double* times, int64_t count,
                                 int64_t n, int64_t* nbr_node, int64_t* nbr_event, double* nbr_dt,
                                 int64_t* nbr_count) {
  API_BEGIN
  tgnn_ctx* ctx = g->ctx;
  ctx->use();
  TGB_REQUIRE(n >= 0 && n <= 32, kConfig, "sample_recent_neighbors: n must lie in [0, 32]");
  if (count == 0) return 0;
  std::vector<int32_t> qn(static_cast<size_t>(count));
  for (int64_t q = 0; q < count; ++q) {
    TGB_REQUIRE(nodes[q] >= 0 && nodes[q] < g->d.N, kConfig, "sample_recent_neighbors: node out of range");
    qn[static_cast<size_t>(q)] = static_cast<int32_t>(nodes[q]);
  }
  const int64_t nn = std::max<int64_t>(n, 1);
  int32_t* d_nodes = dalloc<int32_t>(count);
  double* d_times = dalloc<double>(count);
  int32_t* d_nn = dalloc<int32_t>(count * nn);
  int32_t* d_ne = dalloc<int32_t>(count * nn);
  double* d_nd = dalloc<double>(count * nn);
  int32_t* d_c = dalloc<int32_t>(count);
  h2d(d_nodes, qn.data(), count, ctx->stream);
  h2d(d_times, times, count, ctx->stream);
  sample_queries_launch(g->d, d_nodes, d_times, static_cast<int>(count), static_cast<int>(n), d_nn, d_ne,
                        d_nd, d_c, ctx->stream);
  std::vector<int32_t> hn(static_cast<size_t>(count * nn)), he(static_cast<size_t>(count * nn)),
      hc(static_cast<size_t>(count));
  std::vector<double> hd(static_cast<size_t>(count * nn));
  d2h(hn.data(), d_nn, count * nn, ctx->stream);
  d2h(he.data(), d_ne, count * nn, ctx->stream);
  d2h(hd.data(), d_nd, count * nn, ctx->stream);
  d2h(hc.data(), d_c, count, ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (void* p : {static_cast<void*>(d_nodes), static_cast<void*>(d_times), static_cast<void*>(d_nn),
                  static_cast<void*>(d_ne), static_cast<void*>(d_nd), static_cast<void*>(d_c)})
    cudaFree(p);
  for (int64_t q = 0; q < count; ++q) {
    nbr_count[q] = hc[static_cast<size_t>(q)];
    for (int64_t m = 0; m < n; ++m) {
      const bool ok = m < hc[static_cast<size_t>(q)];
      nbr_node[q * n + m] = ok ? hn[static_cast<size_t>(q * n + m)] : -1;
      nbr_event[q * n + m] = ok ? he[static_cast<size_t>(q * n + m)] : -1;
      nbr_dt[q * n + m] = ok ? hd[static_cast<size_t>(q * n + m)] : 0.0;
    }
  }
  API_END
}

int tgnn_sample_negatives(tgnn_graph* g, int64_t batch_index, int64_t group, int64_t count, uint64_t seed,
                          int64_t* out) {
  API_BEGIN
  tgnn_ctx* ctx = g->ctx;
  ctx->use();
  const int64_t lo = g->d.boundary >= 0 ? g->d.boundary : 0;
  TGB_REQUIRE(g->d.N - lo > 0, kConfig, "negative sampling: empty destination partition");
  if (count <= 0) return 0;
  DPlan pl;  // only args + negs are used
  pl.args = dalloc<PlanArgs>(1);
  int32_t* negs = dalloc<int32_t>(count);
  PlanArgs a;
  a.begin = 0;
  a.end = count;
  a.batch_begin = 0;
  a.batch_index = batch_index;
  a.group = group;
  a.seed = seed;
  a.neg_mode = 1;
  a.valid = 1;
  set_plan_args_launch(pl.args, a, ctx->stream);
  pl.negs = negs;
  pl.cap_B = static_cast<int>(count);
  negatives_only_launch(g->d, pl.args, static_cast<int>(count), negs, ctx->stream);
  std::vector<int32_t> h(static_cast<size_t>(count));
  d2h(h.data(), negs, count, ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(pl.args);
  cudaFree(negs);
  for (int64_t x = 0; x < count; ++x) out[x] = h[static_cast<size_t>(x)];
  API_END
}

int tgnn_plan_sub_batch(tgnn_graph* g, int64_t begin, int64_t end, const int64_t* negatives, int64_t n,
                        int64_t* root_node, double* root_t, int64_t* nbr_count, int64_t* nbr_node,
                        int64_t* nbr_event, double* nbr_dt, int64_t* supports, int64_t* num_supports) {
  API_BEGIN
  tgnn_ctx* ctx = g->ctx;
  ctx->use();
  TGB_REQUIRE(n >= 0 && n <= 32, kConfig, "plan_sub_batch: n must lie in [0, 32]");
  TGB_REQUIRE(begin >= 0 && end <= g->d.E && begin <= end, kConfig,
              "plan_sub_batch: event range out of bounds");
  const int64_t B = end - begin;
  if (B == 0) {
    *num_supports = 0;
    return 0;
  }
  tgnn_trainer tmp;  // plan-only harness: one plan, no model
  tmp.ctx = ctx;
  tmp.g = g;
  tmp.cap_B = static_cast<int>(B);
  tmp.seed = 0;
  tmp.plans.resize(1);
  const int capU = cap_U_for(g->d.N, static_cast<int>(B), n);
  plan_alloc(tmp.plans[0], static_cast<int>(B), static_cast<int>(n), capU, g->d.N);
  plan_explicit(&tmp, 0, begin, end, negatives);
  DPlan& pl = tmp.plans[0];
  const int R = static_cast<int>(3 * B);
  const int nn = static_cast<int>(std::max<int64_t>(n, 1));
  std::vector<int32_t> rn(R), cnt(R), sn(static_cast<size_t>(R) * nn), se(static_cast<size_t>(R) * nn),
      sup(static_cast<size_t>(capU));
  std::vector<double> rt(R), sd(static_cast<size_t>(R) * nn);
  int32_t sz[kSzCount];
  d2h(sz, pl.sizes, kSzCount, ctx->stream);
  d2h(rn.data(), pl.root_node, R, ctx->stream);
  d2h(rt.data(), pl.root_t, R, ctx->stream);
  d2h(cnt.data(), pl.nbr_cnt, R, ctx->stream);
  if (n > 0) {
    d2h(sn.data(), pl.slot_node, static_cast<size_t>(R) * n, ctx->stream);
    d2h(se.data(), pl.slot_event, static_cast<size_t>(R) * n, ctx->stream);
    d2h(sd.data(), pl.slot_dt, static_cast<size_t>(R) * n, ctx->stream);
  }
  d2h(sup.data(), pl.supports, capU, ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int r = 0; r < R; ++r) {
    root_node[r] = rn[r];
    root_t[r] = rt[r];
    nbr_count[r] = cnt[r];
    for (int64_t m = 0; m < n; ++m) {
      const bool ok = m < cnt[r];
      nbr_node[r * n + m] = ok ? sn[r * n + m] : -1;
      nbr_event[r * n + m] = ok ? se[r * n + m] : -1;
      nbr_dt[r * n + m] = ok ? sd[r * n + m] : 0.0;
    }
  }
  *num_supports = sz[kSzU];
  for (int u = 0; u < sz[kSzU]; ++u) supports[u] = sup[static_cast<size_t>(u)];
  plan_free(tmp.plans[0]);
  tmp.plans.clear();
  API_END
}

// ----------------------------------------------------------------- memstore
int tgnn_memstore_create(tgnn_ctx* ctx, int64_t num_nodes, int64_t d_mem, tgnn_memstore** out) {
  API_BEGIN
  ctx->use();
  *out = memstore_new(ctx, num_nodes, d_mem);
  API_END
}

int tgnn_memstore_destroy(tgnn_memstore* m) {
  API_BEGIN
  delete m;
  API_END
}

int tgnn_memstore_reset(tgnn_memstore* m) {
  API_BEGIN
  m->ctx->use();
  reset_state_launch(m->d, m->ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(m->ctx->stream));
  API_END
}

int tgnn_memstore_export(tgnn_memstore* m, double* memory, double* last_update, double* mail_mem,
                         double* mail_t, double* mail_dt, int64_t* mail_event) {
  API_BEGIN
  m->ctx->use();
  const int64_t N = m->d.N, d = m->d.d;
  cudaStream_t s = m->ctx->stream;
  std::vector<float> mem(static_cast<size_t>(N * d)), mail(static_cast<size_t>(N * 2 * d));
  std::vector<double> lu(N), mt(N), mdt(N);
  std::vector<int32_t> ev(N);
  d2h(mem.data(), m->d.memory, mem.size(), s);
  d2h(mail.data(), m->d.mail_mem, mail.size(), s);
  d2h(lu.data(), m->d.last_update, N, s);
  d2h(mt.data(), m->d.mail_t, N, s);
  d2h(mdt.data(), m->d.mail_dt, N, s);
  d2h(ev.data(), m->d.mail_ev, N, s);
  TGB_CUDA(cudaStreamSynchronize(s));
  if (memory) for (size_t x = 0; x < mem.size(); ++x) memory[x] = mem[x];
  if (mail_mem) for (size_t x = 0; x < mail.size(); ++x) mail_mem[x] = mail[x];
  for (int64_t v = 0; v < N; ++v) {
    if (last_update) last_update[v] = lu[v];
    if (mail_t) mail_t[v] = mt[v];
    if (mail_dt) mail_dt[v] = mdt[v];
    if (mail_event) mail_event[v] = ev[v];
  }
  API_END
}

int tgnn_memstore_import(tgnn_memstore* m, const double* memory, const double* last_update,
                         const double* mail_mem, const double* mail_t, const double* mail_dt,
                         const int64_t* mail_event) {
  API_BEGIN
  m->ctx->use();
  const int64_t N = m->d.N, d = m->d.d;
  std::vector<float> mem(static_cast<size_t>(N * d)), mail(static_cast<size_t>(N * 2 * d));
  std::vector<int32_t> ev(N);
  for (size_t x = 0; x < mem.size(); ++x) mem[x] = static_cast<float>(memory[x]);
  for (size_t x = 0; x < mail.size(); ++x) mail[x] = static_cast<float>(mail_mem[x]);
  for (int64_t v = 0; v < N; ++v) ev[v] = static_cast<int32_t>(mail_event[v]);
  TGB_CUDA(cudaMemcpy(m->d.memory, mem.data(), sizeof(float) * mem.size(), cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(m->d.mail_mem, mail.data(), sizeof(float) * mail.size(), cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(m->d.last_update, last_update, sizeof(double) * N, cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(m->d.mail_t, mail_t, sizeof(double) * N, cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(m->d.mail_dt, mail_dt, sizeof(double) * N, cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(m->d.mail_ev, ev.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice));
  API_END
}

int tgnn_memstore_read(tgnn_memstore* m, const int64_t* nodes, int64_t count, double* mem_rows,
                       double* mail_rows) {
  API_BEGIN
  m->ctx->use();
  const int64_t N = m->d.N, d = m->d.d;
  for (int64_t x = 0; x < count; ++x)
    TGB_REQUIRE(nodes[x] >= 0 && nodes[x] < N, kProtocol, "read: index out of range");
  std::vector<double> mem(static_cast<size_t>(N * d)), mail(static_cast<size_t>(N * 2 * d)), mt(N), mdt(N),
      lu(N);
  std::vector<int64_t> ev(N);
  int rc = tgnn_memstore_export(m, mem.data(), lu.data(), mail.data(), mt.data(), mdt.data(), ev.data());
  if (rc) return rc;
  const int64_t mw = 2 * d + 3;
  for (int64_t x = 0; x < count; ++x) {
    const int64_t v = nodes[x];
    for (int64_t q = 0; q < d; ++q) mem_rows[x * d + q] = mem[v * d + q];
    for (int64_t q = 0; q < 2 * d; ++q) mail_rows[x * mw + q] = mail[v * 2 * d + q];
    mail_rows[x * mw + 2 * d] = mt[v];
    mail_rows[x * mw + 2 * d + 1] = mdt[v];
    mail_rows[x * mw + 2 * d + 2] = static_cast<double>(ev[v]);
  }
  API_END
}

int tgnn_memstore_write(tgnn_memstore* m, const int64_t* nodes, int64_t count, const double* mem_rows,
                        const double* mail_rows) {
  API_BEGIN
  m->ctx->use();
  const int64_t N = m->d.N, d = m->d.d, mw = 2 * d + 3;
  if (count == 0) return 0;
  // later rows win (apply_root_write in row order): keep the last row per node
  std::vector<int64_t> keep;
  {
    std::vector<int64_t> last(static_cast<size_t>(N), -1);
    for (int64_t x = 0; x < count; ++x) {
      TGB_REQUIRE(nodes[x] >= 0 && nodes[x] < N, kProtocol, "write: index out of range");
      last[static_cast<size_t>(nodes[x])] = x;
    }
    for (int64_t x = 0; x < count; ++x)
      if (last[static_cast<size_t>(nodes[x])] == x) keep.push_back(x);
  }
  const int K = static_cast<int>(keep.size());
  const size_t bytes = pack_bytes(K, d);
  std::vector<char> host(bytes, 0);
  WriteSet v = pack_view(host.data(), K, d);
  *const_cast<int32_t*>(v.count) = K;
  for (int q = 0; q < K; ++q) {
    const int64_t x = keep[static_cast<size_t>(q)];
    const_cast<int32_t*>(v.node)[q] = static_cast<int32_t>(nodes[x]);
    const_cast<int32_t*>(v.event)[q] = static_cast<int32_t>(mail_rows[x * mw + 2 * d + 2]);
    const_cast<double*>(v.t)[q] = mail_rows[x * mw + 2 * d];
    const_cast<double*>(v.dt)[q] = mail_rows[x * mw + 2 * d + 1];
    for (int64_t i = 0; i < d; ++i) const_cast<float*>(v.mem)[q * d + i] = static_cast<float>(mem_rows[x * d + i]);
    for (int64_t i = 0; i < 2 * d; ++i)
      const_cast<float*>(v.mail)[q * 2 * d + i] = static_cast<float>(mail_rows[x * mw + i]);
  }
  void* dev = nullptr;
  TGB_CUDA(cudaMalloc(&dev, bytes));
  TGB_CUDA(cudaMemcpy(dev, host.data(), bytes, cudaMemcpyHostToDevice));
  apply_writes_launch({pack_view(dev, K, d)}, m->d, m->win, m->ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(m->ctx->stream));
  cudaFree(dev);
  API_END
}

// ----------------------------------------------------------------- trainer
int tgnn_param_count(const tgnn_model_config* m, int64_t* out) {
  API_BEGIN
  *out = ParamLayout::make(dims_of(m)).total;
  API_END
}

int tgnn_init_params(const tgnn_model_config* m, uint64_t seed, double* flat) {
  API_BEGIN
  auto v = host_init_params(dims_of(m), seed);
  std::memcpy(flat, v.data(), sizeof(double) * v.size());
  API_END
}

int tgnn_trainer_create(tgnn_ctx* ctx, tgnn_graph* g, const tgnn_model_config* m, int64_t max_local_batch,
                        uint64_t seed, tgnn_trainer** out) {
  API_BEGIN
  ctx->use();
  auto tr = std::make_unique<tgnn_trainer>();
  tr->init(ctx, g, dims_of(m), max_local_batch, seed, 1);
  *out = tr.release();
  API_END
}

int tgnn_trainer_destroy(tgnn_trainer* tr) {
  API_BEGIN
  delete tr;
  API_END
}

int tgnn_trainer_set_params(tgnn_trainer* tr, const double* flat) {
  API_BEGIN
  tr->ctx->use();
  TGB_CUDA(cudaStreamSynchronize(tr->ctx->stream));
  tr->set_params(flat);
  API_END
}

int tgnn_trainer_get_params(tgnn_trainer* tr, double* flat) {
  API_BEGIN
  tr->ctx->use();
  tr->get_flat(tr->params, flat);
  API_END
}

int tgnn_trainer_get_grads(tgnn_trainer* tr, double* flat) {
  API_BEGIN
  tr->ctx->use();
  tr->get_flat(tr->grads, flat);
  API_END
}

int tgnn_trainer_sub_step(tgnn_trainer* tr, int64_t begin, int64_t end, const int64_t* negatives,
                          const double* view_mem, const double* view_mail, double* loss_out,
                          double* s_hat_out) {
  API_BEGIN
  tgnn_ctx* ctx = tr->ctx;
  ctx->use();
  plan_explicit(tr, 0, begin, end, negatives);
  const int U = plan_size(ctx, tr->plans[0], kSzU);
  upload_view(tr, tr->views[0], U, view_mem, view_mail);
  substep_launch(tr->sc(), tr->plans[0], tr->views[0], tr->d_loss, ctx->stream);
  double loss = 0;
  d2h(&loss, tr->d_loss, 1, ctx->stream);
  ctx->check_numeric();
  *loss_out = loss;
  tr->last_U = U;
  if (s_hat_out) {
    const int64_t d = tr->m.d_mem;
    std::vector<float> sh(static_cast<size_t>(U * d));
    d2h(sh.data(), tr->w.s_hat, sh.size(), ctx->stream);
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (size_t x = 0; x < sh.size(); ++x) s_hat_out[x] = sh[x];
  }
  API_END
}

int tgnn_trainer_root_writes(tgnn_trainer* tr, int64_t* nodes, double* mem_rows, double* mail_rows,
                             int64_t* num_writes) {
  API_BEGIN
  tgnn_ctx* ctx = tr->ctx;
  ctx->use();
  TGB_REQUIRE(tr->last_U >= 0, kProtocol, "root_writes: no sub_step has run");
  root_writes_launch(tr->sc(), tr->plans[0], tr->views[0], ctx->stream);
  const int64_t d = tr->m.d_mem;
  const int cap = 2 * tr->cap_B;
  std::vector<char> host(tr->w.wpack_bytes);
  d2h(host.data(), static_cast<char*>(tr->w.wpack), host.size(), ctx->stream);
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  WriteSet v = pack_view(host.data(), cap, d);
  const int W = *v.count;
  std::vector<int> order(W);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return v.node[a] < v.node[b]; });
  const int64_t mw = 2 * d + 3;
  for (int q = 0; q < W; ++q) {
    const int x = order[q];
    nodes[q] = v.node[x];
    for (int64_t i = 0; i < d; ++i) mem_rows[q * d + i] = v.mem[x * d + i];
    for (int64_t i = 0; i < 2 * d; ++i) mail_rows[q * mw + i] = v.mail[x * 2 * d + i];
    mail_rows[q * mw + 2 * d] = v.t[x];
    mail_rows[q * mw + 2 * d + 1] = v.dt[x];
    mail_rows[q * mw + 2 * d + 2] = static_cast<double>(v.event[x]);
  }
  *num_writes = W;
  API_END
}

int tgnn_trainer_adam_step(tgnn_trainer* tr, double lr) {
  API_BEGIN
  tr->ctx->use();
  tr->adam(lr, 1.0f);
  TGB_CUDA(cudaStreamSynchronize(tr->ctx->stream));
  API_END
}

int tgnn_trainer_iterate(tgnn_trainer* tr, tgnn_memstore* m, int64_t batch_index, int64_t group,
                         int64_t batch_begin, int64_t begin, int64_t end, double lr, double* loss_out) {
  API_BEGIN
  tgnn_ctx* ctx = tr->ctx;
  ctx->use();
  cudaStream_t s = ctx->stream;
  TGB_REQUIRE(begin >= 0 && end <= tr->g->d.E && begin < end && end - begin <= tr->cap_B, kConfig,
              "iterate: slice out of range");
  PlanArgs a;
  a.begin = begin;
  a.end = end;
  a.batch_begin = batch_begin;
  a.batch_index = batch_index;
  a.group = group;
  a.seed = tr->seed;
  a.neg_mode = 1;
  a.valid = 1;
  DPlan& pl = tr->plans[0];
  set_plan_args_launch(pl.args, a, s);
  plan_launch(tr->g->d, pl, s, ctx->side);
  gather_view_launch(pl, m->d, tr->views[0], s);
  StepCtx sc = tr->sc();
  substep_launch(sc, pl, tr->views[0], tr->d_loss, s);
  root_writes_launch(sc, pl, tr->views[0], s, &m->d);
  tr->adam(lr, 1.0f);
  double loss = 0;
  d2h(&loss, tr->d_loss, 1, s);
  ctx->check_numeric();
  *loss_out = loss;
  tr->last_U = -1;
  API_END
}

// ----------------------------------------------------------------- runs
int tgnn_schedule_query(const tgnn_train_config* tc, int64_t train_begin, int64_t train_end, int32_t rank,
                        int64_t first, int64_t count, int64_t* out, int64_t* barriers_out) {
  API_BEGIN
  const host::TrainCfg c = train_of(tc);
  const host::Schedule sc = host::Schedule::build(c, train_begin, train_end);
  TGB_REQUIRE(rank >= 0 && rank < c.trainers(), kConfig, "schedule: rank out of range");
  *barriers_out = sc.barriers;
  for (int64_t x = 0; x < count; ++x) {
    const int64_t b = first + x;
    int64_t* o = out + x * 12;
    for (int q = 0; q < 12; ++q) o[q] = 0;
    if (b < 0 || b >= sc.barriers) continue;
    const host::Task t = sc.task(rank, b);
    o[0] = t.active;
    o[1] = t.sub;
    o[2] = t.subs;
    o[3] = t.batch;
    o[4] = t.batch_begin;
    o[5] = t.batch_end;
    o[6] = t.slice_begin;
    o[7] = t.slice_end;
    o[8] = t.active ? t.neg_group[static_cast<size_t>(t.sub)] : -1;
    o[9] = t.active && t.sub == 0 && t.reset_before;
    o[10] = sc.active_trainers[static_cast<size_t>(b)];
    o[11] = sc.traversed_after[static_cast<size_t>(b)];
  }
  API_END
}

int tgnn_comm_unique_id(char* out128) {
  API_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NCCL_CHECK(nccl::api().GetUniqueId(&id));
  std::memcpy(out128, &id, 128);
  API_END
}

int tgnn_run_create(tgnn_ctx* ctx, tgnn_graph* g, const tgnn_run_options* opt, tgnn_run** out) {
  API_BEGIN
  ctx->use();
  auto r = std::make_unique<tgnn_run>();
  r->ctx = ctx;
  r->g = g;
  r->tc = train_of(&opt->train);
  r->tc.validate();
  r->rank = opt->rank;
  r->nranks = opt->nranks;
  const int T = r->tc.trainers();
  TGB_REQUIRE(r->nranks == T, kConfig, "run: one rank per trainer is required (nranks == i*j*k)");
  TGB_REQUIRE(r->rank >= 0 && r->rank < T, kConfig, "run: rank out of range");
  r->sched = host::Schedule::build(r->tc, opt->train_begin, opt->train_end);
  r->group = r->sched.group_of(r->rank);
  r->team = r->sched.team_of(r->rank);
  r->member = r->sched.member_of(r->rank);
  r->group_size = r->tc.i * r->tc.j;
  ModelDims m = dims_of(&opt->model);
  r->tr = std::make_unique<tgnn_trainer>();
  r->tr->init(ctx, g, m, r->tc.local_batch, r->tc.seed, r->tc.j > 1 ? 2 * r->tc.j : 1);
  r->mem.reset(memstore_new(ctx, g->d.N, m.d_mem));
  r->d_losses = dalloc<double>(static_cast<size_t>(std::max<int64_t>(r->sched.barriers, 1)));
  TGB_CUDA(cudaMemset(r->d_losses, 0, sizeof(double) * std::max<int64_t>(r->sched.barriers, 1)));
  if (r->group_size > 1) {
    TGB_CUDA(cudaMalloc(&r->gathered, r->tr->w.wpack_bytes * static_cast<size_t>(r->tc.i)));
  }
  r->oplog = opt->oplog != 0;
  if (r->oplog) {
    const int64_t nb = std::max<int64_t>(r->sched.barriers, 1);
    r->d_oplog = dalloc<int64_t>(static_cast<size_t>(4 * nb));
    TGB_CUDA(cudaMemset(r->d_oplog, 0, sizeof(int64_t) * 4 * nb));
  }
  r->snaps = opt->segment_snapshots != 0;
  if (r->snaps) {
    const auto& ps = r->sched.groups[static_cast<size_t>(r->group)];
    r->snap_slot.assign(ps.size(), -1);
    for (size_t x = 0; x < ps.size(); ++x) {
      if (!r->sched.snapshot_after(ps[x])) continue;
      r->snap_slot[x] = static_cast<int64_t>(r->snap_meta.size());
      r->snap_meta.push_back({static_cast<int64_t>(ps[x].sweep), static_cast<int64_t>(ps[x].segment)});
    }
    const size_t n = std::max<size_t>(r->snap_meta.size(), 1);
    r->d_snap_mem = dalloc<float>(n * static_cast<size_t>(g->d.N * m.d_mem));
    r->d_snap_lu = dalloc<double>(n * static_cast<size_t>(g->d.N));
  }
  r->val_begin = opt->val_begin;
  r->val_end = opt->val_end;
  r->eval_batch = opt->eval_batch;
  r->eval_negatives = opt->eval_negatives;
  TGB_REQUIRE(r->val_end <= r->val_begin || (r->val_begin >= 0 && r->val_end <= g->d.E), kConfig,
              "run: validation range out of bounds");
  TGB_REQUIRE(r->eval_negatives >= 0 && r->eval_batch >= 0, kConfig, "run: invalid evaluation options");
  TGB_CUDA(cudaEventCreate(&r->ev_t0));
  r->use_graphs = opt->use_graphs != 0 && r->tc.j <= kMaxStintJ && !r->snaps;
  if (r->use_graphs && r->tc.j > 1) {
    std::vector<StintDesc> sd(static_cast<size_t>(r->sched.barriers + r->tc.j + 1));
    for (int64_t b = 0; b < r->sched.barriers; b += r->tc.j) {
      StintDesc& e = sd[static_cast<size_t>(b)];
      const host::Task t = r->sched.task(r->rank, b);
      for (int sub = 0; sub < r->tc.j; ++sub) {
        PlanArgs& a = e.args[sub];
        a.begin = t.slice_begin;
        a.end = t.slice_end;
        a.batch_begin = t.batch_begin;
        a.batch_index = t.batch;
        a.seed = r->tc.seed;
        a.neg_mode = 1;
        a.valid = t.active && sub < t.subs ? 1 : 0;
        a.group = a.valid ? t.neg_group[static_cast<size_t>(sub)] : 0;
      }
      for (int tt = 0; tt < r->tc.j; ++tt) {
        const host::Task tk = r->sched.task(r->group * r->tc.i * r->tc.j + tt * r->tc.i, b);
        e.reset[tt] = tk.active && tk.reset_before ? 1 : 0;
      }
    }
    r->d_stint = dalloc<StintDesc>(sd.size());
    TGB_CUDA(cudaMemcpy(r->d_stint, sd.data(), sizeof(StintDesc) * sd.size(), cudaMemcpyHostToDevice));
    r->h_stint = sd;
  }
  if (r->use_graphs) {
    // one idle entry past the end: the last barrier prepares an empty plan
    const int64_t nb = r->sched.barriers + 1;
    std::vector<BarrierDesc> desc(static_cast<size_t>(nb));
    for (int64_t b = 0; b < r->sched.barriers; ++b) {
      const host::Task t = r->sched.task(r->rank, b);
      BarrierDesc& d = desc[static_cast<size_t>(b)];
      d.args.begin = t.slice_begin;
      d.args.end = t.slice_end;
      d.args.batch_begin = t.batch_begin;
      d.args.batch_index = t.batch;
      d.args.group = t.active ? t.neg_group[0] : 0;
      d.args.seed = r->tc.seed;
      d.args.neg_mode = 1;
      d.args.valid = t.active ? 1 : 0;
      // the group's copy resets before the read of its sweep's first pair; every
      // member of the group sees the same flag (pair index == barrier at j == 1)
      const host::Task t0 = r->sched.task(r->group * r->tc.i * r->tc.j, b);
      d.reset = t0.active && t0.reset_before ? 1 : 0;
      const int64_t active = r->sched.active_trainers[static_cast<size_t>(b)];
      d.lr = static_cast<float>(r->tc.lr_eff());
      d.c1 = static_cast<float>(1.0 - std::pow(0.9, static_cast<double>(b + 1)));
      d.c2 = static_cast<float>(1.0 - std::pow(0.999, static_cast<double>(b + 1)));
      d.scale = 1.0f / static_cast<float>(active > 0 ? active : 1);
    }
    r->d_desc = dalloc<BarrierDesc>(desc.size());
    TGB_CUDA(cudaMemcpy(r->d_desc, desc.data(), sizeof(BarrierDesc) * desc.size(), cudaMemcpyHostToDevice));
    r->d_ctr = dalloc<int>(1);
    TGB_CUDA(cudaMemset(r->d_ctr, 0, sizeof(int)));
    r->d_ctr_tail = dalloc<int>(1);
    TGB_CUDA(cudaMemset(r->d_ctr_tail, 0, sizeof(int)));
  }
  *out = r.release();
  API_END
}

int tgnn_run_comm_init(tgnn_run* r, const char* unique_id128) {
  API_BEGIN
  r->ctx->use();
  if (r->nranks == 1) return 0;
  TGB_REQUIRE(!r->comm_ready, kProtocol, "run: communicator already initialised");
  ncclUniqueId id;
  std::memcpy(&id, unique_id128, 128);
  NCCL_CHECK(nccl::api().CommInitRank(&r->comm, r->nranks, id, r->rank));
  if (r->group_size > 1) {
    NCCL_CHECK(nccl::api().CommSplit(r->comm, r->group, r->rank, &r->gcomm, nullptr));
  }
  NCCL_CHECK(nccl::api().CommSplit(r->comm, 0, r->rank, &r->hcomm, nullptr));
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_tail, cudaEventDisableTiming));
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_head, cudaEventDisableTiming));
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_comm, cudaEventDisableTiming));
  r->comm_ready = true;
  API_END
}

int tgnn_local_hub_create(int32_t nranks, tgnn_local_hub** out) {
  API_BEGIN
  TGB_REQUIRE(nranks >= 1 && nranks <= kLocalMax, kConfig, "local hub: rank count must lie in [1, 16]");
  auto* h = new tgnn_local_hub();
  h->n = nranks;
  h->runs.assign(static_cast<size_t>(nranks), nullptr);
  h->src.assign(static_cast<size_t>(nranks), nullptr);
  *out = h;
  API_END
}

int tgnn_local_hub_destroy(tgnn_local_hub* h) {
  API_BEGIN
  delete h;
  API_END
}

int tgnn_run_local_init(tgnn_run* r, tgnn_local_hub* h) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(h != nullptr && h->n == r->nranks, kConfig, "local hub: rank count differs from the run's");
  TGB_REQUIRE(!r->comm_ready, kProtocol, "run: communicator already initialised");
  if (r->nranks == 1) return 0;
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_lready, cudaEventDisableTiming));
  TGB_CUDA(cudaEventCreateWithFlags(&r->ev_ldone, cudaEventDisableTiming));
  {
    std::lock_guard<std::mutex> lk(h->mu);
    TGB_REQUIRE(h->runs[static_cast<size_t>(r->rank)] == nullptr, kProtocol, "local hub: rank attached twice");
    h->runs[static_cast<size_t>(r->rank)] = r;
  }
  r->hub = h;
  // collectives are host rendezvous at enqueue time: barriers run on the
  // direct (stream-ordered) path, not from captured graphs
  r->use_graphs = false;
  h->rendezvous();  // every rank attached
  for (int q = 0; q < h->n; ++q) {
    const int dev = h->runs[static_cast<size_t>(q)]->ctx->device;
    if (dev == r->ctx->device) continue;
    const cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TGB_CUDA(e);
    cudaGetLastError();
  }
  r->comm_ready = true;
  API_END
}

int tgnn_run_destroy(tgnn_run* r) {
  API_BEGIN
  if (r) {
    cudaSetDevice(r->ctx->device);
    cudaStreamSynchronize(r->ctx->stream);
  }
  delete r;
  API_END
}

int tgnn_run_info(tgnn_run* r, int64_t* barriers, int64_t* param_count) {
  API_BEGIN
  *barriers = r->sched.barriers;
  *param_count = r->tr->L.total;
  API_END
}

int tgnn_run_barriers(tgnn_run* r, int64_t first, int64_t count) {
  API_BEGIN
  r->ctx->use();
  HubGuard guard(r);
  TGB_REQUIRE(first == r->next_barrier, kProtocol, "run: barriers must be issued in order");
  TGB_REQUIRE(first + count <= r->sched.barriers, kConfig, "run: barrier range past the schedule");
  TGB_REQUIRE(r->nranks == 1 || r->comm_ready, kProtocol, "run: communicator not initialised");
  if (first == 0 && count > 0) TGB_CUDA(cudaEventRecord(r->ev_t0, r->ctx->stream));
  const auto& evb = r->sched.eval_barriers;
  int64_t b = first;
  const int64_t stop = first + count;
  while (b < stop) {
    // segments end at eval barriers, where rank 0 evaluates between barriers
    while (r->eval_cursor < evb.size() && evb[r->eval_cursor] < b) ++r->eval_cursor;
    int64_t seg_end = stop;
    bool eval_here = false;
    if (r->eval_cursor < evb.size() && evb[r->eval_cursor] < stop) {
      seg_end = evb[r->eval_cursor] + 1;
      eval_here = true;
    }
    if (r->use_graphs && r->tc.j > 1) {
      if (r->sexec.empty()) build_stint_graphs(r);
      set_int_kernel<<<1, 1, 0, r->ctx->stream>>>(r->d_ctr, static_cast<int>(b));
      set_int_kernel<<<1, 1, 0, r->ctx->stream>>>(r->d_ctr_tail, static_cast<int>(b));
      TGB_CUDA(cudaGetLastError());
      pack_weights(r->tr->sc(), r->ctx->stream);  // the stint graphs read packed weights
      const int j = r->tc.j;
      for (int64_t x = b; x < seg_end; ++x) {
        const int sidx = static_cast<int>(x % j);
        const int64_t b0 = x - sidx;
        const int set = static_cast<int>((b0 / j) % 2);
        if (sidx == 0 && r->stint_planned != b0) plan_stint_now(r, b0);
        TGB_CUDA(cudaGraphLaunch(r->sexec[static_cast<size_t>(set * j + sidx)], r->ctx->stream));
        if (sidx == j - 1) r->stint_planned = b0 + j;  // planned ahead by this position
      }
      r->tr->adam_t = seg_end;
    } else if (r->use_graphs) {
      if (!r->exec[0]) build_graph(r);
      if (r->prepared != b) prepare_barrier(r, b);
      for (int64_t x = b; x < seg_end;) {
        if ((x & 1) == 0 && x + kMultiBarrier <= seg_end) {
          TGB_CUDA(cudaGraphLaunch(r->mexec, r->ctx->stream));
          x += kMultiBarrier;
        } else {
          TGB_CUDA(cudaGraphLaunch(r->exec[x & 1], r->ctx->stream));
          ++x;
        }
      }
      r->prepared = seg_end;
      r->tr->adam_t = seg_end;
    } else {
      for (int64_t x = b; x < seg_end; ++x) run_barrier(r, x);
    }
    if (eval_here) {
      run_eval_point(r, seg_end - 1);
      ++r->eval_cursor;
    }
    b = seg_end;
  }
  r->next_barrier = stop;
  guard.ok();
  API_END
}

int tgnn_run_losses(tgnn_run* r, int64_t first, int64_t count, double* out) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(first >= 0 && first + count <= r->next_barrier, kConfig, "run: loss range not yet run");
  HubGuard guard(r);
  cudaStream_t s = r->ctx->stream;
  double* tmp = dalloc<double>(static_cast<size_t>(std::max<int64_t>(count, 1)));
  TGB_CUDA(cudaMemcpyAsync(tmp, r->d_losses + first, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  comm_allreduce(r, tmp, static_cast<size_t>(count), RedTy::F64, RedOp::Sum, s);
  d2h(out, tmp, static_cast<size_t>(count), s);
  r->ctx->check_numeric();
  cudaFree(tmp);
  guard.ok();
  for (int64_t b = 0; b < count; ++b) {
    const int64_t a = r->sched.active_trainers[static_cast<size_t>(first + b)];
    out[b] = a > 0 ? out[b] / static_cast<double>(a) : 0.0;
  }
  API_END
}

int tgnn_run_params(tgnn_run* r, double* flat) {
  API_BEGIN
  r->ctx->use();
  r->tr->get_flat(r->tr->params, flat);
  API_END
}

int tgnn_run_metrics(tgnn_run* r, int64_t* count, double* rows) {
  API_BEGIN
  r->ctx->use();
  *count = static_cast<int64_t>(r->rows.size());
  if (!rows) return 0;
  const int64_t nb = r->next_barrier;
  std::vector<double> loss(static_cast<size_t>(std::max<int64_t>(nb, 1)));
  if (nb > 0) {
    const int rc = tgnn_run_losses(r, 0, nb, loss.data());
    if (rc) return rc;
  }
  TGB_CUDA(cudaStreamSynchronize(r->ctx->stream));
  int64_t prev = 0;
  for (size_t x = 0; x < r->rows.size(); ++x) {
    const tgnn_run::Row& row = r->rows[x];
    double acc = 0.0;
    for (int64_t b = prev; b <= row.barrier; ++b) acc += loss[static_cast<size_t>(b)];
    const int64_t n = row.barrier + 1 - prev;
    prev = row.barrier + 1;
    float ms = 0.0f;
    TGB_CUDA(cudaEventElapsedTime(&ms, r->ev_t0, row.done));
    double* o = rows + 5 * x;
    o[0] = static_cast<double>(row.barrier + 1);
    o[1] = static_cast<double>(r->sched.traversed_after[static_cast<size_t>(row.barrier)]);
    o[2] = n > 0 ? acc / static_cast<double>(n) : 0.0;
    o[3] = row.val_mrr;
    o[4] = static_cast<double>(ms) * 1e-3;
  }
  API_END
}

int tgnn_run_evaluate_mrr(tgnn_run* r, int64_t eval_begin, int64_t eval_end, int64_t batch_size,
                          int32_t n_negatives, uint64_t seed, double* mrr, int64_t* queries) {
  API_BEGIN
  r->ctx->use();
  if (!r->ev || r->ev->cap_B != batch_size || r->ev->n_neg != n_negatives) {
    r->ev = std::make_unique<tgnn_evaluator>();
    r->ev->init(r->ctx, r->g, r->tr->m, batch_size, n_negatives);
  }
  TGB_CUDA(cudaMemcpyAsync(r->ev->params, r->tr->params, sizeof(float) * r->tr->L.total,
                           cudaMemcpyDeviceToDevice, r->ctx->stream));
  *mrr = r->ev->evaluate(eval_begin, eval_end, seed, queries);
  API_END
}

int tgnn_run_eval_barriers(tgnn_run* r, int64_t* count, int64_t* out) {
  API_BEGIN
  const auto& e = r->sched.eval_barriers;
  *count = static_cast<int64_t>(e.size());
  if (out)
    for (size_t x = 0; x < e.size(); ++x) out[x] = e[x];
  API_END
}

int tgnn_run_traversed(tgnn_run* r, int64_t first, int64_t count, int64_t* out) {
  API_BEGIN
  const auto& ta = r->sched.traversed_after;
  TGB_REQUIRE(first >= 0 && first + count <= r->sched.barriers, kConfig, "run: range out of bounds");
  const int64_t hi = count > 0 ? ta[static_cast<size_t>(first + count - 1)] : 0;
  const int64_t lo = first > 0 ? ta[static_cast<size_t>(first - 1)] : 0;
  *out = count > 0 ? hi - lo : 0;
  API_END
}

int tgnn_run_launches_per_barrier(tgnn_run* r, int64_t* out) {
  API_BEGIN
  r->ctx->use();
  if (r->use_graphs) {
    if (r->tc.j > 1) {
      if (r->sexec.empty()) build_stint_graphs(r);
    } else if (!r->exec[0]) {
      build_graph(r);
    }
    *out = r->launches;
    return 0;
  }
  TGB_REQUIRE(r->next_barrier < r->sched.barriers, kConfig, "run: no barrier left to inspect");
  TGB_REQUIRE(r->nranks == 1, kConfig, "run: launch counting is done on single-rank runs");
  cudaStream_t s = r->ctx->stream;
  TGB_CUDA(cudaStreamSynchronize(s));
  const int64_t saved_t = r->tr->adam_t;
  cudaGraph_t graph = nullptr;
  TGB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    run_barrier(r, r->next_barrier);
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    r->tr->adam_t = saved_t;
    throw;
  }
  TGB_CUDA(cudaStreamEndCapture(s, &graph));
  r->tr->adam_t = saved_t;
  size_t n = 0;
  TGB_CUDA(cudaGraphGetNodes(graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  TGB_CUDA(cudaGraphGetNodes(graph, nodes.data(), &n));
  int64_t kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    TGB_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) ++kernels;
  }
  cudaGraphDestroy(graph);
  r->launches = kernels;
  *out = kernels;
  API_END
}

int tgnn_run_profile_barrier(tgnn_run* r, double* phase_ms, int32_t* sizes, int32_t direct) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(r->next_barrier < r->sched.barriers, kConfig, "run: no barrier left to profile");
  TGB_REQUIRE(r->nranks == 1 || r->comm_ready, kProtocol, "run: communicator not initialised");
  if (!r->marks_ready) {
    for (auto& e : r->marks.ev) TGB_CUDA(cudaEventCreate(&e));
    r->marks_ready = true;
  }
  for (auto& h : r->marks.hit) h = false;
  r->marks.on = true;
  const int64_t b = r->next_barrier;
  unsigned long long ts_host[phCount + 1] = {};
  bool have_ts = false;
  try {
    if (r->use_graphs && r->tc.j == 1 && !direct) {
      // the production graph body, captured once more with phase stamps on
      // the main stream, replayed for this barrier
      if (!r->exec[0]) build_graph(r);
      if (r->prepared != b) prepare_barrier(r, b);
      cudaStream_t s = r->ctx->stream;
      cudaGraph_t gph = nullptr;
      cudaGraphExec_t ex = nullptr;
      unsigned long long* d_ts = dalloc<unsigned long long>(phCount + 1);
      r->marks.d_ts = d_ts;
      TGB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        barrier_body_dev(r, static_cast<int>(b & 1));
      } catch (...) {
        cudaStreamEndCapture(s, &gph);
        if (gph) cudaGraphDestroy(gph);
        r->marks.d_ts = nullptr;
        cudaFree(d_ts);
        throw;
      }
      r->marks.d_ts = nullptr;
      TGB_CUDA(cudaStreamEndCapture(s, &gph));
      TGB_CUDA(cudaGraphInstantiate(&ex, gph, 0));
      TGB_CUDA(cudaGraphLaunch(ex, s));
      TGB_CUDA(cudaStreamSynchronize(s));
      cudaGraphExecDestroy(ex);
      cudaGraphDestroy(gph);
      TGB_CUDA(cudaMemcpy(ts_host, d_ts, sizeof(ts_host), cudaMemcpyDeviceToHost));
      cudaFree(d_ts);
      have_ts = true;
      r->prepared = b + 1;
      r->tr->adam_t = b + 1;
    } else {
      run_barrier(r, b);
    }
  } catch (...) {
    r->marks.on = false;
    throw;
  }
  r->marks.on = false;
  ++r->next_barrier;
  TGB_CUDA(cudaStreamSynchronize(r->ctx->stream));
  r->ctx->check_numeric();
  // order the recorded markers by time; each interval belongs to its opening marker
  std::vector<std::pair<float, int>> at;
  for (int x = 0; x <= phCount; ++x) {
    if (!r->marks.hit[x]) continue;
    float ms = 0;
    if (have_ts) ms = static_cast<float>(static_cast<double>(ts_host[x] - ts_host[phPlan]) * 1e-6);
    else TGB_CUDA(cudaEventElapsedTime(&ms, r->marks.ev[phPlan], r->marks.ev[x]));
    at.push_back({ms, x});
  }
  std::stable_sort(at.begin(), at.end());
  for (int x = 0; x < phCount; ++x) phase_ms[x] = 0.0;
  for (size_t q = 0; q + 1 < at.size(); ++q)
    if (at[q].second < phCount) phase_ms[at[q].second] += at[q + 1].first - at[q].first;
  int32_t sz[kSzCount];
  const int jj = r->tc.j;
  const size_t slot = jj > 1 ? static_cast<size_t>(((b / jj) % 2) * jj + b % jj)
                             : (r->use_graphs && !direct ? static_cast<size_t>(b & 1) : 0);
  TGB_CUDA(cudaMemcpy(sz, r->tr->plans[slot].sizes, sizeof(sz), cudaMemcpyDeviceToHost));
  TGB_CUDA(cudaMemcpy(&sz[7], r->tr->w.w_count, sizeof(int32_t), cudaMemcpyDeviceToHost));  // W root writes
  for (int x = 0; x < kSzCount; ++x) sizes[x] = sz[x];
  API_END
}

int tgnn_run_gemm_profile(tgnn_run* r, int64_t cap, int64_t* count, double* rows) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(r->next_barrier < r->sched.barriers, kConfig, "run: no barrier left to profile");
  TGB_REQUIRE(r->nranks == 1 || r->comm_ready, kProtocol, "run: communicator not initialised");
  TGB_REQUIRE(gemm_impl() == kGemmTma, kConfig, "run: the GEMM profile covers the tcgen05 TMA engine");
  HubGuard guard(r);
  const int64_t b = r->next_barrier;
  tc_trace_begin();
  try {
    run_barrier(r, b);
  } catch (...) {
    for (auto& e : tc_trace_end()) {
      cudaEventDestroy(e.e0);
      cudaEventDestroy(e.e1);
    }
    throw;
  }
  std::vector<TcTraceEntry> tr = tc_trace_end();
  ++r->next_barrier;
  r->prepared = -1;
  TGB_CUDA(cudaStreamSynchronize(r->ctx->stream));
  r->ctx->check_numeric();
  *count = static_cast<int64_t>(tr.size());
  for (size_t x = 0; x < tr.size(); ++x) {
    const TcTraceEntry& e = tr[x];
    float ms = 0.0f;
    TGB_CUDA(cudaEventElapsedTime(&ms, e.e0, e.e1));
    double flops = 0.0, bytes = 0.0;
    int maxm = 0, maxs = 1;
    for (int q = 0; q < e.count; ++q) {
      int64_t M = e.M[q], K = e.K[q];
      const int64_t N = e.N[q];
      int v = 0;
      if (e.M_dev[q]) {
        TGB_CUDA(cudaMemcpy(&v, e.M_dev[q], sizeof(int), cudaMemcpyDeviceToHost));
        M = std::min<int64_t>(M, v);
      }
      if (e.K_dev[q]) {
        TGB_CUDA(cudaMemcpy(&v, e.K_dev[q], sizeof(int), cudaMemcpyDeviceToHost));
        K = std::min<int64_t>(K, v);
      }
      flops += 2.0 * static_cast<double>(M) * static_cast<double>(N) * static_cast<double>(K);
      bytes += 4.0 * static_cast<double>(M * K + N * K + M * N);
      maxm = std::max<int>(maxm, static_cast<int>(M));
      maxs = std::max(maxs, e.splits[q]);
    }
    if (static_cast<int64_t>(x) < cap) {
      double* o = rows + 6 * x;
      o[0] = ms;
      o[1] = flops;
      o[2] = bytes;
      o[3] = e.count;
      o[4] = maxm;
      o[5] = maxs;
    }
    cudaEventDestroy(e.e0);
    cudaEventDestroy(e.e1);
  }
  guard.ok();
  API_END
}

int tgnn_graph_ingest(tgnn_graph* g, int64_t first, int64_t count, const int32_t* src, const int32_t* dst,
                      const double* t, const float* efeat) {
  API_BEGIN
  tgnn_ctx* ctx = g->ctx;
  ctx->use();
  TGB_REQUIRE(first >= 0 && count >= 0 && first + count <= g->d.E, kConfig, "ingest: range out of bounds");
  // copies on the ingestion stream: they overlap work enqueued earlier and
  // are ordered before any work enqueued after this call
  cudaStream_t s = ctx->h2d;
  if (count > g->st_cap) {
    TGB_CUDA(cudaStreamSynchronize(s));
    for (void* p : {static_cast<void*>(g->st_src), static_cast<void*>(g->st_dst), static_cast<void*>(g->st_t)})
      if (p) cudaFree(p);
    g->st_src = dalloc<int32_t>(static_cast<size_t>(count));
    g->st_dst = dalloc<int32_t>(static_cast<size_t>(count));
    g->st_t = dalloc<double>(static_cast<size_t>(count));
    g->st_cap = count;
  }
  // the index data lands in staging and is checked against the T-CSR's
  // events (bitwise; a mismatch fails the next synchronising call with
  // TGNN_PROTOCOL); the indexed arrays themselves are never rewritten, so
  // planning work already enqueued cannot race with this copy
  h2d(g->st_src, src, static_cast<size_t>(count), s);
  h2d(g->st_dst, dst, static_cast<size_t>(count), s);
  h2d(g->st_t, t, static_cast<size_t>(count), s);
  if (count > 0) {
    ingest_verify_kernel<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 2 * num_sms())), 256, 0, s>>>(
        g->st_src, g->st_dst, g->st_t, g->d.src + first, g->d.dst + first, g->d.t + first, count, ctx->d_flag);
    TGB_CUDA(cudaGetLastError());
  }
  if (g->d.d_e > 0 && efeat) {
    if (g->d.d_e == g->d.d_e_pad) {
      h2d(g->d.efeat + first * g->d.d_e_pad, efeat, static_cast<size_t>(count * g->d.d_e), s);
    } else {
      TGB_CUDA(cudaMemcpy2DAsync(g->d.efeat + first * g->d.d_e_pad, sizeof(float) * g->d.d_e_pad, efeat,
                                 sizeof(float) * g->d.d_e, sizeof(float) * g->d.d_e, static_cast<size_t>(count),
                                 cudaMemcpyHostToDevice, s));
    }
  }
  TGB_CUDA(cudaEventRecord(ctx->ev_h2d, s));
  TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_h2d, 0));
  API_END
}

int tgnn_set_gemm_impl(int impl) {
  API_BEGIN
  TGB_REQUIRE(impl == kGemmSimt || impl == kGemmTma || impl == kGemmGather, kConfig,
              "gemm impl must be 0 (fp32 SIMT), 1 (TMA tcgen05) or 2 (gather tcgen05)");
  set_gemm_impl(impl);
  API_END
}

int tgnn_get_gemm_impl(int* impl) {
  API_BEGIN
  *impl = gemm_impl();
  API_END
}

int tgnn_debug_gemm(int impl, int64_t M, int64_t N, int64_t K, const float* A, int a_trans, const float* B,
                    int b_trans, float* C, int splits) {
  API_BEGIN
  TGB_REQUIRE(M > 0 && N > 0 && K > 0 && splits >= 1, kConfig, "debug_gemm: bad sizes");
  float *dA = dalloc<float>(M * K), *dB = dalloc<float>(K * N), *dC = dalloc<float>(M * N);
  float* ws = splits > 1 ? dalloc<float>(static_cast<size_t>(splits) * M * ((N + 3) / 4 * 4)) : nullptr;
  TGB_CUDA(cudaMemcpy(dA, A, sizeof(float) * M * K, cudaMemcpyHostToDevice));
  TGB_CUDA(cudaMemcpy(dB, B, sizeof(float) * K * N, cudaMemcpyHostToDevice));
  GemmGroup gg;
  GemmProblem& P = gg.p[gg.count++];
  P.M = static_cast<int>(M);
  P.N = static_cast<int>(N);
  P.K = static_cast<int>(K);
  P.a = a_trans ? A_trans(dA, M, static_cast<int>(K)) : A_rows(dA, K, static_cast<int>(K));
  P.b = b_trans ? B_wT(dB, K, static_cast<int>(K)) : B_w(dB, N, static_cast<int>(K));
  P.C = dC;
  P.ldc = N;
  P.splits = splits;
  P.ws = ws;
  if (impl == kGemmTma) {
    // TMA engine over bf16 hi/lo operands (the step's production path)
    const int64_t ar = a_trans ? K : M, ac = a_trans ? M : K;
    const int64_t br = b_trans ? N : K, bc = b_trans ? K : N;
    BfMat ba = bf_alloc(ar, ac), bb = bf_alloc(br, bc);
    bf_from_f32(ba, dA, ar, ac, ac, nullptr);
    bf_from_f32(bb, dB, br, bc, bc, nullptr);
    TcGroup tg;
    TcProblem& T = tg.p[tg.count++];
    T.M = static_cast<int>(M);
    T.N = static_cast<int>(N);
    T.K = static_cast<int>(K);
    T.ntile = tc_ntile(static_cast<int>(N));
    T.a = tma_view(ba, 0, ac, ar, !a_trans, 128);
    T.b = tma_view(bb, 0, bc, br, b_trans, T.ntile);
    T.C = dC;
    T.ldc = N;
    T.splits = splits;
    T.ws = ws;
    T.ldw = static_cast<int>((N + 3) / 4 * 4);
    tc_group_launch(tg, nullptr);
    TGB_CUDA(cudaDeviceSynchronize());
    bf_free(ba);
    bf_free(bb);
  } else if (impl == kGemmGather) {
    gemm_group_launch_tc(gg, nullptr);
  } else {
    gemm_group_launch_simt(gg, nullptr);
  }
  TGB_CUDA(cudaDeviceSynchronize());
  TGB_CUDA(cudaMemcpy(C, dC, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  if (ws) cudaFree(ws);
  API_END
}

int tgnn_debug_gru_trace(uint64_t* out, int32_t cap_ctas, int32_t* n_ctas) {
  API_BEGIN
  gru_debug_trace(reinterpret_cast<unsigned long long*>(out), cap_ctas, n_ctas);
  API_END
}

int tgnn_pinned_alloc(int64_t bytes, void** out) {
  API_BEGIN
  TGB_CUDA(cudaMallocHost(out, static_cast<size_t>(bytes > 0 ? bytes : 1)));
  API_END
}

int tgnn_pinned_free(void* p) {
  API_BEGIN
  if (p) TGB_CUDA(cudaFreeHost(p));
  API_END
}


int tgnn_evaluator_create(tgnn_ctx* ctx, tgnn_graph* g, const tgnn_model_config* m, int64_t batch_size,
                          int32_t n_negatives, tgnn_evaluator** out) {
  API_BEGIN
  ctx->use();
  auto ev = std::make_unique<tgnn_evaluator>();
  ev->init(ctx, g, dims_of(m), batch_size, n_negatives);
  *out = ev.release();
  API_END
}

int tgnn_evaluator_destroy(tgnn_evaluator* ev) {
  API_BEGIN
  if (ev) {
    cudaSetDevice(ev->ctx->device);
    cudaStreamSynchronize(ev->ctx->stream);
  }
  delete ev;
  API_END
}

int tgnn_evaluate_mrr(tgnn_evaluator* ev, const double* params, int64_t eval_begin, int64_t eval_end,
                      uint64_t seed, double* mrr, int64_t* queries) {
  API_BEGIN
  ev->ctx->use();
  if (params) ev->set_params(params);
  *mrr = ev->evaluate(eval_begin, eval_end, seed, queries);
  API_END
}

int tgnn_replay_batch(tgnn_evaluator* ev, tgnn_memstore* state, const double* params, int64_t begin,
                      int64_t end) {
  API_BEGIN
  ev->ctx->use();
  TGB_REQUIRE(begin >= 0 && end <= ev->g->d.E && begin <= end, kConfig, "replay_batch: event range out of bounds");
  TGB_REQUIRE(end - begin <= ev->cap_B, kConfig, "replay_batch: batch exceeds the evaluator capacity");
  TGB_REQUIRE(state->d.N == ev->m.num_nodes && state->d.d == ev->m.d_mem, kShape,
              "replay_batch: memory store shape does not match the model");
  if (params) ev->set_params(params);
  ev->replay(state->d, begin, end, ev->cap_B);
  TGB_CUDA(cudaStreamSynchronize(ev->ctx->stream));
  ev->ctx->check_numeric();
  API_END
}

int tgnn_eval_candidates(tgnn_evaluator* ev, int64_t begin, int64_t end, uint64_t seed, int64_t* out) {
  API_BEGIN
  ev->ctx->use();
  const DGraph& G = ev->g->d;
  TGB_REQUIRE(begin >= 0 && end <= G.E && begin <= end, kConfig, "eval_candidates: event range out of bounds");
  TGB_REQUIRE(end - begin <= ev->cap_B, kConfig, "eval_candidates: range exceeds the evaluator capacity");
  const int64_t lo = G.boundary >= 0 ? G.boundary : 0;
  TGB_REQUIRE(ev->n_neg == 0 || G.N - lo >= 2, kConfig,
              "evaluate_mrr: destination partition too small to sample distractors");
  const int64_t cnt = (end - begin) * ev->n_neg;
  if (cnt == 0) return 0;
  cudaStream_t s = ev->ctx->stream;
  PlanArgs a;
  a.begin = begin;
  a.end = end;
  a.batch_begin = begin;
  a.seed = seed;
  a.neg_mode = 2;
  a.valid = 1;
  set_plan_args_launch(ev->pe.args, a, s);
  plan_launch(G, ev->pe, s);
  std::vector<int32_t> tmp(static_cast<size_t>(cnt));
  d2h(tmp.data(), ev->pe.negs, static_cast<size_t>(cnt), s);
  TGB_CUDA(cudaStreamSynchronize(s));
  for (int64_t x = 0; x < cnt; ++x) out[x] = tmp[static_cast<size_t>(x)];
  API_END
}


int tgnn_checkpoint_save(const tgnn_model_config* m, const double* flat, const char* path) {
  API_BEGIN
  const auto man = host::ckpt_manifest(m->d_mem, m->d_time, m->d_static, m->d_attn, m->d_hidden, m->d_e,
                                       m->num_nodes);
  const std::string err = host::ckpt_save(man, flat, path);
  TGB_REQUIRE(err.empty(), kConfig, err);
  API_END
}

int tgnn_checkpoint_load(const tgnn_model_config* m, const char* path, double* flat) {
  API_BEGIN
  const auto man = host::ckpt_manifest(m->d_mem, m->d_time, m->d_static, m->d_attn, m->d_hidden, m->d_e,
                                       m->num_nodes);
  const std::string err = host::ckpt_load(man, path, flat);
  TGB_REQUIRE(err.empty(), kConfig, err);
  API_END
}


int tgnn_graph_synthetic(tgnn_ctx* ctx, const tgnn_synth_params* p, int32_t threads, tgnn_graph** out) {
  API_BEGIN
  ctx->use();
  host::SynthConfig c;
  c.nodes = p->nodes;
  c.events = p->events;
  c.burst_prob = p->burst_prob;
  c.pref_prob = p->pref_prob;
  c.prefs_per_src = p->prefs_per_src;
  c.src_frac = p->src_frac;
  c.bipartite = p->bipartite != 0;
  c.d_e = p->d_e;
  c.zipf_s = p->zipf_s;
  c.seed = p->seed;
  const host::Generator probe(c);  // validates and fixes the boundary
  auto g = graph_alloc(ctx, c.nodes, probe.boundary(), c.events, c.d_e);
  if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency() - 1));
  synth_stream_to_device(c, g->d, ctx->stream, threads);
  graph_finalize_device(g->d, ctx->stream);
  *out = g.release();
  API_END
}

int tgnn_graph_load_dataset(tgnn_ctx* ctx, const char* csv_path, int32_t threads, tgnn_graph** out) {
  API_BEGIN
  const std::string path(csv_path);
  const host::DatasetMeta meta = host::load_sidecar(host::sidecar_path(path));
  host::EventTable tab;
  if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
  host::load_events(path, meta, threads, tab);  // parse errors surface before any device work
  TGB_REQUIRE(ctx != nullptr, kConfig, "load_dataset: a device context is required");
  ctx->use();
  const int64_t E = static_cast<int64_t>(tab.t.size());
  const int rc = graph_create_impl(ctx, meta.num_nodes, meta.boundary, E, tab.src.data(), tab.dst.data(),
                                   tab.t.data(), tab.efeat.data(), nullptr, meta.d_e, out);
  if (rc) return rc;
  API_END
}

int tgnn_write_dataset(const char* csv_path, int64_t num_nodes, int64_t bipartite_boundary, int64_t num_events,
                       const int64_t* src, const int64_t* dst, const double* t, const double* efeat, int64_t d_e) {
  API_BEGIN
  host::write_dataset(csv_path, num_nodes, bipartite_boundary, num_events, src, dst, t, efeat, d_e);
  API_END
}

int tgnn_chronological_split(int64_t num_events, double train_frac, double val_frac, int64_t* train_end,
                             int64_t* val_end) {
  API_BEGIN
  host::chronological_split(num_events, train_frac, val_frac, train_end, val_end);
  API_END
}


int tgnn_graph_edge_feats(tgnn_graph* g, int64_t first, int64_t count, float* out) {
  API_BEGIN
  g->ctx->use();
  const DGraph& D = g->d;
  TGB_REQUIRE(first >= 0 && count >= 0 && first + count <= D.E, kConfig, "edge_feats: range out of bounds");
  if (D.d_e == 0 || count == 0) return 0;
  TGB_CUDA(cudaMemcpy2DAsync(out, sizeof(float) * D.d_e, D.efeat + first * D.d_e_pad, sizeof(float) * D.d_e_pad,
                             sizeof(float) * D.d_e, static_cast<size_t>(count), cudaMemcpyDeviceToHost, g->ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(g->ctx->stream));
  API_END
}


int tgnn_debug_gemm_bench(int64_t M, int64_t N, int64_t K, int32_t ntile, int32_t iters, double* us,
                          uint64_t* trace, int32_t* grid) {
  API_BEGIN
  tc_debug_bench(static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), ntile, iters, us,
                 reinterpret_cast<unsigned long long*>(trace), grid);
  API_END
}


int tgnn_run_oplog(tgnn_run* r, int64_t* count, int64_t* rows) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(r->oplog, kConfig, "run: op-log recording was not enabled (tgnn_run_options.oplog)");
  std::vector<int64_t> log(static_cast<size_t>(4 * std::max<int64_t>(r->sched.barriers, 1)));
  TGB_CUDA(cudaStreamSynchronize(r->ctx->stream));
  TGB_CUDA(cudaMemcpy(log.data(), r->d_oplog, sizeof(int64_t) * log.size(), cudaMemcpyDeviceToHost));
  const int local = r->rank % (r->tc.i * r->tc.j);
  int64_t n = 0;
  for (int64_t b = 0; b < r->next_barrier; ++b) {
    const host::Task t = r->sched.task(r->rank, b);
    if (!t.active || t.sub != 0) continue;
    if (rows) {
      const int64_t* l = log.data() + 4 * b;
      const int64_t rr[2][6] = {{t.sweep, t.pair, 0, local, l[0], l[1]}, {t.sweep, t.pair, 1, local, l[2], l[3]}};
      std::memcpy(rows + 6 * n, rr, sizeof(rr));
    }
    n += 2;
  }
  *count = n;
  API_END
}


int tgnn_run_loss_async(tgnn_run* r, int64_t b, double* dst) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(b >= 0 && b < r->next_barrier, kConfig, "run: loss of a barrier not yet enqueued");
  // on the read-back stream once the barrier's loss is written: the compute
  // stream never waits for the copy (tgnn_ctx_synchronize joins it)
  TGB_CUDA(cudaEventRecord(r->ctx->ev_d2h, r->ctx->stream));
  TGB_CUDA(cudaStreamWaitEvent(r->ctx->d2h, r->ctx->ev_d2h, 0));
  TGB_CUDA(cudaMemcpyAsync(dst, r->d_losses + b, sizeof(double), cudaMemcpyDeviceToHost, r->ctx->d2h));
  API_END
}


int tgnn_run_snapshots(tgnn_run* r, int64_t* count, int64_t* meta, double* memory, double* last_update) {
  API_BEGIN
  r->ctx->use();
  *count = r->snap_taken;
  if (!meta && !memory && !last_update) return 0;
  TGB_CUDA(cudaStreamSynchronize(r->ctx->stream));
  const int64_t N = r->mem->d.N, d = r->mem->d.d;
  std::vector<float> mf(static_cast<size_t>(N * d));
  for (int64_t x = 0; x < r->snap_taken; ++x) {
    if (meta) {
      meta[2 * x] = r->snap_meta[static_cast<size_t>(x)][0];
      meta[2 * x + 1] = r->snap_meta[static_cast<size_t>(x)][1];
    }
    if (memory) {
      TGB_CUDA(cudaMemcpy(mf.data(), r->d_snap_mem + x * N * d, sizeof(float) * mf.size(), cudaMemcpyDeviceToHost));
      for (int64_t q = 0; q < N * d; ++q) memory[x * N * d + q] = mf[static_cast<size_t>(q)];
    }
    if (last_update)
      TGB_CUDA(cudaMemcpy(last_update + x * N, r->d_snap_lu + x * N, sizeof(double) * N, cudaMemcpyDeviceToHost));
  }
  API_END
}

int tgnn_run_check_replicas(tgnn_run* r, uint64_t* hash_out) {
  API_BEGIN
  r->ctx->use();
  TGB_REQUIRE(r->nranks == 1 || r->comm_ready, kProtocol, "run: communicator not initialised");
  HubGuard guard(r);
  *hash_out = check_replicas(r);
  guard.ok();
  API_END
}

}  // extern "C"
