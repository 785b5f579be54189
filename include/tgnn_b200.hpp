// tgnn_b200.hpp -- the reference-side drop-in: the reference's own C++
// interfaces (namespace tgnn, /root/reference/proj/include/tgnn) served by the
// B200 training step behind the C ABI of tgnn_b200.h.
//
// A maintainer adds this header next to proj/include/tgnn/ and redirects the
// call sites they choose; nothing in the reference changes. Include it after
// (or instead of) tgnn/trainer.hpp and link libtgnn_b200.so:
//
//   g++ -std=c++20 -I<ref>/proj/include -I<repo>/include app.cpp
//       -L<repo>/paper_2307_07649_b200 -ltgnn_b200 -Wl,-rpath,<repo>/paper_2307_07649_b200
//
// Two levels:
//  * parity level -- sample_recent_neighbors, sample_negatives, plan_sub_batch,
//    DeviceMemoryClient (a MemoryClient), evaluate_mrr, replay_batch: the
//    reference signatures on a device graph, f64 <-> fp32 at the boundary;
//  * performance level -- run_training / run_sequential taking the reference's
//    RunOptions and returning its RunResult (barrier losses, metrics rows and
//    the metrics_out CSV, per-memory-copy op-logs into oplog_out, on_eval with
//    the weights of every eval point, segment snapshots). Like the reference,
//    the i*j*k trainers are threads of this process (trainer.hpp:748-760); the
//    ranks exchange through the in-process hub (tgnn_run_local_init), spread
//    round-robin over DeviceOptions::devices. One process per GPU over NCCL is
//    the tgnn_run_comm_init path of the C ABI (bench.py, tests/mp_worker.py).
// Errors come back as the reference's exception types (common.hpp:16-34).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <exception>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "tgnn/memory_daemon.hpp"
#include "tgnn/oplog.hpp"
#include "tgnn/trainer.hpp"
#include "tgnn_b200.h"

namespace tgnn::b200 {

// Status code -> the reference's exception taxonomy.
inline void check(int rc) {
  if (rc == 0) return;
  const std::string m = tgnn_last_error();
  switch (rc) {
    case TGNN_CONFIG_ERROR: throw config_error(m);
    case TGNN_PARSE_ERROR: throw parse_error(m);
    case TGNN_NUMERIC_ERROR: throw numeric_error(m);
    case TGNN_PROTOCOL_ERROR: throw protocol_error(m);
    case TGNN_SHAPE_ERROR: throw shape_error(m);
    default: throw std::runtime_error(m);
  }
}

inline tgnn_model_config to_c(const ModelConfig& m) {
  tgnn_model_config c{};
  c.d_mem = static_cast<int64_t>(m.d_mem);
  c.d_time = static_cast<int64_t>(m.d_time);
  c.d_static = static_cast<int64_t>(m.d_static);
  c.d_attn = static_cast<int64_t>(m.d_attn);
  c.d_hidden = static_cast<int64_t>(m.d_hidden);
  c.d_e = static_cast<int64_t>(m.d_e);
  c.n_neighbors = static_cast<int64_t>(m.n_neighbors);
  c.num_nodes = m.num_nodes;
  c.max_t = m.max_t;
  return c;
}

inline tgnn_train_config to_c(const TrainConfig& t) {
  tgnn_train_config c{};
  c.i = t.i;
  c.j = t.j;
  c.k = t.k;
  c.p = t.p;
  c.q = t.q;
  c.epochs = t.epochs;
  c.local_batch = t.local_batch;
  c.lr_base = t.lr_base;
  c.seed = t.seed;
  c.local_batch_ref = t.local_batch_ref;
  c.neg_groups = t.neg_groups;
  return c;
}

// Flat f64 weights in for_each_tensor order (model.hpp:56-76) <-> ModelParams.
inline std::vector<double> flatten(const ModelParams& p) {
  std::vector<double> flat;
  for_each_tensor(const_cast<ModelParams&>(p), [&](const char*, Tensor& t) {
    flat.insert(flat.end(), t.data(), t.data() + t.numel());
  });
  return flat;
}

inline ModelParams unflatten(const ModelConfig& cfg, std::span<const double> flat) {
  ModelParams p;
  shape_params(cfg, p);
  std::size_t at = 0;
  for_each_tensor(p, [&](const char*, Tensor& t) {
    if (at + t.numel() > flat.size()) throw shape_error("b200: flat parameter vector too short");
    std::copy(flat.begin() + static_cast<std::ptrdiff_t>(at),
              flat.begin() + static_cast<std::ptrdiff_t>(at + t.numel()), t.data());
    at += t.numel();
  });
  if (at != flat.size()) throw shape_error("b200: flat parameter vector too long");
  return p;
}

// One device context (its CUDA streams); use it from one host thread.
class Context {
 public:
  explicit Context(int device = 0) { check(tgnn_ctx_create(device, &h_)); }
  ~Context() {
    if (h_) tgnn_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tgnn_ctx* get() const { return h_; }

 private:
  tgnn_ctx* h_ = nullptr;
};

// Device copy of a finalized TemporalGraph (temporal_graph.hpp:33-95): the
// T-CSR is rebuilt on device, features are stored as fp32.
class Graph {
 public:
  Graph(Context& ctx, const TemporalGraph& tg) {
    const std::size_t E = tg.events.size();
    std::vector<int64_t> s(E), d(E);
    std::vector<double> t(E);
    for (std::size_t e = 0; e < E; ++e) {
      s[e] = tg.events[e].src;
      d[e] = tg.events[e].dst;
      t[e] = tg.events[e].t;
    }
    check(tgnn_graph_create_f64(ctx.get(), tg.num_nodes, tg.bipartite_boundary, static_cast<int64_t>(E), s.data(),
                                d.data(), t.data(), tg.d_e ? tg.edge_feats.data() : nullptr,
                                static_cast<int64_t>(tg.d_e), &h_));
  }
  ~Graph() {
    if (h_) tgnn_graph_destroy(h_);
  }
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;
  tgnn_graph* get() const { return h_; }

 private:
  tgnn_graph* h_ = nullptr;
};

// ---------------------------------------------------------------- parity level
// sample_recent_neighbors (temporal_graph.hpp:296-318).
inline std::vector<NeighborRef> sample_recent_neighbors(Graph& g, NodeId v, TimeT t, std::size_t n) {
  const int64_t nn = static_cast<int64_t>(std::max<std::size_t>(n, 1));
  std::vector<int64_t> node{std::vector<int64_t>(static_cast<std::size_t>(nn))};
  std::vector<int64_t> ev{std::vector<int64_t>(static_cast<std::size_t>(nn))};
  std::vector<double> dt{std::vector<double>(static_cast<std::size_t>(nn))};
  int64_t cnt = 0;
  const int64_t q = v;
  const double qt = t;
  check(tgnn_sample_recent_neighbors(g.get(), &q, &qt, 1, static_cast<int64_t>(n), node.data(), ev.data(), dt.data(),
                                     &cnt));
  std::vector<NeighborRef> out{std::vector<NeighborRef>(static_cast<std::size_t>(cnt))};
  for (std::size_t m = 0; m < out.size(); ++m) out[m] = NeighborRef{node[m], ev[m], dt[m]};
  return out;
}

// sample_negatives (temporal_graph.hpp:355-370).
inline std::vector<NodeId> sample_negatives(Graph& g, EventId batch_index, std::int64_t group, EventId count,
                                            std::uint64_t seed) {
  std::vector<int64_t> out{std::vector<int64_t>(static_cast<std::size_t>(std::max<EventId>(count, 0)))};
  check(tgnn_sample_negatives(g.get(), batch_index, group, count, seed, out.data()));
  return std::vector<NodeId>(out.begin(), out.end());
}

// plan_sub_batch (trainer.hpp:76-106).
inline SubBatchPlan plan_sub_batch(Graph& g, EventId begin, EventId end, std::span<const NodeId> negatives,
                                   std::size_t n) {
  if (begin < 0 || begin > end) throw config_error("plan_sub_batch: event range out of bounds");
  if (negatives.size() != static_cast<std::size_t>(end - begin))
    throw config_error("plan_sub_batch: one negative per event required");
  const std::size_t R = 3 * static_cast<std::size_t>(end - begin), nn = std::max<std::size_t>(n, 1);
  std::vector<int64_t> negs(negatives.begin(), negatives.end());
  std::vector<int64_t> rn{std::vector<int64_t>(R)}, cnt{std::vector<int64_t>(R)};
  std::vector<double> rt{std::vector<double>(R)};
  std::vector<int64_t> nb{std::vector<int64_t>(R * nn)}, ne{std::vector<int64_t>(R * nn)};
  std::vector<double> nd{std::vector<double>(R * nn)};
  std::vector<int64_t> sup{std::vector<int64_t>(R * (n + 1) + 1)};
  int64_t U = 0;
  check(tgnn_plan_sub_batch(g.get(), begin, end, negs.data(), static_cast<int64_t>(n), rn.data(), rt.data(), cnt.data(),
                            nb.data(), ne.data(), nd.data(), sup.data(), &U));
  SubBatchPlan plan;
  plan.begin = begin;
  plan.end = end;
  plan.roots.resize(R);
  for (std::size_t x = 0; x < R; ++x) {
    RootEmbed& re = plan.roots[x];
    re.node = rn[x];
    re.t = rt[x];
    for (int64_t m = 0; m < cnt[x]; ++m) {
      const std::size_t at = x * n + static_cast<std::size_t>(m);
      re.nbrs.push_back(NeighborRef{nb[at], ne[at], nd[at]});
    }
  }
  plan.supports.assign(sup.begin(), sup.begin() + U);
  return plan;
}

// A MemoryClient (shared_buffers.hpp:124-130) over a node-memory state that
// lives in HBM (NodeMemoryState, memory_store.hpp:16-50).
class DeviceMemoryClient final : public MemoryClient {
 public:
  DeviceMemoryClient(Context& ctx, NodeId num_nodes, std::size_t d_mem) : d_mem_(d_mem) {
    check(tgnn_memstore_create(ctx.get(), num_nodes, static_cast<int64_t>(d_mem), &h_));
  }
  ~DeviceMemoryClient() override {
    if (h_) tgnn_memstore_destroy(h_);
  }
  DeviceMemoryClient(const DeviceMemoryClient&) = delete;
  DeviceMemoryClient& operator=(const DeviceMemoryClient&) = delete;

  std::vector<ReadView> read(const std::vector<std::vector<NodeId>>& subs) override {
    std::vector<ReadView> out;
    for (const auto& nodes : subs) {
      ReadView v;
      v.nodes = nodes;
      v.mem = Tensor({nodes.size(), d_mem_});
      v.mail = Tensor({nodes.size(), 2 * d_mem_ + 3});
      std::vector<int64_t> ids(nodes.begin(), nodes.end());
      if (!ids.empty())
        check(tgnn_memstore_read(h_, ids.data(), static_cast<int64_t>(ids.size()), v.mem.data(), v.mail.data()));
      out.push_back(std::move(v));
    }
    return out;
  }
  void write(const std::vector<NodeId>& nodes, const Tensor& mem_rows, const Tensor& mail_rows) override {
    std::vector<int64_t> ids(nodes.begin(), nodes.end());
    if (!ids.empty())
      check(tgnn_memstore_write(h_, ids.data(), static_cast<int64_t>(ids.size()), mem_rows.data(), mail_rows.data()));
  }
  void reset() { check(tgnn_memstore_reset(h_)); }  // reset_state (memory_store.hpp:43-50)
  void export_state(NodeMemoryState& s) const {
    std::vector<int64_t> ev{std::vector<int64_t>(static_cast<std::size_t>(s.num_nodes))};
    check(tgnn_memstore_export(h_, s.memory.data(), s.last_update.data(), s.mail_mem.data(), s.mail_t.data(),
                               s.mail_dt.data(), ev.data()));
    std::copy(ev.begin(), ev.end(), s.mail_event.begin());
  }
  tgnn_memstore* get() const { return h_; }

 private:
  tgnn_memstore* h_ = nullptr;
  std::size_t d_mem_ = 0;
};

// evaluate_mrr (trainer.hpp:383-468) on device.
inline EvalResult evaluate_mrr(Context& ctx, Graph& g, const ModelParams& p, EventId eval_begin, EventId eval_end,
                               EventId batch_size, int n_negatives, std::uint64_t seed) {
  tgnn_evaluator* ev = nullptr;
  const tgnn_model_config mc = to_c(p.cfg);
  check(tgnn_evaluator_create(ctx.get(), g.get(), &mc, batch_size, n_negatives, &ev));
  const std::vector<double> flat = flatten(p);
  EvalResult r;
  const int rc = tgnn_evaluate_mrr(ev, flat.data(), eval_begin, eval_end, seed, &r.mrr, &r.queries);
  tgnn_evaluator_destroy(ev);
  check(rc);
  return r;
}

// replay_batch (trainer.hpp:336-371) into a device memory state.
inline void replay_batch(Context& ctx, Graph& g, const ModelParams& p, DeviceMemoryClient& state, EventId begin,
                         EventId end) {
  if (begin >= end) return;
  tgnn_evaluator* ev = nullptr;
  const tgnn_model_config mc = to_c(p.cfg);
  check(tgnn_evaluator_create(ctx.get(), g.get(), &mc, end - begin, 0, &ev));
  const std::vector<double> flat = flatten(p);
  const int rc = tgnn_replay_batch(ev, state.get(), flat.data(), begin, end);
  tgnn_evaluator_destroy(ev);
  check(rc);
}

// ---------------------------------------------------------------- performance level
struct DeviceOptions {
  std::vector<int> devices{0};  // ranks are placed round-robin over these
  bool use_graphs = true;       // CUDA-graph barriers (single-rank runs)
};

namespace detail {

// Rank r of a run in its own thread. Rank 0 produces the metrics rows, the
// on_eval calls and the final weights, as the reference's evaluating trainer.
struct Job {
  Job(const TemporalGraph& graph, const RunOptions& o, const TrainConfig& c, const ModelConfig& m)
      : g(graph), opt(o), cfg(c), mcfg(m) {}
  const TemporalGraph& g;
  const RunOptions& opt;
  TrainConfig cfg;
  ModelConfig mcfg;
  int T = 1, K = 1;
  std::vector<int> devices;
  bool use_graphs = true;
  tgnn_local_hub* hub = nullptr;
  std::vector<tgnn_graph*> graphs;  // one device graph per entry of devices
  RunResult res;
  std::mutex mu;
  std::vector<std::vector<std::array<int64_t, 6>>> oplog;  // per memory copy
  std::exception_ptr first;
  bool first_is_root = false;

  void fail(std::exception_ptr e, bool root_cause) {
    std::lock_guard<std::mutex> lk(mu);
    if (!first || (root_cause && !first_is_root)) {
      first = e;
      first_is_root = root_cause;
    }
  }
};

inline bool is_secondary(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const std::exception& x) {
    return std::string(x.what()).find("another rank failed") != std::string::npos;
  } catch (...) {
  }
  return false;
}

inline void rank_body(Job& J, int rank, tgnn_ctx* ctx, tgnn_graph* graph) {
  const RunOptions& opt = J.opt;
  tgnn_run_options o{};
  o.model = to_c(J.mcfg);
  o.train = to_c(J.cfg);
  o.train_begin = opt.train_begin;
  o.train_end = opt.train_end;
  o.rank = rank;
  o.nranks = J.T;
  o.use_graphs = J.use_graphs ? 1 : 0;
  o.val_begin = opt.val_begin;
  o.val_end = opt.val_end;
  o.eval_negatives = opt.eval_negatives;
  o.eval_batch = opt.eval_batch;
  o.oplog = opt.oplog_out.empty() ? 0 : 1;
  o.segment_snapshots = opt.segment_snapshots ? 1 : 0;
  tgnn_run* r = nullptr;
  check(tgnn_run_create(ctx, graph, &o, &r));
  struct Guard {
    tgnn_run* r;
    ~Guard() { tgnn_run_destroy(r); }
  } guard{r};
  if (J.T > 1) check(tgnn_run_local_init(r, J.hub));
  int64_t barriers = 0, nparam = 0;
  check(tgnn_run_info(r, &barriers, &nparam));
  int64_t ne = 0;
  check(tgnn_run_eval_barriers(r, &ne, nullptr));
  std::vector<int64_t> evb{std::vector<int64_t>(static_cast<std::size_t>(ne))};
  if (ne) check(tgnn_run_eval_barriers(r, &ne, evb.data()));
  int64_t next = 0;
  std::vector<double> rows;
  std::vector<double> flat{std::vector<double>(static_cast<std::size_t>(nparam))};
  for (int64_t e : evb) {
    check(tgnn_run_barriers(r, next, e + 1 - next));
    next = e + 1;
    int64_t nrow = 0;
    check(tgnn_run_metrics(r, &nrow, nullptr));
    rows.assign(static_cast<std::size_t>(5 * nrow), 0.0);
    check(tgnn_run_metrics(r, &nrow, rows.data()));  // collective: every rank
    if (rank != 0 || nrow == 0) continue;
    const double* q = rows.data() + 5 * (nrow - 1);
    MetricsRow row;
    row.iter = static_cast<std::int64_t>(q[0]);
    row.traversed = static_cast<std::int64_t>(q[1]);
    row.loss = q[2];
    row.val_mrr = q[3];
    row.elapsed_s = q[4];
    J.res.metrics.push_back(row);
    tgnn::detail::write_metrics_row(opt.metrics_out, row);
    if (opt.on_eval) {
      check(tgnn_run_params(r, flat.data()));
      opt.on_eval(row, unflatten(J.mcfg, flat));
    }
  }
  std::vector<double> loss{std::vector<double>(static_cast<std::size_t>(barriers))};
  if (barriers) check(tgnn_run_losses(r, 0, barriers, loss.data()));  // collective
  uint64_t fp = 0;
  if (J.T > 1) check(tgnn_run_check_replicas(r, &fp));  // the replica invariant
  const int per_group = J.cfg.i * J.cfg.j;
  const int group = rank / per_group;
  if (!opt.oplog_out.empty()) {
    int64_t n = 0;
    check(tgnn_run_oplog(r, &n, nullptr));
    std::vector<int64_t> rr{std::vector<int64_t>(static_cast<std::size_t>(6 * n))};
    if (n) check(tgnn_run_oplog(r, &n, rr.data()));
    std::lock_guard<std::mutex> lk(J.mu);
    for (int64_t x = 0; x < n; ++x)
      J.oplog[static_cast<std::size_t>(group)].push_back(
          {rr[6 * x], rr[6 * x + 1], rr[6 * x + 2], rr[6 * x + 3], rr[6 * x + 4], rr[6 * x + 5]});
  }
  if (opt.segment_snapshots && rank % per_group == 0) {  // one replica per memory copy
    int64_t n = 0;
    check(tgnn_run_snapshots(r, &n, nullptr, nullptr, nullptr));
    const std::size_t N = static_cast<std::size_t>(J.g.num_nodes), d = J.mcfg.d_mem;
    std::vector<int64_t> meta{std::vector<int64_t>(static_cast<std::size_t>(2 * n))};
    std::vector<double> mem{std::vector<double>(static_cast<std::size_t>(n) * N * d)};
    std::vector<double> lu{std::vector<double>(static_cast<std::size_t>(n) * N)};
    if (n) check(tgnn_run_snapshots(r, &n, meta.data(), mem.data(), lu.data()));
    std::vector<MemorySnapshot> snaps;
    for (int64_t x = 0; x < n; ++x) {
      MemorySnapshot s;
      s.sweep = static_cast<int>(meta[2 * x]);
      s.segment = static_cast<int>(meta[2 * x + 1]);
      s.memory = Tensor({N, d});
      std::copy(mem.begin() + static_cast<std::ptrdiff_t>(x * N * d),
                mem.begin() + static_cast<std::ptrdiff_t>((x + 1) * N * d), s.memory.data());
      s.last_update.assign(lu.begin() + static_cast<std::ptrdiff_t>(x * N),
                           lu.begin() + static_cast<std::ptrdiff_t>((x + 1) * N));
      snaps.push_back(std::move(s));
    }
    std::lock_guard<std::mutex> lk(J.mu);
    J.res.snapshots[static_cast<std::size_t>(group)] = std::move(snaps);
  }
  if (rank == 0) {
    check(tgnn_run_params(r, flat.data()));
    J.res.params = unflatten(J.mcfg, flat);
    J.res.barrier_loss = std::move(loss);
    J.res.barriers = barriers;
  }
}

}  // namespace detail

// run_training (trainer.hpp:630-772): the threaded i x j x k run.
inline RunResult run_training(const TemporalGraph& g, const RunOptions& opt, const DeviceOptions& dev = {}) {
  TrainConfig cfg = opt.train;
  cfg.validate();
  const ModelConfig mcfg = tgnn::detail::resolve_model(g, opt.model);
  if (dev.devices.empty()) throw config_error("b200: no device given");
  detail::Job J(g, opt, cfg, mcfg);
  J.T = cfg.num_trainers();
  J.K = cfg.k;
  J.devices = dev.devices;
  J.use_graphs = dev.use_graphs;
  if (!opt.oplog_out.empty() && opt.oplog_out.size() != static_cast<std::size_t>(J.K))
    throw config_error("run_training: need one op-log sink per memory copy");
  J.res.snapshots.resize(static_cast<std::size_t>(J.K));
  J.oplog.resize(static_cast<std::size_t>(J.K));
  tgnn::detail::write_metrics_header(opt.metrics_out);
  const auto t0 = std::chrono::steady_clock::now();
  // one context + device graph per device, shared read-only by its ranks
  const std::size_t nd = std::min<std::size_t>(dev.devices.size(), static_cast<std::size_t>(J.T));
  std::vector<std::unique_ptr<Context>> gctx;
  std::vector<std::unique_ptr<Graph>> graphs;
  for (std::size_t x = 0; x < nd; ++x) {
    gctx.push_back(std::make_unique<Context>(dev.devices[x]));
    graphs.push_back(std::make_unique<Graph>(*gctx.back(), g));
  }
  if (J.T > 1) check(tgnn_local_hub_create(J.T, &J.hub));
  auto body = [&](int rank) {
    try {
      const std::size_t slot = static_cast<std::size_t>(rank) % nd;
      Context ctx(dev.devices[slot]);
      detail::rank_body(J, rank, ctx.get(), graphs[slot]->get());
    } catch (...) {
      const std::exception_ptr e = std::current_exception();
      J.fail(e, !detail::is_secondary(e));
    }
  };
  if (J.T == 1) {
    body(0);
  } else {
    std::vector<std::thread> th;
    for (int rank = 0; rank < J.T; ++rank) th.emplace_back(body, rank);
    for (auto& t : th) t.join();
  }
  if (J.hub) tgnn_local_hub_destroy(J.hub);
  graphs.clear();
  gctx.clear();
  if (J.first) std::rethrow_exception(J.first);
  // each memory copy's op-log: its ranks' records ordered by (iter, kind, rank)
  for (std::size_t grp = 0; grp < J.oplog.size() && !opt.oplog_out.empty(); ++grp) {
    auto& recs = J.oplog[grp];
    std::stable_sort(recs.begin(), recs.end(), [](const auto& a, const auto& b) {
      return std::tie(a[1], a[2], a[3]) < std::tie(b[1], b[2], b[3]);
    });
    if (!opt.oplog_out[grp]) continue;
    OpLogWriter w(*opt.oplog_out[grp]);
    for (const auto& q : recs)
      w.append(OpRecord{q[0], q[1], q[2] ? 'W' : 'R', static_cast<int>(q[3]), q[4], q[5]});
    w.flush();
  }
  J.res.elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return std::move(J.res);
}

// run_sequential (trainer.hpp:777-867): the single-trainer run.
inline RunResult run_sequential(const TemporalGraph& g, const RunOptions& opt, const DeviceOptions& dev = {}) {
  if (opt.train.num_trainers() != 1) throw config_error("run_sequential: requires i = j = k = 1");
  return run_training(g, opt, dev);
}

}  // namespace tgnn::b200
