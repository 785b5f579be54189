// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the UNMODIFIED reference headers
// (/root/reference/proj/include/tgnn/*.hpp, included by path at build time,
// never copied). It is compiled by oracle/Makefile into oracle/_ref/libtgnn_ref.so
// and is loaded only by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg. Nothing in the product links it.
//
// Every entry point calls the reference's own function of the same name:
//   gen_synthetic            synthetic.hpp:54-112
//   TemporalGraph::finalize  temporal_graph.hpp:55-91
//   sample_recent_neighbors  temporal_graph.hpp:296-318
//   sample_negatives         temporal_graph.hpp:355-370
//   plan_sub_batch           trainer.hpp:76-106
//   init_params              model.hpp:122-141
//   sub_step                 trainer.hpp:170-272
//   build_root_writes        trainer.hpp:284-330
//   replay_batch             trainer.hpp:336-371
//   evaluate_mrr             trainer.hpp:383-468
//   Adam::step               optimizer.hpp:40-56
//   build_assignment         parallel.hpp:218-331
//   run_sequential/run_training trainer.hpp:630-867
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <cstdio>
#include <string>
#include <vector>

#include "tgnn/synthetic.hpp"
#include "tgnn/trainer.hpp"

using namespace tgnn;

namespace {

thread_local std::string g_err;

int fail_with(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_GUARD(...)                                            \
  try {                                                           \
    __VA_ARGS__                                                   \
  } catch (const parse_error& e) {                                \
    return fail_with(e, 2);                                       \
  } catch (const config_error& e) {                               \
    return fail_with(e, 1);                                       \
  } catch (const numeric_error& e) {                              \
    return fail_with(e, 3);                                       \
  } catch (const protocol_error& e) {                             \
    return fail_with(e, 4);                                       \
  } catch (const shape_error& e) {                                \
    return fail_with(e, 5);                                       \
  } catch (const std::exception& e) {                             \
    return fail_with(e, 9);                                       \
  }                                                               \
  return 0;

}  // namespace

extern "C" {

// Mirrors ModelConfig (model.hpp:19-35) with fixed-width fields.
struct ref_model_cfg {
  int64_t d_mem, d_time, d_static, d_attn, d_hidden, d_e, n_neighbors, num_nodes;
  double max_t;
};

// Mirrors TrainConfig (parallel.hpp:15-26).
struct ref_train_cfg {
  int32_t i, j, k, p, q;
  int32_t epochs;
  int64_t local_batch;
  double lr_base;
  uint64_t seed;
  int64_t local_batch_ref;
  int64_t neg_groups;
};

const char* ref_last_error(void) { return g_err.c_str(); }

static ModelConfig to_mcfg(const ref_model_cfg* c) {
  ModelConfig m;
  m.d_mem = static_cast<std::size_t>(c->d_mem);
  m.d_time = static_cast<std::size_t>(c->d_time);
  m.d_static = static_cast<std::size_t>(c->d_static);
  m.d_attn = static_cast<std::size_t>(c->d_attn);
  m.d_hidden = static_cast<std::size_t>(c->d_hidden);
  m.d_e = static_cast<std::size_t>(c->d_e);
  m.n_neighbors = static_cast<std::size_t>(c->n_neighbors);
  m.num_nodes = c->num_nodes;
  m.max_t = c->max_t;
  return m;
}

static TrainConfig to_tcfg(const ref_train_cfg* c) {
  TrainConfig t;
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

static void params_from_flat(ModelParams& p, const double* flat) {
  std::size_t at = 0;
  for_each_tensor(p, [&](const char*, Tensor& t) {
    std::memcpy(t.data(), flat + at, t.numel() * sizeof(double));
    at += t.numel();
  });
}

static void params_to_flat(const ModelParams& p, double* flat) {
  std::size_t at = 0;
  for_each_tensor(const_cast<ModelParams&>(p), [&](const char*, Tensor& t) {
    std::memcpy(flat + at, t.data(), t.numel() * sizeof(double));
    at += t.numel();
  });
}

// ---------------------------------------------------------------- graph
int ref_graph_synthetic(int64_t nodes, int64_t events, double burst_prob, double pref_prob,
                        int32_t prefs_per_src, double src_frac, int32_t bipartite, int64_t d_e,
                        double zipf_s, uint64_t seed, void** out) {
  REF_GUARD({
    SynthParams p;
    p.nodes = nodes;
    p.events = events;
    p.burst_prob = burst_prob;
    p.pref_prob = pref_prob;
    p.prefs_per_src = prefs_per_src;
    p.src_frac = src_frac;
    p.bipartite = bipartite != 0;
    p.d_e = static_cast<std::size_t>(d_e);
    p.zipf_s = zipf_s;
    p.seed = seed;
    *out = new TemporalGraph(gen_synthetic(p));
  })
}

// load_dataset / write_dataset (temporal_graph.hpp:136-262), unmodified.
int ref_load_dataset(const char* csv_path, void** out) {
  REF_GUARD({ *out = new TemporalGraph(load_dataset(csv_path)); })
}

int ref_write_dataset(void* gp, const char* csv_path) {
  REF_GUARD({ write_dataset(*static_cast<TemporalGraph*>(gp), csv_path); })
}

int ref_chronological_split(void* gp, double train_frac, double val_frac, int64_t* train_end,
                            int64_t* val_end) {
  REF_GUARD({
    SplitRanges r = chronological_split(*static_cast<TemporalGraph*>(gp), train_frac, val_frac);
    *train_end = r.train_end;
    *val_end = r.val_end;
  })
}

int ref_graph_from_events(int64_t num_nodes, int64_t boundary, int64_t num_events,
                          const int64_t* src, const int64_t* dst, const double* t,
                          const double* efeat, int64_t d_e, void** out) {
  REF_GUARD({
    auto* g = new TemporalGraph();
    g->num_nodes = num_nodes;
    g->bipartite_boundary = boundary;
    g->d_e = static_cast<std::size_t>(d_e);
    g->events.resize(static_cast<std::size_t>(num_events));
    for (int64_t e = 0; e < num_events; ++e) g->events[e] = {src[e], dst[e], t[e]};
    g->edge_feats = Tensor({static_cast<std::size_t>(num_events), static_cast<std::size_t>(d_e)});
    if (d_e > 0) std::memcpy(g->edge_feats.data(), efeat, sizeof(double) * num_events * d_e);
    try {
      g->finalize();
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  })
}

void ref_graph_free(void* g) { delete static_cast<TemporalGraph*>(g); }

void ref_graph_info(void* gp, int64_t* num_nodes, int64_t* boundary, int64_t* num_events,
                    int64_t* d_e) {
  auto* g = static_cast<TemporalGraph*>(gp);
  *num_nodes = g->num_nodes;
  *boundary = g->bipartite_boundary;
  *num_events = g->num_events();
  *d_e = static_cast<int64_t>(g->d_e);
}

// Finalized (time-sorted) events; efeat may be null.
void ref_graph_export(void* gp, int64_t* src, int64_t* dst, double* t, double* efeat) {
  auto* g = static_cast<TemporalGraph*>(gp);
  for (int64_t e = 0; e < g->num_events(); ++e) {
    src[e] = g->events[e].src;
    dst[e] = g->events[e].dst;
    t[e] = g->events[e].t;
  }
  if (efeat && g->d_e > 0)
    std::memcpy(efeat, g->edge_feats.data(), sizeof(double) * g->edge_feats.numel());
}

// Export feature rows [begin, end) only (large graphs).
void ref_graph_export_feats(void* gp, int64_t begin, int64_t end, double* efeat) {
  auto* g = static_cast<TemporalGraph*>(gp);
  if (g->d_e == 0) return;
  std::memcpy(efeat, g->edge_feats.data() + begin * g->d_e,
              sizeof(double) * (end - begin) * g->d_e);
}

// ---------------------------------------------------------------- sampler
int64_t ref_sample_recent_neighbors(void* gp, int64_t v, double t, int64_t n, int64_t* node,
                                    int64_t* event, double* dt) {
  auto nb = sample_recent_neighbors(*static_cast<TemporalGraph*>(gp), v, t,
                                    static_cast<std::size_t>(n));
  for (std::size_t m = 0; m < nb.size(); ++m) {
    node[m] = nb[m].node;
    event[m] = nb[m].event;
    dt[m] = nb[m].dt;
  }
  return static_cast<int64_t>(nb.size());
}

int ref_sample_negatives(void* gp, int64_t batch_index, int64_t group, int64_t count,
                         uint64_t seed, int64_t* out) {
  REF_GUARD({
    auto v = sample_negatives(*static_cast<TemporalGraph*>(gp), batch_index, group, count, seed);
    std::memcpy(out, v.data(), sizeof(int64_t) * v.size());
  })
}

// The distractors evaluate_mrr draws (its loop at trainer.hpp:413-423, over
// the reference's own hash64 / Rng / bipartite boundary): evaluate_mrr does
// not expose its candidate lists, so this driver walks the same stream.
int ref_eval_candidates(void* gp, int64_t begin, int64_t end, int32_t n_neg, uint64_t seed,
                        int64_t* out) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    const NodeId lo = g->bipartite() ? g->bipartite_boundary : 0;
    const NodeId span = g->num_nodes - lo;
    for (EventId e = begin; e < end; ++e) {
      const Event& ev = g->events[static_cast<std::size_t>(e)];
      for (int s = 0; s < n_neg; ++s) {
        Rng r(hash64(seed, 0x6576616cull, static_cast<std::uint64_t>(e), static_cast<std::uint64_t>(s)));
        NodeId v;
        do {
          v = lo + r.next_below(span);
        } while (v == ev.dst);
        *out++ = v;
      }
    }
  })
}

// Roots are event-major (src, dst, neg); neighbour arrays are [R x n] padded.
// supports must hold R*(n+1) entries; *num_supports receives U.
int ref_plan_sub_batch(void* gp, int64_t begin, int64_t end, const int64_t* negatives, int64_t n,
                       int64_t* root_node, double* root_t, int64_t* nbr_count, int64_t* nbr_node,
                       int64_t* nbr_event, double* nbr_dt, int64_t* supports,
                       int64_t* num_supports) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    std::span<const NodeId> negs(negatives, static_cast<std::size_t>(end - begin));
    SubBatchPlan plan = plan_sub_batch(*g, begin, end, negs, static_cast<std::size_t>(n));
    for (std::size_t r = 0; r < plan.roots.size(); ++r) {
      const RootEmbed& re = plan.roots[r];
      root_node[r] = re.node;
      root_t[r] = re.t;
      nbr_count[r] = static_cast<int64_t>(re.nbrs.size());
      for (std::size_t m = 0; m < re.nbrs.size(); ++m) {
        nbr_node[r * n + m] = re.nbrs[m].node;
        nbr_event[r * n + m] = re.nbrs[m].event;
        nbr_dt[r * n + m] = re.nbrs[m].dt;
      }
    }
    std::memcpy(supports, plan.supports.data(), sizeof(int64_t) * plan.supports.size());
    *num_supports = static_cast<int64_t>(plan.supports.size());
  })
}

// ---------------------------------------------------------------- model
int64_t ref_param_count(const ref_model_cfg* c) {
  ModelParams p;
  shape_params(to_mcfg(c), p);
  return static_cast<int64_t>(param_count(p));
}

int ref_init_params(const ref_model_cfg* c, uint64_t seed, double* flat) {
  REF_GUARD({ params_to_flat(init_params(to_mcfg(c), seed), flat); })
}

// One sub_step on an injected read view. view_mem [U x d_mem],
// view_mail [U x (2 d_mem + 3)] aligned with the plan's supports (the caller
// obtains U from ref_plan_sub_batch). grads_out [nparam] receives the
// (zero-initialised) accumulated gradients; s_hat_out [U x d_mem].
int ref_sub_step(void* gp, const ref_model_cfg* c, const double* params_flat, int64_t begin,
                 int64_t end, const int64_t* negatives, const double* view_mem,
                 const double* view_mail, double* loss_out, double* grads_out,
                 double* s_hat_out) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    ModelConfig mc = to_mcfg(c);
    ModelParams p;
    shape_params(mc, p);
    params_from_flat(p, params_flat);
    std::span<const NodeId> negs(negatives, static_cast<std::size_t>(end - begin));
    SubBatchPlan plan = plan_sub_batch(*g, begin, end, negs, mc.n_neighbors);
    ReadView view;
    view.nodes = plan.supports;
    const std::size_t U = plan.supports.size(), d = mc.d_mem, mw = mail_row_width(d);
    view.mem = Tensor({U, d});
    view.mail = Tensor({U, mw});
    std::memcpy(view.mem.data(), view_mem, sizeof(double) * U * d);
    std::memcpy(view.mail.data(), view_mail, sizeof(double) * U * mw);
    ModelGrads grads = make_grads(mc);
    zero_grads(grads);
    std::vector<std::vector<double>> s_hat;
    SubStepStats st = sub_step(*g, p, plan, view, grads, &s_hat);
    *loss_out = st.loss;
    std::vector<double> flat(param_count(p));
    flatten_grads(grads, flat);
    std::memcpy(grads_out, flat.data(), sizeof(double) * flat.size());
    for (std::size_t u = 0; u < U; ++u)
      std::memcpy(s_hat_out + u * d, s_hat[u].data(), sizeof(double) * d);
  })
}

// build_root_writes for the same injected view/s_hat. nodes_out [<= 2B],
// mem_out [W x d_mem], mail_out [W x (2 d_mem + 3)].
int ref_build_root_writes(void* gp, int64_t d_mem, int64_t n, int64_t begin, int64_t end,
                          const int64_t* negatives, const double* view_mem,
                          const double* view_mail, const double* s_hat, int64_t* nodes_out,
                          double* mem_out, double* mail_out, int64_t* num_writes) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    std::span<const NodeId> negs(negatives, static_cast<std::size_t>(end - begin));
    SubBatchPlan plan = plan_sub_batch(*g, begin, end, negs, static_cast<std::size_t>(n));
    ReadView view;
    view.nodes = plan.supports;
    const std::size_t U = plan.supports.size(), d = static_cast<std::size_t>(d_mem),
                      mw = mail_row_width(d);
    view.mem = Tensor({U, d});
    view.mail = Tensor({U, mw});
    std::memcpy(view.mem.data(), view_mem, sizeof(double) * U * d);
    std::memcpy(view.mail.data(), view_mail, sizeof(double) * U * mw);
    std::vector<std::vector<double>> sh(U, std::vector<double>(d));
    for (std::size_t u = 0; u < U; ++u) std::memcpy(sh[u].data(), s_hat + u * d, sizeof(double) * d);
    RootWrites w = build_root_writes(*g, d, plan, view, sh);
    for (std::size_t x = 0; x < w.nodes.size(); ++x) nodes_out[x] = w.nodes[x];
    std::memcpy(mem_out, w.mem.data(), sizeof(double) * w.mem.numel());
    std::memcpy(mail_out, w.mail.data(), sizeof(double) * w.mail.numel());
    *num_writes = static_cast<int64_t>(w.nodes.size());
  })
}

// replay_batch on a state held in caller arrays (memory [N x d], last_update [N],
// mail_mem [N x 2d], mail_t [N], mail_dt [N], mail_event [N]); updated in place.
int ref_replay_batch(void* gp, const ref_model_cfg* c, const double* params_flat,
                     double* memory, double* last_update, double* mail_mem, double* mail_t,
                     double* mail_dt, int64_t* mail_event, int64_t begin, int64_t end) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    ModelConfig mc = to_mcfg(c);
    ModelParams p;
    shape_params(mc, p);
    params_from_flat(p, params_flat);
    const std::size_t N = static_cast<std::size_t>(g->num_nodes), d = mc.d_mem;
    NodeMemoryState s = init_state(g->num_nodes, d);
    std::memcpy(s.memory.data(), memory, sizeof(double) * N * d);
    std::memcpy(s.mail_mem.data(), mail_mem, sizeof(double) * N * 2 * d);
    for (std::size_t v = 0; v < N; ++v) {
      s.last_update[v] = last_update[v];
      s.mail_t[v] = mail_t[v];
      s.mail_dt[v] = mail_dt[v];
      s.mail_event[v] = mail_event[v];
    }
    replay_batch(*g, p, s, begin, end);
    std::memcpy(memory, s.memory.data(), sizeof(double) * N * d);
    std::memcpy(mail_mem, s.mail_mem.data(), sizeof(double) * N * 2 * d);
    for (std::size_t v = 0; v < N; ++v) {
      last_update[v] = s.last_update[v];
      mail_t[v] = s.mail_t[v];
      mail_dt[v] = s.mail_dt[v];
      mail_event[v] = s.mail_event[v];
    }
  })
}

int ref_evaluate_mrr(void* gp, const ref_model_cfg* c, const double* params_flat,
                     int64_t eval_begin, int64_t eval_end, int64_t batch, int32_t n_neg,
                     uint64_t seed, double* mrr_out, int64_t* queries_out) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    ModelConfig mc = to_mcfg(c);
    ModelParams p;
    shape_params(mc, p);
    params_from_flat(p, params_flat);
    EvalResult r = evaluate_mrr(*g, p, eval_begin, eval_end, batch, n_neg, seed);
    *mrr_out = r.mrr;
    *queries_out = r.queries;
  })
}

// ---------------------------------------------------------------- checkpoint
int ref_save_checkpoint(const ref_model_cfg* c, const double* params_flat, const char* path) {
  REF_GUARD({
    ModelParams p;
    shape_params(to_mcfg(c), p);
    params_from_flat(p, params_flat);
    save_checkpoint(p, path);
  })
}

int ref_load_checkpoint(const ref_model_cfg* c, const char* path, double* params_flat) {
  REF_GUARD({
    ModelParams p;
    shape_params(to_mcfg(c), p);
    load_checkpoint(p, path);
    params_to_flat(p, params_flat);
  })
}

// ---------------------------------------------------------------- optimizer
void* ref_adam_create(int64_t n) { return new Adam(static_cast<std::size_t>(n)); }
void ref_adam_free(void* a) { delete static_cast<Adam*>(a); }
int ref_adam_step(void* ap, const ref_model_cfg* c, double* params_flat, const double* grads,
                  double lr) {
  REF_GUARD({
    ModelConfig mc = to_mcfg(c);
    ModelParams p;
    shape_params(mc, p);
    params_from_flat(p, params_flat);
    std::span<const double> gs(grads, param_count(p));
    static_cast<Adam*>(ap)->step(p, gs, lr);
    params_to_flat(p, params_flat);
  })
}

// ---------------------------------------------------------------- schedule
// Per (rank, barrier): active, sub, stint batch, slice [begin,end), neg group
// of that sub, sweep, pair. Arrays are [T x barriers] row-major.
int ref_assignment(const ref_train_cfg* tc, int64_t train_begin, int64_t train_end,
                   int64_t* barriers_out, int64_t cap, int32_t* active, int32_t* sub,
                   int64_t* batch, int64_t* slice_begin, int64_t* slice_end,
                   int64_t* neg_group, int64_t* pair, int32_t* sweep, int64_t* active_trainers,
                   int64_t* traversed_after, int64_t* eval_barriers, int64_t* num_eval,
                   int64_t* resets /* [k x cap]: 1 when the group's daemon resets before the
                                       read of that barrier's pair */) {
  REF_GUARD({
    TrainConfig cfg = to_tcfg(tc);
    Assignment a = build_assignment(cfg, train_begin, train_end, false);
    *barriers_out = a.barriers;
    if (a.barriers > cap) throw config_error("ref_assignment: capacity too small");
    const int T = cfg.num_trainers();
    for (int r = 0; r < T; ++r) {
      for (int64_t b = 0; b < a.barriers; ++b) {
        TrainerTask t = a.task(r, b);
        const int64_t x = r * cap + b;
        active[x] = t.active ? 1 : 0;
        sub[x] = t.sub;
        batch[x] = t.active ? t.stint->batch : -1;
        slice_begin[x] = t.slice.begin;
        slice_end[x] = t.slice.end;
        neg_group[x] = t.active ? t.stint->neg_group[static_cast<std::size_t>(t.sub)] : -1;
        pair[x] = t.active ? t.stint->pair : -1;
        sweep[x] = t.active ? t.stint->sweep : -1;
      }
    }
    for (int64_t b = 0; b < a.barriers; ++b) {
      active_trainers[b] = a.active_trainers[b];
      traversed_after[b] = a.traversed_after[b];
    }
    *num_eval = static_cast<int64_t>(a.eval_barriers.size());
    for (std::size_t x = 0; x < a.eval_barriers.size(); ++x) eval_barriers[x] = a.eval_barriers[x];
    for (int g = 0; g < cfg.k; ++g) {
      for (int64_t b = 0; b < cap; ++b) resets[g * cap + b] = 0;
      const auto& pairs = a.groups[static_cast<std::size_t>(g)].pairs;
      for (std::size_t p = 0; p < pairs.size(); ++p) {
        if (p == 0 || pairs[p - 1].sweep != pairs[p].sweep) {
          const int64_t b0 = (pairs[p].pair / cfg.j) * cfg.j;
          resets[g * cap + b0] = 1;
        }
      }
    }
  })
}

// ---------------------------------------------------------------- runs
// Runs run_sequential (when sequential != 0; requires i=j=k=1) or the
// threaded run_training. barrier_loss [cap]; params_out [nparam] (may be null);
// metrics rows (iter, traversed, loss, val_mrr, elapsed_s) into metrics [cap_m x 5].
int ref_run(void* gp, const ref_model_cfg* c, const ref_train_cfg* tc, int64_t train_begin,
            int64_t train_end, int64_t val_begin, int64_t val_end, int32_t eval_negatives,
            int64_t eval_batch, int32_t sequential, double* barrier_loss, int64_t cap,
            int64_t* barriers_out, double* params_out, double* metrics, int64_t cap_m,
            int64_t* num_metrics, double* elapsed_out) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    RunOptions opt;
    opt.model = to_mcfg(c);
    opt.train = to_tcfg(tc);
    opt.train_begin = train_begin;
    opt.train_end = train_end;
    opt.val_begin = val_begin;
    opt.val_end = val_end;
    opt.eval_negatives = eval_negatives;
    opt.eval_batch = eval_batch;
    const auto t0 = std::chrono::steady_clock::now();
    RunResult res = sequential ? run_sequential(*g, opt) : run_training(*g, opt);
    *elapsed_out =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *barriers_out = res.barriers;
    for (int64_t b = 0; b < res.barriers && b < cap; ++b) barrier_loss[b] = res.barrier_loss[b];
    if (params_out) params_to_flat(res.params, params_out);
    *num_metrics = static_cast<int64_t>(res.metrics.size());
    for (std::size_t x = 0; x < res.metrics.size() && static_cast<int64_t>(x) < cap_m; ++x) {
      metrics[x * 5 + 0] = static_cast<double>(res.metrics[x].iter);
      metrics[x * 5 + 1] = static_cast<double>(res.metrics[x].traversed);
      metrics[x * 5 + 2] = res.metrics[x].loss;
      metrics[x * 5 + 3] = res.metrics[x].val_mrr;
      metrics[x * 5 + 4] = res.metrics[x].elapsed_s;
    }
  })
}

// run_training with op-log sinks (trainer.hpp:583, 643-667): one file per
// memory copy, "<prefix>.<r>.oplog"; and validate_oplog (oplog.hpp:105-156).
int ref_run_oplog(void* gp, const ref_model_cfg* c, const ref_train_cfg* tc, int64_t train_begin,
                  int64_t train_end, const char* prefix) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    RunOptions opt;
    opt.model = to_mcfg(c);
    opt.train = to_tcfg(tc);
    opt.train_begin = train_begin;
    opt.train_end = train_end;
    std::vector<std::unique_ptr<std::ofstream>> files;
    for (int r = 0; r < opt.train.k; ++r) {
      files.push_back(std::make_unique<std::ofstream>(std::string(prefix) + "." + std::to_string(r) + ".oplog"));
      opt.oplog_out.push_back(files.back().get());
    }
    run_training(*g, opt);
    for (auto& f : files) f->flush();
  })
}

// run_training with segment_snapshots (trainer.hpp:581,593; parallel.hpp:288-290):
// every memory copy's snapshots in plan order, meta[cap x 3] = copy, sweep,
// segment; memory[cap x N x d_mem]; last_update[cap x N].
int ref_run_snapshots(void* gp, const ref_model_cfg* c, const ref_train_cfg* tc, int64_t train_begin,
                      int64_t train_end, int64_t cap, int64_t* count_out, int64_t* meta, double* memory,
                      double* last_update) {
  REF_GUARD({
    auto* g = static_cast<TemporalGraph*>(gp);
    RunOptions opt;
    opt.model = to_mcfg(c);
    opt.train = to_tcfg(tc);
    opt.train_begin = train_begin;
    opt.train_end = train_end;
    opt.segment_snapshots = true;
    RunResult res = run_training(*g, opt);
    int64_t n = 0;
    for (std::size_t grp = 0; grp < res.snapshots.size(); ++grp) {
      for (const MemorySnapshot& sn : res.snapshots[grp]) {
        if (n < cap) {
          meta[n * 3 + 0] = static_cast<int64_t>(grp);
          meta[n * 3 + 1] = sn.sweep;
          meta[n * 3 + 2] = sn.segment;
          const auto f = sn.memory.flat();
          std::copy(f.begin(), f.end(), memory + n * static_cast<int64_t>(f.size()));
          std::copy(sn.last_update.begin(), sn.last_update.end(),
                    last_update + n * static_cast<int64_t>(sn.last_update.size()));
        }
        ++n;
      }
    }
    *count_out = n;
  })
}

int ref_validate_oplog(const char* path, int32_t i, int32_t j, int64_t* bad_line, char* msg, int64_t msg_cap) {
  REF_GUARD({
    OplogVerdict v = validate_oplog_file(path, i, j);
    *bad_line = v.ok ? 0 : static_cast<int64_t>(v.line);
    std::snprintf(msg, static_cast<size_t>(msg_cap), "%s", v.message.c_str());
  })
}

}  // extern "C"
