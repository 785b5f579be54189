// ORACLE / TEST INFRASTRUCTURE ONLY.
// Exercises the reference-side drop-in (include/tgnn_b200.hpp) exactly as a
// reference user would: the reference's own types (TemporalGraph, RunOptions,
// RunResult, MemoryClient, ...) from the UNMODIFIED headers under
// /root/reference/proj/include, compared with the reference's own functions.
// Built by oracle/Makefile into oracle/_ref/shim_driver; run by
// tests/test_shim_cpp.py:
//   shim_driver cpu   -- no GPU: C ABI host paths through the shim types
//   shim_driver gpu   -- the drop-in on cuda:0 against the reference
// Prints one line per check ("ok ..." / "FAIL ..."); exit status = failures.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "tgnn/parallel.hpp"
#include "tgnn/synthetic.hpp"
#include "tgnn_b200.hpp"

using namespace tgnn;

namespace {

int g_fail = 0;

double g_ref_mean[2] = {0, 0};  // reference mean MRR over seeds 5..12 at (1,1,1), (1,1,4) (argv)

void report(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "ok" : "FAIL", what.c_str());
  std::fflush(stdout);
  if (!ok) ++g_fail;
}

ModelConfig model_for(const TemporalGraph& g, std::size_t d_mem, std::size_t d_time, std::size_t d_static,
                      std::size_t d_attn, std::size_t n) {  // acceptance.cpp:113-126
  ModelConfig m;
  m.d_mem = d_mem;
  m.d_time = d_time;
  m.d_static = d_static;
  m.d_attn = d_attn;
  m.d_hidden = d_attn;
  m.d_e = g.d_e;
  m.n_neighbors = n;
  m.num_nodes = g.num_nodes;
  m.max_t = g.events.empty() ? 1.0 : g.events.back().t;
  return m;
}

double max_abs_diff(std::span<const double> a, std::span<const double> b) {
  double m = 0;
  for (std::size_t x = 0; x < a.size() && x < b.size(); ++x) m = std::max(m, std::fabs(a[x] - b[x]));
  return a.size() == b.size() ? m : INFINITY;
}

double max_abs(std::span<const double> a) {
  double m = 0;
  for (double v : a) m = std::max(m, std::fabs(v));
  return m;
}

// ---------------------------------------------------------------- cpu
void cpu_checks() {
  SynthParams sp;
  sp.nodes = 60;
  sp.events = 800;
  sp.d_e = 4;
  sp.seed = 3;
  const TemporalGraph g = gen_synthetic(sp);
  const ModelConfig mc = model_for(g, 6, 4, 3, 5, 5);
  // init_params through the C ABI, unflattened into the reference's ModelParams
  const ModelParams ref = init_params(mc, 7);
  std::vector<double> flat{std::vector<double>(param_count(ref))};
  const tgnn_model_config c = b200::to_c(mc);
  b200::check(tgnn_init_params(&c, 7, flat.data()));
  const ModelParams ours = b200::unflatten(mc, flat);
  report(b200::flatten(ours) == b200::flatten(ref), "init_params == reference, every tensor bitwise");
  // the schedule (build_assignment + Assignment::task) through the C ABI
  TrainConfig tc;
  tc.i = 2;
  tc.j = 2;
  tc.k = 2;
  tc.q = 8;
  tc.local_batch = 25;
  tc.epochs = 3;
  const Assignment asg = build_assignment(tc, 0, 700);
  const tgnn_train_config tcc = b200::to_c(tc);
  bool same = true;
  for (int r = 0; r < tc.num_trainers(); ++r) {
    std::vector<int64_t> out{std::vector<int64_t>(static_cast<std::size_t>(12 * asg.barriers))};
    int64_t nb = 0;
    b200::check(tgnn_schedule_query(&tcc, 0, 700, r, 0, asg.barriers, out.data(), &nb));
    same &= nb == asg.barriers;
    for (int64_t b = 0; b < asg.barriers && same; ++b) {
      const TrainerTask t = asg.task(r, b);
      const int64_t* o = out.data() + 12 * b;
      same &= o[0] == (t.active ? 1 : 0) &&
              (!t.active || (o[1] == t.sub && o[3] == t.stint->batch && o[6] == t.slice.begin && o[7] == t.slice.end));
      same &= o[10] == asg.active_trainers[static_cast<std::size_t>(b)] &&
              o[11] == asg.traversed_after[static_cast<std::size_t>(b)];
    }
  }
  report(same, "schedule_query == build_assignment / Assignment::task at (2,2,2)");
  // checkpoint files: the shim's weights saved by the C ABI, loaded by the reference
  const std::string path = "/tmp/tgnn_shim_driver.ckpt";
  b200::check(tgnn_checkpoint_save(&c, flat.data(), path.c_str()));
  ModelParams back;
  shape_params(mc, back);
  load_checkpoint(back, path);
  report(b200::flatten(back) == flat, "model.ckpt written through the C ABI loads in the reference");
  // errors map onto the reference's exception types
  bool threw = false;
  try {
    b200::check(tgnn_schedule_query(&tcc, 10, 5, 0, 0, 0, nullptr, nullptr));
  } catch (const config_error&) {
    threw = true;
  }
  report(threw, "status codes rethrow as the reference's config_error");
}

// ---------------------------------------------------------------- gpu
void gpu_checks() {
  // parity level: sampler, negatives, plan, MemoryClient on a device graph
  {
    SynthParams sp;
    sp.nodes = 500;
    sp.events = 20000;
    sp.d_e = 6;
    sp.seed = 9;
    const TemporalGraph g = gen_synthetic(sp);
    b200::Context ctx(0);
    b200::Graph G(ctx, g);
    bool ok = true;
    for (int q = 0; q < 400 && ok; ++q) {
      const NodeId v = (q * 37) % g.num_nodes;
      const TimeT t = g.events[static_cast<std::size_t>((q * 7919) % g.num_events())].t;
      const auto a = b200::sample_recent_neighbors(G, v, t, 10);
      const auto b = sample_recent_neighbors(g, v, t, 10);
      ok &= a.size() == b.size();
      for (std::size_t m = 0; m < a.size() && ok; ++m)
        ok &= a[m].node == b[m].node && a[m].event == b[m].event && a[m].dt == b[m].dt;
    }
    report(ok, "sample_recent_neighbors == reference (400 queries, bitwise)");
    const auto negs = b200::sample_negatives(G, 11, 3, 600, 1);
    report(negs == sample_negatives(g, 11, 3, 600, 1), "sample_negatives == reference");
    const SubBatchPlan pa = b200::plan_sub_batch(G, 9000, 9600, negs, 10);
    const SubBatchPlan pb = plan_sub_batch(g, 9000, 9600, negs, 10);
    ok = pa.supports == pb.supports && pa.roots.size() == pb.roots.size();
    for (std::size_t x = 0; x < pa.roots.size() && ok; ++x) {
      ok &= pa.roots[x].node == pb.roots[x].node && pa.roots[x].t == pb.roots[x].t &&
            pa.roots[x].nbrs.size() == pb.roots[x].nbrs.size();
      for (std::size_t m = 0; m < pa.roots[x].nbrs.size() && ok; ++m)
        ok &= pa.roots[x].nbrs[m].node == pb.roots[x].nbrs[m].node &&
              pa.roots[x].nbrs[m].event == pb.roots[x].nbrs[m].event && pa.roots[x].nbrs[m].dt == pb.roots[x].nbrs[m].dt;
    }
    report(ok, "plan_sub_batch == reference (roots, neighbours, supports)");
    // MemoryClient: a replay through the device client vs the reference's replay
    const ModelConfig mc = model_for(g, 8, 4, 4, 8, 5);
    const ModelParams p = init_params(mc, 3);
    b200::DeviceMemoryClient dm(ctx, g.num_nodes, mc.d_mem);
    NodeMemoryState st = init_state(g.num_nodes, mc.d_mem);
    for (EventId b = 0; b < 3000; b += 300) {
      b200::replay_batch(ctx, G, p, dm, b, b + 300);
      replay_batch(g, p, st, b, b + 300);
    }
    NodeMemoryState ours = init_state(g.num_nodes, mc.d_mem);
    dm.export_state(ours);
    const double err = max_abs_diff(ours.memory.flat(), st.memory.flat());
    report(err <= 1e-4 * max_abs(st.memory.flat()) && ours.last_update == st.last_update &&
               ours.mail_event == st.mail_event && ours.mail_t == st.mail_t,
           "DeviceMemoryClient + replay_batch == reference replay (memory 1e-4, times and mail events exact)");
    const std::vector<std::vector<NodeId>> subs{{3, 17, 250}, {499}};
    const auto views = dm.read(subs);
    DirectMemoryClient dc(st);
    const auto want = dc.read(subs);
    ok = views.size() == 2;
    for (std::size_t s = 0; s < views.size() && ok; ++s)
      ok &= views[s].nodes == want[s].nodes &&
            max_abs_diff(views[s].mem.flat(), want[s].mem.flat()) <= 1e-4 * (max_abs(want[s].mem.flat()) + 1e-6);
    report(ok, "DeviceMemoryClient::read == DirectMemoryClient::read");
    const EvalResult ea = b200::evaluate_mrr(ctx, G, p, 15000, 16000, 200, 19, 5);
    const EvalResult eb = evaluate_mrr(g, p, 15000, 16000, 200, 19, 5);
    report(ea.queries == eb.queries && std::fabs(ea.mrr - eb.mrr) <= 5e-3,
           "evaluate_mrr == reference (" + std::to_string(ea.mrr) + " vs " + std::to_string(eb.mrr) + ")");
  }
  // performance level: run_training with the reference's RunOptions / RunResult
  {
    SynthParams sp;
    sp.nodes = 20;
    sp.events = 120;
    sp.d_e = 2;
    sp.seed = 21;
    const TemporalGraph g = gen_synthetic(sp);
    const int shapes[][4] = {{1, 1, 1, 2}, {1, 1, 2, 2}, {2, 1, 1, 2}, {1, 2, 1, 2}, {2, 2, 1, 2}, {1, 2, 2, 3}};
    for (const auto& s : shapes) {
      RunOptions o;
      o.model = model_for(g, 3, 2, 2, 3, 2);
      o.model.d_hidden = 2;
      o.train.i = s[0];
      o.train.j = s[1];
      o.train.k = s[2];
      o.train.q = s[0] * s[1] * s[2];
      o.train.local_batch = 15;
      o.train.epochs = s[3];
      o.train.seed = 3;
      o.train.lr_base = 1e-3;
      o.train_begin = 0;
      o.train_end = 90;
      o.val_begin = 90;
      o.val_end = 120;
      o.eval_negatives = 5;
      std::vector<std::ostringstream> la(static_cast<std::size_t>(s[2])), lb(static_cast<std::size_t>(s[2]));
      std::ostringstream ma, mb;
      RunOptions oa = o, ob = o;
      for (auto& x : la) oa.oplog_out.push_back(&x);
      for (auto& x : lb) ob.oplog_out.push_back(&x);
      oa.metrics_out = &ma;
      ob.metrics_out = &mb;
      int evals = 0;
      double last_mrr = -1;
      std::vector<double> last_w;
      ob.on_eval = [&](const MetricsRow& row, const ModelParams& p) {
        ++evals;
        last_mrr = row.val_mrr;
        last_w = b200::flatten(p);
      };
      const RunResult ra = run_training(g, oa);
      const RunResult rb = b200::run_training(g, ob);
      const std::string tag = "(" + std::to_string(s[0]) + "," + std::to_string(s[1]) + "," + std::to_string(s[2]) + ")";
      bool logs = true;
      for (std::size_t x = 0; x < la.size(); ++x) logs &= la[x].str() == lb[x].str() && !la[x].str().empty();
      report(logs, tag + " op-log of every memory copy byte-identical to run_training's");
      const double lmax = max_abs(ra.barrier_loss);
      report(rb.barriers == ra.barriers && std::fabs(rb.barrier_loss[0] - ra.barrier_loss[0]) <= 1e-4 * std::fabs(ra.barrier_loss[0]) &&
                 max_abs_diff(rb.barrier_loss, ra.barrier_loss) <= 1e-3 * lmax,
             tag + " barrier_loss (first 1e-4, all 1e-3)");
      const auto wa = b200::flatten(ra.params), wb = b200::flatten(rb.params);
      std::vector<double> dif(wa.size());
      for (std::size_t x = 0; x < wa.size(); ++x) dif[x] = std::fabs(wa[x] - wb[x]);
      std::nth_element(dif.begin(), dif.begin() + static_cast<std::ptrdiff_t>(dif.size() / 2), dif.end());
      report(dif[dif.size() / 2] <= 1e-5, tag + " RunResult.params (median |diff| <= 1e-5)");
      report(rb.metrics.size() == ra.metrics.size() && evals == static_cast<int>(rb.metrics.size()) &&
                 last_w == wb && last_mrr == rb.metrics.back().val_mrr,
             tag + " metrics rows, one on_eval per row with the row's weights");
      // metrics_out: same header, one row per eval point, the reference's formats
      std::istringstream sa(ma.str()), sb(mb.str());
      std::string ha, hb;
      std::getline(sa, ha);
      std::getline(sb, hb);
      int rows = 0;
      bool fmt = ha == hb;
      for (std::string la2, lb2; std::getline(sa, la2) && std::getline(sb, lb2); ++rows) {
        fmt &= la2.substr(0, la2.find(',', la2.find(',') + 1)) == lb2.substr(0, lb2.find(',', lb2.find(',') + 1));
        fmt &= std::count(lb2.begin(), lb2.end(), ',') == 4;
      }
      report(fmt && rows == static_cast<int>(ra.metrics.size()), tag + " metrics_out CSV (header, iter, traversed)");
    }
  }
  // segment snapshots (acceptance criterion 4, acceptance.cpp:265-328)
  {
    SynthParams sp;
    sp.nodes = 120;
    sp.events = 500;
    sp.d_e = 1;
    sp.seed = 41;
    const TemporalGraph g = gen_synthetic(sp);
    RunOptions o;
    o.model = model_for(g, 6, 3, 2, 6, 3);
    o.train.k = 4;
    o.train.q = 4;
    o.train.local_batch = 25;
    o.train.epochs = 4;
    o.train.seed = 9;
    o.train.lr_base = 0.0;
    o.train_begin = 0;
    o.train_end = 400;
    o.segment_snapshots = true;
    const RunResult ra = run_training(g, o);
    const RunResult rb = b200::run_training(g, o);
    bool ok = ra.snapshots.size() == 4 && rb.snapshots.size() == 4;
    int n = 0;
    for (std::size_t c = 0; c < 4 && ok; ++c) {
      ok &= ra.snapshots[c].size() == rb.snapshots[c].size();
      for (std::size_t x = 0; x < ra.snapshots[c].size() && ok; ++x, ++n) {
        const MemorySnapshot &a = ra.snapshots[c][x], &b = rb.snapshots[c][x];
        ok &= a.sweep == b.sweep && a.segment == b.segment && a.last_update == b.last_update &&
              max_abs_diff(a.memory.flat(), b.memory.flat()) <= 1e-4 * max_abs(a.memory.flat());
      }
    }
    report(ok && n == 16, "RunResult.snapshots: 16 segment snapshots of 4 copies == run_training's (1e-4, "
                          "last_update exact)");
  }
  // acceptance criteria 7 and 8 (acceptance.cpp:402-458): the benchmark stream
  // through run_training with validation, metrics_out and on_eval
  {
    SynthParams sp;
    sp.nodes = 300;
    sp.events = 5000;
    sp.pref_prob = 0.95;
    sp.prefs_per_src = 1;
    sp.burst_prob = 0.15;
    sp.zipf_s = 1.1;
    sp.d_e = 0;
    sp.seed = 20260819;
    const TemporalGraph g = gen_synthetic(sp);
    RunOptions o;
    o.model = model_for(g, 24, 8, 8, 24, 8);
    o.train.local_batch = 175;
    o.train.lr_base = 2e-3;
    o.train.epochs = 150;
    o.train.seed = 5;
    o.train_begin = 0;
    o.train_end = 3500;
    o.val_begin = 3500;
    o.val_end = 4500;
    o.eval_negatives = 49;
    double harmonic = 0;
    for (int k = 1; k <= 50; ++k) harmonic += 1.0 / k;
    const double want7 = 3.0 * harmonic / 50.0;
    // (i, j, k), the reference's mean final val MRR at 525,000 traversed events
    // over training seeds 5..12 (tests/golden/convergence_ref.json, passed on
    // the command line by tests/test_shim_cpp.py; seed 5 alone is the
    // reference's anchor 0.8767 / 0.8824), tolerance 0.02 on the mean
    const struct { int i, j, k; double mrr, tol; } runs[] = {{1, 1, 1, g_ref_mean[0], 0.02},
                                                            {1, 1, 4, g_ref_mean[1], 0.02}};
    for (const auto& v : runs) {
      RunOptions x = o;
      x.train.i = v.i;
      x.train.j = v.j;
      x.train.k = v.k;
      x.train.q = v.i * v.j * v.k;  // same epochs: equal traversed events (acceptance.cpp:468-478)
      double best = 0;
      ModelParams best_w;
      x.on_eval = [&](const MetricsRow& row, const ModelParams& p) {
        if (row.val_mrr > best) {
          best = row.val_mrr;
          best_w = p;
        }
      };
      std::ostringstream csv;
      x.metrics_out = &csv;
      const RunResult r = b200::run_training(g, x);
      const std::string tag = "(" + std::to_string(v.i) + "," + std::to_string(v.j) + "," + std::to_string(v.k) + ")";
      double best20 = 0;
      for (std::size_t row = 0; row < std::min<std::size_t>(20, r.metrics.size()); ++row)
        best20 = std::max(best20, r.metrics[row].val_mrr);
      if (v.k == 1)
        report(best20 >= want7, tag + " criterion 7: best val MRR " + std::to_string(best20) +
                                    " within 20 epochs >= " + std::to_string(want7));
      const MetricsRow& last = r.metrics.back();
      // criterion 8 over seeds 5..12: seed 5 is this run, the others train
      // without per-epoch validation and score the final weights the same way
      double sum = last.val_mrr;
      std::string per = std::to_string(last.val_mrr);
      bool traversed_ok = last.traversed == 525000;
      for (std::uint64_t sd = 6; sd <= 12; ++sd) {
        RunOptions y = x;
        y.train.seed = sd;
        y.val_begin = y.val_end = 0;
        y.on_eval = nullptr;
        y.metrics_out = nullptr;
        const RunResult ry = b200::run_training(g, y);
        b200::Context cx(0);
        b200::Graph Gx(cx, g);
        const double m = b200::evaluate_mrr(cx, Gx, ry.params, 3500, 4500, 175, 49, 5).mrr;
        sum += m;
        per += " " + std::to_string(m);
        traversed_ok = traversed_ok && ry.barriers == r.barriers;
      }
      const double mean = sum / 8.0;
      report(traversed_ok && v.mrr > 0 && std::fabs(mean - v.mrr) <= v.tol,
             tag + " criterion 8: final val MRR at " + std::to_string(last.traversed) +
                 " traversed, seeds 5..12: " + per + "; mean " + std::to_string(mean) + " (reference mean " +
                 std::to_string(v.mrr) + ")");
      // checkpoint-on-best through on_eval (trainer.hpp:584-587): the best row's
      // weights score that row's MRR again
      b200::Context ctx(0);
      b200::Graph G(ctx, g);
      const EvalResult e = b200::evaluate_mrr(ctx, G, best_w, 3500, 4500, 175, 49, 5);
      report(std::fabs(e.mrr - best) <= 1e-9, tag + " on_eval weights reproduce the best row's MRR");
      const std::string text = csv.str();
      const std::size_t lines = static_cast<std::size_t>(std::count(text.begin(), text.end(), '\n'));
      report(lines == r.metrics.size() + 1, tag + " metrics_out rows");
    }
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  try {
    if (mode == "cpu") cpu_checks();
    else if (mode == "gpu") {
      if (argc > 3) {
        g_ref_mean[0] = std::atof(argv[2]);
        g_ref_mean[1] = std::atof(argv[3]);
      }
      gpu_checks();
    }
    else {
      std::fprintf(stderr, "usage: shim_driver cpu | gpu [ref_mean_111 ref_mean_114]\n");
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 1 + g_fail;
  }
  std::printf("%s: %d failure(s)\n", mode.c_str(), g_fail);
  return g_fail;
}
