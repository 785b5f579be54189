// Host-side i x j x k schedule: which global batch, slice, negative group and
// sub-iteration each trainer rank runs at each barrier, where memory copies
// reset, and how many trainers are active. Restates the reference planner
// (ref parallel.hpp:15-50 TrainConfig, :92-123 slicing/segments/budget,
// :128-183 Assignment::task, :187-210 negative groups, :218-331
// build_assignment) as flat per-(rank, barrier) descriptors that the device
// runner consumes.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../common.cuh"
#include "synth.hpp"

namespace tgb::host {

struct TrainCfg {
  int i = 1, j = 1, k = 1, p = 1, q = 1;
  int epochs = 1;
  int64_t local_batch = 600;
  double lr_base = 1e-3;
  uint64_t seed = 1;
  int64_t local_batch_ref = 0;
  int64_t neg_groups = 0;

  int trainers() const { return i * j * k; }
  int64_t global_batch() const { return static_cast<int64_t>(i) * local_batch; }
  double lr_eff() const {
    const double ref = static_cast<double>(local_batch_ref > 0 ? local_batch_ref : local_batch);
    return lr_base * (static_cast<double>(trainers()) * static_cast<double>(local_batch)) / ref;
  }
  void validate() const {
    TGB_REQUIRE(i >= 1 && j >= 1 && k >= 1 && p >= 1 && q >= 1, kConfig,
                "config: i, j, k, p, q must all be >= 1");
    TGB_REQUIRE(static_cast<int64_t>(i) * j * k == static_cast<int64_t>(p) * q, kConfig,
                "config: i*j*k must equal p*q");
    TGB_REQUIRE(k >= p, kConfig, "config: memory parallelism k must be >= machine count p");
    TGB_REQUIRE(local_batch >= 1, kConfig, "config: local_batch must be >= 1");
    TGB_REQUIRE(epochs >= 1, kConfig, "config: epochs must be >= 1");
    TGB_REQUIRE(neg_groups == 0 || neg_groups >= j, kConfig,
                "config: neg_groups must be 0 (unlimited) or >= j");
  }
};

// One stint = one global batch held by a team for up to j sub-iterations.
struct Stint {
  int64_t pair = 0, batch = 0;
  int team = 0, sweep = 0, segment = 0, subs = 0;
  std::vector<int64_t> neg_group;
};

// What one rank does at one barrier.
struct Task {
  bool active = false;
  int sub = 0;
  int subs = 0;
  int64_t pair = -1, batch = -1, batch_begin = 0, batch_end = 0, slice_begin = 0, slice_end = 0;
  int sweep = -1;
  bool reset_before = false;  // its group's memory resets before this stint's read
  std::vector<int64_t> neg_group;  // all subs of the stint (read at sub 0)
  std::vector<int64_t> slice_b, slice_e;  // not used (same slice for every sub)
};

class Schedule {
 public:
  TrainCfg cfg;
  int64_t train_begin = 0, train_end = 0, nb = 0, barriers = 0;
  std::vector<std::pair<int64_t, int64_t>> batches;
  std::vector<std::vector<Stint>> groups;          // per memory copy
  std::vector<int64_t> active_trainers, traversed_after, eval_barriers;
  std::vector<std::pair<int64_t, int64_t>> segments;  // k chronological batch ranges

  // DaemonOp::Snapshot placement (ref parallel.hpp:288-290): after the write
  // bracket of a pair whose batch closes its segment.
  bool snapshot_after(const Stint& st) const {
    return st.batch == segments[static_cast<size_t>(st.segment)].second - 1;
  }

  int group_of(int r) const { return r / (cfg.i * cfg.j); }
  int team_of(int r) const { return (r % (cfg.i * cfg.j)) / cfg.i; }
  int member_of(int r) const { return r % cfg.i; }

  static std::pair<int64_t, int64_t> slice_of(int64_t b, int64_t e, int i, int m) {
    const int64_t n = e - b;
    int64_t at = b;
    for (int x = 0; x < m; ++x) at += n / i + (x < n % i ? 1 : 0);
    return {at, at + n / i + (m < n % i ? 1 : 0)};
  }

  Task task(int rank, int64_t barrier) const {
    Task t;
    const int g = group_of(rank);
    const int64_t pair = (barrier / cfg.j) * cfg.j + team_of(rank);
    const auto& ps = groups[static_cast<size_t>(g)];
    if (pair >= static_cast<int64_t>(ps.size())) return t;
    const Stint& st = ps[static_cast<size_t>(pair)];
    const int sub = static_cast<int>(barrier % cfg.j);
    if (sub >= st.subs) return t;
    t.active = true;
    t.sub = sub;
    t.subs = st.subs;
    t.pair = st.pair;
    t.batch = st.batch;
    t.sweep = st.sweep;
    t.batch_begin = batches[static_cast<size_t>(st.batch)].first;
    t.batch_end = batches[static_cast<size_t>(st.batch)].second;
    auto sl = slice_of(t.batch_begin, t.batch_end, cfg.i, member_of(rank));
    t.slice_begin = sl.first;
    t.slice_end = sl.second;
    t.neg_group = st.neg_group;
    t.reset_before = pair == 0 || ps[static_cast<size_t>(pair - 1)].sweep != st.sweep;
    return t;
  }

  static std::vector<int64_t> neg_groups_for(uint64_t seed, int group, int64_t pair, int subs, int j,
                                             int64_t limit) {
    std::vector<int64_t> out(static_cast<size_t>(subs));
    if (limit == 0) {
      for (int s = 0; s < subs; ++s) out[static_cast<size_t>(s)] = pair * j + s;
      return out;
    }
    // partial Fisher-Yates over [0, limit) with a sparse swap map
    Stream st(hash64_4(seed, 0x6e656773ull, static_cast<uint64_t>(group), static_cast<uint64_t>(pair)));
    std::map<int64_t, int64_t> moved;
    auto at = [&](int64_t x) {
      auto it = moved.find(x);
      return it == moved.end() ? x : it->second;
    };
    for (int s = 0; s < subs; ++s) {
      const int64_t pick = s + static_cast<int64_t>(st.u64() % static_cast<uint64_t>(limit - s));
      out[static_cast<size_t>(s)] = at(pick);
      moved[pick] = at(s);
    }
    return out;
  }

  static Schedule build(const TrainCfg& cfg, int64_t train_begin, int64_t train_end) {
    cfg.validate();
    TGB_REQUIRE(train_end > train_begin, kConfig, "assignment: empty training range");
    Schedule a;
    a.cfg = cfg;
    a.train_begin = train_begin;
    a.train_end = train_end;
    const int64_t gb = cfg.global_batch();
    const int64_t total = train_end - train_begin;
    a.nb = (total + gb - 1) / gb;
    for (int64_t b = 0; b < a.nb; ++b) {
      const int64_t lo = train_begin + b * gb;
      a.batches.emplace_back(lo, std::min(train_end, lo + gb));
    }
    // k chronological segments of batch indices (the last may be short)
    std::vector<std::pair<int64_t, int64_t>> seg;
    const int64_t seg_len = (a.nb + cfg.k - 1) / cfg.k;
    for (int64_t s = 0; s < a.nb; s += seg_len) seg.emplace_back(s, std::min(a.nb, s + seg_len));
    while (static_cast<int>(seg.size()) < cfg.k) seg.emplace_back(a.nb, a.nb);
    a.segments = seg;
    // team-iteration budget spread over the k memory copies
    const int64_t iters = static_cast<int64_t>(cfg.epochs) * a.nb;
    a.groups.resize(static_cast<size_t>(cfg.k));
    for (int g = 0; g < cfg.k; ++g) {
      const int64_t n_iters = iters / cfg.k + (g < iters % cfg.k ? 1 : 0);
      if (n_iters == 0) continue;
      const int64_t n_pairs = (n_iters + cfg.j - 1) / cfg.j;
      auto& ps = a.groups[static_cast<size_t>(g)];
      for (int sweep = 0; static_cast<int64_t>(ps.size()) < n_pairs; ++sweep) {
        for (int s = sweep == 0 ? g : 0; s < cfg.k && static_cast<int64_t>(ps.size()) < n_pairs; ++s) {
          for (int64_t b = seg[static_cast<size_t>(s)].first;
               b < seg[static_cast<size_t>(s)].second && static_cast<int64_t>(ps.size()) < n_pairs; ++b) {
            Stint st;
            st.pair = static_cast<int64_t>(ps.size());
            st.team = static_cast<int>(st.pair % cfg.j);
            st.batch = b;
            st.sweep = sweep;
            st.segment = s;
            st.subs = cfg.j;
            ps.push_back(st);
          }
        }
      }
      ps.back().subs = static_cast<int>(n_iters - (n_pairs - 1) * cfg.j);
      for (auto& st : ps)
        st.neg_group = neg_groups_for(cfg.seed, g, st.pair, st.subs, cfg.j, cfg.neg_groups);
    }
    int64_t barriers = 0;
    for (const auto& ps : a.groups)
      for (const auto& st : ps) barriers = std::max(barriers, (st.pair / cfg.j) * cfg.j + st.subs);
    a.barriers = barriers;
    a.active_trainers.assign(static_cast<size_t>(barriers), 0);
    a.traversed_after.assign(static_cast<size_t>(barriers), 0);
    for (const auto& ps : a.groups) {
      for (const auto& st : ps) {
        const int64_t base = (st.pair / cfg.j) * cfg.j;
        const auto& b = a.batches[static_cast<size_t>(st.batch)];
        for (int s = 0; s < st.subs; ++s) {
          a.active_trainers[static_cast<size_t>(base + s)] += cfg.i;
          a.traversed_after[static_cast<size_t>(base + s)] += b.second - b.first;
        }
      }
    }
    for (int64_t b = 1; b < barriers; ++b)
      a.traversed_after[static_cast<size_t>(b)] += a.traversed_after[static_cast<size_t>(b - 1)];
    int64_t mark = total;
    for (int64_t b = 0; b < barriers; ++b) {
      if (a.traversed_after[static_cast<size_t>(b)] >= mark) {
        a.eval_barriers.push_back(b);
        while (mark <= a.traversed_after[static_cast<size_t>(b)]) mark += total;
      }
    }
    if (barriers > 0 && (a.eval_barriers.empty() || a.eval_barriers.back() != barriers - 1))
      a.eval_barriers.push_back(barriers - 1);
    return a;
  }
};

}  // namespace tgb::host
