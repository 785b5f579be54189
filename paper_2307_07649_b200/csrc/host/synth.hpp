// Host-side synthetic event stream, bit-identical to the reference generator
// gen_synthetic (ref synthetic.hpp:54-112): same counter-based streams
// (rng.hpp), same draw order per event, same libm calls. It is input plumbing
// (the reference's own setup path), not part of the timed training step.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../common.cuh"

namespace tgb::host {

// rng.hpp:28-56 -- sequential splitmix chain seeded through one splitmix.
class Stream {
 public:
  explicit Stream(uint64_t seed) : s_(splitmix64(seed ^ 0xa02bdbf7bb3c0a7ull)) {}
  uint64_t u64() { return s_ = splitmix64(s_); }
  double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  int64_t below(int64_t n) { return static_cast<int64_t>(u64() % static_cast<uint64_t>(n)); }
  double normal() {
    double a = unit();
    const double b = unit();
    if (a < 1e-300) a = 1e-300;
    return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
  }

 private:
  uint64_t s_;
};

inline uint64_t hash64_2(uint64_t a, uint64_t b) { return splitmix64(hash_fold(a, b)); }
inline uint64_t hash64_3(uint64_t a, uint64_t b, uint64_t c) {
  return splitmix64(hash_fold(hash_fold(a, b), c));
}
inline uint64_t hash64_4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return splitmix64(hash_fold(hash_fold(hash_fold(a, b), c), d));
}

struct SynthConfig {
  int64_t nodes = 1000, events = 10000;
  double burst_prob = 0.2, pref_prob = 0.85;
  int prefs_per_src = 3;
  double src_frac = 0.5;
  bool bipartite = true;
  int64_t d_e = 0;
  double zipf_s = 1.0;
  uint64_t seed = 1;
};

// Inverse-CDF popularity over ranks [0, n): P(r) ~ 1 / (r + 1)^s.
class Popularity {
 public:
  Popularity(int64_t n, double s) : cum_(static_cast<size_t>(n)) {
    double run = 0;
    for (int64_t r = 0; r < n; ++r) {
      run += 1.0 / std::pow(static_cast<double>(r + 1), s);
      cum_[static_cast<size_t>(r)] = run;
    }
    total_ = run;
  }
  int64_t draw(Stream& st) const {
    const double target = st.unit() * total_;
    return static_cast<int64_t>(std::lower_bound(cum_.begin(), cum_.end(), target) - cum_.begin());
  }

 private:
  std::vector<double> cum_;
  double total_ = 0;
};

// Writes the stream in generation order (already ascending in t: gaps are
// non-negative, so the reference's stable sort is the identity). efeat may be
// null; features are rounded to float32.
inline int64_t synthesize(const SynthConfig& c, int64_t* src, int64_t* dst, double* t,
                          float* efeat) {
  TGB_REQUIRE(c.nodes >= 2, kConfig, "gen: need at least 2 nodes");
  TGB_REQUIRE(c.events > 0, kConfig, "gen: need a positive event count");
  TGB_REQUIRE(c.burst_prob >= 0 && c.burst_prob < 1, kConfig, "gen: burst-prob must be in [0,1)");
  int64_t n_src = c.nodes, lo_dst = 0, n_dst = c.nodes, boundary = -1;
  if (c.bipartite) {
    n_src = std::max<int64_t>(1, static_cast<int64_t>(std::llround(static_cast<double>(c.nodes) * c.src_frac)));
    n_src = std::min(n_src, c.nodes - 1);
    lo_dst = n_src;
    n_dst = c.nodes - n_src;
    boundary = n_src;
  }
  const Popularity src_pop(n_src, c.zipf_s), dst_pop(n_dst, c.zipf_s);
  Stream st(hash64_2(c.seed, 0x67656e65ull));
  double clock = 0;
  int64_t last_src = -1;
  for (int64_t e = 0; e < c.events; ++e) {
    const bool burst = last_src >= 0 && st.unit() < c.burst_prob;
    const int64_t s = burst ? last_src : src_pop.draw(st);
    int64_t d;
    if (c.prefs_per_src > 0 && st.unit() < c.pref_prob) {
      const int64_t slot = st.below(c.prefs_per_src);
      Stream pref(hash64_4(c.seed, 0x70726566ull, static_cast<uint64_t>(s), static_cast<uint64_t>(slot)));
      d = lo_dst + pref.below(n_dst);
    } else {
      d = lo_dst + dst_pop.draw(st);
    }
    if (!c.bipartite && d == s) d = (d + 1) % c.nodes;
    const double gap = -std::log(std::max(st.unit(), 1e-12));
    clock += burst ? gap * 0.01 : gap;
    src[e] = s;
    dst[e] = d;
    t[e] = clock;
    if (efeat) {
      float* row = efeat + e * c.d_e;
      for (int64_t f = 0; f < c.d_e; ++f) row[f] = static_cast<float>(0.1 * st.normal());
    } else {
      for (int64_t f = 0; f < c.d_e; ++f) (void)st.normal();
    }
    last_src = s;
  }
  return boundary;
}

}  // namespace tgb::host
