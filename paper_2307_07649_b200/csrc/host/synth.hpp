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

// Box-Muller of two raw chain outputs (Rng::next_normal, rng.hpp:46-52),
// scaled and rounded as gen_synthetic's features (synthetic.hpp:104).
inline float feature_from(uint64_t ra, uint64_t rb) {
  double a = static_cast<double>(ra >> 11) * 0x1.0p-53;
  const double b = static_cast<double>(rb >> 11) * 0x1.0p-53;
  if (a < 1e-300) a = 1e-300;
  return static_cast<float>(0.1 * (std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b)));
}

// The event part of gen_synthetic's sequential stream: endpoints and time of
// the next event. The caller then consumes 2 * d_e chain outputs for its
// features (next_normal per feature) before asking for the next event.
class Generator {
 public:
  explicit Generator(const SynthConfig& c)
      : c_(c), src_pop_(1, 1.0), dst_pop_(1, 1.0), st_(hash64_2(c.seed, 0x67656e65ull)) {
    TGB_REQUIRE(c.nodes >= 2, kConfig, "gen: need at least 2 nodes");
    TGB_REQUIRE(c.events > 0, kConfig, "gen: need a positive event count");
    TGB_REQUIRE(c.burst_prob >= 0 && c.burst_prob < 1, kConfig, "gen: burst-prob must be in [0,1)");
    n_src_ = c.nodes;
    n_dst_ = c.nodes;
    if (c.bipartite) {
      n_src_ = std::max<int64_t>(1, static_cast<int64_t>(std::llround(static_cast<double>(c.nodes) * c.src_frac)));
      n_src_ = std::min(n_src_, c.nodes - 1);
      lo_dst_ = n_src_;
      n_dst_ = c.nodes - n_src_;
      boundary_ = n_src_;
    }
    src_pop_ = Popularity(n_src_, c.zipf_s);
    dst_pop_ = Popularity(n_dst_, c.zipf_s);
  }
  int64_t boundary() const { return boundary_; }
  Stream& stream() { return st_; }

  void next(int64_t& s, int64_t& d, double& t) {
    const bool burst = last_src_ >= 0 && st_.unit() < c_.burst_prob;
    s = burst ? last_src_ : src_pop_.draw(st_);
    if (c_.prefs_per_src > 0 && st_.unit() < c_.pref_prob) {
      const int64_t slot = st_.below(c_.prefs_per_src);
      Stream pref(hash64_4(c_.seed, 0x70726566ull, static_cast<uint64_t>(s), static_cast<uint64_t>(slot)));
      d = lo_dst_ + pref.below(n_dst_);
    } else {
      d = lo_dst_ + dst_pop_.draw(st_);
    }
    if (!c_.bipartite && d == s) d = (d + 1) % c_.nodes;
    const double gap = -std::log(std::max(st_.unit(), 1e-12));
    clock_ += burst ? gap * 0.01 : gap;
    t = clock_;
    last_src_ = s;
  }

 private:
  SynthConfig c_;
  int64_t n_src_ = 0, lo_dst_ = 0, n_dst_ = 0, boundary_ = -1;
  Popularity src_pop_, dst_pop_;
  Stream st_;
  double clock_ = 0;
  int64_t last_src_ = -1;
};

// Writes the stream in generation order (already ascending in t: gaps are
// non-negative, so the reference's stable sort is the identity). efeat may be
// null; features are rounded to float32.
inline int64_t synthesize(const SynthConfig& c, int64_t* src, int64_t* dst, double* t,
                          float* efeat) {
  Generator gen(c);
  Stream& st = gen.stream();
  for (int64_t e = 0; e < c.events; ++e) {
    gen.next(src[e], dst[e], t[e]);
    float* row = efeat ? efeat + e * c.d_e : nullptr;
    for (int64_t f = 0; f < c.d_e; ++f) {
      const uint64_t a = st.u64();
      const uint64_t b = st.u64();
      if (row) row[f] = feature_from(a, b);
    }
  }
  return gen.boundary();
}

}  // namespace tgb::host
