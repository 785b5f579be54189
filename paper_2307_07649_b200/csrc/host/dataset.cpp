// See dataset.hpp. Compiled by the host C++ compiler (std::from_chars for
// doubles: correctly rounded, the reference's parser).
#include "dataset.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string_view>
#include <thread>

#include "../common.cuh"

namespace tgb::host {

namespace {

std::string_view trim(std::string_view s) {
  auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
  while (!s.empty() && ws(s.front())) s.remove_prefix(1);
  while (!s.empty() && ws(s.back())) s.remove_suffix(1);
  return s;
}

// comma fields of one line (no quoting, as the reference)
void fields(std::string_view line, std::vector<std::string_view>& out) {
  out.clear();
  size_t at = 0;
  for (;;) {
    const size_t comma = line.find(',', at);
    if (comma == std::string_view::npos) {
      out.push_back(line.substr(at));
      return;
    }
    out.push_back(line.substr(at, comma - at));
    at = comma + 1;
  }
}

struct ParseFail {
  int64_t line = -1;
  int code = 0;
  std::string msg;
};

template <typename T>
bool number(std::string_view s, T& v) {
  const char* b = s.data();
  const char* e = b + s.size();
  auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e;
}

template <typename T>
T number_or_throw(std::string_view s, int64_t line_no, const char* what) {
  T v{};
  if (!number(s, v))
    throw Error(kParse, "line " + std::to_string(line_no) + ": bad " + what + " field '" + std::string(s) + "'");
  return v;
}

struct Chunk {
  size_t begin = 0, end = 0;  // byte range, line-aligned
  int64_t first_line = 0;     // line number of the first line in the range
  EventTable rows;
  ParseFail fail;
};

void parse_chunk(const std::string& text, const DatasetMeta& meta, Chunk& c) {
  const size_t ncols = 3 + static_cast<size_t>(meta.d_e);
  std::vector<std::string_view> cols;
  int64_t line_no = c.first_line;
  size_t at = c.begin;
  auto fail = [&](int code, std::string msg) {
    c.fail.line = line_no;
    c.fail.code = code;
    c.fail.msg = std::move(msg);
  };
  const std::string ln = "line ";
  while (at < c.end) {
    size_t nl = text.find('\n', at);
    if (nl == std::string::npos || nl > c.end) nl = c.end;
    std::string_view sv = trim(std::string_view(text).substr(at, nl - at));
    at = nl + 1;
    if (!sv.empty()) {
      fields(sv, cols);
      if (cols.size() != ncols) {
        fail(kParse, ln + std::to_string(line_no) + ": expected " + std::to_string(ncols) + " fields, got " +
                         std::to_string(cols.size()));
        return;
      }
      int64_t s = 0, d = 0;
      double t = 0;
      const char* bad = nullptr;
      std::string_view badv;
      if (!number(trim(cols[0]), s)) bad = "src", badv = trim(cols[0]);
      else if (!number(trim(cols[1]), d)) bad = "dst", badv = trim(cols[1]);
      else if (!number(trim(cols[2]), t)) bad = "t", badv = trim(cols[2]);
      if (bad) {
        fail(kParse, ln + std::to_string(line_no) + ": bad " + bad + " field '" + std::string(badv) + "'");
        return;
      }
      if (s < 0 || s >= meta.num_nodes || d < 0 || d >= meta.num_nodes) {
        fail(kParse, ln + std::to_string(line_no) + ": node id out of range [0, " + std::to_string(meta.num_nodes) + ")");
        return;
      }
      c.rows.src.push_back(s);
      c.rows.dst.push_back(d);
      c.rows.t.push_back(t);
      for (size_t f = 0; f < static_cast<size_t>(meta.d_e); ++f) {
        double v = 0;
        if (!number(trim(cols[3 + f]), v)) {
          fail(kParse, ln + std::to_string(line_no) + ": bad feature field '" + std::string(trim(cols[3 + f])) + "'");
          return;
        }
        c.rows.efeat.push_back(static_cast<float>(v));
      }
    }
    ++line_no;
  }
}

}  // namespace

std::string sidecar_path(const std::string& csv_path) {
  const size_t dot = csv_path.find_last_of('.');
  const size_t slash = csv_path.find_last_of('/');
  if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) return csv_path + ".meta";
  return csv_path.substr(0, dot) + ".meta";
}

DatasetMeta load_sidecar(const std::string& meta_path) {
  std::ifstream in(meta_path);
  if (!in) throw Error(kConfig, "cannot open dataset sidecar: " + meta_path);
  DatasetMeta m;
  bool have_nodes = false;
  std::string line;
  int64_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const std::string_view sv = trim(line);
    if (sv.empty() || sv.front() == '#') continue;
    const size_t eq = sv.find('=');
    if (eq == std::string_view::npos)
      throw Error(kParse, "sidecar line " + std::to_string(line_no) + ": expected key=value");
    const std::string_view key = trim(sv.substr(0, eq)), val = trim(sv.substr(eq + 1));
    if (key == "num_nodes") {
      m.num_nodes = number_or_throw<int64_t>(val, line_no, "num_nodes");
      have_nodes = true;
    } else if (key == "bipartite_boundary") {
      m.boundary = val == "none" ? -1 : number_or_throw<int64_t>(val, line_no, "bipartite_boundary");
    } else if (key == "d_e") {
      m.d_e = static_cast<int64_t>(number_or_throw<uint64_t>(val, line_no, "d_e"));
    } else {
      throw Error(kParse, "sidecar line " + std::to_string(line_no) + ": unknown key '" + std::string(key) + "'");
    }
  }
  if (!have_nodes) throw Error(kConfig, "sidecar missing num_nodes: " + meta_path);
  return m;
}

void load_events(const std::string& csv_path, const DatasetMeta& meta, int threads, EventTable& out) {
  std::ifstream in(csv_path, std::ios::binary);
  if (!in) throw Error(kConfig, "cannot open dataset file: " + csv_path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  // header (line 1)
  if (text.empty()) throw Error(kParse, "line 1: missing header row");
  size_t hdr_end = text.find('\n');
  if (hdr_end == std::string::npos) hdr_end = text.size();
  {
    std::vector<std::string_view> cols;
    fields(trim(std::string_view(text).substr(0, hdr_end)), cols);
    if (cols.size() != 3 + static_cast<size_t>(meta.d_e) || trim(cols[0]) != "src" || trim(cols[1]) != "dst" ||
        trim(cols[2]) != "t")
      throw Error(kParse, "line 1: header must be src,dst,t followed by " + std::to_string(meta.d_e) +
                              " feature columns");
  }
  const size_t body = std::min(text.size(), hdr_end + 1);
  // line-aligned chunks, one per worker
  const int T = std::max(1, threads);
  std::vector<Chunk> chunks(static_cast<size_t>(T));
  size_t at = body;
  for (int w = 0; w < T; ++w) {
    Chunk& c = chunks[static_cast<size_t>(w)];
    c.begin = at;
    size_t cut = w == T - 1 ? text.size() : body + (text.size() - body) * static_cast<size_t>(w + 1) / T;
    if (cut < at) cut = at;
    if (cut < text.size()) {
      const size_t nl = text.find('\n', cut);
      cut = nl == std::string::npos ? text.size() : nl + 1;
    }
    c.end = cut;
    at = cut;
  }
  int64_t line = 2;
  for (Chunk& c : chunks) {
    c.first_line = line;
    line += std::count(text.begin() + static_cast<std::ptrdiff_t>(c.begin),
                       text.begin() + static_cast<std::ptrdiff_t>(c.end), '\n');
  }
  std::vector<std::thread> pool;
  for (Chunk& c : chunks) pool.emplace_back([&text, &meta, &c]() { parse_chunk(text, meta, c); });
  for (auto& th : pool) th.join();
  for (const Chunk& c : chunks)
    if (c.fail.line >= 0) throw Error(c.fail.code, c.fail.msg);  // chunks are in file order
  size_t E = 0;
  for (const Chunk& c : chunks) E += c.rows.t.size();
  out.src.reserve(E);
  out.dst.reserve(E);
  out.t.reserve(E);
  out.efeat.reserve(E * static_cast<size_t>(meta.d_e));
  for (Chunk& c : chunks) {
    out.src.insert(out.src.end(), c.rows.src.begin(), c.rows.src.end());
    out.dst.insert(out.dst.end(), c.rows.dst.begin(), c.rows.dst.end());
    out.t.insert(out.t.end(), c.rows.t.begin(), c.rows.t.end());
    out.efeat.insert(out.efeat.end(), c.rows.efeat.begin(), c.rows.efeat.end());
    c.rows = EventTable{};
  }
}

void write_dataset(const std::string& csv_path, int64_t num_nodes, int64_t boundary, int64_t E,
                   const int64_t* src, const int64_t* dst, const double* t, const double* efeat,
                   int64_t d_e) {
  std::ofstream out(csv_path);
  if (!out) throw Error(kConfig, "cannot write dataset file: " + csv_path);
  std::string line = "src,dst,t";
  for (int64_t f = 0; f < d_e; ++f) line += ",f" + std::to_string(f);
  out << line << "\n";
  char num[64];
  for (int64_t e = 0; e < E; ++e) {
    line.clear();
    line += std::to_string(src[e]);
    line += ',';
    line += std::to_string(dst[e]);
    line += ',';
    std::snprintf(num, sizeof num, "%.17g", t[e]);
    line += num;
    for (int64_t f = 0; f < d_e; ++f) {
      std::snprintf(num, sizeof num, "%.17g", efeat[e * d_e + f]);
      line += ',';
      line += num;
    }
    out << line << '\n';
  }
  std::ofstream meta(sidecar_path(csv_path));
  meta << "num_nodes=" << num_nodes << "\n";
  if (boundary >= 0) meta << "bipartite_boundary=" << boundary << "\n";
  else meta << "bipartite_boundary=none\n";
  meta << "d_e=" << d_e << "\n";
}

void chronological_split(int64_t num_events, double train_frac, double val_frac, int64_t* train_end,
                         int64_t* val_end) {
  if (!(train_frac > 0.0 && train_frac < 1.0) || !(val_frac > 0.0 && val_frac < 1.0) || train_frac + val_frac >= 1.0)
    throw Error(kConfig, "split fractions must lie in (0,1) and sum below 1");
  const double n = static_cast<double>(num_events);
  *train_end = static_cast<int64_t>(std::llround(n * train_frac));
  *val_end = static_cast<int64_t>(std::llround(n * (train_frac + val_frac)));
}

}  // namespace tgb::host
