// model.ckpt compatibility (ref model.hpp:168-222): a text manifest, one
// "tensor <name> <rank> <dims...>" line per tensor in for_each_tensor order
// (model.hpp:56-76), the line "data", then every tensor's f64 payload
// (little-endian) in manifest order. The device keeps fp32 weights; the file
// carries the flat f64 vector the host converts to and from.
#pragma once

#include <cstdint>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

namespace tgb::host {

struct CkptTensor {
  const char* name;
  std::vector<int64_t> shape;
};

// names and reference shapes (shape_params, model.hpp:79-101); rank-1 tensors
// are omega and the biases, dec.W2 is [1, d_h] and dec.b2 is [1]
inline std::vector<CkptTensor> ckpt_manifest(int64_t d_mem, int64_t d_time, int64_t d_static,
                                             int64_t d_attn, int64_t d_hidden, int64_t d_e,
                                             int64_t num_nodes) {
  const int64_t gin = 2 * d_mem + d_time + d_e + d_mem;
  const int64_t q_in = d_mem + d_static + d_time;
  const int64_t kv_in = d_mem + d_static + d_e + d_time;
  const int64_t dh = d_hidden ? d_hidden : d_mem;
  return {{"omega", {d_time}},          {"gru.Wz", {d_mem, gin}}, {"gru.Wr", {d_mem, gin}},
          {"gru.Wh", {d_mem, gin}},     {"gru.bz", {d_mem}},      {"gru.br", {d_mem}},
          {"gru.bh", {d_mem}},          {"attn.Wq", {d_attn, q_in}}, {"attn.bq", {d_attn}},
          {"attn.Wk", {d_attn, kv_in}}, {"attn.bk", {d_attn}},    {"attn.Wv", {d_attn, kv_in}},
          {"attn.bv", {d_attn}},        {"static_table", {num_nodes, d_static}},
          {"dec.W1", {dh, 2 * d_attn}}, {"dec.b1", {dh}},         {"dec.W2", {1, dh}},
          {"dec.b2", {1}}};
}

inline int64_t ckpt_numel(const std::vector<int64_t>& s) {
  int64_t n = 1;
  for (int64_t d : s) n *= d;
  return n;
}

// Returns an empty string on success, else the reference's error text.
inline std::string ckpt_save(const std::vector<CkptTensor>& man, const double* flat, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) return "cannot write checkpoint: " + path;
  out << "tgnn-checkpoint v1\n";
  for (const CkptTensor& t : man) {
    out << "tensor " << t.name << " " << t.shape.size();
    for (int64_t d : t.shape) out << " " << d;
    out << "\n";
  }
  out << "data\n";
  int64_t at = 0;
  for (const CkptTensor& t : man) {
    const int64_t n = ckpt_numel(t.shape);
    out.write(reinterpret_cast<const char*>(flat + at), static_cast<std::streamsize>(n * sizeof(double)));
    at += n;
  }
  if (!out) return "cannot write checkpoint: " + path;
  return {};
}

inline std::string ckpt_load(const std::vector<CkptTensor>& man, const std::string& path, double* flat) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return "cannot open checkpoint: " + path;
  std::string line;
  if (!std::getline(in, line) || line != "tgnn-checkpoint v1") return "checkpoint: bad magic line in " + path;
  std::vector<std::pair<std::string, std::vector<int64_t>>> got;
  while (std::getline(in, line)) {
    if (line == "data") break;
    std::istringstream ls(line);
    std::string kw, name;
    int64_t rank = 0;
    if (!(ls >> kw >> name >> rank) || kw != "tensor" || rank < 0) return "checkpoint: bad manifest line '" + line + "'";
    std::vector<int64_t> shape(static_cast<size_t>(rank));
    for (auto& d : shape)
      if (!(ls >> d)) return "checkpoint: truncated shape in '" + line + "'";
    got.emplace_back(name, shape);
  }
  int64_t at = 0;
  size_t idx = 0;
  for (const CkptTensor& t : man) {
    if (idx >= got.size() || got[idx].first != t.name || got[idx].second != t.shape)
      return std::string("checkpoint: manifest mismatch at tensor ") + t.name;
    const int64_t n = ckpt_numel(t.shape);
    in.read(reinterpret_cast<char*>(flat + at), static_cast<std::streamsize>(n * sizeof(double)));
    if (!in) return std::string("checkpoint: truncated payload at ") + t.name;
    at += n;
    ++idx;
  }
  if (idx != got.size()) return "checkpoint: extra tensors in manifest";
  return {};
}

}  // namespace tgb::host
