// Dataset files either side of the sampler (ref temporal_graph.hpp:96-274):
// the event CSV ("src,dst,t[,f0,...]"), its ".meta" sidecar, write_dataset
// and chronological_split. Same grammar, error classes and messages as the
// reference; the CSV body is parsed by several threads over line-aligned
// chunks and the earliest failing line is reported.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace tgb::host {

struct DatasetMeta {
  int64_t num_nodes = 0;
  int64_t boundary = -1;
  int64_t d_e = 0;
};

struct EventTable {
  std::vector<int64_t> src, dst;
  std::vector<double> t;
  std::vector<float> efeat;  // [E, d_e] (fp32, the device feature type)
};

std::string sidecar_path(const std::string& csv_path);
DatasetMeta load_sidecar(const std::string& meta_path);
void load_events(const std::string& csv_path, const DatasetMeta& meta, int threads, EventTable& out);
void write_dataset(const std::string& csv_path, int64_t num_nodes, int64_t boundary, int64_t E,
                   const int64_t* src, const int64_t* dst, const double* t, const double* efeat,
                   int64_t d_e);
void chronological_split(int64_t num_events, double train_frac, double val_frac, int64_t* train_end,
                         int64_t* val_end);

}  // namespace tgb::host
