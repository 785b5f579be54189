// Device-side finalize (T-CSR build) and the streaming synthetic generator.
//
// finalize (temporal_graph.hpp:55-91) on device:
//   1. ascending-t check; if unsorted, a stable radix sort of (t, index) and a
//      permutation gather of the events and their feature rows;
//   2. validation in sorted order (first failing event, the reference's message);
//   3. T-CSR: 2E (node, 2e + side) pairs radix-sorted by node (stable, so
//      each node's incidence is in ascending event order and a self-loop is
//      listed twice), then gathered into inc_t / inc_eid / inc_nbr, and
//      inc_ptr from the run boundaries of the sorted node keys.
// All of it is integer/f64 data movement: HBM-bound sorts and gathers.
#include <algorithm>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "graph.cuh"

namespace tgb {

namespace {

template <typename T>
T* dmalloc(size_t n) {
  T* p = nullptr;
  TGB_CUDA(cudaMalloc(&p, (n > 0 ? n : 1) * sizeof(T)));
  return p;
}

inline int grid_for(int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 16 * num_sms())));
}

__global__ void unsorted_kernel(const double* __restrict__ t, int64_t E, int* flag) {
  for (int64_t e = blockIdx.x * blockDim.x + threadIdx.x; e + 1 < E; e += gridDim.x * blockDim.x)
    if (t[e + 1] < t[e]) *flag = 1;
}

// keys: t + 0.0 folds -0.0 into +0.0 (equal under the reference's operator<)
__global__ void sort_keys_kernel(const double* __restrict__ t, int64_t E, double* key, int32_t* idx) {
  for (int64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    key[e] = t[e] + 0.0;
    idx[e] = static_cast<int32_t>(e);
  }
}

__global__ void permute_events_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ src,
                                      const int32_t* __restrict__ dst, const double* __restrict__ t, int64_t E,
                                      int32_t* src_o, int32_t* dst_o, double* t_o) {
  for (int64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int64_t o = perm[e];
    src_o[e] = src[o];
    dst_o[e] = dst[o];
    t_o[e] = t[o];
  }
}

// one warp per row, 16-byte vectors (d_pad % 4 == 0)
__global__ void permute_rows_kernel(const int32_t* __restrict__ perm, const float* __restrict__ in, int64_t E,
                                    int64_t d_pad, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t e = warp; e < E; e += nw) {
    const float4* a = reinterpret_cast<const float4*>(in + static_cast<int64_t>(perm[e]) * d_pad);
    float4* b = reinterpret_cast<float4*>(out + e * d_pad);
    for (int64_t x = lane; x < d_pad / 4; x += 32) b[x] = a[x];
  }
}

// first failing event (sorted order); at one event the range check wins
__global__ void validate_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t E,
                                int64_t N, int64_t boundary, unsigned long long* first_bad) {
  for (int64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int64_t s = src[e], d = dst[e];
    unsigned long long code = ~0ull;
    if (s < 0 || s >= N || d < 0 || d >= N) code = static_cast<unsigned long long>(e) << 1;
    else if (boundary >= 0 && !(s < boundary && d >= boundary)) code = (static_cast<unsigned long long>(e) << 1) | 1ull;
    if (code != ~0ull) atomicMin(first_bad, code);
  }
}

__global__ void inc_pairs_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t E,
                                 int32_t* key, int32_t* val) {
  for (int64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    key[2 * e] = src[e];
    val[2 * e] = static_cast<int32_t>(2 * e);
    key[2 * e + 1] = dst[e];
    val[2 * e + 1] = static_cast<int32_t>(2 * e + 1);
  }
}

__global__ void inc_fill_kernel(const int32_t* __restrict__ val, const int32_t* __restrict__ src,
                                const int32_t* __restrict__ dst, const double* __restrict__ t, int64_t M,
                                double* inc_t, int32_t* inc_eid, int32_t* inc_nbr) {
  for (int64_t p = blockIdx.x * blockDim.x + threadIdx.x; p < M; p += gridDim.x * blockDim.x) {
    const int32_t v = val[p];
    const int32_t e = v >> 1;
    inc_eid[p] = e;
    inc_t[p] = t[e];
    inc_nbr[p] = (v & 1) ? src[e] : dst[e];  // listed under src -> neighbour dst, and vice versa
  }
}

// inc_ptr[v] = first position of node v in the sorted keys (M for none after)
__global__ void inc_ptr_kernel(const int32_t* __restrict__ key, int64_t M, int64_t N, int64_t* inc_ptr) {
  for (int64_t p = blockIdx.x * blockDim.x + threadIdx.x; p <= M; p += gridDim.x * blockDim.x) {
    const int64_t prev = p == 0 ? -1 : key[p - 1];
    const int64_t cur = p == M ? N : key[p];
    for (int64_t v = prev + 1; v <= cur; ++v) inc_ptr[v] = p;
  }
}

int radix_bits(int64_t maxval) {
  int b = 1;
  while ((1ll << b) <= maxval) ++b;
  return b;
}

}  // namespace

void graph_finalize_device(DGraph& D, cudaStream_t s) {
  const int64_t E = D.E, N = D.N;
  TGB_REQUIRE(E < (1ll << 30), kConfig, "graph: too many events for int32 incidence ids");
  // 1. stable sort by t when needed
  int* d_flag = dmalloc<int>(1);
  TGB_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
  if (E > 1) unsorted_kernel<<<grid_for(E), 256, 0, s>>>(D.t, E, d_flag);
  int unsorted = 0;
  TGB_CUDA(cudaMemcpyAsync(&unsorted, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  TGB_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_flag);
  if (unsorted) {
    double *key = dmalloc<double>(E), *key_s = dmalloc<double>(E);
    int32_t *idx = dmalloc<int32_t>(E), *perm = dmalloc<int32_t>(E);
    sort_keys_kernel<<<grid_for(E), 256, 0, s>>>(D.t, E, key, idx);
    size_t bytes = 0;
    TGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key_s, idx, perm, E, 0, 64, s));
    void* tmp = nullptr;
    TGB_CUDA(cudaMalloc(&tmp, std::max<size_t>(bytes, 1)));
    TGB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, key, key_s, idx, perm, E, 0, 64, s));
    int32_t *src2 = dmalloc<int32_t>(E), *dst2 = dmalloc<int32_t>(E);
    double* t2 = dmalloc<double>(E);
    permute_events_kernel<<<grid_for(E), 256, 0, s>>>(perm, D.src, D.dst, D.t, E, src2, dst2, t2);
    float* ef2 = nullptr;
    if (D.d_e > 0) {
      ef2 = dmalloc<float>(static_cast<size_t>(E * D.d_e_pad));
      permute_rows_kernel<<<grid_for(E * 32), 256, 0, s>>>(perm, D.efeat, E, D.d_e_pad, ef2);
    }
    TGB_CUDA(cudaGetLastError());
    TGB_CUDA(cudaStreamSynchronize(s));
    cudaFree(D.src);
    cudaFree(D.dst);
    cudaFree(D.t);
    D.src = src2;
    D.dst = dst2;
    D.t = t2;
    if (ef2) {
      cudaFree(D.efeat);
      D.efeat = ef2;
    }
    void* ptrs[] = {key, key_s, idx, perm, tmp};
    for (void* p : ptrs) cudaFree(p);
  }
  // 2. validation (sorted order, temporal_graph.hpp:80-87)
  {
    unsigned long long* d_bad = dmalloc<unsigned long long>(1);
    TGB_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), s));
    if (E > 0) validate_kernel<<<grid_for(E), 256, 0, s>>>(D.src, D.dst, E, N, D.boundary, d_bad);
    unsigned long long bad = 0;
    TGB_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
    TGB_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_bad);
    if (bad != ~0ull) {
      const std::string e = std::to_string(bad >> 1);
      if (bad & 1ull) throw Error(kConfig, "graph: event " + e + " does not cross the bipartite boundary");
      throw Error(kConfig, "graph: node id out of range at event " + e);
    }
  }
  // 3. T-CSR
  const int64_t M = 2 * E;
  D.inc_ptr = dmalloc<int64_t>(static_cast<size_t>(N + 1));
  D.inc_t = dmalloc<double>(static_cast<size_t>(M));
  D.inc_eid = dmalloc<int32_t>(static_cast<size_t>(M));
  D.inc_nbr = dmalloc<int32_t>(static_cast<size_t>(M));
  int32_t *key = dmalloc<int32_t>(M), *key_s = dmalloc<int32_t>(M);
  int32_t *val = dmalloc<int32_t>(M), *val_s = dmalloc<int32_t>(M);
  if (E > 0) inc_pairs_kernel<<<grid_for(E), 256, 0, s>>>(D.src, D.dst, E, key, val);
  const int bits = radix_bits(N);
  size_t bytes = 0;
  TGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key_s, val, val_s, M, 0, bits, s));
  void* tmp = nullptr;
  TGB_CUDA(cudaMalloc(&tmp, std::max<size_t>(bytes, 1)));
  if (M > 0) TGB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, key, key_s, val, val_s, M, 0, bits, s));
  if (M > 0) inc_fill_kernel<<<grid_for(M), 256, 0, s>>>(val_s, D.src, D.dst, D.t, M, D.inc_t, D.inc_eid, D.inc_nbr);
  inc_ptr_kernel<<<grid_for(M + 1), 256, 0, s>>>(key_s, M, N, D.inc_ptr);
  TGB_CUDA(cudaGetLastError());
  TGB_CUDA(cudaStreamSynchronize(s));
  void* ptrs[] = {key, key_s, val, val_s, tmp};
  for (void* p : ptrs) cudaFree(p);
}

// ------------------------------------------------------------ streaming synth
int64_t synth_stream_to_device(const host::SynthConfig& c, DGraph& D, cudaStream_t s, int threads) {
  host::Generator gen(c);
  host::Stream& st = gen.stream();
  const int64_t E = c.events, de = c.d_e, dpad = D.d_e_pad;
  // ~64 MB of features per chunk
  const int64_t chunk = std::max<int64_t>(1024, std::min<int64_t>(E, de > 0 ? (64ll << 20) / (4 * dpad) : (1 << 20)));
  const int64_t nchunks = ceil_div(E, chunk);
  struct Buf {
    int32_t* src = nullptr;
    int32_t* dst = nullptr;
    double* t = nullptr;
    float* ef = nullptr;      // pinned, padded rows
    uint64_t* raw = nullptr;  // chain outputs, 2 per feature
    cudaEvent_t done = nullptr;
    bool pending = false;
  } buf[2];
  for (Buf& b : buf) {
    TGB_CUDA(cudaMallocHost(&b.src, sizeof(int32_t) * chunk));
    TGB_CUDA(cudaMallocHost(&b.dst, sizeof(int32_t) * chunk));
    TGB_CUDA(cudaMallocHost(&b.t, sizeof(double) * chunk));
    if (de > 0) {
      TGB_CUDA(cudaMallocHost(&b.ef, sizeof(float) * chunk * dpad));
      std::fill(b.ef, b.ef + chunk * dpad, 0.0f);
      b.raw = new uint64_t[static_cast<size_t>(chunk * 2 * de)];
    }
    TGB_CUDA(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
  }
  auto release = [&]() {
    for (Buf& b : buf) {
      if (b.done) {
        cudaEventSynchronize(b.done);
        cudaEventDestroy(b.done);
      }
      cudaFreeHost(b.src);
      cudaFreeHost(b.dst);
      cudaFreeHost(b.t);
      if (b.ef) cudaFreeHost(b.ef);
      delete[] b.raw;
    }
  };
  const int T = std::max(1, threads);
  try {
    for (int64_t k = 0; k <= nchunks; ++k) {
      // (a) feature transform of chunk k-1 on worker threads ...
      std::vector<std::thread> pool;
      if (k >= 1 && de > 0) {
        Buf& b = buf[(k - 1) & 1];
        const int64_t n = std::min(chunk, E - (k - 1) * chunk);
        for (int w = 0; w < T; ++w) {
          pool.emplace_back([&b, n, de, dpad, w, T]() {
            for (int64_t e = w; e < n; e += T) {
              const uint64_t* r = b.raw + e * 2 * de;
              float* row = b.ef + e * dpad;
              for (int64_t f = 0; f < de; ++f) row[f] = host::feature_from(r[2 * f], r[2 * f + 1]);
            }
          });
        }
      }
      // (b) ... while this thread walks the sequential chain for chunk k
      if (k < nchunks) {
        Buf& b = buf[k & 1];
        if (b.pending) {
          TGB_CUDA(cudaEventSynchronize(b.done));
          b.pending = false;
        }
        const int64_t e0 = k * chunk, n = std::min(chunk, E - e0);
        for (int64_t x = 0; x < n; ++x) {
          int64_t sv, dv;
          double tv;
          gen.next(sv, dv, tv);
          b.src[x] = static_cast<int32_t>(sv);
          b.dst[x] = static_cast<int32_t>(dv);
          b.t[x] = tv;
          uint64_t* r = b.raw ? b.raw + x * 2 * de : nullptr;
          for (int64_t f = 0; f < 2 * de; ++f) r[f] = st.u64();
        }
      }
      for (auto& th : pool) th.join();
      // (c) upload chunk k-1
      if (k >= 1) {
        Buf& b = buf[(k - 1) & 1];
        const int64_t e0 = (k - 1) * chunk, n = std::min(chunk, E - e0);
        TGB_CUDA(cudaMemcpyAsync(D.src + e0, b.src, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        TGB_CUDA(cudaMemcpyAsync(D.dst + e0, b.dst, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        TGB_CUDA(cudaMemcpyAsync(D.t + e0, b.t, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        if (de > 0)
          TGB_CUDA(cudaMemcpyAsync(D.efeat + e0 * dpad, b.ef, sizeof(float) * n * dpad, cudaMemcpyHostToDevice, s));
        TGB_CUDA(cudaEventRecord(b.done, s));
        b.pending = true;
      }
    }
    TGB_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    release();
    throw;
  }
  release();
  return gen.boundary();
}

}  // namespace tgb
