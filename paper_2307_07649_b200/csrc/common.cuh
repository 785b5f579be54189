// Shared device/host helpers for the B200 DistTGL training step.
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace tgb {

// Status codes of the C ABI (include/tgnn_b200.h); they map 1:1 onto the
// reference exception taxonomy (common.hpp:16-34, tensor.hpp:16).
enum Status : int {
  kOk = 0,
  kConfig = 1,
  kParse = 2,
  kNumeric = 3,
  kProtocol = 4,
  kShape = 5,
  kCuda = 6,
  kNccl = 7,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TGB_CUDA(x)                                                                     \
  do {                                                                                  \
    cudaError_t e__ = (x);                                                              \
    if (e__ != cudaSuccess)                                                             \
      throw ::tgb::Error(::tgb::kCuda, std::string(#x) + ": " + cudaGetErrorString(e__)); \
  } while (0)

#define TGB_REQUIRE(cond, code, msg)                     \
  do {                                                   \
    if (!(cond)) throw ::tgb::Error((code), (msg));      \
  } while (0)

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

// rng.hpp:12-17
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// One fold step of rng.hpp:21-24: hash64(a, b, rest...) = hash64(fold(a, b), rest...).
__host__ __device__ __forceinline__ uint64_t hash_fold(uint64_t a, uint64_t b) {
  return splitmix64(a ^ (b + kGamma + (a << 6) + (a >> 2)));
}

__host__ __device__ __forceinline__ uint64_t hash64_5(uint64_t a, uint64_t b, uint64_t c,
                                                       uint64_t d, uint64_t e) {
  return splitmix64(hash_fold(hash_fold(hash_fold(hash_fold(a, b), c), d), e));
}

// First draw of Rng(seed) (rng.hpp:30-35).
__host__ __device__ __forceinline__ uint64_t rng_first_u64(uint64_t seed) {
  return splitmix64(splitmix64(seed ^ 0xa02bdbf7bb3c0a7ull));
}

constexpr uint64_t kTagNegatives = 0x6e656761ull;  // "nega", temporal_graph.hpp:365
constexpr uint64_t kTagEval = 0x6576616cull;       // "eval", trainer.hpp:417

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#ifdef __CUDACC__
// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl
// may start while its stream predecessor drains; pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible, pdl_trigger()
// lets the successor's CTAs be scheduled early. Every hot-path kernel calls
// both first thing, so reading a predecessor's output is always safe.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }
// sigma'(a) = sigma(a) sigma(-a) and tanh'(a) = 1 - tanh(a)^2, from the
// pre-activation: z (1 - z) from a rounded z loses every digit of 1 - z once
// the gate saturates (z = 1 - 1e-5 in fp32 leaves 1 - z with 6e-3 relative
// error), while e^-|a| keeps the derivative to fp32 precision.
__device__ __forceinline__ float dsigmoidf_(float a) {
  const float e = expf(-fabsf(a));
  const float d = 1.0f + e;
  return e / (d * d);
}
__device__ __forceinline__ float dtanhf_(float a) {
  const float e = expf(-2.0f * fabsf(a));
  const float d = 1.0f + e;
  return 4.0f * e / (d * d);
}

#endif  // __CUDACC__

// SM count of the current device (cudaDevAttrMultiProcessorCount; 148 on
// B200), cached per device: every grid size, split-K policy and CTA budget
// scales with it.
inline int num_sms() {
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  int& c = cache[dev & 63];
  if (c == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    c = v;
  }
  return c;
}

// Validated integer knob from the environment (A/B switches): the default
// unless the variable parses completely as an integer in [lo, hi].
inline int env_knob(const char* name, int def, int lo, int hi) {
  const char* e = std::getenv(name);
  if (!e || !*e) return def;
  char* end = nullptr;
  const long v = std::strtol(e, &end, 10);
  if (end == e || *end != '\0' || v < lo || v > hi) return def;
  return static_cast<int>(v);
}

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  // carry the stream's priority into the launch (and into captured graph
  // nodes): the critical path outranks the overlapped branches for SMs
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = prio;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  TGB_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}
#endif

}  // namespace tgb
