// See peer.cuh. Push model: remote NVLink stores are fire-and-forget, remote
// loads are latency-bound, so every cross-GPU transfer here is a store.
//   phase 1: rank r stores its slice q of the bucket into rank q's receive
//            buffer row r (for every q);               -> flag "pushed"
//   phase 2: rank q sums its receive rows in ascending rank order (local
//            loads) and stores the reduced chunk into every rank's gradient
//            buffer;                                    -> flag "reduced"
// The final wait (all chunks arrived) also guarantees that every rank has
// finished reading its receive buffer, so the next call may reuse them.
#include <algorithm>

#include "peer.cuh"

namespace tgb {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 waits for every rank's flag of this phase, then the block proceeds
__device__ void wait_phase(const PeerAR& p, int phase, unsigned e) {
  if (threadIdx.x == 0) {
    const unsigned* f = p.flags[p.rank] + phase * kPeerMax;
    for (int q = 0; q < p.n; ++q) {
      long long spins = 0;
      while (ld_acquire_sys(f + q) < e) {
        __nanosleep(32);
        if (++spins > (1ll << 26)) {  // ~ seconds: a peer is gone
          atomicExch(p.err, 1);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// the last CTA of this rank to arrive publishes the phase to every peer
__device__ void arrive_phase(const PeerAR& p, int phase, unsigned e) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(p.cnt + phase, 1u);
    if (old == gridDim.x - 1) {
      p.cnt[phase] = 0;
      __threadfence_system();
      for (int q = 0; q < p.n; ++q) st_release_sys(p.flags[q] + phase * kPeerMax + p.rank, e);
    }
  }
}

__global__ void __launch_bounds__(512) peer_allreduce_kernel(PeerAR p, int64_t lo, int64_t n,
                                                             const int* __restrict__ ctr, int bucket) {
  pdl_wait();
  // no early pdl_trigger: this kernel waits on other GPUs, and dependents
  // launched early would hold SM slots the compute streams need meanwhile
  const unsigned e = static_cast<unsigned>((*ctr + 1) * 2 + bucket + 1);
  // chunks of 4-float multiples; slice q = [lo + q*chunk, min(lo + n, ...))
  const int64_t chunk = ((n + p.n - 1) / p.n + 3) / 4 * 4;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const float* mine = p.buf[p.rank];
  // phase 1: push slice q of this rank's gradient into rank q's receive row
  // `rank` (16-byte stores; lo and chunk are multiples of 4 floats)
  for (int q = 0; q < p.n; ++q) {
    const int64_t a = lo + q * chunk, len = std::max<int64_t>(0, std::min(lo + n, a + chunk) - a);
    float* dst = p.recv[q] + static_cast<int64_t>(p.rank) * chunk;
    const int64_t l4 = len / 4;
    for (int64_t x = tid; x < l4; x += stride)
      reinterpret_cast<float4*>(dst)[x] = reinterpret_cast<const float4*>(mine + a)[x];
    for (int64_t x = 4 * l4 + tid; x < len; x += stride) dst[x] = mine[a + x];
  }
  arrive_phase(p, 0, e);
  wait_phase(p, 0, e);
  // phase 2: reduce this rank's slice over the receive rows (ascending rank
  // order) and push the result into every rank's gradient buffer
  {
    const int64_t a = lo + p.rank * chunk, len = std::max<int64_t>(0, std::min(lo + n, a + chunk) - a);
    const float* rv = p.recv[p.rank];
    const int64_t l4 = len / 4;
    for (int64_t x = tid; x < l4; x += stride) {
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < p.n; ++q) {
        const float4 v = reinterpret_cast<const float4*>(rv + static_cast<int64_t>(q) * chunk)[x];
        s4.x += v.x;
        s4.y += v.y;
        s4.z += v.z;
        s4.w += v.w;
      }
      for (int q = 0; q < p.n; ++q) reinterpret_cast<float4*>(p.buf[q] + a)[x] = s4;
    }
    for (int64_t x = 4 * l4 + tid; x < len; x += stride) {
      float s1 = 0.0f;
      for (int q = 0; q < p.n; ++q) s1 += rv[static_cast<int64_t>(q) * chunk + x];
      for (int q = 0; q < p.n; ++q) p.buf[q][a + x] = s1;
    }
  }
  arrive_phase(p, 1, e);
  wait_phase(p, 1, e);
}

}  // namespace

void peer_allreduce_launch(const PeerAR& p, int64_t lo, int64_t n, const int* ctr, int bucket, cudaStream_t s) {
  if (n <= 0) return;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kSMs, ceil_div(n, 512 * 2))));
  launch_pdl(peer_allreduce_kernel, dim3(blocks), dim3(512), 0, s, p, lo, n, ctr, bucket);
}

}  // namespace tgb
