// Gradient all-reduce over NVLink / NVSwitch peer memory (single node).
//
// Every rank's flat gradient buffer and a receive buffer are mapped into every
// other rank with CUDA IPC. One kernel per bucket does a two-shot all-reduce
// with remote stores only: each rank pushes slice q of its gradient into rank
// q's receive buffer, rank q sums the rows in ascending rank order (the
// reference's average_active_grads order, trainer.hpp:473-483) and pushes the
// reduced slice into every rank's gradient buffer. Phases are separated by
// release/acquire flags in the peers' flag blocks. Every rank ends with
// bitwise the same sums. Spins are bounded: a stuck peer raises the numeric
// flag instead of hanging the GPU.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace tgb {

constexpr int kPeerMax = 8;

struct PeerAR {
  int rank = 0, n = 1;
  float* buf[kPeerMax] = {};         // each rank's gradient buffer (buf[rank] is local)
  float* recv[kPeerMax] = {};        // each rank's receive buffer [n rows x chunk]
  unsigned* flags[kPeerMax] = {};    // each rank's flag block [3 phases x kPeerMax sources]
  unsigned* cnt = nullptr;           // local CTA arrival counters [2]
  int* err = nullptr;                // set on a timed-out wait
};

// All-reduce (sum) of elements [lo, lo + n) of the gradient buffers (lo a
// multiple of 4: 16-byte transfers). The epoch
// of the call is ((*ctr) + 1) * 2 + bucket + 1 (strictly increasing when the
// tail bucket 0 precedes the head bucket 1 in every barrier).
void peer_allreduce_launch(const PeerAR& p, int64_t lo, int64_t n, const int* ctr, int bucket, cudaStream_t s);

}  // namespace tgb
