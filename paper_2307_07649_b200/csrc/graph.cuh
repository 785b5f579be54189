// Device-side TemporalGraph::finalize (temporal_graph.hpp:55-91) and the
// streaming synthetic input pipeline (synthetic.hpp:54-112) at GDELT scale.
#pragma once

#include <string>

#include "common.cuh"
#include "device_types.cuh"
#include "host/synth.hpp"

namespace tgb {

// D.src / D.dst / D.t (E events, any order) and D.efeat (E padded rows) are
// filled. Stable-sorts events by t when they are not already ascending
// (permuting the feature rows along), validates node ranges and the bipartite
// boundary in sorted order (the reference's first failing event and message),
// and builds the T-CSR: inc_ptr / inc_t / inc_eid / inc_nbr, each event listed
// under src then dst in ascending event order. Allocates the inc_* arrays.
void graph_finalize_device(DGraph& D, cudaStream_t s);

// Generates the gen_synthetic stream (bit-identical to the reference) straight
// into D's device arrays chunk by chunk: the sequential splitmix chain runs on
// the calling thread, the Box-Muller feature transform on worker threads, the
// host->device copies from pinned double buffers overlap both. Host memory is
// O(chunk); D.src/dst/t/efeat must be allocated for c.events events.
// Returns the bipartite boundary (-1 when not bipartite).
int64_t synth_stream_to_device(const host::SynthConfig& c, DGraph& D, cudaStream_t s, int threads);

}  // namespace tgb
