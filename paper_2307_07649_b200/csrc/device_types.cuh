// Device-resident data structures of the B200 training step.
//
// Layout choices (HBM, per GPU):
//  * events: SoA src/dst (int32) + t (f64). Times stay f64 on device: the
//    strict t_e < t sampler cutoff (temporal_graph.hpp:301-303) and the COMB
//    (t, event) order (memory_store.hpp:121-136) are not representable in f32.
//  * T-CSR: per-node ascending incidence (temporal_graph.hpp:78-90) as
//    inc_ptr[N+1] (int64) + parallel arrays inc_t (f64), inc_eid/inc_nbr (int32).
//  * edge features: fp32 rows padded to a multiple of 4 floats (16 B) so row
//    gathers are 128-bit vectorised.
//  * node memory / mailbox (memory_store.hpp:16-28): memory [N, d] fp32,
//    mail_mem [N, 2d] fp32, mail_t / mail_dt / last_update f64, mail_event int32.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tgb {

struct DGraph {
  int64_t N = 0, boundary = -1, E = 0, d_e = 0, d_e_pad = 0;
  int32_t* src = nullptr;
  int32_t* dst = nullptr;
  double* t = nullptr;
  int64_t* inc_ptr = nullptr;
  double* inc_t = nullptr;
  int32_t* inc_eid = nullptr;
  int32_t* inc_nbr = nullptr;
  float* efeat = nullptr;  // [E, d_e_pad]
};

struct DMem {
  int64_t N = 0, d = 0;
  float* memory = nullptr;     // [N, d]
  float* mail_mem = nullptr;   // [N, 2d]
  double* last_update = nullptr;
  double* mail_t = nullptr;
  double* mail_dt = nullptr;
  int32_t* mail_ev = nullptr;  // -1: no cached mail
  unsigned long long* win = nullptr;  // COMB winner stamps (stamp << 32 | event)
};

// Arguments of one plan (one sub-iteration of one trainer), device-resident so
// the whole step can be replayed as a CUDA graph.
struct PlanArgs {
  int64_t begin = 0, end = 0;      // local slice [begin, end)
  int64_t batch_begin = 0;         // first event of the global batch (negative index base)
  int64_t batch_index = 0;         // stint batch index (sample_negatives batch_index)
  int64_t group = 0;               // negative group
  uint64_t seed = 0;
  int32_t neg_mode = 1;            // 1: sample_negatives on device, 0: use provided,
                                   // 2: evaluate_mrr distractors (rpe - 2 per event)
  int32_t valid = 0;               // 0: empty plan (idle trainer)
};

// Per-barrier parameters of one rank, resident in HBM so a whole barrier can
// be captured once as a CUDA graph and replayed: kernels read the entry of the
// device barrier counter.
struct BarrierDesc {
  PlanArgs args;      // this rank's sub-0 plan (valid = 0 when the rank is idle)
  int32_t reset = 0;  // the group's memory copy resets before this read
  int32_t pad = 0;
  float lr = 0, c1 = 1, c2 = 1, scale = 1;  // Adam step (lr_eff, bias corrections, 1/active)
};

// Per-plan runtime sizes, device-resident.
enum SizeIdx { kSzB = 0, kSzR = 1, kSzP = 2, kSzU = 3, kSzUm = 4, kSzItems = 5, kSz2B = 6, kSzCount = 8 };

struct DPlan {
  int cap_B = 0, n = 0, cap_R = 0, cap_P = 0, cap_U = 0;
  // roots per event: 3 for training (src, dst, negative), 2 + n_negatives for
  // evaluate_mrr candidates, 2 for replay_batch (trainer.hpp:336-468)
  int rpe = 3;
  int routing = 1;               // 0: forward-only plan, no backward routing CSR
  int eval_negs = 0;             // 1: the rpe - 2 negatives are evaluate_mrr distractors
  PlanArgs* args = nullptr;
  int32_t* sizes = nullptr;      // [kSzCount]
  int32_t* negs = nullptr;       // [cap_B * max(rpe - 2, 1)]
  int32_t* root_node = nullptr;  // [cap_R]
  double* root_t = nullptr;      // [cap_R]
  int32_t* nbr_cnt = nullptr;    // [cap_R]
  int32_t* slot_node = nullptr;  // [cap_R * n] padded sampler output
  int32_t* slot_event = nullptr;
  double* slot_dt = nullptr;
  int32_t* pair_ptr = nullptr;   // [cap_R + 1]
  int32_t* pair_node = nullptr;  // [cap_P] compacted (root-major)
  int32_t* pair_event = nullptr;
  int32_t* pair_root = nullptr;
  int32_t* pair_sup = nullptr;
  double* pair_dt = nullptr;
  int32_t* root_sup = nullptr;   // [cap_R]
  int32_t* supports = nullptr;   // [cap_U] ascending node ids
  int32_t* sup_row = nullptr;    // [N] node -> support row (valid for marked nodes)
  // routing CSR: items (roots then pairs) grouped by support row
  int32_t* item_key = nullptr;   // [cap_R + cap_P]
  int32_t* item_val = nullptr;
  int32_t* item_key_s = nullptr;
  int32_t* item_val_s = nullptr;
  int32_t* sup_item_ptr = nullptr;  // [cap_U + 1]
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  int sort_bits = 1;
  uint32_t* bitmap = nullptr;    // [ceil(N / 32)] support marks, cleared by finalize
  // The routing sort only depends on the plan: it runs on a side stream,
  // overlapped with the forward pass; the backward waits on ev_sorted.
  cudaEvent_t ev_pairs = nullptr, ev_sorted = nullptr;
};

// Read view (ReadView, shared_buffers.hpp:118-122) in device form.
struct DView {
  int cap_U = 0;
  float* mem = nullptr;      // [cap_U, d]
  float* mail_mem = nullptr; // [cap_U, 2d]
  double* mail_t = nullptr;
  double* mail_dt = nullptr;
  int32_t* mail_ev = nullptr;
};

}  // namespace tgb
