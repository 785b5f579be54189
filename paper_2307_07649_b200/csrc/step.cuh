// The TGN training sub-step on device (trainer.hpp:170-272) and the root
// memory writes (trainer.hpp:284-330).
#pragma once

#include <vector>

#include "common.cuh"
#include "device_types.cuh"
#include "gemm_simt.cuh"
#include "gemm_tma.cuh"

namespace tgb {

// ModelConfig (model.hpp:19-35) and the canonical flat parameter layout
// (for_each_tensor order, model.hpp:56-76).
struct ModelDims {
  int64_t d_mem = 100, d_time = 100, d_static = 100, d_attn = 100, d_hidden = 0, d_e = 0;
  int64_t n_neighbors = 10, num_nodes = 0;
  double max_t = 1.0;

  int64_t mail_dim() const { return 2 * d_mem + d_time + d_e; }
  int64_t gin() const { return mail_dim() + d_mem; }
  int64_t node_dim() const { return d_mem + d_static; }
  int64_t q_in() const { return node_dim() + d_time; }
  int64_t kv_in() const { return node_dim() + d_e + d_time; }
  int64_t dh() const { return d_hidden ? d_hidden : d_mem; }
};

enum TensorId {
  tOmega = 0, tWz, tWr, tWh, tBz, tBr, tBh, tWq, tBq, tWk, tBk, tWv, tBv, tStatic, tW1, tB1, tW2,
  tB2, tNumTensors
};

struct ParamLayout {
  int64_t off[tNumTensors + 1] = {};
  int64_t rows[tNumTensors] = {}, cols[tNumTensors] = {};
  int64_t total = 0;
  static ParamLayout make(const ModelDims& m);
};

// Pre-split (bf16 hi/lo) GEMM operands of the TMA engine. Layouts (columns):
//  Xg [mail2 | phi | ef | mem | 1], RS [r*s | 1], Qin [s_hat | static | 1..1 | 1],
//  KVin [s_hat | static | ef | cos | 1], Hin [h_u | h_v | 1] -- the trailing 1
//  column carries the bias: forward GEMMs use packed [W | b] weights, and the
//  weight-gradient GEMMs emit db as their last output column.
//  dKV [dK | pad | dV], Dg [da_z | pad | da_r | pad | da_h] (blocks 8-aligned).
//  TMA engine, node / edge split of the attention projections (linearity):
//  NF [s_hat | static | 1] per support, EF [e | cos(dt w) | 1] per pair;
//  Wst = [Wq_n ; Wk_n ; Wv_n] (node columns, row blocks d8a apart) gives the
//  per-support node parts QKVn = NF Wst^T, Wkve = [Wk_e Wk_t bk ; Wv_e Wv_t bv]
//  the per-pair edge parts; dNA [dq | pad | dK | pad | dV] per support.
struct StepBf {
  BfMat Xg, GU, RS, Qin, KVin, Gt, H, Hin, Dhid, dQ, dKV, dNA, Dg, NF, EF;
  BfMat Wzr, Whm, Whs, Wq, Wkv, W1a, W1b, W1, Wst, Wkve;  // Wkv = [Wk | bk ; Wv | bv]
  int d8a = 0, d8d = 0;
};

// Per-trainer activation workspace (capacities fixed at creation).
struct StepWork {
  StepBf bf;
  int cap_B = 0, cap_R = 0, cap_P = 0, cap_U = 0;
  bool fwd_only = false;
  int64_t ldx = 0, ldq = 0, ldkv = 0;
  float *Xg = nullptr, *GU = nullptr, *Gates = nullptr, *RS = nullptr, *s_hat = nullptr;
  float *Qin = nullptr, *KVin = nullptr, *Gt = nullptr, *Q = nullptr, *KV = nullptr;
  float *attn_a = nullptr, *H = nullptr, *AB = nullptr, *HID = nullptr, *Dhid = nullptr;
  float *Hin = nullptr, *dlogit = nullptr, *logits = nullptr, *dIn = nullptr, *dQ = nullptr;
  float *dKV = nullptr, *dNodeAcc = nullptr, *dNode = nullptr, *Dg = nullptr, *T1 = nullptr;
  float *DMT = nullptr, *Mom = nullptr, *omega_part = nullptr, *ones = nullptr;
  float *QKVn = nullptr, *cq = nullptr;
  BfMat xg_alt;  // second GRU-input operand: graph slots alternate (bf.Xg is the current one)
  float* omega_att = nullptr;  // attention part of the omega gradient [d_t]  // node parts [U, 3 d8a]; query constant W_q,t 1 + b_q [d_a]
  double* loss_terms = nullptr;
  float* splitk_ws = nullptr;
  size_t splitk_ws_floats = 0;
  int omega_chunks = 0;
  // root writes (compact rows) live in one packed buffer so they can be
  // exchanged with a single collective: see pack_layout().
  void* wpack = nullptr;
  size_t wpack_bytes = 0;
  int32_t* w_count = nullptr;   // [1]
  int32_t* w_node = nullptr;    // [2 cap_B]
  int32_t* w_event = nullptr;
  double* w_t = nullptr;
  double* w_dt = nullptr;
  float* w_mem = nullptr;       // [2 cap_B, d]
  float* w_mail = nullptr;      // [2 cap_B, 2d]
  int32_t* win = nullptr;       // [N] COMB scratch (0 = empty, else event + 1)
};

// Optional CUDA-event phase markers (bench.py reads per-phase device time).
enum Phase {
  phPlan = 0, phGruFwd, phAttnAssemble, phAttnProj, phAttnSoftmax, phDecoder, phDecoderBwd,
  phAttnBwd, phAttnBwdGemm, phGruBwd, phWrites, phAllreduce, phAdam, phCount
};
// Graph-captured barriers stamp %globaltimer from a one-thread kernel instead
// (event records inside a graph are not timing events).
void stamp_launch(unsigned long long* dst, cudaStream_t s);
struct PhaseMarks {
  bool on = false;
  unsigned long long* d_ts = nullptr;  // set: stamp kernels (graph capture); null: events
  cudaEvent_t ev[phCount + 1] = {};
  bool hit[phCount + 1] = {};
  void mark(int slot, cudaStream_t s) {
    if (on) {
      if (d_ts) stamp_launch(d_ts + slot, s);
      else cudaEventRecord(ev[slot], s);
      hit[slot] = true;
    }
  }
};

struct StepCtx {
  ModelDims m;
  ParamLayout L;
  const DGraph* g = nullptr;
  float* params = nullptr;
  float* grads = nullptr;
  StepWork* w = nullptr;
  int* d_numeric_flag = nullptr;  // set when a non-finite value escapes a kernel
  PhaseMarks* marks = nullptr;
  const int* d_ctr = nullptr;  // graph mode: the loss goes to loss_out[*d_ctr]
  // When set, recorded once the gradient range [off[tWq], end) is final (after
  // the attention / decoder weight gradients and the static-table scatter), so
  // its all-reduce can overlap the rest of the GRU backward.
  cudaEvent_t ev_tail_grads = nullptr;
  // Branch stream (graph mode): the caller zeroes the gradients on it
  // (recording ev_g_zero); substep_rest runs the loss and the W2 / b2
  // gradient there (ev_br_dec -> ev_br_join), off the critical path.
  cudaStream_t br = nullptr;
  bool packed = false;  // the TMA weight operands are current (packed by the fused Adam)
  // the GRU input operand's view-only columns were assembled ahead (on the aux
  // stream, assemble_gru_view_launch): only the time-encoding columns remain
  bool xg_pre = false;
  // graph pipeline: ev_mid is recorded on the main stream at point mid_at (1
  // after the decoder, 2 after the attention backward kernel, 3 after the
  // attention backward GEMMs); the next barrier's read starts after it
  cudaEvent_t ev_mid = nullptr;
  int mid_at = 0;
  // Graph mode: the per-pair edge half of the attention projection was
  // enqueued on another stream (attn_edge_launch); wait for ev_edge first.
  cudaEvent_t ev_edge = nullptr;
  cudaEvent_t ev_g_zero = nullptr, ev_br_dec = nullptr, ev_br_join = nullptr;
  cudaEvent_t ev_red = nullptr;  // split-K reductions of the weight gradients on the branch
  // graph pipeline: the previous barrier's tail-range update (static table,
  // attention, decoder) was deferred; wait for it before the first reader on
  // the main stream (gru_out's static columns of NF)
  cudaEvent_t ev_params_tail = nullptr;
  // the per-pair edge projection GEMM joins the node projection's launch (the
  // edge branch only assembles the operands): see attn_edge_launch
  bool edge_gemm_joined = false;
  void mark(int slot, cudaStream_t s) const {
    if (marks) marks->mark(slot, s);
  }
};

// rpe: roots per event of the plans this workspace serves (3 in training,
// 2 + n_negatives for evaluation); fwd_only skips the backward buffers.
void step_alloc(StepWork& w, const ModelDims& m, int cap_B, int cap_U, int64_t num_nodes, int rpe = 3,
                bool fwd_only = false);
void step_free(StepWork& w);
// The view-dependent columns {mail_mem | . | e(mail event) | s | 1} of the GRU
// input operand xg for a prepared plan and read view (everything but the
// time encoding, which depends on omega and is written in the step).
void assemble_gru_view_launch(const StepCtx& c, const DPlan& pl, const DView& vw, const BfMat& xg,
                              cudaStream_t s);

// Forward + backward of one sub-iteration on (plan, view). Writes the loss to
// *loss_out (device double) and the flat gradient (grads zeroed first).
void substep_launch(const StepCtx& c, const DPlan& pl, const DView& vw, double* loss_out,
                    cudaStream_t s);
// The same split in two: the GRU freshen (s_hat, all the root writes need)
// and everything after it. substep_launch == gru + rest.
void substep_gru_launch(const StepCtx& c, const DPlan& pl, const DView& vw, cudaStream_t s);
void substep_rest_launch(const StepCtx& c, const DPlan& pl, const DView& vw, double* loss_out,
                         cudaStream_t s);
// Forward-only evaluation pieces (evaluate_mrr, trainer.hpp:383-468).
// attention embedding of every root (embed_root + attention_forward) into w.H
void attn_forward_launch(const StepCtx& c, const DPlan& pl, cudaStream_t s);
// TMA engine: the plan-only half of it -- edge operands EF / Gt, the query
// constant and the per-pair edge projection KE = EF Wkve^T (into w.KV).
void attn_edge_launch(const StepCtx& c, const DPlan& pl, cudaStream_t s, bool gemm = true);
// The fused GRU freshen kernel serves this memory width (TGNN_GRU_FUSED, default on).
bool gru_fused_enabled(int64_t d);
// The edge-join schedule (TGNN_EDGE_JOIN, default: with the fused GRU): the
// per-pair edge GEMM is launched together with the node projection instead of
// on the edge branch.
bool edge_join_enabled(int64_t d);
// decode_link of (src, dst) and (src, candidate) per event of an evaluation
// plan (rpe = 2 + n_neg); cnt_out[e - base] = #candidates with logit >= truth.
void eval_rank_launch(const StepCtx& c, const DPlan& pl, int32_t* cnt_out, int64_t base, cudaStream_t s);
// build_root_writes + COMB for the plan's slice into w.w_* (compact rows), or
// straight into `direct` when this trainer is its memory copy's only writer.
void root_writes_launch(const StepCtx& c, const DPlan& pl, const DView& vw, cudaStream_t s,
                        DMem* direct = nullptr);
// Applies compact write rows (one or more row sets, later sets win on equal
// nodes -- ascending-rank application, memory_daemon.hpp:35-38) to the state.
struct WriteSet {
  const int32_t* count;
  const int32_t* node;
  const int32_t* event;
  const double* t;
  const double* dt;
  const float* mem;
  const float* mail;
  int cap;
};
// Op-log record (sub plans of the stint + this rank's write rows) into
// log[(*ctr or b) * 4 .. +4): {R first, R len, W first, W len}.
struct OplogPlans {
  const int32_t* sizes[8];
  const int32_t* supports[8];
  int n = 0;
};
void oplog_record_launch(const StepCtx& c, const OplogPlans& op, int64_t* log, int64_t b, cudaStream_t s);
void apply_writes_launch(const std::vector<WriteSet>& sets, DMem& st, int32_t* win,
                         cudaStream_t s);

// Packed write-row buffer: {count | node[cap] | event[cap] | t[cap] | dt[cap] |
// mem[cap, d] | mail[cap, 2d]}, every segment 16-byte aligned.
size_t pack_bytes(int cap, int64_t d);
WriteSet pack_view(void* base, int cap, int64_t d);
void reset_state_launch(DMem& st, cudaStream_t s);

// Dense Adam over the flat parameters (optimizer.hpp:40-56). Gradients are
// scaled by grad_scale first (1 / active trainers after an all-reduce sum).
void adam_launch(float* params, const float* grads, float* m, float* v, int64_t n, float lr,
                 float c1, float c2, float grad_scale, cudaStream_t s,
                 const BarrierDesc* desc = nullptr, const int* ctr = nullptr);
// Graph mode: Adam with the step scalars of desc[*ctr] that also refreshes the
// packed bf16 hi/lo weight operands of the TMA engine (pack_weights), so the
// next step's GEMMs need no separate pack.
// r_lo / r_hi: the flat parameter range [r_lo, r_hi) this launch updates
// (r_hi < 0: to the end), for the split-phase update of the graph barrier.
void adam_pack_launch(const StepCtx& c, float* m, float* v, cudaStream_t s, const BarrierDesc* desc,
                      const int* ctr, int64_t r_lo = 0, int64_t r_hi = -1);
// Packs the TMA engine's weight operands from the fp32 parameters.
void pack_weights(const StepCtx& c, cudaStream_t s);
// Order-independent 64-bit fingerprint of n floats into *out (device).
void params_hash_launch(const float* p, int64_t n, unsigned long long* out, cudaStream_t s);
// Graph mode helpers: reset the memory copy if desc[*ctr].reset; ++*ctr.
void reset_cond_launch(DMem& st, const BarrierDesc* desc, const int* ctr, cudaStream_t s, int offset = 0);
void incr_launch(int* ctr, cudaStream_t s);

}  // namespace tgb
