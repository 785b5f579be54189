/*
 * tgnn_b200.h -- C ABI of the B200-native DistTGL training step.
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj/include/tgnn,
 * "ref" below). Every entry point names the reference interface it replaces.
 * POD arguments only, opaque handles, int status + thread-local message:
 *   0 ok, 1 config_error, 2 parse_error, 3 numeric_error, 4 protocol_error,
 *   5 shape_error, 6 CUDA error, 7 NCCL error      (ref common.hpp:16-34, tensor.hpp:16)
 * Threading: one context per host thread and device; all calls on a context
 * are ordered on its CUDA stream; collectives are enqueued on the same stream.
 * Ownership: handles own device memory; host inputs are copied during the
 * call; outputs go to caller-provided buffers.
 */
#ifndef TGNN_B200_H
#define TGNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (ref common.hpp:16-34, tensor.hpp:16). */
enum {
  TGNN_OK = 0,
  TGNN_CONFIG_ERROR = 1,   /* config_error */
  TGNN_PARSE_ERROR = 2,    /* parse_error (a config_error) */
  TGNN_NUMERIC_ERROR = 3,  /* numeric_error */
  TGNN_PROTOCOL_ERROR = 4, /* protocol_error */
  TGNN_SHAPE_ERROR = 5,    /* shape_error */
  TGNN_CUDA_ERROR = 6,
  TGNN_NCCL_ERROR = 7
};

typedef struct tgnn_ctx tgnn_ctx;
typedef struct tgnn_graph tgnn_graph;
typedef struct tgnn_memstore tgnn_memstore;
typedef struct tgnn_trainer tgnn_trainer;
typedef struct tgnn_run tgnn_run;

/* ModelConfig, ref model.hpp:19-35 (d_hidden 0 => d_mem). */
typedef struct tgnn_model_config {
  int64_t d_mem, d_time, d_static, d_attn, d_hidden, d_e, n_neighbors, num_nodes;
  double max_t;
} tgnn_model_config;

/* TrainConfig, ref parallel.hpp:15-26. */
typedef struct tgnn_train_config {
  int32_t i, j, k, p, q;
  int32_t epochs;
  int64_t local_batch;
  double lr_base;
  uint64_t seed;
  int64_t local_batch_ref;
  int64_t neg_groups;
} tgnn_train_config;

/* SynthParams, ref synthetic.hpp:14-25. */
typedef struct tgnn_synth_params {
  int64_t nodes, events;
  double burst_prob, pref_prob;
  int32_t prefs_per_src;
  double src_frac;
  int32_t bipartite;
  int64_t d_e;
  double zipf_s;
  uint64_t seed;
} tgnn_synth_params;

/* ------------------------------------------------------------------ basics */
const char* tgnn_last_error(void);
int tgnn_version(void);
int tgnn_device_count(int* out);
int tgnn_ctx_create(int device, tgnn_ctx** out);
int tgnn_ctx_destroy(tgnn_ctx* ctx);
int tgnn_ctx_synchronize(tgnn_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for event timing by callers. */
int tgnn_ctx_stream(tgnn_ctx* ctx, void** stream_out);

/* ------------------------------------------------------------------ input
 * gen_synthetic (ref synthetic.hpp:54-112), bit-identical host generator.
 * Events come out finalized (time-sorted); efeat is [events x d_e] float32
 * (the reference's f64 values rounded to f32) and may be NULL. */
int tgnn_gen_synthetic(const tgnn_synth_params* p, int64_t* src, int64_t* dst, double* t,
                       float* efeat, int64_t* bipartite_boundary);

/* ------------------------------------------------------------------ graph
 * TemporalGraph + finalize (ref temporal_graph.hpp:33-95): stable sort by t,
 * validate (config_error), build the device T-CSR. efeat float32 [E x d_e]. */
int tgnn_graph_create(tgnn_ctx* ctx, int64_t num_nodes, int64_t bipartite_boundary,
                      int64_t num_events, const int64_t* src, const int64_t* dst,
                      const double* t, const float* efeat, int64_t d_e, tgnn_graph** out);
/* Same, with float64 features (converted on upload). */
int tgnn_graph_create_f64(tgnn_ctx* ctx, int64_t num_nodes, int64_t bipartite_boundary,
                          int64_t num_events, const int64_t* src, const int64_t* dst,
                          const double* t, const double* efeat, int64_t d_e, tgnn_graph** out);
int tgnn_graph_destroy(tgnn_graph* g);
int tgnn_graph_info(tgnn_graph* g, int64_t* num_nodes, int64_t* boundary, int64_t* num_events,
                    int64_t* d_e);
/* Finalized events back to host (parity checks). */
int tgnn_graph_events(tgnn_graph* g, int64_t* src, int64_t* dst, double* t);

/* sample_recent_neighbors (ref temporal_graph.hpp:296-318), batched over
 * (node, time) queries. Outputs [count x n], most recent first; counts[count]. */
int tgnn_sample_recent_neighbors(tgnn_graph* g, const int64_t* nodes, const double* times,
                                 int64_t count, int64_t n, int64_t* nbr_node,
                                 int64_t* nbr_event, double* nbr_dt, int64_t* nbr_count);
/* sample_negatives (ref temporal_graph.hpp:355-370). */
int tgnn_sample_negatives(tgnn_graph* g, int64_t batch_index, int64_t group, int64_t count,
                          uint64_t seed, int64_t* out);
/* plan_sub_batch (ref trainer.hpp:76-106). Roots event-major (src, dst, neg);
 * neighbour arrays [3B x n]; supports (ascending) needs 3B(n+1) slots. */
int tgnn_plan_sub_batch(tgnn_graph* g, int64_t begin, int64_t end, const int64_t* negatives,
                        int64_t n, int64_t* root_node, double* root_t, int64_t* nbr_count,
                        int64_t* nbr_node, int64_t* nbr_event, double* nbr_dt,
                        int64_t* supports, int64_t* num_supports);

/* ------------------------------------------------------------------ memory store
 * NodeMemoryState (ref memory_store.hpp:16-50) resident in HBM, with the
 * MemoryClient read/write semantics (ref shared_buffers.hpp:124-165). Mail
 * rows are packed {mem2 (2 d_mem) | t | dt | event} (ref memory_store.hpp:52-80). */
int tgnn_memstore_create(tgnn_ctx* ctx, int64_t num_nodes, int64_t d_mem, tgnn_memstore** out);
int tgnn_memstore_destroy(tgnn_memstore* m);
int tgnn_memstore_reset(tgnn_memstore* m);                        /* reset_state */
int tgnn_memstore_read(tgnn_memstore* m, const int64_t* nodes, int64_t count, double* mem_rows,
                       double* mail_rows);                         /* MemoryClient::read */
int tgnn_memstore_write(tgnn_memstore* m, const int64_t* nodes, int64_t count,
                        const double* mem_rows, const double* mail_rows); /* ::write */
/* Full state export: memory [N x d], last_update [N], mail_mem [N x 2d],
 * mail_t [N], mail_dt [N], mail_event [N] (any pointer may be NULL). */
int tgnn_memstore_export(tgnn_memstore* m, double* memory, double* last_update, double* mail_mem,
                         double* mail_t, double* mail_dt, int64_t* mail_event);
int tgnn_memstore_import(tgnn_memstore* m, const double* memory, const double* last_update,
                         const double* mail_mem, const double* mail_t, const double* mail_dt,
                         const int64_t* mail_event);

/* ------------------------------------------------------------------ trainer core
 * TrainerCore (ref trainer.hpp:490-562): parameter replica, gradients and
 * Adam state in HBM, plus the step workspace. max_local_batch bounds the
 * slice length. */
int tgnn_param_count(const tgnn_model_config* m, int64_t* out);   /* param_count */
/* init_params (ref model.hpp:122-141), bit-identical, canonical flat order. */
int tgnn_init_params(const tgnn_model_config* m, uint64_t seed, double* flat);
int tgnn_trainer_create(tgnn_ctx* ctx, tgnn_graph* g, const tgnn_model_config* m,
                        int64_t max_local_batch, uint64_t seed, tgnn_trainer** out);
int tgnn_trainer_destroy(tgnn_trainer* tr);
int tgnn_trainer_set_params(tgnn_trainer* tr, const double* flat);
int tgnn_trainer_get_params(tgnn_trainer* tr, double* flat);
int tgnn_trainer_get_grads(tgnn_trainer* tr, double* flat);
/* sub_step (ref trainer.hpp:170-272) on an injected read view aligned with
 * plan_sub_batch(begin, end, negatives).supports. Gradients are zeroed, then
 * filled; s_hat_out [U x d_mem] may be NULL. */
int tgnn_trainer_sub_step(tgnn_trainer* tr, int64_t begin, int64_t end,
                          const int64_t* negatives, const double* view_mem,
                          const double* view_mail, double* loss_out, double* s_hat_out);
/* build_root_writes (ref trainer.hpp:284-330) for the last sub_step; rows in
 * ascending node order; arrays sized 2B. */
int tgnn_trainer_root_writes(tgnn_trainer* tr, int64_t* nodes, double* mem_rows,
                             double* mail_rows, int64_t* num_writes);
/* Adam::step (ref optimizer.hpp:40-56) with the trainer's current gradients. */
int tgnn_trainer_adam_step(tgnn_trainer* tr, double lr);
/* One full (1,1,1) barrier against a memory store: plan (device negatives),
 * read, sub_step, root writes, Adam -- TrainerCore::iterate + apply. */
int tgnn_trainer_iterate(tgnn_trainer* tr, tgnn_memstore* m, int64_t batch_index,
                         int64_t group, int64_t batch_begin, int64_t begin, int64_t end,
                         double lr, double* loss_out);

/* ------------------------------------------------------------------ runs
 * run_training / run_sequential (ref trainer.hpp:630-867) for one rank of an
 * i x j x k job. With nranks == 1 the whole job runs here; otherwise call
 * tgnn_run_comm_init first (one process per GPU). */
typedef struct tgnn_run_options {
  tgnn_model_config model;
  tgnn_train_config train;
  int64_t train_begin, train_end;
  int32_t rank, nranks;
  int32_t use_graphs; /* capture barrier steps as CUDA graphs */
  /* RunOptions validation (ref trainer.hpp:572-588): an empty [val_begin,
   * val_end) disables MRR evaluation; eval_batch 0 = train.local_batch. */
  int64_t val_begin, val_end;
  int32_t eval_negatives, pad0;
  int64_t eval_batch;
  /* record the daemon op-log of this rank's reads and writes (ref
   * memory_daemon.hpp:73,90, oplog.hpp:15-45); read with tgnn_run_oplog */
  int32_t oplog;
  /* RunOptions.segment_snapshots (ref trainer.hpp:581, parallel.hpp:288-290):
   * copy this rank's memory replica (memory + last_update) after the write
   * bracket of every pair that ends a segment (DaemonOp::Snapshot,
   * memory_daemon.hpp:94-105); read with tgnn_run_snapshots. An oracle
   * feature: the run uses the direct (uncaptured) barrier path. */
  int32_t segment_snapshots;
} tgnn_run_options;

/* build_assignment + Assignment::task (ref parallel.hpp:150-331), host only.
 * For barriers [first, first+count) of `rank`, out[count x 12] holds:
 * active, sub, subs, batch, batch_begin, batch_end, slice_begin, slice_end,
 * neg_group(sub), reset_before(stint read), active_trainers(b), traversed_after(b). */
int tgnn_schedule_query(const tgnn_train_config* tc, int64_t train_begin, int64_t train_end,
                        int32_t rank, int64_t first, int64_t count, int64_t* out,
                        int64_t* barriers_out);

int tgnn_comm_unique_id(char* out128);
int tgnn_run_create(tgnn_ctx* ctx, tgnn_graph* g, const tgnn_run_options* opt, tgnn_run** out);
/* One process per GPU: NCCL communicator over all ranks (+ ncclCommSplit per
 * memory group), from a unique id every rank received out of band. */
int tgnn_run_comm_init(tgnn_run* r, const char* unique_id128);
/* In-process alternative (the reference's threading model: run_training's
 * trainer threads share host arrays, trainer.hpp:671-674): the ranks are host
 * threads of one process, on one device or several. Each rank's thread
 * attaches its run to one shared hub; every collective then becomes a host
 * rendezvous plus cross-stream events and an ascending-rank device reduction
 * (the reference's summation order). Barriers run on the direct path (no
 * CUDA-graph capture). Destroy the hub after every attached run. */
typedef struct tgnn_local_hub tgnn_local_hub;
int tgnn_local_hub_create(int32_t nranks, tgnn_local_hub** out);
int tgnn_local_hub_destroy(tgnn_local_hub* hub);
int tgnn_run_local_init(tgnn_run* r, tgnn_local_hub* hub);
int tgnn_run_destroy(tgnn_run* r);
int tgnn_run_info(tgnn_run* r, int64_t* barriers, int64_t* param_count);
/* Enqueue barriers [first, first + count) on the context stream (no host sync). */
int tgnn_run_barriers(tgnn_run* r, int64_t first, int64_t count);
/* Sync, check numeric flag, copy barrier losses [first, first+count) (mean
 * over active trainers, ref trainer.hpp:713-722; valid on every rank). */
int tgnn_run_losses(tgnn_run* r, int64_t first, int64_t count, double* out);
int tgnn_run_params(tgnn_run* r, double* flat);
/* Enqueue (no sync) the D2H copy of this rank's loss of barrier b into dst
 * (pinned host memory) on the context's read-back stream, after the barrier's
 * loss is written; valid after the next tgnn_ctx_synchronize. */
int tgnn_run_loss_async(tgnn_run* r, int64_t b, double* dst);
/* MetricsRow list (ref trainer.hpp:562-570, one row per eval barrier reached
 * so far, rank 0 evaluates with its device weights as run_training does,
 * trainer.hpp:725-743). rows[count x 5] = iter, traversed, loss (mean barrier
 * loss since the previous row), val_mrr, elapsed_s. Collective when nranks > 1
 * (the loss means need every rank's slot); rows == NULL returns the count only. */
int tgnn_run_metrics(tgnn_run* r, int64_t* count, double* rows);
/* This rank's op-log records so far, rows[count x 6] = epoch (sweep), iter
 * (pair), kind (0 = 'R', 1 = 'W'), rank within the memory copy, first, len
 * (ref OpRecord, oplog.hpp:15-24). A memory copy's op-log is the union of its
 * ranks' rows ordered by (iter, kind, rank). rows == NULL returns the count. */
int tgnn_run_oplog(tgnn_run* r, int64_t* count, int64_t* rows);
/* RunResult.snapshots of this rank's memory copy (ref trainer.hpp:593,
 * MemorySnapshot memory_daemon.hpp:12-17), in plan order: meta[count x 2] =
 * sweep, segment; memory[count x N x d_mem]; last_update[count x N]. Any
 * output may be NULL; count receives the number of snapshots taken so far. */
int tgnn_run_snapshots(tgnn_run* r, int64_t* count, int64_t* meta, double* memory, double* last_update);
/* Replica invariant (ref SPEC.md:397): collective over all ranks; fails with
 * TGNN_PROTOCOL_ERROR if any rank's parameters differ bitwise; hash_out receives the
 * order-independent 64-bit parameter fingerprint. Also checked automatically at
 * every eval point of a multi-rank run. */
int tgnn_run_check_replicas(tgnn_run* r, uint64_t* hash_out);
/* evaluate_mrr of the run's current weights (rank-local, no collective). */
int tgnn_run_evaluate_mrr(tgnn_run* r, int64_t eval_begin, int64_t eval_end, int64_t batch_size,
                          int32_t n_negatives, uint64_t seed, double* mrr, int64_t* queries);
/* Assignment::eval_barriers (ref parallel.hpp:316-329): the barriers after
 * which run_training records a metrics row (one per epoch-equivalent of
 * traversed events, plus the last barrier). out may be NULL (count only). */
int tgnn_run_eval_barriers(tgnn_run* r, int64_t* count, int64_t* out);
/* Events traversed by ALL ranks in barriers [first, first+count) (ref parallel.hpp:302-314). */
int tgnn_run_traversed(tgnn_run* r, int64_t first, int64_t count, int64_t* out);
/* Kernel launches issued per barrier by this rank (counted by capturing the
 * next barrier's enqueue sequence into a CUDA graph; nothing is executed). */
int tgnn_run_launches_per_barrier(tgnn_run* r, int64_t* out);
/* Runs the next barrier with CUDA-event phase markers and returns per-phase
 * device milliseconds [TGNN_PHASES] (plan, gru_fwd, attn_assemble, attn_proj,
 * attn_softmax, decoder, decoder_bwd, attn_bwd, attn_bwd_gemm, gru_bwd,
 * writes, allreduce, adam) and the plan sizes [8] (B, R, P, U, -, items, 2B, W).
 * direct != 0: the single-stream path (each phase alone); 0: the production
 * CUDA-graph schedule (markers on the critical-path stream). */
#define TGNN_PHASES 13
int tgnn_run_profile_barrier(tgnn_run* r, double* phase_ms, int32_t* sizes, int32_t direct);
/* Runs the next barrier on the direct path with every tcgen05 GEMM launch
 * bracketed by CUDA events (the kernel roofline of bench.py). rows[cap x 6]
 * per launch, in launch order: device ms, algorithmic FLOPs (sum of 2 M N K
 * over the launch's problems at their runtime row counts), algorithmic bytes
 * (bf16 hi/lo operands 4 B per element in, fp32 out), problems, largest M,
 * largest split count. *count receives the number of launches. */
int tgnn_run_gemm_profile(tgnn_run* r, int64_t cap, int64_t* count, double* rows);

/* ------------------------------------------------------------------ GEMM engine
 * Process-wide choice for the step's dense contractions:
 *   1 (default) tcgen05 tensor cores, bf16x3 split (hi*hi + hi*lo + lo*hi,
 *     fp32 accumulate in TMEM), operands pre-split by their producers and
 *     loaded by TMA -- fp32-class accuracy;
 *   0 fp32 FMA on CUDA cores -- the exact fp32 path;
 *   2 tcgen05 bf16x3 that gathers and splits fp32 operands inside the GEMM. */
int tgnn_set_gemm_impl(int impl);
int tgnn_get_gemm_impl(int* impl);
/* Test hook: C[M x N] = A . B on device with the chosen engine. A is [M x K]
 * (a_trans = 0) or stored [K x M] (a_trans = 1); B is [K x N] (b_trans = 0) or
 * stored [N x K] (b_trans = 1); all row-major float32 host buffers. splits > 1
 * exercises the split-K path. */
int tgnn_debug_gemm(int impl, int64_t M, int64_t N, int64_t K, const float* A, int a_trans,
                    const float* B, int b_trans, float* C, int splits);

/* ------------------------------------------------------------------ host I/O
 * Streaming ingestion of events [first, first+count) from host buffers: the
 * edge features (float32 [count x d_e]) overwrite the device rows; src / dst /
 * t are uploaded and verified bitwise against the finalized (T-CSR indexed)
 * events -- they are never rewritten, and a mismatch fails the next
 * synchronising call with TGNN_PROTOCOL_ERROR. Used to stream feature windows and
 * by the end-to-end measurement. Pinned buffers make the copies asynchronous:
 * they run on the context's copy stream, overlap work enqueued before the call
 * and are ordered before any work enqueued after it. Ordering contract: in
 * CUDA-graph runs barrier b plans barrier b + 1 (reads its events) while b
 * runs, so the rows of barrier b + 1 must be ingested BEFORE the
 * tgnn_run_barriers call that runs barrier b. */
int tgnn_graph_ingest(tgnn_graph* g, int64_t first, int64_t count, const int32_t* src,
                      const int32_t* dst, const double* t, const float* efeat);
/* Debug: timing (us per launch) of the tcgen05 engine on an M x N x K
 * K-major problem; trace (nullable) receives 16 globaltimer stamps per CTA for
 * up to 296 CTAs: entry, setup done, first TMA landed (MMA), last MMA issued,
 * epilogue start, epilogue end, exit, first TMA issued. */
int tgnn_debug_gemm_bench(int64_t M, int64_t N, int64_t K, int32_t ntile, int32_t iters, double* us,
                          uint64_t* trace, int32_t* grid);
/* Debug: per-CTA globaltimer timeline of the fused GRU kernel. out == NULL
 * arms it for up to cap_ctas CTAs; otherwise synchronises, copies [cap x 16]
 * stamps (entry, after the dependency wait, producer done, MMA done, GEMM2
 * operands ready, epilogue start, epilogue mid, GEMM2 seen, epilogue end,
 * CTA sync, exit) and disarms. */
int tgnn_debug_gru_trace(uint64_t* out, int32_t cap_ctas, int32_t* n_ctas);
int tgnn_pinned_alloc(int64_t bytes, void** out);
int tgnn_pinned_free(void* p);


/* ---- validation path: evaluate_mrr + replay_batch (ref trainer.hpp:336-468) */
typedef struct tgnn_evaluator tgnn_evaluator;
/* Forward-only workspaces for batches of up to batch_size events with
 * n_negatives distractors per event, plus a private node-memory copy. */
int tgnn_evaluator_create(tgnn_ctx* ctx, tgnn_graph* g, const tgnn_model_config* m, int64_t batch_size,
                          int32_t n_negatives, tgnn_evaluator** out);
int tgnn_evaluator_destroy(tgnn_evaluator* ev);
/* Replaces evaluate_mrr(g, p, eval_begin, eval_end, batch_size, n_negatives, seed)
 * (ref trainer.hpp:383-468): memory rebuilt from scratch by replaying
 * [0, eval_begin), then every event ranks its destination against the
 * distractors; params = flat f64 weights in canonical order. */
int tgnn_evaluate_mrr(tgnn_evaluator* ev, const double* params, int64_t eval_begin, int64_t eval_end,
                      uint64_t seed, double* mrr, int64_t* queries);
/* Replaces replay_batch(g, p, state, begin, end) (ref trainer.hpp:336-371) on a
 * memstore; end - begin <= batch_size. params NULL keeps the loaded weights. */
int tgnn_replay_batch(tgnn_evaluator* ev, tgnn_memstore* state, const double* params, int64_t begin,
                      int64_t end);
/* The distractors evaluate_mrr draws for events [begin, end) (ref
 * trainer.hpp:413-423): out[(end - begin) x n_negatives]; end - begin <= batch_size. */
int tgnn_eval_candidates(tgnn_evaluator* ev, int64_t begin, int64_t end, uint64_t seed, int64_t* out);


/* ---- artifacts: model.ckpt (ref model.hpp:168-222), byte-compatible with
 * save_checkpoint / load_checkpoint; flat = f64 weights in canonical order.
 * Load refuses a manifest that does not match the config (TGNN_CONFIG_ERROR). */
int tgnn_checkpoint_save(const tgnn_model_config* m, const double* flat, const char* path);
int tgnn_checkpoint_load(const tgnn_model_config* m, const char* path, double* flat);


/* ---- input pipeline (ref temporal_graph.hpp:96-274, synthetic.hpp:54-112) */
/* gen_synthetic streamed straight into a device graph: bit-identical events
 * and fp32 features, generated chunk by chunk (sequential chain on the calling
 * thread, feature transform on `threads` workers, overlapped H2D copies), then
 * the device finalize. Host memory stays O(chunk) at GDELT scale. */
int tgnn_graph_synthetic(tgnn_ctx* ctx, const tgnn_synth_params* p, int32_t threads, tgnn_graph** out);
/* load_dataset (ref temporal_graph.hpp:136-258): the event CSV plus its
 * ".meta" sidecar, parsed by `threads` workers; the reference's grammar and
 * errors (TGNN_PARSE_ERROR for malformed input, TGNN_CONFIG_ERROR for missing files). */
int tgnn_graph_load_dataset(tgnn_ctx* ctx, const char* csv_path, int32_t threads, tgnn_graph** out);
/* write_dataset (ref temporal_graph.hpp:237-262): CSV + sidecar, %.17g numbers. */
int tgnn_write_dataset(const char* csv_path, int64_t num_nodes, int64_t bipartite_boundary, int64_t num_events,
                       const int64_t* src, const int64_t* dst, const double* t, const double* efeat, int64_t d_e);
/* TemporalGraph::edge_feat rows [first, first+count) as fp32 (ref temporal_graph.hpp:46-48). */
int tgnn_graph_edge_feats(tgnn_graph* g, int64_t first, int64_t count, float* out);
/* chronological_split (ref temporal_graph.hpp:264-279): event-index quantiles. */
int tgnn_chronological_split(int64_t num_events, double train_frac, double val_frac, int64_t* train_end,
                             int64_t* val_end);

#ifdef __cplusplus
}
#endif

#endif /* TGNN_B200_H */
