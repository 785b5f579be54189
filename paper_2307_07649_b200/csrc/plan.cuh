// Sampler / planning launchers (see plan.cu).
#pragma once

#include "common.cuh"
#include "device_types.cuh"

namespace tgb {

size_t plan_sort_tmp_bytes(int cap_items, int bits);
// negatives -> sampler -> support dedup -> pair compaction -> routing CSR
void plan_launch(const DGraph& g, DPlan& pl, cudaStream_t s, cudaStream_t side = nullptr);
void negatives_only_launch(const DGraph& g, const PlanArgs* args, int count, int32_t* negs,
                           cudaStream_t s);
void set_plan_args_launch(PlanArgs* dst, const PlanArgs& a, cudaStream_t s);
// Graph mode: the plan args of barrier *ctr from the descriptor table.
// (offset 1: the next barrier's plan, prepared one barrier ahead)
void select_plan_args_launch(PlanArgs* dst, const BarrierDesc* desc, const int* ctr, cudaStream_t s,
                             int offset = 0);
// Batched sample_recent_neighbors over arbitrary (node, time) queries.
void sample_queries_launch(const DGraph& g, const int32_t* nodes, const double* times, int count,
                           int n, int32_t* nbr_node, int32_t* nbr_event, double* nbr_dt,
                           int32_t* nbr_count, cudaStream_t s);
void gather_view_launch(const DPlan& pl, const DMem& st, DView& vw, cudaStream_t s);

}  // namespace tgb
