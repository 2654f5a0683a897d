// kernels.h -- launchers for the explore() pipeline kernels.
#pragma once
#include <cuda_runtime.h>

#include "batch.cuh"

namespace bpk {

// K1 cost_prefix: per network, prefix sums of fp, bp, fp+bp per type and of w.
void launch_cost_prefix(const NetDesc* nets, int n_nets, const int64_t* fp, const int64_t* bp, const int64_t* w,
                        int64_t* Pfp, int64_t* Pbp, int64_t* Pc, int64_t* Pw, cudaStream_t st, int max_T);
void launch_setup(const BatchDev& B, cudaStream_t st);
void launch_sched(const BatchDev& B, cudaStream_t st);
size_t sched_temp_bytes(int nq);
void launch_partition(const BatchDev& B, int which, int grid, int max_units, int max_N, int T_slots,
                      cudaStream_t st);
size_t partition_smem_bytes(int max_units, int max_N, int T_slots);
void launch_bottleneck(const BatchDev& B, cudaStream_t st);
void launch_dedup(const BatchDev& B, cudaStream_t st);
void launch_coarse_copy(const BatchDev& B, cudaStream_t st);
void launch_dedup_copy_dp(const BatchDev& B, cudaStream_t st);
void launch_dedup_copy_refine(const BatchDev& B, cudaStream_t st);
void launch_refine_list(const BatchDev& B, int fast_grid, cudaStream_t st);
void launch_refine(const BatchDev& B, int sms, int fast_grid, int fast_warps, size_t fast_bytes, int max_L, int max_T,
                   cudaStream_t st);
int refine_setup(int max_N, int max_L, int max_T, size_t* fast_bytes, int* fast_warps);
cudaError_t kernel_attributes_init(int optin_bytes);
cudaError_t partition_attributes_init(int optin_bytes);
size_t refine_region_bytes(int max_N);
// part: bit 0 = keys + work list, bit 1 = representatives, bit 2 = members (copy
// the shared estimate, or list), bit 3 = the listed members
void launch_prune(const BatchDev& B, int pass, cudaStream_t st, int part = 15);
void launch_prune_reset(const BatchDev& B, cudaStream_t st);
void launch_sim_prep(const BatchDev& B, cudaStream_t st);
void launch_lb_bound(const BatchDev& B, cudaStream_t st);
void launch_lb_round1(const BatchDev& B, cudaStream_t st);
void launch_lb_round2(const BatchDev& B, cudaStream_t st);
void launch_lb_finish(const BatchDev& B, cudaStream_t st);
void launch_sim_share(const BatchDev& B, cudaStream_t st);
void launch_sim_fast(const BatchDev& B, int cls, int sms, cudaStream_t st);
void launch_sim_exact(const BatchDev& B, int sms, cudaStream_t st);
void launch_sim_flow(const BatchDev& B, int k, int sms, cudaStream_t st);
size_t sim_exact_state_bytes(int sms, int max_N);
void launch_rank(const BatchDev& B, cudaStream_t st);
void launch_plan_finish(const BatchDev& B, cudaStream_t st);
// one caller-given plan (timeline.cu)
cudaError_t timeline_simulate(const Pools& P, int clusterN, const bp_plan_request& q, bp_timeline_result* res,
                              bp_event* events, int64_t cap, bp_rat* highwater, bp_rat* wstatic, bp_rat* busy,
                              int64_t* h2d, int64_t* d2h);
cudaError_t timeline_estimate(const Pools& P, int clusterN, const bp_plan_request& q, bp_estimate_result* res,
                              bp_stage* stages, int32_t* infeasible, int64_t* h2d, int64_t* d2h);
void refine_trace_collect();
void launch_scatter_results(const bp_query_result* src, int n, const int64_t* ids, bp_query_result* dst,
                            cudaStream_t st);
void launch_scatter_records(const BatchDev& P, const int64_t* woff, bp_candidate* cand, bp_stage* st,
                            cudaStream_t s);   // diagnostics: BP_REFINE_TRACE (kernels.cu)
void launch_best_merge(const bp_best_record* recs, int n, bp_best_record* out, cudaStream_t st);
void launch_best(const BatchDev& B, bp_best_record* out, int64_t query_base, const int64_t* query_ids,
                 cudaStream_t st);

}  // namespace bpk
