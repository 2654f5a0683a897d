/* oracle/bapipe_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference explore() path in plain C (gnu11,
 * __int128).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker.  Same SoA input /
 * output records as the product ABI (include/bapipe_b200.h). */
#ifndef BAPIPE_ORACLE_H
#define BAPIPE_ORACLE_H
#include "bapipe_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int bpo_abi_version(void);

/* explore() per query + per-candidate replay (see oracle/ref_driver.cpp for
 * the same contract on the real reference). */
int bpo_explore_batch(const bp_network* nets, int n_nets, const bp_cluster* cls, int n_cls,
                      const bp_query* q, int nq, bp_query_result* res, bp_candidate* cand,
                      bp_stage* stages);

/* inter_layer_partition (partition.hpp:206-212) on the first n_stages
 * accelerators: writes lo/hi per stage and the min-max stage time.
 * Returns 0, or BP_C_REJ_SHAPE when U < N. */
int bpo_partition(const bp_network* net, const bp_cluster* cl, int n_stages, int64_t a_th,
                  int use_coarse, int64_t* lo, int64_t* hi, int64_t* t_opt);

/* simulate_chain (simulator.hpp:81-246) makespan for one ChainInstance.
 * Returns BP_C_OK or BP_C_ERR_OVERFLOW / BP_C_ERR_DOMAIN. */
int bpo_simulate_chain(int kind, int n, const bp_rat* F, const bp_rat* B, const int64_t* SR,
                       const int64_t* a, const bp_rat* w, int64_t M, bp_rat* makespan);

/* Closed forms (cost_models.hpp:50-82). */
int bpo_minibatch_time(int kind, int64_t M, int64_t N, bp_rat F, bp_rat B, bp_rat SR, bp_rat* out);
int bpo_bubble_fraction(int kind, int64_t M, int64_t N, bp_rat F, bp_rat B, bp_rat SR, bp_rat* out);

#ifdef __cplusplus
}
#endif
#endif
