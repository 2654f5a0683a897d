// xwave.cu -- K4x: exact (Rat) dataflow simulation for the heavy exact
// candidates (simulator.hpp:81-246).
//
// The thread-per-candidate exact kernel (sim.cu k_sim_exact) is throughput-
// efficient, but its latency is one thread's serial walk over 2NM(+2(N-1)M)
// events with per-stage state in global memory, and after the batch dedup the
// candidates with N = 64, M = 128 set the kernel time.  Here a thread block
// owns one candidate and thread s runs stage s: it walks the stage's own op
// sequence (F or B at every position p = 0..2M-1, fixed by its warm-up depth,
// simulator.hpp:87-100) and exchanges arrivals with its neighbours through
// shared-memory FIFOs (F outputs flow s -> s+1, B outputs s+1 -> s, both in
// micro-batch order).  The block advances in rounds: in each round every
// stage whose next op has its arrival (and room for its output) runs it.  The
// number of rounds is the depth of the op DAG -- about 2M + 2N -- instead of
// the event count, and no same-position chain is resolved serially.
//
// Exactness: every thread performs the reference's own Rat operations on the
// same operands -- end = max(free, arrival) + F (or + B), and in sync mode the
// arrival end + SR -- so a candidate overflows here iff it does in the
// reference; overflow is the only error a simulation can raise, so the order
// in which the (independent) stages evaluate does not change the status.
#include "kernels.h"
#include "phases.cuh"

namespace bpk {

namespace {

// FIFO slots per link and direction.  A producer runs at most a few ops ahead
// of its consumer (their warm-up depths differ by 1 or 2), and a full FIFO
// only makes it wait a round; 4 slots halve the shared memory of 8 and let
// twice as many candidates share an SM.
constexpr int FLOW_Q = 4;

// Block-wide sync and OR-reduction of per-thread flags.  One warp (NT = 32):
// a warp reduction, no barrier.  Two warps: each warp reduces its flags
// (REDUX) and lane 0 stores the warp's word; one barrier per round; the words
// rotate over three rounds so that a fast warp's next store never races with
// a slow reader of the previous round.
template <int NT>
__device__ __forceinline__ void flow_sync() {
    if constexpr (NT == 32) __syncwarp();
    else __syncthreads();
}
template <int NT>
__device__ __forceinline__ unsigned flow_or(unsigned f, unsigned* red, int round) {
    const unsigned w = __reduce_or_sync(0xffffffffu, f);
    if constexpr (NT == 32) {
        return w;
    } else {
        unsigned* slot = red + 2 * (round % 3);
        if ((threadIdx.x & 31) == 0) slot[threadIdx.x >> 5] = w;
        __syncthreads();
        return slot[0] | slot[1];
    }
}

template <int NT>
struct FlowSmem {
    Rat qF[NT][FLOW_Q];     // qF[s]: arrivals into stage s from s-1
    Rat qB[NT][FLOW_Q];     // qB[s]: arrivals into stage s from s+1
    int prodF[NT], consF[NT];
    int prodB[NT], consB[NT];
    Rat fr[NT];
    unsigned red[6];        // flow_or: two warp words per round, three rounds
    int next;               // the block's next candidate (dynamic assignment)
};

template <int NT>
__global__ void __launch_bounds__(NT) k_sim_flow(BatchDev B, int cls) {
    __shared__ FlowSmem<NT> sm;
    const int s = threadIdx.x;
    const int count = B.sim_count[cls];
    // candidates are handed out dynamically (their event counts differ by
    // orders of magnitude): a block that finishes takes the next one
    int* ctr = B.sim_count + SIM_CLASSES + cls;
    for (int idx = blockIdx.x; idx < count; idx = sm.next) {
        const int64_t ci = B.sim_list[(int64_t)cls * B.ncand + idx];
        const bp_candidate& cd = B.cand[ci];
        const CState cs = B.cs[ci];
        const QDesc Q = B.q[B.cq[ci]];
        const int N = Q.N;
        const int kind = cd.kind;
        const int64_t M = cd.M, micro = cd.micro;
        const bool async = kind_async(kind);
        sm.prodF[s] = sm.consF[s] = sm.prodB[s] = sm.consB[s] = 0;
        Err e{ERR_NONE};
        Rat fr{0, 1}, Fd{0, 1}, Bd{0, 1};
        int64_t w = 0, act = 0, srin = 0, srlink = 0;
        if (s < N) {
            const NetView v = net_view(B.P, Q.net);
            const ChainView c = chain_view(B.P, Q.cl, N);
            const int64_t slot = Q.stage_off + (ci - Q.cand_off) * N;
            const int64_t qo = Q.qstage_off;
            const bool refined = cs.plan_kind == PLAN_REFINED;
            const int32_t* hi = refined ? B.qhi + qo : B.chi + slot;
            if (refined) {
                Fd = B.qF[qo + s];
                Bd = B.qB[qo + s];
            } else {   // chain_instance (simulator.hpp:248-262)
                const int32_t t = c.type[s];
                Fd = R(stage_sum_whole(B.clo[slot + s], B.chi[slot + s], v.Pfp + (int64_t)t * (v.L + 1)));
                Bd = R(stage_sum_whole(B.clo[slot + s], B.chi[slot + s], v.Pbp + (int64_t)t * (v.L + 1)));
            }
            act = (s >= 1 ? v.a[hi[s - 1] - 1] : v.a[hi[0] - 1]) * micro;
            if (s > 0) {
                const int64_t a = v.a[hi[s - 1] - 1] * micro;
                srin = a == 0 ? 0 : ceil_div64(a, c.bw[s - 1]);
            }
            if (s + 1 < N) {
                const int64_t a = v.a[hi[s] - 1] * micro;
                srlink = a == 0 ? 0 : ceil_div64(a, c.bw[s]);
            }
            w = warmup_depth(kind, N, s + 1);
            if (w > M) w = M;
        }
        flow_sync<NT>();
        int64_t p = 0;                 // this stage's next position
        bool done = s >= N;
        bool aborted = false;
        volatile FlowSmem<NT>& vs = sm;
        int round = 0;
        for (;; ++round) {
            bool ran = false;
            if (!done) {
                const StageOp op = op_at(p, w, M);
                const int m = (int)op.m;
                const int k = (m - 1) % FLOW_Q;
                // arrival present and room downstream for this op's output
                const bool in_ok = op.is_f ? (s == 0 || vs.prodF[s] >= m) : (s + 1 >= N || vs.prodB[s] >= m);
                const bool out_ok = op.is_f ? (s + 1 >= N || vs.consF[s + 1] >= m - FLOW_Q)
                                            : (s == 0 || vs.consB[s - 1] >= m - FLOW_Q);
                if (in_ok && out_ok) {
                    // one code path for F and B lanes (operands selected, not
                    // branched), so a warp with both kinds of op runs each
                    // Rat operation once
                    __threadfence_block();
                    const bool f = op.is_f;
                    const bool has_in = f ? s > 0 : s + 1 < N;
                    const bool has_out = f ? s + 1 < N : s > 0;
                    Rat ready = fr;
                    if (has_in) {
                        volatile Rat* q = f ? &vs.qF[s][k] : &vs.qB[s][k];
                        const Rat arr{q->n, q->d};
                        *(f ? &vs.consF[s] : &vs.consB[s]) = m;
                        if (rat_gt(arr, ready)) ready = arr;
                    }
                    fr = rat_addsub_body(ready, f ? Fd : Bd, +1, e);
                    if (has_out) {
                        const Rat out = async ? fr : rat_addsub_body(fr, R(f ? srlink : srin), +1, e);
                        const int t = f ? s + 1 : s - 1;
                        volatile Rat* q = f ? &vs.qF[t][k] : &vs.qB[t][k];
                        q->n = out.n;
                        q->d = out.d;
                        __threadfence_block();
                        *(f ? &vs.prodF[t] : &vs.prodB[t]) = m;
                    }
                    ran = true;
                    if (++p == 2 * M) done = true;
                }
            }
            // bit 0: an error, bit 1: a stage not done, bit 2: a stage moved
            const unsigned f = flow_or<NT>((e.bad() ? 1u : 0u) | (done ? 0u : 2u) | (ran ? 4u : 0u), sm.red, round);
            if (f & 1u) {
                aborted = true;
                break;
            }
            if (!(f & 2u)) break;
            if (!(f & 4u)) __trap();   // no stage could move: impossible for a valid schedule
        }
        sm.fr[s] = fr;
        flow_sync<NT>();
        // makespan (simulator.hpp:173-180)
        Rat mk{0, 1};
        for (int t = 0; t < N; ++t)
            if (rat_gt(sm.fr[t], mk)) mk = sm.fr[t];
        // feature high-water: min(M, depth) * a (219-238)
        if (!aborted && s < N && (i128)w * act > (i128)INT64_MAX) e.set(ERR_OVERFLOW);
        // (every thread left the loop in the same round: the next words are clean)
        const bool core_bad = flow_or<NT>((aborted || e.bad()) ? 1u : 0u, sm.red, round + 1) != 0;
        // link busy fraction Rat(M * SR) / makespan (239-244): this
        // candidate's own (asynchronous members sharing the events form theirs)
        if (!core_bad && s + 1 < N && mk.n != 0) (void)rat_div(R(M * srlink), mk, e);
        const bool bad = core_bad || flow_or<NT>(e.bad() ? 1u : 0u, sm.red, round + 2) != 0;
        if (s == 0) {
            B.cs[ci].sim_core = core_bad ? 2 : 1;
            B.cs[ci].sim_mk = mk;
            bp_candidate& out = B.cand[ci];
            if (bad) {
                out.status = BP_C_ERR_OVERFLOW;
            } else {
                out.makespan = bp_rat{mk.n, mk.d};
                out.status = BP_C_OK;
            }
            sm.next = (int)gridDim.x + atomicAdd(ctr, 1);
        }
        flow_sync<NT>();
    }
}

}  // namespace

void launch_sim_flow(const BatchDev& B, int k, int sms, cudaStream_t st) {
    if (k == 0) k_sim_flow<32><<<sms * 32, 32, 0, st>>>(B, SIM_FLOW);
    else k_sim_flow<64><<<sms * 24, 64, 0, st>>>(B, SIM_FLOW + 1);
}

}  // namespace bpk
