// sim.cu -- K4 sim_wavefront: the 1F1B-family schedule simulation
// (simulator.hpp:81-246) for every candidate that passed its estimate.
//
// Fast path (k_sim_fast): a group of G lanes owns one candidate, S stages per
// lane; time is scaled by D (lcm of the stage denominators) so every event is
// an exact int64 (sim_classify proves no reference Rat can overflow there).
// The groups walk the sequence positions p = 0..2M-1 in lockstep.  At each
// position every stage runs exactly one op (F or B, fixed by its warm-up
// depth, simulator.hpp:87-100):
//     endF(m,s) = max(free_s, arrival_F) + F_s     arrival from stage s-1
//     endB(m,s) = max(free_s, arrival_B) + B_s     arrival from stage s+1
// An arrival produced at an earlier position waits in a one-slot mailbox
// (at most one is ever outstanding per link direction); arrivals produced at
// the same position form a chain along the stages (warm-up F chains, drain B
// chains).  y_s = max(a_s, y_{s-1} + b_s) is max-plus affine, so a chain is
// resolved by a segmented inclusive scan over the lanes (shuffles, width G):
// ascending for F, descending for B.  This is the reference's sorted-op
// recurrence (the (pos, sub) order is a topological order of the same DAG),
// computed position-parallel instead of op-serial.
//
// Slow path (k_sim_exact): thread per candidate, exact Rat events
// (phases.cuh:sim_exact), for candidates whose scaled times could exceed int64
// -- exactly where the reference's Rats might overflow.
#include <cstdlib>

#include "kernels.h"
#include "phases.cuh"

namespace bpk {

constexpr int64_t NEGV = -((int64_t)1 << 61);   // values stay below 2^61 (sim_classify)
constexpr int SIM_THREADS = 128;

__device__ __forceinline__ int64_t smax(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t sat(int64_t x) { return x < NEGV ? NEGV : x; }

// ---- batch-level deduplication of identical simulations.  simulate()'s
// inputs are the plan (layer ranges + fractions, through F/B per stage), the
// chain's types, kind, M, micro and the link bandwidths (SR per link);
// capacities only decide WHETHER a candidate is simulated.  Candidates whose
// inputs coincide (e.g. cluster mixes differing only in memory) are
// simulated once, by the smallest candidate index, inside the run; the hash
// only groups, inputs are compared exactly.
__device__ uint64_t sim_hash(const BatchDev& B, int64_t ci) {
    const bp_candidate& cd = B.cand[ci];
    const CState& cs = B.cs[ci];
    const int qi = B.cq[ci];
    const QDesc Q = B.q[qi];
    const ChainView c = chain_view(B.P, Q.cl, Q.N);
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&](uint64_t x) { h ^= x; h *= 0x100000001b3ull; h ^= h >> 29; };
    mix((uint64_t)(uint32_t)B.qrep[qi]);
    mix((uint64_t)cs.plan_kind * 8 + (uint64_t)cd.kind);
    mix((uint64_t)cd.M);
    mix((uint64_t)cd.micro);
    // an asynchronous schedule has no transfer ops (simulator.hpp:111-117):
    // its events do not depend on the links, only its busy fractions do
    // (recomputed per candidate when the outcome is shared, sim_copy)
    if (!kind_async(cd.kind))
        for (int k = 0; k + 1 < Q.N; ++k) mix((uint64_t)c.bw[k]);
    if (cs.plan_kind != PLAN_REFINED) {
        const int64_t slot = Q.stage_off + (ci - Q.cand_off) * Q.N;
        for (int s = 0; s < Q.N; ++s) mix(((uint64_t)(uint32_t)B.clo[slot + s] << 32) | (uint32_t)B.chi[slot + s]);
    }
    return h ? h : 1;
}

__device__ bool same_sim(const BatchDev& B, int64_t a, int64_t b) {
    const bp_candidate &x = B.cand[a], &y = B.cand[b];
    const CState &cx = B.cs[a], &cy = B.cs[b];
    const int qa = B.cq[a], qb = B.cq[b];
    if (B.qrep[qa] != B.qrep[qb] || cx.plan_kind != cy.plan_kind || x.kind != y.kind || x.M != y.M ||
        x.micro != y.micro)
        return false;
    const QDesc A = B.q[qa], Q = B.q[qb];   // same class: same network, N and stage types
    const ChainView ca = chain_view(B.P, A.cl, A.N), cb = chain_view(B.P, Q.cl, Q.N);
    if (!kind_async(x.kind))
        for (int k = 0; k + 1 < A.N; ++k)
            if (ca.bw[k] != cb.bw[k]) return false;
    if (cx.plan_kind != PLAN_REFINED) {
        const int64_t sa = A.stage_off + (a - A.cand_off) * A.N, sb = Q.stage_off + (b - Q.cand_off) * Q.N;
        for (int s = 0; s < A.N; ++s)
            if (B.clo[sa + s] != B.clo[sb + s] || B.chi[sa + s] != B.chi[sb + s]) return false;
    }
    return true;
}

__device__ __forceinline__ uint32_t sim_slot(const BatchDev& B, uint64_t h) {
    return (uint32_t)(h ^ (h >> 32)) & (uint32_t)B.smask;
}

__global__ void k_sim_classify(BatchDev B) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.ncand) return;
    const int64_t ci = B.cperm[i];
    int cls = sim_classify(B, ci);
    if (cls == SIM_EXACT) {
        const bp_candidate& c = B.cand[ci];
        const int64_t N = c.n_stages, ev = 2 * N * c.M + (c.kind >= 2 ? 2 * (N - 1) * c.M : 0);
        if (N >= FLOW_MIN_N && N <= 64 && ev >= FLOW_MIN_EVENTS) cls = SIM_FLOW + (N <= 32 ? 0 : 1);
    }
    B.cs[ci].sim_cls = cls;
    B.cs[ci].sim_rep = -1;
    if (cls < 0) return;
    const uint64_t h = sim_hash(B, ci);
    for (uint32_t slot = sim_slot(B, h);; slot = (slot + 1) & (uint32_t)B.smask) {
        const unsigned long long prev = atomicCAS(&B.skey[slot], 0ull, (unsigned long long)h);
        if (prev == 0ull || prev == h) {
            atomicMin(&B.srep[slot], (int32_t)ci);
            return;
        }
    }
}

// simulated candidates whose inputs equal an earlier candidate's copy its
// outcome after the simulators ran
// A member's outcome from its representative's simulation.  Synchronous
// kinds share only with identical links: the record is copied.  An
// asynchronous member may differ from its representative in the links: it
// takes the representative's events outcome (sim_core, sim_mk) and forms its
// own link busy fractions Rat(M * SR) / makespan (simulator.hpp:239-244).
__device__ void sim_copy(const BatchDev& B, int64_t ci, int64_t r) {
    bp_candidate& cd = B.cand[ci];
    if (!kind_async(cd.kind)) {
        cd.status = B.cand[r].status;
        cd.makespan = B.cand[r].makespan;
        return;
    }
    const CState& rs = B.cs[r];
    if (rs.sim_core != 1) {   // the shared events (or high-water) overflowed
        cd.status = BP_C_ERR_OVERFLOW;
        return;
    }
    const Rat mk = rs.sim_mk;
    const CState& cs = B.cs[ci];
    const QDesc Q = B.q[B.cq[ci]];
    const int N = Q.N;
    const NetView v = net_view(B.P, Q.net);
    const ChainView c = chain_view(B.P, Q.cl, N);
    const int32_t* hi = cs.plan_kind == PLAN_REFINED ? B.qhi + Q.qstage_off
                                                     : B.chi + Q.stage_off + (ci - Q.cand_off) * N;
    Err e{ERR_NONE};
    for (int k = 0; k + 1 < N && !e.bad(); ++k) {
        if (mk.n == 0) break;
        const int64_t a = v.a[hi[k] - 1] * cd.micro;
        const int64_t sr = a == 0 ? 0 : ceil_div64(a, c.bw[k]);
        (void)rat_div(R(cd.M * sr), mk, e);
    }
    if (e.bad()) {
        cd.status = BP_C_ERR_OVERFLOW;
    } else {
        cd.makespan = bp_rat{mk.n, mk.d};
        cd.status = BP_C_OK;
    }
}

__global__ void k_sim_share(BatchDev B) {
    int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ci >= B.ncand) return;
    const int32_t r = B.cs[ci].sim_rep;
    if (r < 0) return;
    if (B.prune_lb && B.cs[r].lbstate == LB_DEFERRED) return;   // not simulated (yet)
    sim_copy(B, ci, r);
}

__global__ void k_sim_prep(BatchDev B) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int cls = -1;
    uint64_t ev = 0;
    if (i < B.ncand) {
        int64_t ci = B.cperm[i];
        cls = B.cs[ci].sim_cls;
        if (cls >= 0) {
            const uint64_t h = sim_hash(B, ci);
            uint32_t slot = sim_slot(B, h);
            while (B.skey[slot] != h) slot = (slot + 1) & (uint32_t)B.smask;
            const int32_t r = B.srep[slot];
            if (B.dedup && r != ci && same_sim(B, ci, r)) {
                B.cs[ci].sim_rep = r;
                // an asynchronous member may classify apart from its
                // representative (its link term in the bound differs): it
                // follows the representative's class (BP_OPT_PRUNE_LB rounds)
                B.cs[ci].sim_cls = B.cs[r].sim_cls;
                cls = -1;
            }
        }
        // BP_OPT_PRUNE_LB: scaled-integer representatives wait for their
        // query's best (k_lb_round1 / k_lb_decide list them)
        if (cls >= 0 && cls < SIM_EXACT && B.prune_lb) cls = -1;
        if (cls >= 0) {
            int pos = atomicAdd(&B.sim_count[cls], 1);
            B.sim_list[(int64_t)cls * B.ncand + pos] = (int32_t)ci;
            // simulated events (SURVEY.md 8d X_sim): 2NM ops, + 2(N-1)M transfers when sync
            const bp_candidate& c = B.cand[ci];
            const uint64_t N = (uint64_t)c.n_stages, M = (uint64_t)c.M;
            ev = 2 * N * M + (c.kind >= 2 ? 2 * (N - 1) * M : 0);
        }
    }
    // instrumentation: warp-aggregated event counts per simulator class
    uint32_t ev32 = ev < (1u << 26) ? (uint32_t)ev : 0;
    if (ev32 != ev) atomicAdd(&B.work[WORK_SIM_EVENTS + cls], (unsigned long long)ev);
    const unsigned grp = __match_any_sync(0xffffffffu, cls);
    const uint32_t sum = __reduce_add_sync(grp, ev32);
    if (cls >= 0 && (int)(threadIdx.x & 31) == __ffs(grp) - 1)
        atomicAdd(&B.work[WORK_SIM_EVENTS + cls], (unsigned long long)sum);
}

// ---- exact path scheduling: counting sort of the exact list by
// (stage count, log2 M), heaviest bucket first, so that the 32 lanes of a
// warp run candidates with the same N and similar M (same loop structure).
__device__ __forceinline__ int xbucket(int N, int64_t M, int kind) {
    int lg = 63 - __clzll((long long)M);
    if (lg > 31) lg = 31;
    int n = N > 255 ? 255 : N;
    return XBUCKETS - 1 - ((n * 32 + lg) * 4 + kind);
}

__global__ void k_xsort_count(BatchDev B) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.sim_count[SIM_EXACT]) return;
    int32_t ci = B.sim_list[(int64_t)SIM_EXACT * B.ncand + i];
    int k = xbucket(B.cand[ci].n_stages, B.cand[ci].M, B.cand[ci].kind);
    B.xkey[i] = k;
    atomicAdd(&B.xhist[k], 1);
}

__global__ void __launch_bounds__(1024) k_xsort_scan(BatchDev B) {
    __shared__ int32_t part[1024];
    const int per = XBUCKETS / 1024;
    int base = threadIdx.x * per, s = 0;
    for (int k = 0; k < per; ++k) s += B.xhist[base + k];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = part[threadIdx.x] - s;   // exclusive
    for (int k = 0; k < per; ++k) {
        int c = B.xhist[base + k];
        B.xhist[base + k] = run;
        run += c;
    }
}

__global__ void k_xsort_scatter(BatchDev B) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.sim_count[SIM_EXACT]) return;
    int pos = atomicAdd(&B.xhist[B.xkey[i]], 1);
    B.xsorted[pos] = B.sim_list[(int64_t)SIM_EXACT * B.ncand + i];
}

// Persistent warps take chunks of 32 from the sorted exact list (heaviest
// first) off a global counter, so the long candidates start first and the
// rest fill in behind them; each lane runs one candidate's exact simulation
// with its per-stage state interleaved across the warp (element (s, lane) at
// s*32 + lane: coalesced accesses).
__global__ void __launch_bounds__(256) k_sim_exact(BatchDev B) {
    const int count = B.sim_count[SIM_EXACT];
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t per_stage = 32;                    // lanes interleaved
    const int64_t arr = per_stage * (int64_t)B.max_N; // one array of a warp's state
    Rat* base = B.simbuf + warp * 5 * arr;
    int64_t* ibase = reinterpret_cast<int64_t*>(B.simbuf + nwarps * 5 * arr) + warp * 2 * arr;
    SimState S{base + lane, base + arr + lane, base + 2 * arr + lane, base + 3 * arr + lane, base + 4 * arr + lane,
               ibase + lane, ibase + arr + lane, 32};
    int32_t* next = B.xhist + XBUCKETS;   // chunk counter, zeroed with the histogram
    for (;;) {
        int chunk = 0;
        if (lane == 0) chunk = atomicAdd(next, 1);
        chunk = __shfl_sync(0xffffffffu, chunk, 0);
        if ((int64_t)chunk * 32 >= count) break;
        const int64_t i = (int64_t)chunk * 32 + lane;
        if (i < count) sim_exact(B, B.xsorted[i], S);
    }
}

template <int G, int S>
__global__ void __launch_bounds__(SIM_THREADS) k_sim_fast(BatchDev B, int cls) {
    const unsigned FULL = 0xffffffffu;
    const int count = B.sim_count[cls];
    const int lane = threadIdx.x & 31;
    const int r = lane % G;
    const int gpw = 32 / G;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t warp_global = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    // persistent warps; after the first chunk, chunks of gpw candidates are
    // handed out dynamically (event counts differ by orders of magnitude)
    int* ctr = B.sim_count + SIM_CLASSES + cls;
    auto next_chunk = [&]() -> int64_t {
        int nb = 0;
        if (lane == 0) nb = atomicAdd(ctr, 1);
        nb = __shfl_sync(FULL, nb, 0);
        return (warps_total + nb) * gpw;
    };
    for (int64_t base = warp_global * gpw; base < count; base = next_chunk()) {
    const int64_t gid = base + lane / G;
    const bool active = gid < count;
    int64_t ci = active ? B.sim_list[(int64_t)cls * B.ncand + gid] : -1;
    int N = 1, kind = 0;
    int64_t M = 0, micro = 1, D = 1;
    bool async = true;
    int64_t Fd[S], Bd[S], SRin[S], SRout[S], fr[S], pF[S], pB[S], A[S];
    int64_t wv[S], wprev[S], wnext[S];
    bool has[S];
#pragma unroll
    for (int i = 0; i < S; ++i) {
        has[i] = false;
        Fd[i] = Bd[i] = SRin[i] = SRout[i] = fr[i] = A[i] = 0;
        pF[i] = pB[i] = NEGV;
        wv[i] = wprev[i] = wnext[i] = 0;
    }
    int64_t slot = 0, qo = 0;
    int plan_kind = PLAN_WHOLE;
    if (active) {
        const bp_candidate& cd = B.cand[ci];
        const CState cs = B.cs[ci];
        const int qi = B.cq[ci];
        const QDesc Q = B.q[qi];
        N = Q.N;
        kind = cd.kind;
        M = cd.M;
        micro = cd.micro;
        D = cs.D;
        async = kind_async(kind);
        plan_kind = cs.plan_kind;
        NetView v = net_view(B.P, Q.net);
        ChainView c = chain_view(B.P, Q.cl, N);
        slot = Q.stage_off + (ci - Q.cand_off) * N;
        qo = Q.qstage_off;
        const int32_t* hi = plan_kind == PLAN_REFINED ? B.qhi + qo : B.chi + slot;
        const int32_t* lo = plan_kind == PLAN_REFINED ? B.qlo + qo : B.clo + slot;
#pragma unroll
        for (int i = 0; i < S; ++i) {
            const int s = r * S + i;
            if (s >= N) continue;
            has[i] = true;
            if (plan_kind == PLAN_REFINED) {
                Rat f = B.qF[qo + s], b = B.qB[qo + s];
                Fd[i] = f.n * (D / f.d);
                Bd[i] = b.n * (D / b.d);
            } else {
                int32_t t = c.type[s];
                Fd[i] = stage_sum_whole(lo[s], hi[s], v.Pfp + (int64_t)t * (v.L + 1));
                Bd[i] = stage_sum_whole(lo[s], hi[s], v.Pbp + (int64_t)t * (v.L + 1));
            }
            if (s > 0) {
                int64_t a = v.a[hi[s - 1] - 1] * micro;
                SRin[i] = (a == 0 ? 0 : ceil_div64(a, c.bw[s - 1])) * D;
                A[i] = a;
            } else {
                A[i] = v.a[hi[0] - 1] * micro;
            }
            if (s + 1 < N) {
                int64_t a = v.a[hi[s] - 1] * micro;
                SRout[i] = (a == 0 ? 0 : ceil_div64(a, c.bw[s])) * D;
            }
            int64_t w = warmup_depth(kind, N, s + 1);
            wv[i] = w < M ? w : M;
            if (s > 0) { w = warmup_depth(kind, N, s); wprev[i] = w < M ? w : M; }
            if (s + 1 < N) { w = warmup_depth(kind, N, s + 2); wnext[i] = w < M ? w : M; }
        }
    }
    int64_t Mloop = active ? M : 0;
    for (int o = 16; o > 0; o >>= 1) Mloop = smax(Mloop, __shfl_xor_sync(FULL, Mloop, o));
    const int64_t syncF = async ? 0 : 1;
    for (int64_t p = 0; p < 2 * Mloop; ++p) {
        const bool live = active && p < 2 * M;
        bool isF[S], isB[S], chF[S], chB[S];
        int64_t mm[S];
        bool anyF = false, anyB = false;
#pragma unroll
        for (int i = 0; i < S; ++i) {
            isF[i] = isB[i] = chF[i] = chB[i] = false;
            mm[i] = 0;
            if (has[i] && live) {
                const int s = r * S + i;
                StageOp op = op_at(p, wv[i], M);
                mm[i] = op.m;
                isF[i] = op.is_f;
                isB[i] = !op.is_f;
                if (isF[i] && s > 0) {
                    StageOp q = op_at(p, wprev[i], M);
                    chF[i] = q.is_f && q.m == op.m;
                }
                if (isB[i] && s + 1 < N) {
                    StageOp q = op_at(p, wnext[i], M);
                    chB[i] = !q.is_f && q.m == op.m;
                }
            }
            anyF |= chF[i];
            anyB |= chB[i];
        }
        const unsigned balF = __ballot_sync(FULL, anyF), balB = __ballot_sync(FULL, anyB);
        // ---- forward ops (ascending stages)
        int64_t eF[S];
#pragma unroll
        for (int i = 0; i < S; ++i) {
            const int s = r * S + i;
            int64_t dep = (isF[i] && !chF[i] && s > 0) ? pF[i] : NEGV;
            eF[i] = isF[i] ? smax(fr[i], dep) + Fd[i] : NEGV;
        }
        if (balF) {
            // local inclusive composition of f_i(y) = max(a_i, y + b_i)
            int64_t cA[S], cB[S];
#pragma unroll
            for (int i = 0; i < S; ++i) {
                int64_t a = eF[i];
                int64_t b = chF[i] ? SRin[i] * syncF + Fd[i] : NEGV;
                if (i == 0) { cA[i] = a; cB[i] = b; }
                else { cA[i] = smax(a, sat(cA[i - 1] + b)); cB[i] = sat(cB[i - 1] + b); }
            }
            int64_t gA = cA[S - 1], gB = cB[S - 1];
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                int64_t pa = __shfl_up_sync(FULL, gA, o, G), pb = __shfl_up_sync(FULL, gB, o, G);
                if (r >= o) { gA = smax(gA, sat(pa + gB)); gB = sat(pb + gB); }
            }
            int64_t xA = __shfl_up_sync(FULL, gA, 1, G);
            if (r == 0) xA = NEGV;
#pragma unroll
            for (int i = 0; i < S; ++i) eF[i] = smax(cA[i], sat(xA + cB[i]));
        }
#pragma unroll
        for (int i = 0; i < S; ++i)
            if (isF[i]) fr[i] = eF[i];
        // ---- backward ops (descending stages)
        int64_t eB[S];
#pragma unroll
        for (int i = 0; i < S; ++i) {
            const int s = r * S + i;
            int64_t dep = (isB[i] && !chB[i] && s + 1 < N) ? pB[i] : NEGV;
            eB[i] = isB[i] ? smax(fr[i], dep) + Bd[i] : NEGV;
        }
        if (balB) {
            int64_t cA[S], cB[S];
#pragma unroll
            for (int i = S - 1; i >= 0; --i) {
                int64_t a = eB[i];
                int64_t b = chB[i] ? SRout[i] * syncF + Bd[i] : NEGV;
                if (i == S - 1) { cA[i] = a; cB[i] = b; }
                else { cA[i] = smax(a, sat(cA[i + 1] + b)); cB[i] = sat(cB[i + 1] + b); }
            }
            int64_t gA = cA[0], gB = cB[0];
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                int64_t pa = __shfl_down_sync(FULL, gA, o, G), pb = __shfl_down_sync(FULL, gB, o, G);
                if (r + o < G) { gA = smax(gA, sat(pa + gB)); gB = sat(pb + gB); }
            }
            int64_t xA = __shfl_down_sync(FULL, gA, 1, G);
            if (r == G - 1) xA = NEGV;
#pragma unroll
            for (int i = 0; i < S; ++i) eB[i] = smax(cA[i], sat(xA + cB[i]));
        }
#pragma unroll
        for (int i = 0; i < S; ++i)
            if (isB[i]) fr[i] = eB[i];
        // ---- mailboxes: F from stage s-1, B from stage s+1
        {
            int64_t vF = isF[S - 1] ? eF[S - 1] + SRout[S - 1] * syncF : 0;
            int64_t mF = isF[S - 1] ? mm[S - 1] : -1;
            int64_t inF = __shfl_up_sync(FULL, vF, 1, G), inFm = __shfl_up_sync(FULL, mF, 1, G);
            int64_t vB = isB[0] ? eB[0] + SRin[0] * syncF : 0;
            int64_t mB = isB[0] ? mm[0] : -1;
            int64_t inB = __shfl_down_sync(FULL, vB, 1, G), inBm = __shfl_down_sync(FULL, mB, 1, G);
#pragma unroll
            for (int i = 0; i < S; ++i) {
                const int s = r * S + i;
                if (!has[i] || !live) continue;
                // from s-1
                int64_t v_in, m_in;
                if (i > 0) { v_in = isF[i - 1] ? eF[i - 1] + SRout[i - 1] * syncF : 0; m_in = isF[i - 1] ? mm[i - 1] : -1; }
                else { v_in = inF; m_in = r > 0 ? inFm : -1; }
                if (s > 0 && m_in >= 0 && !(chF[i] && mm[i] == m_in)) pF[i] = v_in;
                // from s+1
                if (i + 1 < S) { v_in = isB[i + 1] ? eB[i + 1] + SRin[i + 1] * syncF : 0; m_in = isB[i + 1] ? mm[i + 1] : -1; }
                else { v_in = inB; m_in = r + 1 < G ? inBm : -1; }
                if (s + 1 < N && m_in >= 0 && !(chB[i] && mm[i] == m_in)) pB[i] = v_in;
            }
        }
    }
    // ---- makespan (simulator.hpp:173-180) and the post-simulation Rat checks
    int64_t X = 0;
#pragma unroll
    for (int i = 0; i < S; ++i)
        if (has[i]) X = smax(X, fr[i]);
    for (int o = 1; o < G; o <<= 1) X = smax(X, __shfl_xor_sync(FULL, X, o, G));
    Err e{ERR_NONE};
    Rat mk{0, 1};
    if (active) {
        uint64_t g = gcd_u64((uint64_t)X, (uint64_t)D);
        mk = Rat{X / (int64_t)g, D / (int64_t)g};
#pragma unroll
        for (int i = 0; i < S; ++i) {
            if (!has[i]) continue;
            // feature high-water: min(M, depth) * a (219-238)
            if ((i128)wv[i] * A[i] > (i128)INT64_MAX) e.set(ERR_OVERFLOW);
        }
    }
    // the events and high-water (shared with asynchronous members), then this
    // candidate's own link busy fractions
    const unsigned core_bad = __ballot_sync(FULL, e.bad());
    if (active) {
#pragma unroll
        for (int i = 0; i < S; ++i) {
            const int s = r * S + i;
            if (!has[i]) continue;
            // busy fraction Rat(M * SR) / makespan (239-244)
            if (s + 1 < N && mk.n != 0) (void)rat_div(R(M * (SRout[i] / D)), mk, e);
        }
    }
    unsigned bad = __ballot_sync(FULL, e.bad());
    if (active && r == 0) {
        bp_candidate& cd = B.cand[ci];
        const unsigned gm = G == 32 ? FULL : ((1u << (G & 31)) - 1u) << (lane - r);
        B.cs[ci].sim_core = (core_bad & gm) ? 2 : 1;
        B.cs[ci].sim_mk = mk;
        if (bad & gm) {
            cd.status = BP_C_ERR_OVERFLOW;
        } else {
            cd.makespan = bp_rat{mk.n, mk.d};
            cd.status = BP_C_OK;
        }
    }
    }  // persistent loop
}

// ---- BP_OPT_PRUNE_LB: estimate-based pruning (the reference's
// explore() simulates every candidate, explorer.hpp:96-132).
//
// Only the scaled-integer class is ever skipped: its simulation provably
// cannot raise (k_sim_prep's bound), so skipping it cannot change a query's
// outcome, and a skipped candidate is feasible, hence ranked, either way.  It
// is skipped when its makespan lower bound exceeds its query's best
// simulated makespan, so it cannot be ranked first: the query's best record
// is unchanged.  Every stage runs its M F and M B ops one after another, and
// before the first of them micro-batch 1 must cross the stages before it,
// after the last of them micro-batch M must cross them back (sync transfers
// on both paths, simulator.hpp:134-171):
//   makespan >= max_b [ sum_{s<b} (F_s + B_s + 2 SR_s [sync]) + M (F_b + B_b) ].
// Scaled by the candidate's D this is an integer below the class's 2^61
// bound.
__device__ int64_t sim_lower_bound_scaled(const BatchDev& B, int64_t ci) {
    const bp_candidate& cd = B.cand[ci];
    const CState& cs = B.cs[ci];
    const int qi = B.cq[ci];
    const QDesc Q = B.q[qi];
    const int N = Q.N;
    const int64_t M = cd.M, micro = cd.micro, D = cs.D;
    const bool sync = !kind_async(cd.kind);
    const NetView v = net_view(B.P, Q.net);
    const ChainView c = chain_view(B.P, Q.cl, N);
    const int64_t slot = Q.stage_off + (ci - Q.cand_off) * N, qo = Q.qstage_off;
    const bool refined = cs.plan_kind == PLAN_REFINED;
    const int32_t* hi = refined ? B.qhi + qo : B.chi + slot;
    const int32_t* lo = refined ? B.qlo + qo : B.clo + slot;
    int64_t prefix = 0, best = 0;
    for (int s = 0; s < N; ++s) {
        int64_t F, Bt;
        if (refined) {
            const Rat f = B.qF[qo + s], b = B.qB[qo + s];
            F = f.n * (D / f.d);
            Bt = b.n * (D / b.d);
        } else {
            const int32_t t = c.type[s];
            F = stage_sum_whole(lo[s], hi[s], v.Pfp + (int64_t)t * (v.L + 1));
            Bt = stage_sum_whole(lo[s], hi[s], v.Pbp + (int64_t)t * (v.L + 1));
        }
        const int64_t here = prefix + M * (F + Bt);
        best = here > best ? here : best;
        int64_t sr = 0;
        if (sync && s + 1 < N) {
            const int64_t a = v.a[hi[s] - 1] * micro;
            sr = (a == 0 ? 0 : ceil_div64(a, c.bw[s])) * D;
        }
        prefix += F + Bt + 2 * sr;
    }
    return best;
}

__device__ __forceinline__ bool lb_class(int cls) { return cls >= 0 && cls < SIM_EXACT; }

// bound of every scaled-integer candidate; per query, the smallest bound's
// candidate (the seed, simulated first)
__global__ void k_lb_bound(BatchDev B) {
    const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ci >= B.ncand) return;
    CState& cs = B.cs[ci];
    cs.lb = -1;
    cs.lbstate = LB_NONE;
    if (!lb_class(cs.sim_cls)) return;
    const int64_t lb = sim_lower_bound_scaled(B, ci);
    cs.lb = lb;
    cs.lbstate = LB_DEFERRED;
    const int qi = B.cq[ci];
    const float key = (float)lb / (float)cs.D;
    atomicMin(&B.qseed[qi], ((unsigned long long)__float_as_uint(key) << 32) |
                                (unsigned long long)(uint32_t)(ci - B.q[qi].cand_off));
}

__device__ void lb_list(const BatchDev& B, int64_t r) {
    const int cls = B.cs[r].sim_cls;
    const int pos = atomicAdd(&B.sim_count[cls], 1);
    B.sim_list[(int64_t)cls * B.ncand + pos] = (int32_t)r;
    const bp_candidate& c = B.cand[r];
    const uint64_t N = (uint64_t)c.n_stages, M = (uint64_t)c.M;
    atomicAdd(&B.work[WORK_SIM_EVENTS + cls], (unsigned long long)(2 * N * M + (c.kind >= 2 ? 2 * (N - 1) * M : 0)));
}

// round 1: each query's seed (its simulation representative) is simulated
// with the exact classes
__global__ void k_lb_round1(BatchDev B) {
    const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ci >= B.ncand || !lb_class(B.cs[ci].sim_cls)) return;
    const int qi = B.cq[ci];
    if ((uint32_t)(B.qseed[qi] & 0xffffffffull) != (uint32_t)(ci - B.q[qi].cand_off)) return;
    const int64_t r = B.cs[ci].sim_rep >= 0 ? B.cs[ci].sim_rep : ci;
    if (atomicCAS(&B.cs[r].lbstate, LB_DEFERRED, LB_ROUND1) == LB_DEFERRED) lb_list(B, r);
}

// each query's best simulated makespan so far (thread per query)
__global__ void k_lb_incumbent(BatchDev B) {
    const int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= B.nq) return;
    const QDesc Q = B.q[qi];
    bp_rat inc{0, 0};
    for (int i = 0; i < 2 * Q.nbase; ++i) {
        const bp_candidate& c = B.cand[Q.cand_off + i];
        if (c.status != BP_C_OK) continue;
        const Rat m{c.makespan.num, c.makespan.den};
        if (inc.den == 0 || rat_lt(m, Rat{inc.num, inc.den})) inc = c.makespan;
    }
    B.qinc[qi] = inc;
}

// round 2: the deferred representatives some member of which has a bound
// not above its query's best
__global__ void k_lb_decide(BatchDev B) {
    const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ci >= B.ncand) return;
    const CState cs = B.cs[ci];
    if (!lb_class(cs.sim_cls)) return;
    const int64_t r = cs.sim_rep >= 0 ? cs.sim_rep : ci;
    if (B.cs[r].lbstate != LB_DEFERRED) return;
    const bp_rat inc = B.qinc[B.cq[ci]];
    // lb / D <= inc.num / inc.den, exactly
    const bool need = inc.den == 0 || (i128)cs.lb * inc.den <= (i128)inc.num * cs.D;
    if (need && atomicCAS(&B.cs[r].lbstate, LB_DEFERRED, LB_ROUND2) == LB_DEFERRED) lb_list(B, r);
}

// the skipped candidates' records; members of round-2 representatives copy
// their outcome
__global__ void k_lb_finish(BatchDev B) {
    const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ci >= B.ncand) return;
    const CState cs = B.cs[ci];
    if (!lb_class(cs.sim_cls)) return;
    const int64_t r = cs.sim_rep >= 0 ? cs.sim_rep : ci;
    bp_candidate& cd = B.cand[ci];
    if (B.cs[r].lbstate == LB_DEFERRED) {
        cd.status = BP_C_PRUNED_LB;
        cd.makespan = bp_rat{0, 0};
    } else if (cs.sim_rep >= 0 && cd.status == C_PENDING) {
        sim_copy(B, ci, r);
    }
}

// The dataflow lists in decreasing op-DAG depth (2M + 2N rounds, 16 log2
// buckets): their blocks take candidates from a counter in list order, so the
// heaviest start first and the phase ends on light ones (LPT).
__global__ void __launch_bounds__(1024) k_flow_sort(BatchDev B, int cls) {
    __shared__ int cnt[16], off[16];
    const int n = B.sim_count[cls];
    int32_t* list = B.sim_list + (int64_t)cls * B.ncand;
    if (threadIdx.x < 16) cnt[threadIdx.x] = 0;
    __syncthreads();
    auto key = [&](int32_t ci) {
        const bp_candidate& c = B.cand[ci];
        const int64_t r = 2 * c.M + 2 * (int64_t)c.n_stages;
        const int lg = 63 - __clzll((long long)r);
        return 15 - (lg > 15 ? 15 : lg);
    };
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cnt[key(list[i])], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0;
        for (int k = 0; k < 16; ++k) { off[k] = a; a += cnt[k]; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int32_t ci = list[i];
        B.flow_tmp[atomicAdd(&off[key(ci)], 1)] = ci;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) list[i] = B.flow_tmp[i];
}

static inline int blocks_for(int64_t n, int t) { return (int)((n + t - 1) / t); }

void launch_sim_prep(const BatchDev& B, cudaStream_t st) {
    cudaMemsetAsync(B.sim_count, 0, 2 * SIM_CLASSES * sizeof(int32_t), st);
    cudaMemsetAsync(B.skey, 0, ((size_t)B.smask + 1) * sizeof(unsigned long long), st);
    cudaMemsetAsync(B.srep, 0x7f, ((size_t)B.smask + 1) * sizeof(int32_t), st);
    if (B.ncand) {
        k_sim_classify<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
        k_sim_prep<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
        k_flow_sort<<<1, 1024, 0, st>>>(B, SIM_FLOW);
        k_flow_sort<<<1, 1024, 0, st>>>(B, SIM_FLOW + 1);
    }
}

void launch_sim_share(const BatchDev& B, cudaStream_t st) {
    if (B.ncand) k_sim_share<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
}

void launch_lb_bound(const BatchDev& B, cudaStream_t st) {
    if (!B.ncand) return;
    cudaMemsetAsync(B.qseed, 0xff, (size_t)B.nq * sizeof(unsigned long long), st);
    k_lb_bound<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
}
void launch_lb_round1(const BatchDev& B, cudaStream_t st) {
    if (B.ncand) k_lb_round1<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
}
// after round 1 (and its k_sim_share): the round-2 lists of the scaled-integer
// classes, replacing their round-1 lists
void launch_lb_round2(const BatchDev& B, cudaStream_t st) {
    if (!B.ncand) return;
    cudaMemsetAsync(B.sim_count, 0, SIM_EXACT * sizeof(int32_t), st);
    cudaMemsetAsync(B.sim_count + SIM_CLASSES, 0, SIM_EXACT * sizeof(int32_t), st);
    k_lb_incumbent<<<blocks_for(B.nq, 128), 128, 0, st>>>(B);
    k_lb_decide<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
}
void launch_lb_finish(const BatchDev& B, cudaStream_t st) {
    if (B.ncand) k_lb_finish<<<blocks_for(B.ncand, 128), 128, 0, st>>>(B);
}

void launch_sim_fast(const BatchDev& B, int cls, int sms, cudaStream_t st) {
    const int grid = sms * 8;   // persistent warps
    switch (cls) {
        case 0: k_sim_fast<2, 1><<<grid, SIM_THREADS, 0, st>>>(B, 0); break;
        case 1: k_sim_fast<4, 1><<<grid, SIM_THREADS, 0, st>>>(B, 1); break;
        case 2: k_sim_fast<8, 1><<<grid, SIM_THREADS, 0, st>>>(B, 2); break;
        case 3: k_sim_fast<16, 1><<<grid, SIM_THREADS, 0, st>>>(B, 3); break;
        case 4: k_sim_fast<32, 1><<<grid, SIM_THREADS, 0, st>>>(B, 4); break;
        case 5: k_sim_fast<32, 2><<<grid, SIM_THREADS, 0, st>>>(B, 5); break;
        case 6: k_sim_fast<32, 4><<<grid, SIM_THREADS, 0, st>>>(B, 6); break;
        case 7: k_sim_fast<32, 8><<<grid, SIM_THREADS, 0, st>>>(B, 7); break;
        default: break;
    }
}

// Bytes of exact-simulator state for `sms` SMs (5 Rat + 2 int64 arrays per
// stage per lane per persistent warp).
size_t sim_exact_state_bytes(int sms, int max_N) {
    const size_t warps = (size_t)sms * XSIM_WARPS_PER_SM;
    return warps * 32 * (size_t)(max_N > 0 ? max_N : 1) * (5 * sizeof(Rat) + 2 * sizeof(int64_t));
}

void launch_sim_exact(const BatchDev& B, int sms, cudaStream_t st) {
    if (!B.ncand) return;
    cudaMemsetAsync(B.xhist, 0, (XBUCKETS + 1) * sizeof(int32_t), st);
    k_xsort_count<<<blocks_for(B.ncand, 256), 256, 0, st>>>(B);
    k_xsort_scan<<<1, 1024, 0, st>>>(B);
    k_xsort_scatter<<<blocks_for(B.ncand, 256), 256, 0, st>>>(B);
    const int wps = XSIM_WARPS_PER_SM;
    k_sim_exact<<<sms * wps / 8, 256, 0, st>>>(B);
}

}  // namespace bpk
