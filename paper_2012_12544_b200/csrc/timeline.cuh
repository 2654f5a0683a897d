// timeline.cuh -- one caller-given plan: the full-timeline simulate and the
// estimate (`bapipe simulate` / `bapipe plan`).
//
//   tl_chain      chain_instance (simulator.hpp:248-262) after validate_plan
//                 (plan.hpp:41-85): per-stage F, B, w, a, per-link SR
//   tl_walk       simulate_chain's op walk (simulator.hpp:81-171), every
//                 start / end kept, and the event list (182-216) written in
//                 per-stage segments
//   tl_stage      one stage's segment sorted by (start, kind, micro-batch),
//                 its feature high-water and static weights (217-238)
//   tl_busy       link busy fractions (239-244)
//   tl_estimate   estimate() on the plan (cost_models.hpp:124-166)
//
// Host + device functions on plain arrays: the kernels in timeline.cu run
// them on the GPU (tl_stage one thread per stage); the test emulator
// (tests/cpp/emu_abi_shim.cpp) replays them on the host.  Every Rat operation
// is the reference's, on the same operands, so overflow is reported exactly
// where the reference throws.
#pragma once
#include "phases.cuh"

namespace bpk {

struct TlArgs {
    NetView v;
    ChainView c;              // the first N accelerators of the cluster
    int N, kind, clusterN;
    int64_t M, micro, mini;
    const int32_t *lo, *hi;
    const Rat *lead, *trail;
    // chain instance
    Rat *F, *B, *W;           // [N]
    int64_t *a, *SR;          // [N] (SR[k-1] = link k)
    // op times, index (s-1)*M + (m-1) / (k-1)*M + (m-1)
    Rat *sF, *eF, *sB, *eB;   // [N*M]
    Rat *tFs, *tFe, *tBs, *tBe;   // [(N-1)*M], sync only
    Rat* makespan1;           // [1] one mini-batch's makespan
    // events: stage s's segment is ev[off[s-1] .. off[s])
    bp_event *ev, *ev_tmp;
    int64_t* off;             // [N+1]
};

BPK_HD void tl_fail(bp_timeline_result& r, const Err& e) { r.status = (int32_t)e.code; }

// validate_plan, stage count, chain_instance, M >= 1 (simulator.hpp:264-274,
// 83).  Returns false when the outcome is already decided (r.status set).
BPK_HDNI bool tl_chain(const TlArgs& A, bp_timeline_result& r) {
    Err e{ERR_NONE};
    int64_t where = 0;
    Rat aux{0, 1};
    const int code = validate_frac(A.lo, A.hi, A.lead, A.trail, A.N, A.v.L, &where, &aux, e);
    if (e.bad()) { tl_fail(r, e); return false; }
    if (code) {
        r.status = BP_C_ERR_INVALID_PLAN;
        r.detail = code;
        r.detail2 = where;
        r.aux = bp_rat{aux.n, aux.d};
        return false;
    }
    if (A.N != A.clusterN) {
        r.status = BP_C_ERR_INVALID_PLAN;
        r.detail = BP_IP_STAGE_COUNT;
        return false;
    }
    const NetView& v = A.v;
    for (int s = 0; s < A.N; ++s) {   // F, B, a, w per stage, in chain_instance's order
        const int64_t t = A.c.type[s];
        A.F[s] = stage_sum_frac(A.lo[s], A.hi[s], A.lead[s], A.trail[s], v.Pfp + t * (v.L + 1), e);
        A.B[s] = stage_sum_frac(A.lo[s], A.hi[s], A.lead[s], A.trail[s], v.Pbp + t * (v.L + 1), e);
        const int64_t act = act_at(v, s >= 1 ? A.hi[s - 1] : A.hi[0], e);   // plan.hpp:144-148
        A.a[s] = act * A.micro;
        A.W[s] = stage_sum_frac(A.lo[s], A.hi[s], A.lead[s], A.trail[s], v.Pw, e);
        if (e.bad()) { tl_fail(r, e); return false; }
    }
    for (int k = 1; k < A.N; ++k) {   // link_sr_time (plan.hpp:152-158)
        const int64_t x = act_at(v, A.hi[k - 1], e) * A.micro;
        if (e.bad()) { tl_fail(r, e); return false; }
        A.SR[k - 1] = x == 0 ? 0 : ceil_div64(x, A.c.bw[k - 1]);
    }
    if (A.M < 1) {
        r.status = BP_C_ERR_INVALID_PLAN;
        r.detail = BP_IP_M;
        return false;
    }
    return true;
}

// Events of stage s (1-based) per mini-batch: FP and BP for every m, plus
// SEND_F / RECV_B on link s and RECV_F / SEND_B on link s-1 when that link's
// transfer time is not 0 (simulator.hpp:193-211).
BPK_HD int64_t tl_stage_events(const TlArgs& A, int s) {
    int64_t n = 2 * A.M;
    if (s <= A.N - 1 && A.SR[s - 1] != 0) n += 2 * A.M;
    if (s >= 2 && A.SR[s - 2] != 0) n += 2 * A.M;
    return n * A.mini;
}

// The op walk and the event list.  Ops run position by position; inside a
// position in the reference's (sub, type, stage, m) order (simulator.hpp:
// 105-125): stage s's compute op has sub 2s (F) or 2(N+1-s) (B), a forward
// transfer on link k sub 2k+1 (after F(m,k)), a backward one sub 2(N-k)+1
// (after B(m,k+1)); equal subs order by type.
BPK_HDNI bool tl_walk(const TlArgs& A, bp_timeline_result& r) {
    Err e{ERR_NONE};
    const int N = A.N;
    const int64_t M = A.M;
    const bool async = kind_async(A.kind);
    auto w_of = [&](int s) {   // 1-based stage
        int64_t w = warmup_depth(A.kind, N, s);
        return w < M ? w : M;
    };
    auto ix = [&](int64_t m, int s) { return (int64_t)(s - 1) * M + (m - 1); };
    // stage_free is the end of the stage's previous op (one op per position)
    for (int64_t p = 0; p < 2 * M; ++p) {
        for (int x = 2; x <= 2 * N + 1; ++x) {
            if ((x & 1) == 0) {
                const int s1 = x / 2;                   // F op of stage s1 at sub 2*s1
                const StageOp o1 = op_at(p, w_of(s1), M);
                if (o1.is_f) {
                    const int64_t m = o1.m;
                    // ready = stage_free: the previous op's end on this stage
                    Rat ready{0, 1};
                    if (p > 0) {
                        const StageOp pr = op_at(p - 1, w_of(s1), M);
                        ready = pr.is_f ? A.eF[ix(pr.m, s1)] : A.eB[ix(pr.m, s1)];
                    }
                    if (s1 > 1) {
                        const Rat arr = async ? A.eF[ix(m, s1 - 1)] : A.tFe[ix(m, s1 - 1)];
                        if (rat_gt(arr, ready)) ready = arr;
                    }
                    A.sF[ix(m, s1)] = ready;
                    A.eF[ix(m, s1)] = rat_add(ready, A.F[s1 - 1], e);
                    if (e.bad()) { tl_fail(r, e); return false; }
                }
                const int s2 = N + 1 - x / 2;           // B op of stage s2 at sub 2(N+1-s2)
                const StageOp o2 = op_at(p, w_of(s2), M);
                if (!o2.is_f) {
                    const int64_t m = o2.m;
                    Rat ready{0, 1};
                    if (p > 0) {
                        const StageOp pr = op_at(p - 1, w_of(s2), M);
                        ready = pr.is_f ? A.eF[ix(pr.m, s2)] : A.eB[ix(pr.m, s2)];
                    }
                    if (rat_gt(A.eF[ix(m, s2)], ready)) ready = A.eF[ix(m, s2)];
                    if (s2 < N) {
                        const Rat arr = async ? A.eB[ix(m, s2 + 1)] : A.tBe[ix(m, s2)];
                        if (rat_gt(arr, ready)) ready = arr;
                    }
                    A.sB[ix(m, s2)] = ready;
                    A.eB[ix(m, s2)] = rat_add(ready, A.B[s2 - 1], e);
                    if (e.bad()) { tl_fail(r, e); return false; }
                }
            } else if (!async) {
                const int k1 = (x - 1) / 2;             // forward transfer on link k1, after F(m, k1)
                if (k1 <= N - 1) {
                    const StageOp o = op_at(p, w_of(k1), M);
                    if (o.is_f) {
                        const Rat ready = A.eF[ix(o.m, k1)];
                        A.tFs[ix(o.m, k1)] = ready;
                        A.tFe[ix(o.m, k1)] = rat_add(ready, R(A.SR[k1 - 1]), e);
                        if (e.bad()) { tl_fail(r, e); return false; }
                    }
                }
                const int k2 = N - (x - 1) / 2;         // backward transfer on link k2, after B(m, k2+1)
                if (k2 >= 1) {
                    const StageOp o = op_at(p, w_of(k2 + 1), M);
                    if (!o.is_f) {
                        const Rat ready = A.eB[ix(o.m, k2 + 1)];
                        A.tBs[ix(o.m, k2)] = ready;
                        A.tBe[ix(o.m, k2)] = rat_add(ready, R(A.SR[k2 - 1]), e);
                        if (e.bad()) { tl_fail(r, e); return false; }
                    }
                }
            }
        }
    }
    // makespan (173-180): the stages' last ends, and in sync mode the last
    // micro-batch's transfers
    Rat mk{0, 1};
    for (int s = 1; s <= N; ++s) {
        const StageOp last = op_at(2 * M - 1, w_of(s), M);
        const Rat f = last.is_f ? A.eF[ix(last.m, s)] : A.eB[ix(last.m, s)];
        if (rat_gt(f, mk)) mk = f;
    }
    if (!async)
        for (int k = 1; k <= N - 1; ++k) {
            if (rat_gt(A.tFe[ix(M, k)], mk)) mk = A.tFe[ix(M, k)];
            if (rat_gt(A.tBe[ix(M, k)], mk)) mk = A.tBe[ix(M, k)];
        }
    *A.makespan1 = mk;
    // events (182-211) into per-stage segments; times + r * makespan
    int64_t o = 0;
    for (int s = 1; s <= N; ++s) {
        A.off[s - 1] = o;
        o += tl_stage_events(A, s);
    }
    A.off[N] = o;
    for (int64_t rr = 0; rr < A.mini; ++rr) {
        const Rat offr = rat_mul(R(rr), mk, e);
        if (e.bad()) { tl_fail(r, e); return false; }
        const int64_t moff = rr * M;
        auto put = [&](int st, int kind, int64_t m, Rat a0, Rat a1) {
            // slot: segment of stage st, block rr, then a fixed place per
            // (kind, m) -- the segment is sorted afterwards
            const int64_t per = tl_stage_events(A, st) / A.mini;
            int64_t base = A.off[st - 1] + rr * per;
            int64_t k;
            const bool out_link = st <= N - 1 && A.SR[st - 1] != 0;   // SEND_F / RECV_B here
            switch (kind) {
                case 0: k = m - 1; break;
                case 1: k = M + m - 1; break;
                case 2: k = 2 * M + m - 1; break;                                 // SEND_F (link st)
                case 5: k = 3 * M + m - 1; break;                                 // RECV_B (link st)
                case 3: k = (out_link ? 4 * M : 2 * M) + m - 1; break;            // RECV_F (link st-1)
                default: k = (out_link ? 5 * M : 3 * M) + m - 1; break;           // SEND_B (link st-1)
            }
            bp_event& x = A.ev[base + k];
            x.stage = st;
            x.kind = kind;
            x.pad = 0;
            x.micro_batch = m + moff;
            const Rat b0 = rat_add(a0, offr, e), b1 = rat_add(a1, offr, e);
            x.start = bp_rat{b0.n, b0.d};
            x.end = bp_rat{b1.n, b1.d};
        };
        for (int s = 1; s <= N; ++s)
            for (int64_t m = 1; m <= M; ++m) {
                put(s, 0, m, A.sF[ix(m, s)], A.eF[ix(m, s)]);
                put(s, 1, m, A.sB[ix(m, s)], A.eB[ix(m, s)]);
                if (e.bad()) { tl_fail(r, e); return false; }
            }
        for (int k = 1; k <= N - 1; ++k) {
            if (A.SR[k - 1] == 0) continue;
            for (int64_t m = 1; m <= M; ++m) {
                Rat fs, fe, bs, be;
                if (async) {
                    fs = A.sF[ix(m, k)], fe = A.eF[ix(m, k)];
                    bs = A.sB[ix(m, k + 1)], be = A.eB[ix(m, k + 1)];
                } else {
                    fs = A.tFs[ix(m, k)], fe = A.tFe[ix(m, k)];
                    bs = A.tBs[ix(m, k)], be = A.tBe[ix(m, k)];
                }
                put(k, 2, m, fs, fe);
                put(k + 1, 3, m, fs, fe);
                put(k + 1, 4, m, bs, be);
                put(k, 5, m, bs, be);
                if (e.bad()) { tl_fail(r, e); return false; }
            }
        }
    }
    const Rat total = rat_mul(R(A.mini), mk, e);   // t.makespan (213)
    if (e.bad()) { tl_fail(r, e); return false; }
    r.makespan = bp_rat{total.n, total.d};
    r.n_events = o;
    return true;
}

// (start, kind, micro-batch) within one stage (simulator.hpp:207-212)
BPK_HD bool ev_less(const bp_event& x, const bp_event& y) {
    const Rat a{x.start.num, x.start.den}, b{y.start.num, y.start.den};
    if (!rat_eq(a, b)) return rat_lt(a, b);
    if (x.kind != y.kind) return x.kind < y.kind;
    return x.micro_batch < y.micro_batch;
}

// bottom-up merge sort of v[0..n) with scratch t; less(a, b) strict
template <class T, class Less>
BPK_HD void tl_msort(T* v, T* t, int64_t n, Less less) {
    T* src = v;
    T* dst = t;
    for (int64_t w = 1; w < n; w *= 2) {
        for (int64_t i = 0; i < n; i += 2 * w) {
            const int64_t mid = i + w < n ? i + w : n, hi = i + 2 * w < n ? i + 2 * w : n;
            int64_t a = i, b = mid, k = i;
            while (a < mid && b < hi) dst[k++] = less(src[b], src[a]) ? src[b++] : src[a++];
            while (a < mid) dst[k++] = src[a++];
            while (b < hi) dst[k++] = src[b++];
        }
        T* x = src;
        src = dst;
        dst = x;
    }
    if (src != v)
        for (int64_t i = 0; i < n; ++i) v[i] = src[i];
}

struct TlPoint {
    Rat t;
    int32_t d;
};

// Stage s (1-based): sort its events; feature high-water = peak number of
// live activation buffers (FP start .. BP end, half-open, frees first at
// equal times) times a_s; static weights = 2 w_s (217-238).  Returns the
// error code (0 = none).
BPK_HDNI uint32_t tl_stage(const TlArgs& A, int s, TlPoint* pts, TlPoint* tmp, Rat* highwater, Rat* wstatic) {
    const int64_t b = A.off[s - 1], n = A.off[s] - b;
    tl_msort(A.ev + b, A.ev_tmp + b, n, [](const bp_event& x, const bp_event& y) { return ev_less(x, y); });
    const int64_t M = A.M;
    for (int64_t m = 1; m <= M; ++m) {
        pts[2 * (m - 1)] = TlPoint{A.sF[(int64_t)(s - 1) * M + (m - 1)], +1};
        pts[2 * (m - 1) + 1] = TlPoint{A.eB[(int64_t)(s - 1) * M + (m - 1)], -1};
    }
    tl_msort(pts, tmp, 2 * M, [](const TlPoint& x, const TlPoint& y) {
        if (!rat_eq(x.t, y.t)) return rat_lt(x.t, y.t);
        return x.d < y.d;
    });
    int64_t cur = 0, peak = 0;
    for (int64_t i = 0; i < 2 * M; ++i) {
        cur += pts[i].d;
        if (cur > peak) peak = cur;
    }
    Err e{ERR_NONE};
    highwater[s - 1] = rat_mul(R(peak), R(A.a[s - 1]), e);
    wstatic[s - 1] = rat_mul(R(2), A.W[s - 1], e);
    return e.code;
}

// per_link_busy_fraction (239-244)
BPK_HDNI uint32_t tl_busy(const TlArgs& A, Rat* busy) {
    Err e{ERR_NONE};
    const Rat mk = *A.makespan1;
    for (int k = 1; k <= A.N - 1; ++k) {
        if (mk.n == 0) busy[k - 1] = R(0);
        else busy[k - 1] = rat_div(R(A.M * A.SR[k - 1]), mk, e);
        if (e.bad()) break;
    }
    return e.code;
}

// estimate(kind, plan, ...) (cost_models.hpp:124-166) on a caller's plan:
// stage_costs (103-119) on the fractional plan, then the shared estimate
// code.  The caller checked the kind's mode and the stage count.
// scr: [7N] Rats, scr64: [2N].
BPK_HDNI void tl_estimate(const TlArgs& A, bp_estimate_result& r, bp_stage* st, int32_t* infeasible, Rat* scr,
                          int64_t* scr64) {
    Err e{ERR_NONE};
    const NetView& v = A.v;
    const int N = A.N;
    Rat *F = scr, *Bc = scr + N, *W = scr + 2 * N, *feat = scr + 3 * N, *wts = scr + 4 * N, *bw = scr + 5 * N,
        *Mem = scr + 6 * N;
    for (int s = 0; s < N; ++s) {
        const int64_t l = A.lo[s], h = A.hi[s];
        // a non-empty stage outside [1, L] reads past net.layers: UB there
        if (l <= h && (l < 1 || h > v.L)) { e.set(ERR_UB); break; }
        const int64_t t = A.c.type[s];
        F[s] = stage_sum_frac(l, h, A.lead[s], A.trail[s], v.Pfp + t * (v.L + 1), e);
        Bc[s] = stage_sum_frac(l, h, A.lead[s], A.trail[s], v.Pbp + t * (v.L + 1), e);
        W[s] = stage_sum_frac(l, h, A.lead[s], A.trail[s], v.Pw, e);
        if (e.bad()) break;
    }
    if (e.bad()) { r.status = (int32_t)e.code; return; }
    CachedPlan cp{A.hi, F, Bc, W};
    // estimate() writes its per-stage F/B/W copies, memory, a and SR here
    EstScratch S{feat, wts, bw, Mem, scr64, scr64 + N};
    EstOut o;
    estimate(cp, v, A.c, A.kind, A.M, A.micro, S, o, nullptr, e);
    if (e.bad()) { r.status = (int32_t)e.code; return; }
    // features / weights / bandwidth demand exactly as estimate formed them
    const bool dbl = (A.kind == KIND_FBP || A.kind == KIND_SO);
    Err dummy{ERR_NONE};
    r.status = BP_C_OK;
    r.heuristic = o.heuristic;
    r.minibatch_time = bp_rat{o.minibatch.n, o.minibatch.d};
    r.bubble_fraction = bp_rat{o.bubble.n, o.bubble.d};
    for (int s = 0; s < N; ++s) {
        Rat fm = rat_mul(R(N - s), R(S.A[s]), dummy);
        if (dbl) fm = rat_mul(R(2), fm, dummy);
        const Rat wm = rat_mul(R(2), W[s], dummy);
        st[s].lo = A.lo[s];
        st[s].hi = A.hi[s];
        st[s].lead = bp_rat{A.lead[s].n, A.lead[s].d};
        st[s].trail = bp_rat{A.trail[s].n, A.trail[s].d};
        st[s].features = bp_rat{fm.n, fm.d};
        st[s].weights = bp_rat{wm.n, wm.d};
        if (s + 1 < N) {
            const Rat d = (A.kind == KIND_FBP)
                              ? rat_div(rat_mul(R(2), R(S.A[s + 1]), dummy), rat_add(o.Fm, o.Bm, dummy), dummy)
                              : rat_div(R(S.A[s + 1]), o.Fm, dummy);
            st[s].bw_demand = bp_rat{d.n, d.d};
        } else {
            st[s].bw_demand = bp_rat{0, 1};
        }
        infeasible[s] = rat_gt(Mem[s], R(A.c.cap[s])) ? 1 : 0;
    }
}

}  // namespace bpk
