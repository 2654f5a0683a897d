// model.cuh -- exact device emulation of the reference's per-candidate logic:
//   estimate           cost_models.hpp:124-166 (+ stage_costs 103-119)
//   validate_plan      plan.hpp:41-85
//   memory_fine_tune   partition.hpp:339-435
//   intra_layer_refine partition.hpp:248-333
// Every Rat operation the reference performs on a path is performed here on
// the same values (so overflow/domain errors match), and every layer read
// the reference performs is bounds-checked (so its undefined behaviour is
// reported, not silently different).  The first error wins.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace bpk {

struct IntE {
    int r;
    uint32_t err;
};

// ---------------------------------------------------------------------------
// Plan sources for estimate(): per-stage F, B, W and the stage's hi.
struct WholePlan {          // fractions all 1 (DP / coarse / fine-tuned plans)
    const NetView* v;
    const ChainView* c;
    const int32_t* lo;
    const int32_t* hi;
    BPK_HD int64_t H(int s) const { return hi[s]; }
    // stage_fp_time etc. for a whole-layer stage; a non-empty stage outside
    // [1, L] would read past net.layers (UB in the reference).
    BPK_HD void FBW(int s, Rat& F, Rat& B, Rat& W, Err& e) const {
        int64_t l = lo[s], h = hi[s];
        if (l <= h && (l < 1 || h > v->L)) { e.set(ERR_UB); F = B = W = Rat{0, 1}; return; }
        int32_t t = c->type[s];
        F = R(stage_sum_whole(l, h, v->Pfp + (int64_t)t * (v->L + 1)));
        B = R(stage_sum_whole(l, h, v->Pbp + (int64_t)t * (v->L + 1)));
        W = R(stage_sum_whole(l, h, v->Pw));
    }
};

struct CachedPlan {         // refined plan: F/B/W computed once per query
    const int32_t* hi;
    const Rat *F, *B, *W;
    BPK_HD int64_t H(int s) const { return hi[s]; }
    BPK_HD void FBW(int s, Rat& f, Rat& b, Rat& w, Err&) const {
        f = F[s];
        b = B[s];
        w = W[s];
    }
};

struct EstOut {
    Rat minibatch, bubble, Fm, Bm;
    int heuristic;
    int feasible;
    // overloads() (partition.hpp:344-356), computed after the estimate
    Rat total_over;     // sum of max(mem - cap, 0)
    int worst;          // first index of the maximal overload
    Rat peak_mem;       // max_i(features_i + weights_i) (explorer.hpp:405-408)
    Rat max_bw;         // max bandwidth demand (explorer.hpp:409-410)
    int trials = 0;     // memory_fine_tune trial moves (instrumentation)
    int fb_balanced = 1;   // all stages' F equal and all B equal (heuristic's link-independent part)
};

// Optional per-stage outputs (features, weights, bw demand), may be null.
struct EstStageOut {
    Rat *features, *weights, *bw;
};

// Per-stage scratch of length N (caller-provided; local or global memory).
struct EstScratch {
    Rat *F, *B, *W, *Mem;
    int64_t *A, *SR;
};

// minibatch_time, cost_models.hpp:50-63
BPK_HD Rat minibatch_time(int kind, int64_t M, int64_t N, Rat F, Rat B, Rat SR, Err& e) {
    Rat base = rat_mul(R(M + N - 1), rat_add(F, B, e), e);
    if (kind == KIND_SNO)
        return rat_add(base, rat_mul(rat_mul(R(N + M - 2 - ceil_div64(M - 1, N)), R(2), e), SR, e), e);
    if (kind == KIND_SO) return rat_add(base, rat_mul(rat_mul(R(N - 1), R(2), e), SR, e), e);
    return base;
}

// bubble_fraction, cost_models.hpp:65-82
BPK_HD Rat bubble_fraction(int kind, int64_t M, int64_t N, Rat F, Rat B, Rat SR, Err& e) {
    if (N == 1) return Rat{0, 1};
    Rat total = minibatch_time(kind, M, N, F, B, SR, e);
    if (kind == KIND_SNO) {
        Rat inner = rat_add(rat_add(F, B, e), rat_mul(R(2), SR, e), e);
        Rat num = rat_add(rat_mul(R(N - 1), inner, e),
                          rat_mul(rat_mul(R(M - 1 - ceil_div64(M - 1, N)), R(2), e), SR, e), e);
        return rat_div(num, total, e);
    }
    if (kind == KIND_SO) {
        Rat inner = rat_add(rat_add(F, B, e), rat_mul(R(2), SR, e), e);
        return rat_div(rat_mul(R(N - 1), inner, e), total, e);
    }
    return rat_nd(N - 1, M + N - 1, e);
}

// link_sr_time (plan.hpp:152-158) for the link after stage index k0 (0-based).
template <class PS>
BPK_HD int64_t link_sr(const PS& p, const NetView& v, const ChainView& c, int k0,
                                           int64_t micro, Err& e) {
    int64_t a = act_at(v, p.H(k0), e) * micro;
    if (a == 0) return 0;
    return ceil_div64(a, c.bw[k0]);
}

// estimate(kind, plan, net, cluster, M, micro), cost_models.hpp:124-166.
BPK_HD bool ft_int_ok(const NetView& v, const ChainView& c, int64_t M, int64_t micro);
BPK_HD void estimate_whole_int(const WholePlan& p, const NetView& v, const ChainView& c, int kind, int64_t M,
                               int64_t micro, const EstScratch& s, EstOut& o, Err& e);

template <class PS>
BPK_HD void estimate_body(const PS& p, const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro,
                         const EstScratch& s, EstOut& o, const EstStageOut* so, Err& e) {
    if constexpr (std::is_same<PS, WholePlan>::value) {
        if (!so && ft_int_ok(v, c, M, micro)) {   // every value an integer in range: int64 (below)
            estimate_whole_int(p, v, c, kind, M, micro, s, o, e);
            return;
        }
    }
    const int N = c.N;
    // stage_costs (103-119), stage order F, B, w, a, SR
    for (int i = 0; i < N; ++i) {
        p.FBW(i, s.F[i], s.B[i], s.W[i], e);
        if (e.bad()) return;
        int64_t act = (i >= 1) ? act_at(v, p.H(i - 1), e) : act_at(v, p.H(0), e);
        if (e.bad()) return;
        s.A[i] = act * micro;
        s.SR[i] = (i >= 1) ? link_sr(p, v, c, i - 1, micro, e) : 0;
        if (e.bad()) return;
    }
    Rat Fm{0, 1}, Bm{0, 1};
    int64_t SRm = 0;
    bool balanced = true;
    for (int i = 0; i < N; ++i) {
        if (!rat_eq(s.F[i], s.F[0]) || !rat_eq(s.B[i], s.B[0])) balanced = false;
        if (rat_gt(s.F[i], Fm)) Fm = s.F[i];
        if (rat_gt(s.B[i], Bm)) Bm = s.B[i];
        if (s.SR[i] > SRm) SRm = s.SR[i];
    }
    const bool fb_bal = balanced;   // F and B (the SR part depends on the links)
    for (int i = 1; i < N; ++i)
        if (s.SR[i] != s.SR[N > 1 ? 1 : 0]) balanced = false;
    o.Fm = Fm;
    o.Bm = Bm;
    o.minibatch = minibatch_time(kind, M, N, Fm, Bm, R(SRm), e);
    o.bubble = bubble_fraction(kind, M, N, Fm, Bm, R(SRm), e);
    o.heuristic = (!balanced || M < N) ? 1 : 0;
    o.fb_balanced = fb_bal ? 1 : 0;
    if (e.bad()) return;
    o.feasible = 1;
    o.peak_mem = Rat{0, 1};
    const bool dbl = (kind == KIND_FBP || kind == KIND_SO);
    for (int i = 0; i < N; ++i) {
        // features_memory (86-91), weights_memory (94), mem check (152-160)
        Rat fm = rat_mul(R(N - i), R(s.A[i]), e);
        if (dbl) fm = rat_mul(R(2), fm, e);
        Rat wm = rat_mul(R(2), s.W[i], e);
        Rat mem = rat_add(fm, wm, e);
        if (e.bad()) return;
        s.Mem[i] = mem;
        if (rat_gt(mem, R(c.cap[i]))) o.feasible = 0;
        if (so) { so->features[i] = fm; so->weights[i] = wm; }
        if (rat_gt(mem, o.peak_mem)) o.peak_mem = mem;
    }
    // bandwidth_demand (97-100) per link (161-164)
    o.max_bw = Rat{0, 1};
    if (!so && N > 1) {
        // every link's demand is a / Fm (2a / (Fm + Bm) for fbp-as): one
        // denominator, so the largest cut activation gives the largest
        // demand.  When a_max * den(Fm) < 2^62 no link's quotient can leave
        // int64, and the first error (if any) is the first out-of-range layer
        // read, exactly as the per-link loop would raise them.
        int64_t amax = 0;
        int kub = N - 1;
        for (int k = 0; k + 1 < N; ++k) {
            const int64_t j = p.H(k);
            if (j < 1 || j > v.L) { kub = k; break; }
            const int64_t a = v.a[j - 1] * micro;
            if (a > amax) amax = a;
        }
        Err le{ERR_NONE};
        const Rat den = (kind == KIND_FBP) ? rat_add(Fm, Bm, le) : Fm;
        const i128 top = (kind == KIND_FBP) ? 2 * (i128)amax : (i128)amax;
        if (!le.bad() && den.n > 0 && amax >= 0 && top * den.d < ((i128)1 << 62)) {
            if (kub < N - 1) { e.set(ERR_UB); return; }
            o.max_bw = rat_div(R((int64_t)top), den, e);
            return;
        }
    }
    for (int k = 0; k + 1 < N; ++k) {
        Rat a = R(act_at(v, p.H(k), e) * micro);
        Rat d;
        if (kind == KIND_FBP) d = rat_div(rat_mul(R(2), a, e), rat_add(Fm, Bm, e), e);
        else d = rat_div(a, Fm, e);
        if (e.bad()) return;
        if (so) so->bw[k] = d;
        if (rat_gt(d, o.max_bw)) o.max_bw = d;
    }
}

// out of line; the error latch travels by value (see RatE in rat.cuh)
template <class PS>
BPK_HDNI uint32_t estimate_v(const PS& p, const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, const EstScratch& s, EstOut& o, const EstStageOut* so, uint32_t ecode) {
    Err e{ecode};
    estimate_body(p, v, c, kind, M, micro, s, o, so, e);
    return e.code;
}
template <class PS>
BPK_HD void estimate(const PS& p, const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, const EstScratch& s, EstOut& o, const EstStageOut* so, Err& e) { e.code = estimate_v(p, v, c, kind, M, micro, s, o, so, e.code); }

// estimate() of a whole-layer plan that differs from the one whose estimate
// is in s / o only in the adjacent stages i0 < i1 (a memory_fine_tune trial
// move, partition.hpp:403-410).  The reference recomputes the whole estimate
// (cost_models.hpp:124-166) for every trial; the per-stage values of the
// other stages are the ones it computed before, with the same (absent)
// errors, so only stages i0, i1, the cut between them and the aggregates are
// recomputed here.  On a whole-layer plan F, B, W are integers, so the
// per-link bandwidth demands a / Fm (or 2a / (Fm + Bm) for fbp-as) cannot
// leave int64 once 2a and Fm + Bm fit: they are not formed during trials
// (o.max_bw is left stale; the caller recomputes it for the final plan).
BPK_HD void estimate_move_body(const WholePlan& p, const NetView& v, const ChainView& c, int kind, int64_t M,
                            int64_t micro, const EstScratch& s, EstOut& o, int i0, int i1, Err& e) {
    const int N = c.N;
    const bool dbl = (kind == KIND_FBP || kind == KIND_SO);
    // stage_costs (103-119) for the two stages, in the reference's order; the
    // cut between them is stage i1's input (and stage 0's own activation unit
    // is its output cut, plan.hpp:144-148)
    for (int i = i0; i <= i1; ++i) {
        p.FBW(i, s.F[i], s.B[i], s.W[i], e);
        if (e.bad()) return;
        if (i == i1 || i == 0) {
            const int64_t act = (i >= 1) ? act_at(v, p.H(i - 1), e) : act_at(v, p.H(0), e);
            if (e.bad()) return;
            s.A[i] = act * micro;
            if (i >= 1) {
                s.SR[i] = link_sr(p, v, c, i - 1, micro, e);
                if (e.bad()) return;
            }
        }
    }
    Rat Fm{0, 1}, Bm{0, 1};
    int64_t SRm = 0;
    bool balanced = true;
    for (int i = 0; i < N; ++i) {
        if (!rat_eq(s.F[i], s.F[0]) || !rat_eq(s.B[i], s.B[0])) balanced = false;
        if (rat_gt(s.F[i], Fm)) Fm = s.F[i];
        if (rat_gt(s.B[i], Bm)) Bm = s.B[i];
        if (s.SR[i] > SRm) SRm = s.SR[i];
    }
    const bool fb_bal = balanced;   // F and B (the SR part depends on the links)
    for (int i = 1; i < N; ++i)
        if (s.SR[i] != s.SR[N > 1 ? 1 : 0]) balanced = false;
    o.Fm = Fm;
    o.Bm = Bm;
    o.minibatch = minibatch_time(kind, M, N, Fm, Bm, R(SRm), e);
    o.bubble = bubble_fraction(kind, M, N, Fm, Bm, R(SRm), e);
    o.heuristic = (!balanced || M < N) ? 1 : 0;
    o.fb_balanced = fb_bal ? 1 : 0;
    if (e.bad()) return;
    for (int i = i0; i <= i1; ++i) {
        Rat fm = rat_mul(R(N - i), R(s.A[i]), e);
        if (dbl) fm = rat_mul(R(2), fm, e);
        Rat wm = rat_mul(R(2), s.W[i], e);
        s.Mem[i] = rat_add(fm, wm, e);
        if (e.bad()) return;
    }
    o.feasible = 1;
    o.peak_mem = Rat{0, 1};
    for (int i = 0; i < N; ++i) {
        if (rat_gt(s.Mem[i], R(c.cap[i]))) o.feasible = 0;
        if (rat_gt(s.Mem[i], o.peak_mem)) o.peak_mem = s.Mem[i];
    }
    // the bandwidth-demand operations that could overflow (see above)
    if (kind == KIND_FBP) {
        (void)rat_add(Fm, Bm, e);
        for (int k = 0; k + 1 < N; ++k) (void)rat_mul(R(2), R(s.A[k + 1]), e);
    }
}

// out of line; the error latch travels by value (see RatE in rat.cuh)
BPK_HDNI uint32_t estimate_move_v(const WholePlan& p, const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, const EstScratch& s, EstOut& o, int i0, int i1, uint32_t ecode) {
    Err e{ecode};
    estimate_move_body(p, v, c, kind, M, micro, s, o, i0, i1, e);
    return e.code;
}
BPK_HD void estimate_move(const WholePlan& p, const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, const EstScratch& s, EstOut& o, int i0, int i1, Err& e) { e.code = estimate_move_v(p, v, c, kind, M, micro, s, o, i0, i1, e.code); }

// overloads() bookkeeping (partition.hpp:344-356) on the estimate in s.Mem:
// ov = mem > cap ? mem - cap : 0; total += ov; worst = first max (381-383).
// Only memory_fine_tune performs these Rat operations in the reference, so
// only its call sites run this.
BPK_HD void overloads_from_mem(const ChainView& c, const EstScratch& s, EstOut& o, Err& e) {
    o.total_over = Rat{0, 1};
    o.worst = 0;
    Rat worst_over{0, 1};
    for (int i = 0; i < c.N; ++i) {
        Rat cap = R(c.cap[i]);
        Rat ov = rat_gt(s.Mem[i], cap) ? rat_sub(s.Mem[i], cap, e) : Rat{0, 1};
        o.total_over = rat_add(o.total_over, ov, e);
        if (i > 0 && rat_gt(ov, worst_over)) o.worst = i;
        if (i == 0 || rat_gt(ov, worst_over)) worst_over = ov;
    }
}

// Note on the mem values: overloads() (partition.hpp:349) and explore()
// (explorer.hpp:406) recompute features + weights -- identical values to the
// estimate's own sum, hence identical overflow behaviour; computed once here.

// ---------------------------------------------------------------------------
// validate_plan (plan.hpp:41-85) for a whole-layer plan (all fractions 1).
// Returns 0 or BP_IP_* with *where = stage (1-based) / layer.
BPK_HD int validate_whole(const int32_t* lo, const int32_t* hi, int N, int64_t L,
                                              int64_t* where) {
    int64_t prev_hi = 0;
    for (int n = 0; n < N; ++n) {
        if (lo[n] < 1 || hi[n] > L || lo[n] > hi[n]) { *where = n + 1; return 1; }   // RANGE
        if (n == 0) {
            if (lo[n] != 1) { *where = 1; return 3; }                                // FIRST
        } else {
            bool shared = (lo[n] == prev_hi);
            if (!shared && lo[n] != prev_hi + 1) { *where = n + 1; return 4; }      // CONTIG
            if (shared) { *where = n + 1; return 5; }                                // SHARED_FULL (lead == 1)
        }
        prev_hi = hi[n];
    }
    if (hi[N - 1] != L) { *where = 0; return 7; }                                    // LAST
    return 0;   // coverage of a contiguous whole plan sums to exactly 1
}

// validate_plan for a fractional (refined) plan, including the exact Rat
// coverage sums of the reference's O(L*N) loop (78-84): only layers on a
// stage boundary can have more than one owner; their sums are formed in
// stage order exactly as `sum += owned_fraction(s, j)` does.
BPK_HDNI int validate_frac(const int32_t* lo, const int32_t* hi, const Rat* lead, const Rat* trail, int N,
                             int64_t L, int64_t* where, Rat* aux, Err& e) {
    int64_t prev_hi = 0;
    const Rat one{1, 1}, zero{0, 1};
    for (int n = 0; n < N; ++n) {
        if (lo[n] < 1 || hi[n] > L || lo[n] > hi[n]) { *where = n + 1; return 1; }
        if (!rat_gt(lead[n], zero) || rat_gt(lead[n], one) || !rat_gt(trail[n], zero) || rat_gt(trail[n], one)) {
            *where = n + 1;
            return 2;
        }
        if (n == 0) {
            if (lo[n] != 1 || !rat_eq(lead[n], one)) { *where = 1; return 3; }
        } else {
            bool shared = (lo[n] == prev_hi);
            if (!shared && lo[n] != prev_hi + 1) { *where = n + 1; return 4; }
            if (shared && rat_eq(lead[n], one)) { *where = n + 1; return 5; }
            if (!shared && !rat_eq(lead[n], one)) { *where = n + 1; return 6; }
        }
        prev_hi = hi[n];
    }
    if (hi[N - 1] != L || !rat_eq(trail[N - 1], one)) { *where = 0; return 7; }
    // coverage: walk layers in order; a layer j is owned by the run of
    // consecutive stages whose range contains it.
    int n = 0;
    for (int64_t j = 1; j <= L;) {
        while (n < N && hi[n] < j) ++n;           // first stage containing j
        // interior layer of a single stage: owned fraction 1, sum = 1
        if (lo[n] < j && j < hi[n]) { j = hi[n]; continue; }
        Rat sum{0, 1};
        for (int m = n; m < N && lo[m] <= j; ++m) {
            if (hi[m] < j) continue;
            Rat own;
            if (lo[m] == hi[m]) own = rat_sub(rat_add(lead[m], trail[m], e), R(1), e);
            else if (j == lo[m]) own = lead[m];
            else if (j == hi[m]) own = trail[m];
            else own = R(1);
            sum = rat_add(sum, own, e);
            if (e.bad()) return 0;
        }
        if (!rat_eq(sum, one)) { *where = j; *aux = sum; return 8; }
        ++j;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// memory_fine_tune (partition.hpp:339-435) on a plan held in lo/hi.
// o / s must hold the estimate of the input plan (the caller computed it with
// the same scratch); overloads() bookkeeping is added here.  frac_lead / frac_trail (nullable) are the input plan's
// fractions, used by the collapse step (359-373); at boundary n the loop
// only ever compares the ORIGINAL trail[n] and lead[n+1] (each is mutated
// only by its own boundary), so the originals suffice.
// Returns FT_OK (plan in lo/hi, estimate of it in o/scratch) or FT_REJ /
// FT_NOCONV; errors go to e.
enum { FT_OK = 0, FT_REJ = 3, FT_NOCONV = 4 };

// Once memory_fine_tune has collapsed the plan to whole layers, every Rat its
// trial estimates form is an integer (sums of layer costs, products with
// integers, quotients that are only compared).  ft_int_ok bounds all of them
// for this candidate from the network totals (costs, weights and activations
// are >= 0, fp/bp >= 1: profiles.hpp:83-98), so that none can leave int64:
//   features + weights of a stage  <= 2 N amax micro + 2 W_total
//   total overload                 <= N * that
//   minibatch_time, bubble_fraction terms <= (M + N)(F_tot + B_tot) + 4 (M + N) amax micro
// (bandwidth demands a / Fm, 2a / (Fm + Bm) are quotients of such integers,
// Fm >= 1).  Under the bound the reference's trials cannot raise, so they can
// be decided with int64 arithmetic (fine_tune_int).
BPK_HD bool ft_int_ok(const NetView& v, const ChainView& c, int64_t M, int64_t micro) {
    const int N = c.N;
    if (micro < 0 || M < 1 || v.L < 1) return false;
    int64_t amax = v.a[v.L - 1];
    if (v.L >= 2 && v.asort[v.L - 2] > amax) amax = v.asort[v.L - 2];   // asort: first L-1, ascending
    int64_t ft = 0, bt = 0;
    for (int s = 0; s < N; ++s) {
        const int64_t o = (int64_t)c.type[s] * (v.L + 1) + v.L;
        if (v.Pfp[o] > ft) ft = v.Pfp[o];
        if (v.Pbp[o] > bt) bt = v.Pbp[o];
    }
    const i128 lim = (i128)1 << 61;
    const i128 A = (i128)amax * micro;
    if (amax < 0 || A >= lim) return false;
    const i128 mem = 2 * (i128)N * A + 2 * (i128)v.Pw[v.L];
    if ((i128)N * mem >= lim) return false;
    return (i128)(M + N) * ((i128)ft + bt) + 4 * (i128)(M + N) * A < lim;
}

// estimate() (cost_models.hpp:124-166) of a whole-layer plan under ft_int_ok:
// every value it forms is an integer below 2^61, so the same values come from
// int64 arithmetic and no operation can raise (the UB reads are checked as
// in the exact path, in the same order).  Of the outputs only the bubble
// fraction and the largest bandwidth demand are fractions: every link's
// demand has the same denominator (Fm, or Fm + Bm for fbp-as), so the largest
// cut activation gives the largest demand -- one reduction each instead of
// one per link.
BPK_HD void estimate_whole_int(const WholePlan& p, const NetView& v, const ChainView& c, int kind, int64_t M,
                               int64_t micro, const EstScratch& s, EstOut& o, Err& e) {
    const int N = c.N;
    for (int i = 0; i < N; ++i) {   // stage_costs (103-119)
        p.FBW(i, s.F[i], s.B[i], s.W[i], e);
        if (e.bad()) return;
        const int64_t act = (i >= 1) ? act_at(v, p.H(i - 1), e) : act_at(v, p.H(0), e);
        if (e.bad()) return;
        s.A[i] = act * micro;
        s.SR[i] = (i >= 1) ? link_sr(p, v, c, i - 1, micro, e) : 0;
        if (e.bad()) return;
    }
    int64_t Fm = 0, Bm = 0, SRm = 0;
    bool balanced = true;
    for (int i = 0; i < N; ++i) {
        if (s.F[i].n != s.F[0].n || s.B[i].n != s.B[0].n) balanced = false;
        if (s.F[i].n > Fm) Fm = s.F[i].n;
        if (s.B[i].n > Bm) Bm = s.B[i].n;
        if (s.SR[i] > SRm) SRm = s.SR[i];
    }
    const bool fb_bal = balanced;   // F and B (the SR part depends on the links)
    for (int i = 1; i < N; ++i)
        if (s.SR[i] != s.SR[N > 1 ? 1 : 0]) balanced = false;
    o.Fm = R(Fm);
    o.Bm = R(Bm);
    int64_t mb = (M + N - 1) * (Fm + Bm);                         // minibatch_time (50-63)
    if (kind == KIND_SNO) mb += (N + M - 2 - ceil_div64(M - 1, N)) * 2 * SRm;
    else if (kind == KIND_SO) mb += (int64_t)(N - 1) * 2 * SRm;
    o.minibatch = R(mb);
    if (N == 1) o.bubble = Rat{0, 1};                               // bubble_fraction (65-82)
    else if (kind == KIND_SNO)
        o.bubble = rat_div(R((int64_t)(N - 1) * (Fm + Bm + 2 * SRm) + (M - 1 - ceil_div64(M - 1, N)) * 2 * SRm),
                           R(mb), e);
    else if (kind == KIND_SO) o.bubble = rat_div(R((int64_t)(N - 1) * (Fm + Bm + 2 * SRm)), R(mb), e);
    else o.bubble = rat_nd(N - 1, M + N - 1, e);
    o.heuristic = (!balanced || M < N) ? 1 : 0;
    o.fb_balanced = fb_bal ? 1 : 0;
    if (e.bad()) return;
    o.feasible = 1;
    const int64_t fmul = (kind == KIND_FBP || kind == KIND_SO) ? 2 : 1;
    int64_t peak = 0;
    for (int i = 0; i < N; ++i) {                                   // memory check (152-160)
        const int64_t mem = (int64_t)(N - i) * s.A[i] * fmul + 2 * s.W[i].n;
        s.Mem[i] = R(mem);
        if (mem > c.cap[i]) o.feasible = 0;
        if (mem > peak) peak = mem;
    }
    o.peak_mem = R(peak);
    int64_t amax = 0;                                               // bandwidth_demand (161-164)
    for (int k = 0; k + 1 < N; ++k) {
        const int64_t a = act_at(v, p.H(k), e) * micro;
        if (e.bad()) return;
        if (a > amax) amax = a;
    }
    if (N < 2) o.max_bw = Rat{0, 1};
    else if (kind == KIND_FBP) o.max_bw = rat_div(R(2 * amax), R(Fm + Bm), e);
    else o.max_bw = rat_div(R(amax), R(Fm), e);
}

// memory_fine_tune's trial loop (partition.hpp:375-433) under ft_int_ok: the
// same moves, in the same order, accepted on the same comparisons, but only
// the values a decision reads are formed -- stage i0/i1 costs, the overloads,
// and on a non-relaxed improvement max(F + B) against the link times.  The
// accepted plan's full estimate is then recomputed exactly.
BPK_HD int fine_tune_int(const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, int32_t* lo,
                           int32_t* hi, const EstScratch& s, EstOut& o, Err& e, int64_t total, int worst,
                           int limit) {
    const int N = c.N;
    const int64_t fmul = (kind == KIND_FBP || kind == KIND_SO) ? 2 : 1;
    WholePlan wp{&v, &c, lo, hi};
    int guard = 0, trials = 0;
    // a trial changes stages i0, i1 only: its total overload is the current
    // one with their two terms replaced (exact: every value is an integer
    // below 2^61, ft_int_ok); the worst stage and the bottleneck test are
    // formed over all stages only for a trial whose total improves
    auto over = [&](int i, int64_t mem) { return mem > c.cap[i] ? mem - c.cap[i] : (int64_t)0; };
    while (total > 0) {
        if (++guard > limit) { o.trials = trials; return FT_NOCONV; }
        int cn[2], cd[2], nc = 0;
        if (worst > 0) { cn[nc] = worst - 1; cd[nc] = -1; ++nc; }
        if (worst < N - 1) { cn[nc] = worst + 1; cd[nc] = +1; ++nc; }
        if (nc == 2 && c.cap[worst + 1] - s.Mem[worst + 1].n > c.cap[worst - 1] - s.Mem[worst - 1].n) {
            int t = cn[0]; cn[0] = cn[1]; cn[1] = t;
            t = cd[0]; cd[0] = cd[1]; cd[1] = t;
        }
        bool moved = false;
        for (int relax = 0; relax < 2 && !moved; ++relax) {
            for (int ci = 0; ci < nc; ++ci) {
                if (lo[worst] == hi[worst]) continue;
                const int nb = cn[ci];
                const int32_t sw_lo = lo[worst], sw_hi = hi[worst], sn_lo = lo[nb], sn_hi = hi[nb];
                if (cd[ci] < 0) { lo[worst] += 1; hi[nb] += 1; }
                else { hi[worst] -= 1; lo[nb] -= 1; }
                const int i0 = worst < nb ? worst : nb, i1 = i0 + 1;
                const Rat kF[2] = {s.F[i0], s.F[i1]}, kB[2] = {s.B[i0], s.B[i1]}, kW[2] = {s.W[i0], s.W[i1]},
                          kM[2] = {s.Mem[i0], s.Mem[i1]};
                const int64_t kA[3] = {s.A[0], s.A[i1], s.SR[i1]};
                for (int i = i0; i <= i1; ++i) {           // stage_costs (cost_models.hpp:103-119)
                    wp.FBW(i, s.F[i], s.B[i], s.W[i], e);
                    if (i == i1 || i == 0) {
                        const int64_t act = (i >= 1) ? act_at(v, wp.H(i - 1), e) : act_at(v, wp.H(0), e);
                        s.A[i] = act * micro;
                        if (i >= 1) s.SR[i] = link_sr(wp, v, c, i - 1, micro, e);
                    }
                    if (e.bad()) return FT_OK;
                    s.Mem[i] = R((int64_t)(N - i) * s.A[i] * fmul + 2 * s.W[i].n);
                }
                ++trials;
                // overloads (partition.hpp:344-356, 381-383)
                const int64_t tot = total - over(i0, kM[0].n) - over(i1, kM[1].n) + over(i0, s.Mem[i0].n) +
                                    over(i1, s.Mem[i1].n);
                bool ok = tot < total;
                int wi = 0;
                if (ok) {
                    int64_t wo = 0;
                    for (int i = 0; i < N; ++i) {
                        const int64_t ov = over(i, s.Mem[i].n);
                        if (i == 0 || ov > wo) { wo = ov; wi = i; }
                    }
                }
                if (ok && !relax) {
                    int64_t target = 0;                         // max_stage_compute_time
                    for (int n = 0; n < N; ++n) {
                        const int64_t t = s.F[n].n + s.B[n].n;
                        if (t > target) target = t;
                    }
                    for (int k = 0; k + 1 < N; ++k)             // detect_comm_bottleneck
                        if (s.SR[k + 1] > target) ok = false;
                }
                if (ok) {
                    total = tot;
                    worst = wi;
                    moved = true;
                    break;
                }
                lo[worst] = sw_lo; hi[worst] = sw_hi; lo[nb] = sn_lo; hi[nb] = sn_hi;
                s.F[i0] = kF[0]; s.F[i1] = kF[1];
                s.B[i0] = kB[0]; s.B[i1] = kB[1];
                s.W[i0] = kW[0]; s.W[i1] = kW[1];
                s.Mem[i0] = kM[0]; s.Mem[i1] = kM[1];
                s.A[0] = kA[0]; s.A[i1] = kA[1]; s.SR[i1] = kA[2];
            }
        }
        if (!moved) { o.trials = trials; return FT_REJ; }
    }
    o.trials = trials;
    if (trials) estimate(wp, v, c, kind, M, micro, s, o, nullptr, e);
    return FT_OK;
}

BPK_HD int memory_fine_tune_body(const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro,
                                 int32_t* lo, int32_t* hi, const Rat* frac_lead, const Rat* frac_trail,
                                 const EstScratch& s, EstOut& o, Err& e) {
    const int N = c.N;
    overloads_from_mem(c, s, o, e);                        // first overloads() (357)
    if (e.bad()) return FT_OK;
    if (rat_eq(o.total_over, Rat{0, 1})) return FT_OK;   // identity
    if (frac_lead) {
        for (int n = 0; n < N - 1; ++n) {
            if (hi[n] != lo[n + 1]) continue;
            if (rat_ge(frac_trail[n], frac_lead[n + 1])) lo[n + 1] = hi[n] + 1;
            else hi[n] = hi[n] - 1;
        }
    }
    WholePlan wp{&v, &c, lo, hi};
    estimate(wp, v, c, kind, M, micro, s, o, nullptr, e);
    if (!e.bad()) overloads_from_mem(c, s, o, e);
    if (e.bad()) return FT_OK;
    Rat total = o.total_over;
    int worst = o.worst;
    int guard = 0, trials = 0;
    const int limit = 8 * (int)((int64_t)N * v.L + 4);
    if (total.d == 1 && ft_int_ok(v, c, M, micro))
        return fine_tune_int(v, c, kind, M, micro, lo, hi, s, o, e, total.n, worst, limit);
    const Rat zero{0, 1};
    while (rat_gt(total, zero)) {
        if (++guard > limit) { o.trials = trials; return FT_NOCONV; }
        int cn[2], cd[2], nc = 0;
        if (worst > 0) { cn[nc] = worst - 1; cd[nc] = -1; ++nc; }
        if (worst < N - 1) { cn[nc] = worst + 1; cd[nc] = +1; ++nc; }
        if (nc == 2) {
            // headroom(i) = cap_i - (features_i + weights_i) on the current
            // plan, whose estimate is the one in the scratch right now.
            Rat hr = rat_sub(R(c.cap[worst + 1]), s.Mem[worst + 1], e);
            Rat hl = rat_sub(R(c.cap[worst - 1]), s.Mem[worst - 1], e);
            if (e.bad()) return FT_OK;
            if (rat_gt(hr, hl)) {
                int t = cn[0]; cn[0] = cn[1]; cn[1] = t;
                t = cd[0]; cd[0] = cd[1]; cd[1] = t;
            }
        }
        bool moved = false;
        for (int relax = 0; relax < 2 && !moved; ++relax) {
            for (int ci = 0; ci < nc; ++ci) {
                if (lo[worst] == hi[worst]) continue;
                int nb = cn[ci];
                int32_t sw_lo = lo[worst], sw_hi = hi[worst], sn_lo = lo[nb], sn_hi = hi[nb];
                if (cd[ci] < 0) { lo[worst] += 1; hi[nb] += 1; }
                else { hi[worst] -= 1; lo[nb] -= 1; }
                // the trial changes stages i0 < i1 only: incremental estimate,
                // with their scratch entries saved for the undo below
                const int i0 = worst < nb ? worst : nb, i1 = i0 + 1;
                const Rat kF[2] = {s.F[i0], s.F[i1]}, kB[2] = {s.B[i0], s.B[i1]}, kW[2] = {s.W[i0], s.W[i1]},
                          kM[2] = {s.Mem[i0], s.Mem[i1]};
                const int64_t kA[3] = {s.A[0], s.A[i1], s.SR[i1]};
                estimate_move(wp, v, c, kind, M, micro, s, o, i0, i1, e);
                ++trials;
                if (!e.bad()) overloads_from_mem(c, s, o, e);
                if (e.bad()) return FT_OK;
                bool ok = rat_lt(o.total_over, total);
                if (ok && !relax) {
                    // max_stage_compute_time (plan.hpp:115-123), then
                    // detect_comm_bottleneck (partition.hpp:228-241)
                    Rat target{0, 1};
                    for (int n = 0; n < N; ++n) {
                        Rat t = rat_add(s.F[n], s.B[n], e);
                        if (rat_gt(t, target)) target = t;
                    }
                    // link_sr(k) of this plan is s.SR[k + 1] (the trial's
                    // estimate formed it; the reference forms it again here)
                    bool bott = false;
                    for (int k = 0; k + 1 < N; ++k)
                        if (rat_gt(R(s.SR[k + 1]), target)) bott = true;
                    ok = !bott;
                }
                if (ok) {
                    total = o.total_over;
                    worst = o.worst;
                    moved = true;
                    break;
                }
                lo[worst] = sw_lo; hi[worst] = sw_hi; lo[nb] = sn_lo; hi[nb] = sn_hi;
                s.F[i0] = kF[0]; s.F[i1] = kF[1];
                s.B[i0] = kB[0]; s.B[i1] = kB[1];
                s.W[i0] = kW[0]; s.W[i1] = kW[1];
                s.Mem[i0] = kM[0]; s.Mem[i1] = kM[1];
                s.A[0] = kA[0]; s.A[i1] = kA[1]; s.SR[i1] = kA[2];
            }
        }
        if (!moved) { o.trials = trials; return FT_REJ; }
    }
    // the accepted plan's full estimate (the bandwidth demands were not
    // formed during the trials; same values, no new errors)
    o.trials = trials;
    if (trials) estimate(wp, v, c, kind, M, micro, s, o, nullptr, e);
    return FT_OK;
}

// out of line; the error latch travels by value (see RatE in rat.cuh)
BPK_HDNI IntE memory_fine_tune_v(const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, int32_t* lo,
                                 int32_t* hi, const Rat* frac_lead, const Rat* frac_trail, const EstScratch& s,
                                 EstOut& o, uint32_t ecode) {
    Err e{ecode};
    const int r = memory_fine_tune_body(v, c, kind, M, micro, lo, hi, frac_lead, frac_trail, s, o, e);
    return IntE{r, e.code};
}
BPK_HD int memory_fine_tune(const NetView& v, const ChainView& c, int kind, int64_t M, int64_t micro, int32_t* lo,
                            int32_t* hi, const Rat* frac_lead, const Rat* frac_trail, const EstScratch& s, EstOut& o,
                            Err& e) {
    const IntE x = memory_fine_tune_v(v, c, kind, M, micro, lo, hi, frac_lead, frac_trail, s, o, e.code);
    e.code = x.err;
    return x.r;
}

// ---------------------------------------------------------------------------
// intra_layer_refine (partition.hpp:248-333) on one query's plan.
// lo/hi/lead/trail: the plan (in/out).  tF/tB/tT: per-stage fp, bp and
// compute time caches, recomputed lazily when a stage is marked dirty (the
// reference recomputes them at every use; the values, hence the overflow
// outcome, are the same).
BPK_HD void stage_times(const NetView& v, const ChainView& c, int s, const int32_t* lo,
                                            const int32_t* hi, const Rat* lead, const Rat* trail, Rat& F, Rat& B,
                                            Err& e) {
    int32_t t = c.type[s];
    F = stage_sum_frac(lo[s], hi[s], lead[s], trail[s], v.Pfp + (int64_t)t * (v.L + 1), e);
    B = stage_sum_frac(lo[s], hi[s], lead[s], trail[s], v.Pbp + (int64_t)t * (v.L + 1), e);
}

#ifdef BPK_REFINE_TRACE
void bpk_refine_trace(Rat t_hi, Rat t_lo, int64_t c_from, int64_t c_to, Rat avail, Rat x, Rat nh, Rat nl,
                      Rat lead, Rat trail);
#endif

// One boundary step of intra_layer_refine (partition.hpp:302-327) decided on
// scaled integers.  With D = lcm(den t_hi, den t_lo), every Rat the reference
// forms in the step (t_hi - t_lo, x, x*1024, the quantization scores, t -
// x*c) has a value whose denominator divides D*cs, D*1024 or D*den(x); when
// those scales and the scaled numerators stay below 2^62, no reduced value
// can exceed int64, so the reference cannot overflow and the decisions can
// be made with integer compares.  Returns FS_FALLBACK when a bound fails (the
// caller then runs the exact Rat step), FS_NOMOVE, or FS_MOVE with the
// reduced x and the two new stage times.  ~4 gcds instead of ~60.
enum { FS_FALLBACK = 0, FS_NOMOVE = 1, FS_MOVE = 2 };

BPK_HD Rat reduce_pos(i128 n, i128 d) {       // n >= 0, d > 0, both < 2^62
    uint64_t g = gcd_u64((uint64_t)n, (uint64_t)d);
    return Rat{(int64_t)udiv_exact64((uint64_t)n, g), (int64_t)udiv_exact64((uint64_t)d, g)};
}

// The same step when the common scale D < 2^31, both stage times are below
// 2^20 and c_from + c_to < 2^20: then every scaled quantity below is under
// 2^62 by construction (Th, Tl < 2^51; D*cs < 2^51; x*1024 and the scores
// < 2^62; at acceptance den(x) <= 1024), so the step runs in int64 with no
// per-product checks.  Returns -1 when the bounds do not hold.
BPK_HD int refine_small_step(Rat t_hi, Rat t_lo, int64_t c_from, int64_t c_to, Rat avail, Rat& x, Rat& nh, Rat& nl) {
    const int64_t B31 = (int64_t)1 << 31, B20 = (int64_t)1 << 20;
    if (t_hi.d >= B31 || t_lo.d >= B31 || c_from >= B20 / 2 || c_to >= B20 / 2) return -1;
    if (t_hi.n >= (t_hi.d << 20) || t_lo.n >= (t_lo.d << 20)) return -1;
    const uint32_t g = gcd_u32((uint32_t)t_hi.d, (uint32_t)t_lo.d);
    const int64_t mh = (uint32_t)t_lo.d / g, ml = (uint32_t)t_hi.d / g;
    const int64_t D = t_hi.d * mh;
    if (D >= B31) return -1;
    const int64_t cs = c_from + c_to;
    const int64_t Th = t_hi.n * mh, Tl = t_lo.n * ml;   // < 2^20 * D < 2^51
    x = reduce_pos(Th - Tl, D * cs);
    if (!rat_lt(x, avail)) {
        // x = avail - Rat(1, 1024)
        if (avail.d >= ((int64_t)1 << 40) || avail.n >= ((int64_t)1 << 40)) return -1;
        Err le{ERR_NONE};
        x = rat_sub(avail, Rat{1, 1024}, le);
        if (le.bad()) return -1;
        if (x.n <= 0) return FS_NOMOVE;
    }
    if (x.d > 1024) {                                     // quantize (257-265)
        if (x.d >= ((int64_t)1 << 51)) return -1;
        const int64_t num = x.n * 1024;                   // x < avail <= 1: x.n < x.d
        const uint64_t un = (uint64_t)num, ud = (uint64_t)x.d;
        uint64_t uk = (uint64_t)((double)un / (double)ud);
        while (uk * ud > un) --uk;
        while ((uk + 1) * ud <= un) ++uk;
        const int64_t k = (int64_t)uk, kc = k + (uk * ud != un ? 1 : 0);
        auto over1024 = [](int64_t q) {
            if (q == 0) return Rat{0, 1};
            int tz = bpk_ffs64((long long)q) - 1;
            tz = tz < 10 ? tz : 10;
            return Rat{q >> tz, (int64_t)1024 >> tz};
        };
        const Rat qlo = over1024(k), qhi = over1024(kc);
        if (rat_ge(qhi, avail)) {
            x = qlo;
        } else {
            const int64_t a1 = Th * 1024 - k * c_from * D, a2 = Tl * 1024 + k * c_to * D;
            const int64_t b1 = Th * 1024 - kc * c_from * D, b2 = Tl * 1024 + kc * c_to * D;
            const int64_t s_lo = a1 > a2 ? a1 : a2, s_hi = b1 > b2 ? b1 : b2;
            x = s_lo <= s_hi ? qlo : qhi;
        }
    }
    if (x.n <= 0 || !rat_lt(x, avail)) return FS_NOMOVE;
    if (x.d > 1024) return -1;                            // (not reached: den(x) <= 1024 here)
    const int64_t Dx = D * x.d;
    const int64_t TH = Th * x.d, NH = TH - x.n * c_from * D, NL = Tl * x.d + x.n * c_to * D;
    if ((NH > NL ? NH : NL) >= TH) return FS_NOMOVE;
    if (NH < 0) return -1;
    nh = reduce_pos(NH, Dx);
    nl = reduce_pos(NL, Dx);
    return FS_MOVE;
}

// Every product below is formed from two int64 factors already checked
// against 2^62 (64x64 -> 128-bit multiplies only: a 128x128 product is ~60
// instructions and this step runs millions of times).
BPK_HD int refine_fast_step_body(Rat t_hi, Rat t_lo, int64_t c_from, int64_t c_to, Rat avail, Rat& x, Rat& nh,
                                 Rat& nl) {
    const i128 B62 = (i128)1 << 62;
    if (t_hi.n < 0 || t_lo.n < 0 || avail.n <= 0) return FS_FALLBACK;
    const int small = refine_small_step(t_hi, t_lo, c_from, c_to, avail, x, nh, nl);
    if (small >= 0) return small;
    const uint64_t g = gcd_u64((uint64_t)t_hi.d, (uint64_t)t_lo.d);
    const int64_t mh = (int64_t)udiv_exact64((uint64_t)t_lo.d, g), ml = (int64_t)udiv_exact64((uint64_t)t_hi.d, g);
    const i128 D128 = (i128)t_hi.d * mh;
    if (D128 >= B62) return FS_FALLBACK;
    const int64_t D = (int64_t)D128;
    const int64_t cs = c_from + c_to;
    if ((i128)D * cs >= B62 || (i128)D * 1024 >= B62) return FS_FALLBACK;
    const i128 Th128 = (i128)t_hi.n * mh, Tl128 = (i128)t_lo.n * ml;
    if (Th128 >= B62 || Tl128 >= B62) return FS_FALLBACK;
    const int64_t Th = (int64_t)Th128, Tl = (int64_t)Tl128;
    // x = (t_hi - t_lo) / (c_from + c_to), reduced
    x = reduce_pos(Th - Tl, D * cs);
    if (!rat_lt(x, avail)) {
        // x = avail - Rat(1, 1024)
        if ((i128)avail.d * 1024 >= B62 || (i128)avail.n * 1024 >= B62) return FS_FALLBACK;
        Err le{ERR_NONE};
        x = rat_sub(avail, Rat{1, 1024}, le);
        if (le.bad()) return FS_FALLBACK;
        if (x.n <= 0) return FS_NOMOVE;
    }
    if (x.d > 1024) {                                     // quantize (257-265)
        if ((i128)x.n * 1024 >= B62) return FS_FALLBACK;
        const int64_t num = x.n * 1024;
        // k = floor(num / x.d) < 1024 (0 < x < avail <= 1): a double
        // estimate, corrected exactly, instead of a 64-bit software divide
        const uint64_t un = (uint64_t)num, ud = (uint64_t)x.d;
        uint64_t uk = (uint64_t)((double)un / (double)ud);
        while (uk * ud > un) --uk;
        while ((uk + 1) * ud <= un) ++uk;
        const int64_t k = (int64_t)uk, kc = k + (uk * ud != un ? 1 : 0);
        // k / 1024 reduced: the gcd is a power of two (0 <= k <= 1024)
        auto over1024 = [](int64_t q) {
            if (q == 0) return Rat{0, 1};
            int tz = bpk_ffs64((long long)q) - 1;
            tz = tz < 10 ? tz : 10;
            return Rat{q >> tz, (int64_t)1024 >> tz};
        };
        const Rat qlo = over1024(k), qhi = over1024(kc);
        if (rat_ge(qhi, avail)) {
            x = qlo;
        } else {
            // score(f) = max(t_hi - f*c_from, t_lo + f*c_to), all scaled by D*1024
            const i128 kf = (i128)k * c_from, kt = (i128)k * c_to, kcf = (i128)kc * c_from, kct = (i128)kc * c_to;
            if (kf >= B62 || kt >= B62 || kcf >= B62 || kct >= B62) return FS_FALLBACK;
            const i128 a1 = (i128)Th * 1024 - (i128)(int64_t)kf * D, a2 = (i128)Tl * 1024 + (i128)(int64_t)kt * D;
            const i128 b1 = (i128)Th * 1024 - (i128)(int64_t)kcf * D, b2 = (i128)Tl * 1024 + (i128)(int64_t)kct * D;
            if (a1 >= B62 || a2 >= B62 || b1 >= B62 || b2 >= B62 || a1 <= -B62 || b1 <= -B62) return FS_FALLBACK;
            const i128 s_lo = a1 > a2 ? a1 : a2, s_hi = b1 > b2 ? b1 : b2;
            x = s_lo <= s_hi ? qlo : qhi;
        }
    }
    if (x.n <= 0 || !rat_lt(x, avail)) return FS_NOMOVE;
    // acceptance: max(t_hi - x*c_from, t_lo + x*c_to) < t_hi, scaled by D*den(x)
    const i128 Dx = (i128)D * x.d;
    const i128 xf = (i128)x.n * c_from, xt = (i128)x.n * c_to;
    if (Dx >= B62 || xf >= B62 || xt >= B62) return FS_FALLBACK;
    const i128 TH = (i128)Th * x.d, NH = TH - (i128)(int64_t)xf * D, NL = (i128)Tl * x.d + (i128)(int64_t)xt * D;
    if (TH >= B62 || NL >= B62 || NH <= -B62) return FS_FALLBACK;
    if ((NH > NL ? NH : NL) >= TH) return FS_NOMOVE;
    if (NH < 0) return FS_FALLBACK;
    nh = reduce_pos(NH, Dx);
    nl = reduce_pos(NL, Dx);
    return FS_MOVE;
}

// out of line, results by value (see RatE in rat.cuh)
struct StepOut {
    int fs;
    uint32_t err;
    Rat x, nh, nl;
};
BPK_HD StepOut refine_fast_step(Rat t_hi, Rat t_lo, int64_t c_from, int64_t c_to, Rat avail) {
    StepOut o{};
    o.fs = refine_fast_step_body(t_hi, t_lo, c_from, c_to, avail, o.x, o.nh, o.nl);
    return o;
}

// The reference's boundary step on exact Rats (partition.hpp:302-327), for
// the steps refine_fast_step cannot bound; out of line so that the common
// path's code stays small.  Returns FS_NOMOVE or FS_MOVE (errors go to e,
// which the caller checks first).
BPK_HD int refine_exact_step_body(Rat t_hi, Rat t_lo, int64_t c_from, int64_t c_to, Rat avail, Rat& x, Rat& nh,
                                  Rat& nl, Err& e) {
    const Rat zero{0, 1}, step{1, 1024};
    x = rat_div(rat_sub(t_hi, t_lo, e), rat_add(R(c_from), R(c_to), e), e);
    if (rat_ge(x, avail)) x = rat_sub(avail, step, e);
    if (e.bad() || !rat_gt(x, zero)) return FS_NOMOVE;
    if (x.d > 1024) {                                       // quantize (257-265)
        const Rat y = rat_mul(x, R(1024), e);
        if (e.bad()) return FS_NOMOVE;
        const Rat qlo = rat_nd(rat_floor(y), 1024, e);
        const Rat qhi = rat_nd(rat_ceil(y), 1024, e);
        if (rat_ge(qhi, avail)) {
            x = qlo;
        } else {
            const Rat s_lo = rat_max(rat_sub(t_hi, rat_mul(qlo, R(c_from), e), e),
                                     rat_add(t_lo, rat_mul(qlo, R(c_to), e), e));
            const Rat s_hi = rat_max(rat_sub(t_hi, rat_mul(qhi, R(c_from), e), e),
                                     rat_add(t_lo, rat_mul(qhi, R(c_to), e), e));
            if (e.bad()) return FS_NOMOVE;
            x = rat_le(s_lo, s_hi) ? qlo : qhi;
        }
    }
    if (!rat_gt(x, zero) || rat_ge(x, avail)) return FS_NOMOVE;
    nh = rat_sub(t_hi, rat_mul(x, R(c_from), e), e);
    nl = rat_add(t_lo, rat_mul(x, R(c_to), e), e);
    if (e.bad() || rat_ge(rat_max(nh, nl), t_hi)) return FS_NOMOVE;
    return FS_MOVE;
}
BPK_HDNI StepOut refine_exact_step(Rat t_hi, Rat t_lo, int64_t c_from, int64_t c_to, Rat avail) {
    StepOut o{};
    Err e{ERR_NONE};
    o.fs = refine_exact_step_body(t_hi, t_lo, c_from, c_to, avail, o.x, o.nh, o.nl, e);
    o.err = e.code;
    return o;
}

// True when recomputing the stage time from the plan (stage_fp_time +
// stage_bp_time, plan.hpp:90-113) cannot overflow: every partial sum is at
// most t and its reduced denominator divides den(lead) * den(trail).
BPK_HD bool stage_time_safe(Rat t, Rat lead, Rat trail) {
    // a double estimate settles all but the borderline cases
    const double x = (double)t.n * (double)lead.d * (double)trail.d, y = 0x1p62 * (double)t.d;
    if (x < y * (1 - 0x1p-40)) return true;
    if (x > y * (1 + 0x1p-40)) return false;
    return (i128)t.n * lead.d * trail.d < ((i128)1 << 62) * t.d;
}

BPK_HD void refine_body(const NetView& v, const ChainView& c, int32_t* lo, int32_t* hi, Rat* lead, Rat* trail,
                        Rat* tF, Rat* tB, Rat* tT, uint8_t* dirty, int64_t* stats, Err& e) {
    const int N = c.N;
    stats[0] = stats[1] = stats[2] = stats[3] = 0;   // iterations, evaluated steps, moves, exact steps
    if (N <= 1) return;
    for (int s = 0; s < N; ++s) dirty[s] = 1;
    auto T = [&](int s) -> Rat {
        if (dirty[s] & 1) {
            stage_times(v, c, s, lo, hi, lead, trail, tF[s], tB[s], e);
            tT[s] = rat_add(tF[s], tB[s], e);
            dirty[s] &= (uint8_t)~1u;
        }
        return tT[s];
    };
    // bit 1 of dirty[b]: boundary b (stages b, b+1) was evaluated without a
    // move and neither stage changed since.  A boundary step is a pure
    // function of its two stages, so the reference would recompute the same
    // values and again not move: skipping it is exact.
    bool changed = true;
    int guard = 0;
    while (changed && ++guard < 1000) {
        changed = false;
        ++stats[0];
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = 0; i < N - 1; ++i) {
                int n0 = (pass == 0) ? i : (N - 2 - i);
                if (dirty[n0] & 2) continue;
                dirty[n0] |= 2;   // cleared below if this step moves
                ++stats[1];
                Rat t_a = T(n0);
                if (e.bad()) return;
                Rat t_b = T(n0 + 1);
                if (e.bad()) return;
                if (rat_eq(t_a, t_b)) continue;
                int dir = rat_gt(t_a, t_b) ? +1 : -1;
                int from = dir > 0 ? n0 : n0 + 1;
                int to = dir > 0 ? n0 + 1 : n0;
                int64_t j = dir > 0 ? hi[from] : lo[from];
                bool shared = (hi[n0] == lo[n0 + 1]);
                if (dir < 0 && !shared) {
                    int64_t cur_cut = act_at(v, hi[n0], e);
                    int64_t aj = act_at(v, j, e);
                    if (e.bad()) return;
                    if (aj > cur_cut) continue;
                }
                if (j < 1 || j > v.L) { e.set(ERR_UB); return; }
                int64_t c_from = fpbp_at(v, j, c.type[from]);
                int64_t c_to = fpbp_at(v, j, c.type[to]);
                Rat t_hi = rat_max(t_a, t_b), t_lo = rat_min(t_a, t_b);
                // avail = owned_fraction(from, j) (plan.hpp:33-39)
                Rat avail;
                if (lo[from] == hi[from]) avail = rat_sub(rat_add(lead[from], trail[from], e), R(1), e);
                else if (j == lo[from]) avail = lead[from];
                else avail = trail[from];
                if (e.bad()) return;
                StepOut st = refine_fast_step(t_hi, t_lo, c_from, c_to, avail);
                if (st.fs == FS_NOMOVE) continue;
                if (st.fs == FS_FALLBACK) {                // the reference's Rat step, verbatim
                    ++stats[3];
                    st = refine_exact_step(t_hi, t_lo, c_from, c_to, avail);
                    if (st.err) { e.set(st.err); return; }
                    if (st.fs == FS_NOMOVE) continue;
                }
                const Rat x = st.x, nh = st.nh, nl = st.nl;
#ifdef BPK_REFINE_TRACE
                bpk_refine_trace(t_hi, t_lo, c_from, c_to, avail, x, nh, nl, lead[from], trail[from]);
#endif
                // apply_move (269-292)
                int a = n0, b = n0 + 1;
                if (dir > 0) {
                    if (shared) {
                        trail[a] = rat_sub(trail[a], x, e);
                        lead[b] = rat_add(lead[b], x, e);
                    } else {
                        trail[a] = rat_sub(R(1), x, e);
                        lo[b] = hi[a];
                        lead[b] = x;
                    }
                } else {
                    if (shared) {
                        lead[b] = rat_sub(lead[b], x, e);
                        trail[a] = rat_add(trail[a], x, e);
                    } else {
                        lead[b] = rat_sub(R(1), x, e);
                        hi[a] = lo[b];
                        trail[a] = x;
                    }
                }
                if (e.bad()) return;
                dirty[a] = dirty[b] = 1;                 // stage times stale, boundaries a, b unstable
                if (a > 0) dirty[a - 1] &= 1;            // boundary a-1 touches stage a
                // The new stage times are nh (from) and nl (to) exactly; keep
                // them unless recomputing from the plan could overflow, in
                // which case the lazy exact recomputation decides (as the
                // reference does at its next use).
                if (stage_time_safe(nh, lead[from], trail[from])) { tT[from] = nh; dirty[from] &= (uint8_t)~1u; }
                if (stage_time_safe(nl, lead[to], trail[to])) { tT[to] = nl; dirty[to] &= (uint8_t)~1u; }
                changed = true;
                ++stats[2];
            }
        }
    }
}

// out of line with the error latch in a register (see RatE in rat.cuh)
BPK_HDNI uint32_t refine_v(const NetView& v, const ChainView& c, int32_t* lo, int32_t* hi, Rat* lead, Rat* trail,
                           Rat* tF, Rat* tB, Rat* tT, uint8_t* dirty, int64_t* stats, uint32_t ecode) {
    Err e{ecode};
    // register copies: through the references (and the stats pointer) every
    // field access after an out-of-line call was a reload from local memory
    const NetView vv = v;
    const ChainView cc = c;
    int64_t st[4];
    refine_body(vv, cc, lo, hi, lead, trail, tF, tB, tT, dirty, st, e);
    for (int k = 0; k < 4; ++k) stats[k] = st[k];
    return e.code;
}
BPK_HD void refine(const NetView& v, const ChainView& c, int32_t* lo, int32_t* hi, Rat* lead, Rat* trail, Rat* tF,
                   Rat* tB, Rat* tT, uint8_t* dirty, int64_t* stats, Err& e) {
    e.code = refine_v(v, c, lo, hi, lead, trail, tF, tB, tT, dirty, stats, e.code);
}

}  // namespace bpk
