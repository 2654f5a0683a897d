// common.cuh -- device-side data layout and the exact per-stage cost model.
//
// HBM layout (all int64 unless noted; "pool" = one array for all networks):
//   per network i (NetDesc): L layers, T accelerator types
//     fp, bp            [T][L]    raw times (0 = type missing)
//     w, a              [L]       weight_bytes, out_activation_bytes
//     Pfp, Pbp, Pc      [T][L+1]  prefix sums of fp, bp, fp+bp     (K1 cost_prefix)
//     Pw                [L+1]     prefix sums of w
//     asort             [L-1]     a[0..L-2] sorted (coarse block counting)
//     type_ok           [T] u8    every layer has fp and bp for the type
//   per cluster (ClDesc): N accelerators; type, cap, minm[N][4], bw[N-1]
//
// Stage sums replace the reference's O(stage length) Rat loops
// (plan.hpp:90-132) by O(1) prefix differences.  The values are identical;
// the overflow predicate of every intermediate partial sum the reference
// forms is reproduced exactly (see stage_sum_frac below).
#pragma once
#include <stdint.h>

#include "rat.cuh"

namespace bpk {

enum { KIND_AS = 0, KIND_FBP = 1, KIND_SNO = 2, KIND_SO = 3 };
enum { MODE_SYNC = 0, MODE_ASYNC = 1 };

struct NetDesc {
    int32_t L, T;
    int64_t off_layer;   // w, a, asort (asort uses L-1 of the L slots)
    int64_t off_typed;   // fp, bp: [T][L]
    int64_t off_pref;    // Pw: L+1
    int64_t off_tpref;   // Pfp, Pbp, Pc: [T][L+1]
    int64_t off_tflag;   // type_ok: T
    int32_t valid;       // network-level schema checks (profiles.hpp:83-98)
    int32_t pad;
};

struct ClDesc {
    int32_t N, mode;
    int64_t off_acc;        // type, cap, minm (x4)
    int64_t off_link;       // bw
    int32_t first_bad_acc;  // first accelerator failing validate_cluster (N if none)
    int32_t first_bad_link; // first link with bw <= 0 (N-1 if none)
};

struct Pools {
    const NetDesc* nets;
    const ClDesc* cls;
    const int64_t *fp, *bp, *w, *a, *asort, *Pfp, *Pbp, *Pc, *Pw;
    const uint8_t* type_ok;
    const int32_t* ctype;
    const int64_t *cap, *minm, *bw;
};

// One network + chain prefix as seen by a query.
struct NetView {
    int64_t L;
    int32_t T;
    const int64_t *fp, *bp, *w, *a, *Pfp, *Pbp, *Pc, *Pw, *asort;
};

struct ChainView {
    int32_t N, mode;
    const int32_t* type;
    const int64_t *cap, *minm, *bw;
};

BPK_HD NetView net_view(const Pools& P, int i) {
    NetDesc d = P.nets[i];
    NetView v;
    v.L = d.L;
    v.T = d.T;
    v.fp = P.fp + d.off_typed;
    v.bp = P.bp + d.off_typed;
    v.w = P.w + d.off_layer;
    v.a = P.a + d.off_layer;
    v.asort = P.asort + d.off_layer;
    v.Pfp = P.Pfp + d.off_tpref;
    v.Pbp = P.Pbp + d.off_tpref;
    v.Pc = P.Pc + d.off_tpref;
    v.Pw = P.Pw + d.off_pref;
    return v;
}

BPK_HD ChainView chain_view(const Pools& P, int i, int N) {
    ClDesc d = P.cls[i];
    ChainView c;
    c.N = N;
    c.mode = d.mode;
    c.type = P.ctype + d.off_acc;
    c.cap = P.cap + d.off_acc;
    c.minm = P.minm + 4 * d.off_acc;
    c.bw = P.bw + d.off_link;
    return c;
}

// net.layers[j-1].out_activation_bytes with the reference's UB made explicit.
BPK_HD int64_t act_at(const NetView& v, int64_t j, Err& e) {
    if (j < 1 || j > v.L) { e.set(ERR_UB); return 0; }
    return v.a[j - 1];
}

// fp + bp of layer j on type t, from the prefix sums (the refine kernel keeps
// only those in shared memory)
BPK_HD int64_t fpbp_at(const NetView& v, int64_t j, int32_t t) {
    const int64_t o = (int64_t)t * (v.L + 1) + j;
    return (v.Pfp[o] - v.Pfp[o - 1]) + (v.Pbp[o] - v.Pbp[o - 1]);
}

BPK_HD int64_t pref(const int64_t* P, int64_t L, int32_t t, int64_t j) {
    return P[(int64_t)t * (L + 1) + j];
}

// warmup_depth, schedule_kind.hpp:52-57
BPK_HD int64_t warmup_depth(int kind, int64_t N, int64_t s) {
    int64_t d = N - s + 1;
    if (kind == KIND_FBP || kind == KIND_SO) d *= 2;
    return d;
}

BPK_HD bool kind_async(int kind) { return kind == KIND_AS || kind == KIND_FBP; }

// ---------------------------------------------------------------------------
// Exact stage sums.  Reference (plan.hpp:90-132): t = 0; for j = lo..hi:
//   t += owned_fraction(s, j) * Rat(v_j).
// owned = lead (j == lo), trail (j == hi), 1 inside, lead + trail - 1 when
// lo == hi.  With v_j >= 0 every partial sum of the interior run is
// monotone, so the largest one (just before the trailing term) decides
// whether any of them overflows; its reduced denominator is that of
// lead * v_lo (adding integers keeps the denominator).
//   P: prefix sums of v over layers (P[j] = v_1 + ... + v_j).
BPK_HD Rat stage_sum_frac_body(int64_t lo, int64_t hi, Rat lead, Rat trail, const int64_t* P, Err& e) {
    if (lo > hi) return Rat{0, 1};
    if (lo == hi) {
        Rat own = rat_sub(rat_add(lead, trail, e), R(1), e);
        return rat_mul(own, R(P[lo] - P[lo - 1]), e);   // 0 + own * v: same value
    }
    Rat t = rat_mul(lead, R(P[lo] - P[lo - 1]), e);
    if (hi - lo >= 2) {
        int64_t S = P[hi - 1] - P[lo];                    // interior, owned = 1 each
        i128 num = (i128)t.n + (i128)S * t.d;             // largest partial sum, den t.d
        if (num > (i128)INT64_MAX || num < (i128)INT64_MIN) { e.set(ERR_OVERFLOW); return Rat{0, 1}; }
        t = Rat{(int64_t)num, t.d};
    }
    Rat th = rat_mul(trail, R(P[hi] - P[hi - 1]), e);
    return rat_add(t, th, e);
}
// out of line, error by value (see RatE in rat.cuh)
BPK_HDNI RatE stage_sum_frac_v(int64_t lo, int64_t hi, Rat lead, Rat trail, const int64_t* P) {
    Err e{ERR_NONE};
    const Rat r = stage_sum_frac_body(lo, hi, lead, trail, P, e);
    return RatE{r, e.code};
}
BPK_HD Rat stage_sum_frac(int64_t lo, int64_t hi, Rat lead, Rat trail, const int64_t* P, Err& e) {
    const RatE x = stage_sum_frac_v(lo, hi, lead, trail, P);
    if (x.err) e.set(x.err);
    return x.r;
}

// Whole-layer stage (fractions 1): plain prefix difference.  Partial sums are
// bounded by the network totals, which upload checks keep below 2^62.
BPK_HD int64_t stage_sum_whole(int64_t lo, int64_t hi, const int64_t* P) {
    return lo > hi ? 0 : P[hi] - P[lo - 1];
}

}  // namespace bpk
