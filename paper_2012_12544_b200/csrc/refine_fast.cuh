// refine_fast.cuh -- intra_layer_refine (partition.hpp:248-333) in one
// bounded regime, for the slim refine kernel (k_refine_fast, kernels.cu).
//
// The walk is the reference's: while (changed && ++guard < 1000) a forward
// then a backward pass over the N-1 boundaries, each boundary step deciding
// a move of fraction x of one boundary layer (302-327, apply_move 269-292).
// It is serial, so the kernel's time is one query's walk; this version makes
// each step short:
//   * the layer tables it reads (fp+bp per type, out_act) are int32 copies in
//     shared memory (the general kernel reads int64 prefix sums from L2);
//   * stage times, fractions and x stay reduced rationals, but every
//     reduction is split Knuth-style (4.5.1) so that the only gcd on
//     denominators of stage size is gcd(den t_a, den t_b); all others have
//     one operand <= 1024 (den x) or <= c_from + c_to;
//   * no 128-bit, exact-Rat or error-latch code: every step first checks the
//     regime below, and a query leaving it returns RF_BAIL, after which the
//     general kernel (k_refine_smem) re-runs it from the DP plan.  The walk is
//     a pure function of (plan, network, chain), so that re-run is exact.
//
// Regime (checked before use; same proof as refine_small_step in model.cuh):
//   every stage time t = n/d has d < 2^31 and value < 2^20; every fraction
//   (lead / trail) has den < 2^31; fp + bp of every layer < 2^19; the common
//   scale D = lcm(d_a, d_b) < 2^31.  Then every Rat the reference forms in a
//   step is below 2^62 in reduced form (so it cannot throw), and every scaled
//   integer below fits int64.  Stage times are updated to the reduced
//   t -+ x*c directly; stage_time_safe() (model.cuh) proves that the
//   reference's recomputation of that stage from the plan cannot overflow,
//   else the walk bails.
#pragma once
#include "model.cuh"

namespace bpk {

enum { RF_DONE = 0, RF_BAIL = 1 };

// Shared-memory view of one query for the walk.
struct FastRefine {
    const int32_t* cost;   // [T][L] fp + bp (< 2^19)
    const int32_t* act;    // [L] out_activation_bytes (< 2^31)
    const int32_t* type;   // [N] accelerator type of each stage
    int32_t L, N;
    int32_t *lo, *hi;      // plan (in / out)
    Rat *lead, *trail;     // fractions (in / out)
    Rat* t;                // stage compute times (in: the DP plan's, integers)
    uint8_t* memo;         // 1: boundary evaluated without a move, both stages unchanged since
};

// Integer helpers with no 64-bit software division: every divisor here is
// below 2^32 and every division is exact, and the divisors are mostly powers
// of two (the 1/1024 grid), which take a shift.
BPK_HD bool rf_pow2(uint32_t m) { return (m & (m - 1)) == 0; }
BPK_HD int rf_ctz(uint32_t m) { return bpk_ffs64((long long)m) - 1; }

BPK_HDNI uint32_t rf_udiv32(uint32_t a, uint32_t g) { return a / g; }

// a / g for a 32-bit a that g divides exactly
BPK_HD uint32_t rf_div32(uint32_t a, uint32_t g) { return rf_pow2(g) ? a >> rf_ctz(g) : rf_udiv32(a, g); }

// a / o for an odd o > 1 dividing a exactly: the inverse of o modulo 2^64.
// Out of line, like every path below that is not taken on most steps: the
// walk is one thread's serial chain, and instruction-cache misses on a large
// inlined body cost more than the calls.
BPK_HDNI int64_t rf_div_odd(int64_t a, uint32_t o) {
    if ((uint64_t)a < ((uint64_t)1 << 32)) return (int64_t)((uint32_t)a / o);
    const uint64_t inv = inv64_lift(o, inv32_odd(o));
    return (int64_t)((uint64_t)a * inv);
}

// a / g for a 64-bit a (any sign) that g < 2^32 divides exactly: shift out the
// twos, then the odd part
BPK_HD int64_t rf_div64(int64_t a, uint32_t g) {
    const int tz = rf_ctz(g);
    a >>= tz;                                   // exact: arithmetic shift of a multiple of 2^tz
    const uint32_t o = g >> tz;
    return o == 1 ? a : rf_div_odd(a, o);
}

BPK_HDNI uint32_t rf_gcd_mod_odd(uint64_t a, uint32_t m) { return gcd_u32(umod_u64_u32(a, m), m); }

// gcd(a, m) for a >= 0 and 0 < m < 2^32 (a power-of-two m: the lowest set bit)
BPK_HD uint32_t gcd_mod(uint64_t a, uint32_t m) {
    BPK_COUNT(12);
    if (rf_pow2(m)) {
        if (a == 0) return m;
        const uint64_t lb = a & (0ull - a);
        return lb < m ? (uint32_t)lb : m;
    }
    BPK_COUNT(13);
    return rf_gcd_mod_odd(a, m);
}

// a + s*b (s = +1 / -1) for reduced a, b with 0 < a.d, b.d < 2^31, |a.n| <
// 2^52, |b.n| < 2^32 and b.d <= 2^11; Knuth 4.5.1: g = gcd(a.d, b.d),
// t = a.n*(b.d/g) + s*b.n*(a.d/g), g2 = gcd(t, g): (t/g2) / ((a.d/g)*(b.d/g2)).
// Both gcds have an operand <= b.d.
BPK_HD Rat rf_add_small(Rat a, Rat b, int s) {
    const uint32_t g = gcd_mod((uint64_t)a.d, (uint32_t)b.d);
    const int64_t bg = rf_div32((uint32_t)b.d, g), ag = rf_div32((uint32_t)a.d, g);
    const int64_t t = a.n * bg + (s > 0 ? b.n : -b.n) * ag;
    const uint32_t g2 = gcd_mod(uabs64(t), g);
    return Rat{rf_div64(t, g2), ag * rf_div32((uint32_t)b.d, g2)};
}

// x * c for a reduced x with x.d <= 2^11 and 0 < c < 2^19
BPK_HD Rat rf_mul_int(Rat x, int64_t c) {
    const uint32_t g = gcd_mod((uint64_t)c, (uint32_t)x.d);
    return Rat{x.n * rf_div32((uint32_t)c, g), rf_div32((uint32_t)x.d, g)};
}

// a < b for 0 <= a.n, b.n < 2^63 and dens < 2^63: exact 128-bit cross products
BPK_HD bool rf_lt(Rat a, Rat b) { return (u128)(uint64_t)a.n * (uint64_t)b.d < (u128)(uint64_t)b.n * (uint64_t)a.d; }

BPK_HD bool rf_time_ok(Rat t) {
    return t.d > 0 && t.d < ((int64_t)1 << 31) && t.n >= 0 && t.n < (t.d << 20);
}
BPK_HD bool rf_frac_ok(Rat f) { return f.d > 0 && f.d < ((int64_t)1 << 31) && f.n >= 0 && f.n <= f.d; }

// owned_fraction of a stage's only layer: lead + trail - 1 (Knuth 4.5.1)
BPK_HDNI Rat rf_single_owned(Rat ld, Rat tr) {
    const uint32_t gg = gcd_u32((uint32_t)ld.d, (uint32_t)tr.d);
    const int64_t lg = rf_div32((uint32_t)ld.d, gg), tg = rf_div32((uint32_t)tr.d, gg);
    const int64_t tt = ld.n * tg + tr.n * lg - lg * tr.d;   // over lg * tr.d
    const uint32_t g2 = gcd_mod(uabs64(tt), gg);
    return Rat{rf_div64(tt, g2), lg * rf_div32((uint32_t)tr.d, g2)};
}

// ---- the common case, branch-light: powers of two --------------------------
// Most denominators in a walk are powers of two (every quantized x is k/1024),
// and adding a fraction whose denominator is a power of two to a reduced
// value never leaves a common ODD factor: only twos need cancelling.
BPK_HD int rf_ctz64(uint64_t v) { return bpk_ffs64((long long)v) - 1; }

// a + s * bn / 2^m for a reduced a (0 < a.d < 2^31, |a.n| < 2^52) and a
// reduced bn / 2^m (m <= 11, |bn| < 2^30): Knuth 4.5.1 with g = 2^min(e_a, m)
// and g2 = 2^min(ctz t, log g)
BPK_HD Rat rf_add_p2(Rat a, int64_t bn, int m, int s) {
    const int ea = rf_ctz((uint32_t)a.d);
    const int l = ea < m ? ea : m;
    const int64_t ad = a.d >> l;
    const int64_t t = (a.n << (m - l)) + (s > 0 ? bn : -bn) * ad;
    // branch-free (the commit's four sums interleave): t == 0 gives 0/1
    const uint64_t ut = uabs64(t);
    int z = rf_ctz64(ut | ((uint64_t)1 << 62));
    z = z < l ? z : l;
    return Rat{t >> z, t == 0 ? 1 : ad << (m - z)};
}

// x * c for x = xn / 2^m reduced (xn odd unless m = 0) and 0 < c < 2^19
BPK_HD Rat rf_mul_p2(int64_t xn, int m, int64_t c) {
    int z = rf_ctz((uint32_t)c);
    z = z < m ? z : m;
    return Rat{xn * (c >> z), (int64_t)1 << (m - z)};
}

// divisibility of a >= 0 by an odd o (o < 2^52): a * o^-1 mod 2^64 is the
// exact quotient iff it times o does not wrap
BPK_HD uint64_t rf_inv64(uint64_t o) {
    uint64_t x = (3 * o) ^ 2;                 // 5 bits
    x *= 2 - o * x;                           // 10
    x *= 2 - o * x;                           // 20
    x *= 2 - o * x;                           // 40
    x *= 2 - o * x;                           // 80
    return x;
}
BPK_HD bool rf_divides(uint64_t a, uint64_t o, uint64_t inv, uint64_t* quot) {
    const uint64_t q = a * inv;
#ifdef __CUDA_ARCH__
    const bool ok = __umul64hi(q, o) == 0;
#else
    const bool ok = (uint64_t)(((u128)q * o) >> 64) == 0;
#endif
    *quot = q;
    return ok;
}

// floor(num / den) for 0 <= num < 2^62, 0 < den < 2^62, quotient <= 2^11:
// a float estimate, corrected exactly
BPK_HD float rf_rcp(float x) {
#ifdef __CUDA_ARCH__
    return __frcp_rn(x);
#else
    return 1.0f / x;
#endif
}
BPK_HD int64_t rf_small_quot(int64_t num, int64_t den) {
    int64_t k = (int64_t)((float)num * rf_rcp((float)den));
    if (k > 2048) k = 2048;
    if (k < 0) k = 0;
    while (k > 0 && k * den > num) --k;
    while ((k + 1) * den <= num) ++k;
    return k;
}

// ---- the general cases, out of line ---------------------------------------
struct RfCmp {
    int64_t D, A, Bv;
    uint32_t g;
};
// t_a, t_b over their common scale D = lcm(d_a, d_b) (Knuth: gcd(d_a, d_b))
BPK_HDNI RfCmp rf_compare_general(Rat ta, Rat tb) {
    RfCmp r;
    r.g = gcd_u32((uint32_t)ta.d, (uint32_t)tb.d);
    const int64_t mb = rf_div32((uint32_t)tb.d, r.g), ma = rf_div32((uint32_t)ta.d, r.g);
    r.D = ta.d * mb;
    r.A = ta.n * mb;
    r.Bv = tb.n * ma;
    return r;
}

// x0 = Nd / (D * cs) reduced, the general way (gcd(Nd, D) = gcd(Nd, g) by
// Knuth, then the cs part)
BPK_HDNI Rat rf_x0_general(int64_t Nd, int64_t D, uint32_t g, int64_t cs) {
    const uint32_t g2 = gcd_mod((uint64_t)Nd, g);
    const int64_t n1 = rf_div64(Nd, g2);
    const uint32_t g3 = gcd_mod((uint64_t)n1, (uint32_t)cs);
    return Rat{rf_div64(n1, g3), (int64_t)rf_div32((uint32_t)D, g2) * rf_div32((uint32_t)cs, g3)};
}

struct RfCommit {
    Rat nh, nl, fa, fb;
};
// the move's new stage times and fractions for an x whose denominator is
// not a power of two (x kept exact, den <= 1024)
BPK_HDNI RfCommit rf_commit_general(Rat t_hi, Rat t_lo, Rat x, int64_t c_from, int64_t c_to, Rat trail_a,
                                    Rat lead_b, int dir, int shared) {
    RfCommit o;
    o.nh = rf_add_small(t_hi, rf_mul_int(x, c_from), -1);
    o.nl = rf_add_small(t_lo, rf_mul_int(x, c_to), +1);
    if (shared) {
        o.fa = rf_add_small(trail_a, x, dir > 0 ? -1 : +1);
        o.fb = rf_add_small(lead_b, x, dir > 0 ? +1 : -1);
    } else {
        o.fa = dir > 0 ? Rat{x.d - x.n, x.d} : x;
        o.fb = dir > 0 ? x : Rat{x.d - x.n, x.d};
    }
    return o;
}

// ---- the walk ---------------------------------------------------------------
// Section timers for tests/cpp/refine_walk_bench.cu (RF_PROF builds only).
#if defined(RF_PROF) && defined(__CUDA_ARCH__)
#define RF_MARK(k)                          \
    do {                                    \
        const long long t1_ = clock64();    \
        rf_prof[k] += t1_ - rf_t0;          \
        rf_t0 = t1_;                        \
    } while (0)
#define RF_PROF_DECL long long rf_prof[8] = {0, 0, 0, 0, 0, 0, 0, 0}, rf_t0 = clock64();
#else
#define RF_MARK(k) ((void)0)
#define RF_PROF_DECL
#endif

// next boundary >= from (forward) / <= from (backward) whose memo bit is clear
BPK_HD int rf_next_fwd(uint64_t open, int from) {
    if (from >= 64) return -1;
    const uint64_t m = open & (~0ull << from);
    return m ? rf_ctz64(m) : -1;
}
BPK_HD int rf_next_bwd(uint64_t open, int from) {
    if (from < 0) return -1;
    const uint64_t m = open & (from >= 63 ? ~0ull : ((2ull << from) - 1));
#ifdef __CUDA_ARCH__
    return m ? 63 - __clzll((long long)m) : -1;
#else
    return m ? 63 - __builtin_clzll(m) : -1;
#endif
}

// The walk.  stats: iterations, evaluated boundary steps, moves.
BPK_HD int refine_fast_walk(const FastRefine& q, int64_t* stats, long long* prof_out = nullptr) {
    RF_PROF_DECL
    const int N = q.N;
    if (N > 64) return RF_BAIL;
    const uint64_t all = N - 1 >= 64 ? ~0ull : ((1ull << (N - 1)) - 1);
    uint64_t memo = 0;    // bit n0: boundary n0 evaluated without a move, both stages unchanged since
    int64_t iters = 0, evals = 0, moves = 0;
    bool changed = true;
    int guard = 0;
    while (changed && ++guard < 1000) {
        changed = false;
        ++iters;
        for (int pass = 0; pass < 2; ++pass) {
            for (int n0 = pass == 0 ? rf_next_fwd(all & ~memo, 0) : rf_next_bwd(all & ~memo, N - 2); n0 >= 0;
                 n0 = pass == 0 ? rf_next_fwd(all & ~memo, n0 + 1) : rf_next_bwd(all & ~memo, n0 - 1)) {
                memo |= 1ull << n0;                       // cleared below if this step moves
                ++evals;
                RF_MARK(7);
                const Rat ta = q.t[n0], tb = q.t[n0 + 1];
                const int32_t lo0 = q.lo[n0], hi0 = q.hi[n0], lo1 = q.lo[n0 + 1], hi1 = q.hi[n0 + 1];
                const int32_t ty0 = q.type[n0], ty1 = q.type[n0 + 1];
                // t_a vs t_b over the common scale D = lcm(d_a, d_b)
                int64_t D, A, Bv;
                uint32_t g;
                if (rf_pow2((uint32_t)ta.d) && rf_pow2((uint32_t)tb.d)) {
                    const bool ga = ta.d >= tb.d;
                    D = ga ? ta.d : tb.d;
                    g = (uint32_t)(ga ? tb.d : ta.d);
                    const int sh = rf_ctz((uint32_t)D) - rf_ctz(g);
                    A = ga ? ta.n : ta.n << sh;
                    Bv = ga ? tb.n << sh : tb.n;
                } else {
                    BPK_COUNT(22);
                    const RfCmp r = rf_compare_general(ta, tb);
                    D = r.D;
                    A = r.A;
                    Bv = r.Bv;
                    g = r.g;
                }
                if (D >= ((int64_t)1 << 31)) return RF_BAIL;
                if (A == Bv) continue;                    // t_a == t_b
                const int dir = A > Bv ? +1 : -1;
                RF_MARK(0);
                const int from = dir > 0 ? n0 : n0 + 1, to = dir > 0 ? n0 + 1 : n0;
                const int32_t j = dir > 0 ? hi0 : lo1;
                const bool shared = hi0 == lo1;
                if (j < 1 || j > q.L) return RF_BAIL;     // (the reference's UB case; the general kernel reports it)
                if (dir < 0 && !shared && q.act[j - 1] > q.act[hi0 - 1]) continue;
                const int64_t c_from = q.cost[(dir > 0 ? ty0 : ty1) * q.L + (j - 1)];
                const int64_t c_to = q.cost[(dir > 0 ? ty1 : ty0) * q.L + (j - 1)];
                const Rat t_hi = dir > 0 ? ta : tb, t_lo = dir > 0 ? tb : ta;
                const int64_t Th = dir > 0 ? A : Bv, Tl = dir > 0 ? Bv : A;
                // avail = owned_fraction(from, j) (plan.hpp:33-39)
                const int32_t lof = dir > 0 ? lo0 : lo1, hif = dir > 0 ? hi0 : hi1;
                const Rat ld = q.lead[from], tr = q.trail[from];
                const Rat avail = lof == hif ? rf_single_owned(ld, tr) : (j == lof ? ld : tr);
                if (avail.n <= 0 || avail.d >= ((int64_t)1 << 31)) return RF_BAIL;
                const int64_t cs = c_from + c_to;
                RF_MARK(1);
                // x = (t_hi - t_lo) / (c_from + c_to) = Nd / (D*cs), then quantize (257-265)
                const int64_t Nd = Th - Tl;
                Rat x{0, 1};
                bool quant;
                int eD = -1;                              // log2 D when x is x0 and D a power of two
                int64_t qn = Nd, qd = D * cs;             // the value to quantize (need not be reduced)
                if (!rf_lt(Rat{Nd, D * cs}, avail)) {
                    BPK_COUNT(21);
                    // x = avail - 1/1024
                    x = rf_add_p2(avail, 1, 10, -1);
                    if (x.n <= 0) continue;
                    quant = x.d > 1024;
                    qn = x.n;
                    qd = x.d;
                } else {
                    // den(x0) = 2^E2 * O / gcd(Nd, O), O the odd part of D * cs
                    eD = rf_ctz((uint32_t)D);
                    const int ec = rf_ctz((uint32_t)cs);
                    const int eN = rf_ctz64((uint64_t)Nd);
                    const int E2 = eD + ec - (eN < eD + ec ? eN : eD + ec);
                    const uint64_t O = (uint64_t)(D >> eD) * (uint64_t)(cs >> ec);
                    BPK_COUNT(16);
                    if (E2 > 10) {
                        BPK_COUNT(17);
                        quant = true;                     // den(x0) > 1024
                    } else if (O == 1) {
                        BPK_COUNT(18);
                        quant = false;                    // den(x0) = 2^E2 <= 1024
                        x = Rat{Nd >> (eN < eD + ec ? eN : eD + ec), (int64_t)1 << E2};
                    } else if ((1024 >> E2) < 3) {
                        BPK_COUNT(19);
                        // den(x0) <= 1024 only if O divides Nd
                        uint64_t qo;
                        // O is the odd part of cs (< 2^20) unless D has an odd factor:
                        // the inverse mod 2^32 then one lift is half the work of mod 2^64
                        const uint64_t inv = O >> 32 ? rf_inv64(O) : inv64_lift((uint32_t)O, inv32_odd((uint32_t)O));
                        quant = !rf_divides((uint64_t)Nd, O, inv, &qo);
                        if (!quant) x = Rat{(int64_t)qo >> (eN < eD + ec ? eN : eD + ec), (int64_t)1 << E2};
                    } else {
                        BPK_COUNT(20);
                        x = rf_x0_general(Nd, D, g, cs);
                        quant = x.d > 1024;
                    }
                }
                RF_MARK(2);
                int64_t k = 0, kc = 0;
                if (quant) {
                    // k = floor(1024 x), kc = ceil(1024 x)
                    const int64_t num = qn * 1024, den = qd;
                    if (eD >= 0 && qd == D * cs && rf_pow2((uint32_t)D)) {
                        // x0 with D = 2^eD: floor(1024 Nd / D) is a shift, below 1024 cs < 2^30,
                        // and k = that / cs a 32-bit division
                        const uint32_t Y = (uint32_t)(eD >= 10 ? (Nd >> (eD - 10)) : (Nd << (10 - eD)));
                        k = (int64_t)(Y / (uint32_t)cs);
                    } else {
                        k = rf_small_quot(num, den);
                    }
                    kc = k + (k * den != num ? 1 : 0);
                    const int zl = k ? (rf_ctz((uint32_t)k) < 10 ? rf_ctz((uint32_t)k) : 10) : 10;
                    const int zh = rf_ctz((uint32_t)kc) < 10 ? rf_ctz((uint32_t)kc) : 10;
                    const Rat qlo = k ? Rat{k >> zl, (int64_t)1024 >> zl} : Rat{0, 1};
                    const Rat qhi = Rat{kc >> zh, (int64_t)1024 >> zh};
                    if (!rf_lt(qhi, avail)) {
                        x = qlo;
                    } else {
                        // score(f) = max(t_hi - f*c_from, t_lo + f*c_to), scaled by D*1024
                        const int64_t a1 = Th * 1024 - k * c_from * D, a2 = Tl * 1024 + k * c_to * D;
                        const int64_t b1 = Th * 1024 - kc * c_from * D, b2 = Tl * 1024 + kc * c_to * D;
                        const int64_t s_lo = a1 > a2 ? a1 : a2, s_hi = b1 > b2 ? b1 : b2;
                        x = s_lo <= s_hi ? qlo : qhi;
                    }
                }
                RF_MARK(3);
                if (x.n <= 0 || !rf_lt(x, avail)) continue;
                // acceptance: max(t_hi - x*c_from, t_lo + x*c_to) < t_hi, scaled by D*den(x)
                const int64_t TH = Th * x.d, NH = TH - x.n * c_from * D, NL = Tl * x.d + x.n * c_to * D;
                if ((NH > NL ? NH : NL) >= TH) continue;
                if (NH < 0) return RF_BAIL;
                RF_MARK(4);
                // commit: new stage times (reduced), apply_move (269-292)
                const int a = n0, b = n0 + 1;
                const Rat trail_a = q.trail[a], lead_b = q.lead[b];
                Rat nh, nl, fa, fb;
                if (rf_pow2((uint32_t)x.d)) {
                    const int m = rf_ctz((uint32_t)x.d);
                    const Rat yf = rf_mul_p2(x.n, m, c_from), yt = rf_mul_p2(x.n, m, c_to);
                    nh = rf_add_p2(t_hi, yf.n, rf_ctz((uint32_t)yf.d), -1);
                    nl = rf_add_p2(t_lo, yt.n, rf_ctz((uint32_t)yt.d), +1);
                    if (shared) {
                        fa = rf_add_p2(trail_a, x.n, m, dir > 0 ? -1 : +1);
                        fb = rf_add_p2(lead_b, x.n, m, dir > 0 ? +1 : -1);
                    } else {
                        fa = dir > 0 ? Rat{x.d - x.n, x.d} : x;
                        fb = dir > 0 ? x : Rat{x.d - x.n, x.d};
                    }
                } else {
                    BPK_COUNT(23);
                    const RfCommit o = rf_commit_general(t_hi, t_lo, x, c_from, c_to, trail_a, lead_b, dir, shared);
                    nh = o.nh;
                    nl = o.nl;
                    fa = o.fa;
                    fb = o.fb;
                }
                if (!rf_frac_ok(fa) || !rf_frac_ok(fb) || !rf_time_ok(nh) || !rf_time_ok(nl)) return RF_BAIL;
                if (!shared) {
                    if (dir > 0) q.lo[b] = hi0;
                    else q.hi[a] = lo1;
                }
                q.trail[a] = fa;
                q.lead[b] = fb;
                // the reference recomputes these stage times from the plan at
                // their next use; its partial sums cannot overflow when
                // value * den(lead) * den(trail) < 2^62 (value < 2^20 here)
                const Rat lf = from == b ? fb : q.lead[from], tf = from == a ? fa : q.trail[from];
                const Rat lt = to == b ? fb : q.lead[to], tt = to == a ? fa : q.trail[to];
                if (((lf.d | tf.d | lt.d | tt.d) >> 21) != 0 &&
                    (!stage_time_safe(nh, lf, tf) || !stage_time_safe(nl, lt, tt)))
                    return RF_BAIL;
                q.t[from] = nh;
                q.t[to] = nl;
                // boundaries a - 1, a, b are unstable
                memo &= ~(1ull << a);
                if (a > 0) memo &= ~(1ull << (a - 1));
                if (b < N - 1) memo &= ~(1ull << b);
                changed = true;
                ++moves;
                RF_MARK(5);
            }
        }
    }
    stats[0] = iters;
    stats[1] = evals;
    stats[2] = moves;
#if defined(RF_PROF) && defined(__CUDA_ARCH__)
    if (prof_out)
        for (int k = 0; k < 8; ++k) prof_out[k] = rf_prof[k];
#endif
    return RF_DONE;
}

}  // namespace bpk
