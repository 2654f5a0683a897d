/* oracle/bapipe_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the
 * product).  A plain-C restatement of the reference explore() path, written
 * for readability, not speed: every function follows the reference function
 * named beside it (paths relative to /root/reference/proj/include/bapipe/).
 * It deliberately keeps the reference's algorithms (O(N*U^2) DP, O(len) stage
 * sums, sort-based simulation) so it checks the CUDA path's shortcuts.
 *
 * Exceptions are emulated with setjmp/longjmp per candidate; allocations are
 * tracked per candidate so a longjmp never leaks.  Out-of-range layer reads
 * (undefined behaviour in the reference) raise
 * E_UB at the exact read the reference performs.
 *
 * Pinning: tests/test_oracle.py checks this file against (a) the reference's
 * own golden vectors (restated inline in tests/test_oracle.py from
 * proj/tests/test_*.cpp) and (b) the compiled reference (oracle/_ref) on thousands
 * of seeded random queries and the BASELINE configs.
 */
#include "bapipe_oracle.h"

#include <setjmp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;
typedef struct { int64_t n, d; } rat;

enum {
    E_NONE = 0, E_OVERFLOW, E_DOMAIN, E_INVALID_PLAN, E_INF_COARSEN, E_INF_FINETUNE,
    E_INF_NOCONV, E_SHAPE, E_UB, E_NOMEM
};

typedef struct {
    jmp_buf jb;
    int64_t detail, detail2;
    rat aux;
    void** allocs;
    int n_allocs, cap_allocs;
} exc_t;

static __thread exc_t* X;

static void raise_(int code) { longjmp(X->jb, code); }

static void* amalloc(size_t bytes) {
    if (X->n_allocs == X->cap_allocs) {
        int nc = X->cap_allocs ? 2 * X->cap_allocs : 64;
        void** na = (void**)realloc(X->allocs, sizeof(void*) * (size_t)nc);
        if (!na) raise_(E_NOMEM);
        X->allocs = na;
        X->cap_allocs = nc;
    }
    void* p = calloc(1, bytes ? bytes : 1);
    if (!p) raise_(E_NOMEM);
    X->allocs[X->n_allocs++] = p;
    return p;
}

static void afree_all(exc_t* e) {
    for (int i = 0; i < e->n_allocs; ++i) free(e->allocs[i]);
    free(e->allocs);
    e->allocs = NULL;
    e->n_allocs = e->cap_allocs = 0;
}

/* ---------------------------------------------------------------- Rat
 * rational.hpp:14-114.  from128 reduces with a 128-bit Euclid gcd and then
 * checks that the reduced numerator/denominator fit int64 (lines 83-95). */
static i128 gcd128(i128 a, i128 b) {
    while (b != 0) { i128 t = a % b; a = b; b = t; }
    return a == 0 ? 1 : a;
}

static rat from128(i128 n, i128 d) {
    if (d == 0) raise_(E_DOMAIN);
    if (d < 0) { n = -n; d = -d; }
    i128 an = n < 0 ? -n : n;
    i128 g = gcd128(an, d);
    if (g > 1) { n /= g; d /= g; }
    if (n > (i128)INT64_MAX || n < (i128)INT64_MIN || d > (i128)INT64_MAX) raise_(E_OVERFLOW);
    rat r = {(int64_t)n, (int64_t)d};
    return r;
}

static rat R(int64_t v) { rat r = {v, 1}; return r; }

static int64_t gcd64(int64_t a, int64_t b) {   /* std::gcd on non-negatives */
    while (b != 0) { int64_t t = a % b; a = b; b = t; }
    return a;
}

/* Rat(n, d) constructor -> normalize() (rational.hpp:18, 100-106). */
static rat Rnd(int64_t n, int64_t d) {
    if (d == 0) raise_(E_DOMAIN);
    if (d < 0) { n = -n; d = -d; }
    int64_t g = gcd64(n < 0 ? -n : n, d);
    if (g > 1) { n /= g; d /= g; }
    if (d == 0) d = 1;
    rat r = {n, d};
    return r;
}

static rat radd(rat a, rat b) { return from128((i128)a.n * b.d + (i128)b.n * a.d, (i128)a.d * b.d); }
static rat rsub(rat a, rat b) { return from128((i128)a.n * b.d - (i128)b.n * a.d, (i128)a.d * b.d); }
static rat rmul(rat a, rat b) { return from128((i128)a.n * b.n, (i128)a.d * b.d); }
static rat rdiv(rat a, rat b) {
    if (b.n == 0) raise_(E_DOMAIN);
    return from128((i128)a.n * b.d, (i128)a.d * b.n);
}
static int req(rat a, rat b) { return a.n == b.n && a.d == b.d; }
static int rlt(rat a, rat b) { return (i128)a.n * b.d < (i128)b.n * a.d; }
static int rgt(rat a, rat b) { return rlt(b, a); }
static int rle(rat a, rat b) { return !rlt(b, a); }
static int rge(rat a, rat b) { return !rlt(a, b); }
static rat rmax(rat a, rat b) { return rlt(a, b) ? b : a; }   /* std::max */
static rat rmin(rat a, rat b) { return rlt(b, a) ? b : a; }   /* std::min */
static int64_t rfloor(rat a) {                                  /* 59-63 */
    int64_t q = a.n / a.d;
    if (a.n % a.d != 0 && a.n < 0) --q;
    return q;
}
static int64_t rceil(rat a) {                                   /* 64-68 */
    int64_t q = a.n / a.d;
    if (a.n % a.d != 0 && a.n > 0) ++q;
    return q;
}
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }  /* 112-114 */
static bp_rat BR(rat r) { bp_rat o = {r.n, r.d}; return o; }
static rat RB(bp_rat r) { rat o = {r.num, r.den}; return o; }

/* ---------------------------------------------------------------- inputs */
typedef struct {
    int64_t L;
    int32_t T;
    const int64_t *fp, *bp, *w, *a;
} net_t;

typedef struct {
    int64_t N;
    int mode;
    const int32_t* type;
    const int64_t *cap, *minm, *bw;
} cl_t;

/* net.layers[j - 1] with j 1-based: any out-of-range read is the reference's UB. */
static int64_t L_idx(const net_t* net, int64_t j) {
    if (j < 1 || j > net->L) raise_(E_UB);
    return j - 1;
}
static int64_t fp_at(const net_t* net, int64_t j, int32_t t) { return net->fp[(size_t)t * net->L + L_idx(net, j)]; }
static int64_t bp_at(const net_t* net, int64_t j, int32_t t) { return net->bp[(size_t)t * net->L + L_idx(net, j)]; }
static int64_t w_at(const net_t* net, int64_t j) { return net->w[L_idx(net, j)]; }
static int64_t a_at(const net_t* net, int64_t j) { return net->a[L_idx(net, j)]; }

/* schedule_kind.hpp:52-57 */
static int64_t warmup_depth(int kind, int64_t N, int64_t s) {
    int64_t d = N - s + 1;
    if (kind == BP_KIND_FBP_AS || kind == BP_KIND_1F1B_SO) d *= 2;
    return d;
}

/* ---------------------------------------------------------------- plan
 * plan.hpp:16-28 */
typedef struct {
    int64_t N;
    int64_t *lo, *hi;
    rat *lead, *trail;
} plan_t;

static plan_t plan_new(int64_t N) {
    plan_t p;
    p.N = N;
    p.lo = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    p.hi = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    p.lead = (rat*)amalloc(sizeof(rat) * (size_t)N);
    p.trail = (rat*)amalloc(sizeof(rat) * (size_t)N);
    for (int64_t i = 0; i < N; ++i) { p.lo[i] = p.hi[i] = 1; p.lead[i] = R(1); p.trail[i] = R(1); }
    return p;
}

static void plan_copy(plan_t* dst, const plan_t* src) {
    memcpy(dst->lo, src->lo, sizeof(int64_t) * (size_t)src->N);
    memcpy(dst->hi, src->hi, sizeof(int64_t) * (size_t)src->N);
    memcpy(dst->lead, src->lead, sizeof(rat) * (size_t)src->N);
    memcpy(dst->trail, src->trail, sizeof(rat) * (size_t)src->N);
}

static plan_t plan_dup(const plan_t* src) {
    plan_t p = plan_new(src->N);
    plan_copy(&p, src);
    return p;
}

/* owned_fraction, plan.hpp:33-39 */
static rat owned_fraction(const plan_t* p, int64_t n, int64_t j) {
    if (j < p->lo[n] || j > p->hi[n]) return R(0);
    if (p->lo[n] == p->hi[n]) return rsub(radd(p->lead[n], p->trail[n]), R(1));
    if (j == p->lo[n]) return p->lead[n];
    if (j == p->hi[n]) return p->trail[n];
    return R(1);
}

/* validate_plan, plan.hpp:41-85 */
static void invalid(int code, int64_t idx) {
    X->detail = code;
    X->detail2 = idx;
    raise_(E_INVALID_PLAN);
}

static void validate_plan(const plan_t* p, const net_t* net) {
    if (p->N == 0) invalid(0, 0);
    int64_t L = net->L, prev_hi = 0;
    for (int64_t n = 0; n < p->N; ++n) {
        if (p->lo[n] < 1 || p->hi[n] > L || p->lo[n] > p->hi[n]) invalid(BP_IP_RANGE, n + 1);
        rat zero = R(0), one = R(1);
        if (!rgt(p->lead[n], zero) || rgt(p->lead[n], one) || !rgt(p->trail[n], zero) ||
            rgt(p->trail[n], one))
            invalid(BP_IP_FRACTION, n + 1);
        if (n == 0) {
            if (p->lo[n] != 1 || !req(p->lead[n], one)) invalid(BP_IP_FIRST, 1);
        } else {
            int shared = (p->lo[n] == prev_hi);
            if (!shared && p->lo[n] != prev_hi + 1) invalid(BP_IP_CONTIG, n + 1);
            if (shared && req(p->lead[n], one)) invalid(BP_IP_SHARED_FULL, n + 1);
            if (!shared && !req(p->lead[n], one)) invalid(BP_IP_LEAD_UNSHARED, n + 1);
        }
        prev_hi = p->hi[n];
    }
    if (p->hi[p->N - 1] != L || !req(p->trail[p->N - 1], R(1))) invalid(BP_IP_LAST, 0);
    for (int64_t j = 1; j <= L; ++j) {
        rat sum = R(0);
        for (int64_t n = 0; n < p->N; ++n) sum = radd(sum, owned_fraction(p, n, j));
        if (!req(sum, R(1))) { X->aux = sum; invalid(BP_IP_COVERAGE, j); }
    }
}

/* stage_fp_time / stage_bp_time / stage_compute_time, plan.hpp:90-113 */
static rat stage_fp_time(const plan_t* p, int64_t n, const net_t* net, const cl_t* cl) {
    rat t = R(0);
    for (int64_t j = p->lo[n]; j <= p->hi[n]; ++j)
        t = radd(t, rmul(owned_fraction(p, n, j), R(fp_at(net, j, cl->type[n]))));
    return t;
}
static rat stage_bp_time(const plan_t* p, int64_t n, const net_t* net, const cl_t* cl) {
    rat t = R(0);
    for (int64_t j = p->lo[n]; j <= p->hi[n]; ++j)
        t = radd(t, rmul(owned_fraction(p, n, j), R(bp_at(net, j, cl->type[n]))));
    return t;
}
static rat stage_compute_time(const plan_t* p, int64_t n, const net_t* net, const cl_t* cl) {
    rat f = stage_fp_time(p, n, net, cl);
    rat b = stage_bp_time(p, n, net, cl);
    return radd(f, b);
}
/* plan.hpp:115-123 */
static rat max_stage_compute_time(const plan_t* p, const net_t* net, const cl_t* cl) {
    rat m = R(0);
    for (int64_t n = 0; n < p->N; ++n) {
        rat t = stage_compute_time(p, n, net, cl);
        if (rgt(t, m)) m = t;
    }
    return m;
}
/* plan.hpp:125-132 */
static rat stage_weight_bytes(const plan_t* p, int64_t n, const net_t* net) {
    rat w = R(0);
    for (int64_t j = p->lo[n]; j <= p->hi[n]; ++j)
        w = radd(w, rmul(owned_fraction(p, n, j), R(w_at(net, j))));
    return w;
}
/* plan.hpp:136-148 (k, i 1-based) */
static int64_t cut_activation_bytes(const plan_t* p, int64_t k, const net_t* net) {
    return a_at(net, p->hi[k - 1]);
}
static int64_t stage_activation_bytes(const plan_t* p, int64_t i, const net_t* net) {
    if (i >= 2) return cut_activation_bytes(p, i - 1, net);
    return a_at(net, p->hi[0]);
}
/* plan.hpp:152-158 */
static int64_t link_sr_time(const plan_t* p, int64_t k, const net_t* net, const cl_t* cl, int64_t micro) {
    int64_t a = cut_activation_bytes(p, k, net) * micro;
    if (a == 0) return 0;
    return ceil_div(a, cl->bw[k - 1]);
}

/* ---------------------------------------------------------------- cost models
 * cost_models.hpp:50-100 */
static rat minibatch_time(int kind, int64_t M, int64_t N, rat F, rat B, rat SR) {
    rat base = rmul(R(M + N - 1), radd(F, B));
    switch (kind) {
        case BP_KIND_1F1B_SNO:
            return radd(base, rmul(rmul(R(N + M - 2 - ceil_div(M - 1, N)), R(2)), SR));
        case BP_KIND_1F1B_SO:
            return radd(base, rmul(rmul(R(N - 1), R(2)), SR));
        default:
            return base;
    }
}

static rat bubble_fraction(int kind, int64_t M, int64_t N, rat F, rat B, rat SR) {
    if (N == 1) return R(0);
    rat total = minibatch_time(kind, M, N, F, B, SR);
    switch (kind) {
        case BP_KIND_1F1B_SNO: {
            rat inner = radd(radd(F, B), rmul(R(2), SR));
            rat num = radd(rmul(R(N - 1), inner),
                           rmul(rmul(R(M - 1 - ceil_div(M - 1, N)), R(2)), SR));
            return rdiv(num, total);
        }
        case BP_KIND_1F1B_SO: {
            rat inner = radd(radd(F, B), rmul(R(2), SR));
            return rdiv(rmul(R(N - 1), inner), total);
        }
        default:
            return Rnd(N - 1, M + N - 1);
    }
}

static rat features_memory(int kind, int64_t N, int64_t i, rat a) {
    rat m = rmul(R(N - i + 1), a);
    if (kind == BP_KIND_FBP_AS || kind == BP_KIND_1F1B_SO) m = rmul(R(2), m);
    return m;
}
static rat weights_memory(rat w) { return rmul(R(2), w); }
static rat bandwidth_demand(int kind, rat a, rat F, rat B) {
    if (kind == BP_KIND_FBP_AS) return rdiv(rmul(R(2), a), radd(F, B));
    return rdiv(a, F);
}

typedef struct {
    rat minibatch, bubble;
    rat *features, *weights, *bw;
    int* infeasible;
    int heuristic;
} est_t;

/* estimate, cost_models.hpp:124-166 (with stage_costs, 103-119) */
static est_t estimate(int kind, const plan_t* p, const net_t* net, const cl_t* cl, int64_t M,
                      int64_t micro) {
    int64_t N = p->N;
    rat* F = (rat*)amalloc(sizeof(rat) * (size_t)N);
    rat* B = (rat*)amalloc(sizeof(rat) * (size_t)N);
    rat* W = (rat*)amalloc(sizeof(rat) * (size_t)N);
    int64_t* A = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    int64_t* S = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    for (int64_t i = 1; i <= N; ++i) {
        F[i - 1] = stage_fp_time(p, i - 1, net, cl);
        B[i - 1] = stage_bp_time(p, i - 1, net, cl);
        W[i - 1] = stage_weight_bytes(p, i - 1, net);
        A[i - 1] = stage_activation_bytes(p, i, net) * micro;
        S[i - 1] = (i >= 2) ? link_sr_time(p, i - 1, net, cl, micro) : 0;
    }
    rat Fm = R(0), Bm = R(0);
    int64_t SRm = 0;
    int balanced = 1;
    for (int64_t i = 0; i < N; ++i) {
        if (!req(F[i], F[0]) || !req(B[i], B[0])) balanced = 0;
        if (rgt(F[i], Fm)) Fm = F[i];
        if (rgt(B[i], Bm)) Bm = B[i];
        if (S[i] > SRm) SRm = S[i];
    }
    for (int64_t i = 2; i <= N; ++i)
        if (S[i - 1] != S[N > 1 ? 1 : 0]) balanced = 0;
    est_t e;
    e.minibatch = minibatch_time(kind, M, N, Fm, Bm, R(SRm));
    e.bubble = bubble_fraction(kind, M, N, Fm, Bm, R(SRm));
    e.heuristic = !balanced || M < N;
    e.features = (rat*)amalloc(sizeof(rat) * (size_t)N);
    e.weights = (rat*)amalloc(sizeof(rat) * (size_t)N);
    e.bw = (rat*)amalloc(sizeof(rat) * (size_t)(N > 1 ? N - 1 : 1));
    e.infeasible = (int*)amalloc(sizeof(int) * (size_t)N);
    for (int64_t i = 1; i <= N; ++i) {
        rat fm = features_memory(kind, N, i, R(A[i - 1]));
        rat wm = weights_memory(W[i - 1]);
        e.features[i - 1] = fm;
        e.weights[i - 1] = wm;
        e.infeasible[i - 1] = rgt(radd(fm, wm), R(cl->cap[i - 1]));
    }
    for (int64_t k = 1; k <= N - 1; ++k) {
        rat a = R(cut_activation_bytes(p, k, net) * micro);
        e.bw[k - 1] = bandwidth_demand(kind, a, Fm, Bm);
    }
    return e;
}

static int memory_feasible(const est_t* e, int64_t N) {
    for (int64_t i = 0; i < N; ++i)
        if (e->infeasible[i]) return 0;
    return 1;
}

/* ---------------------------------------------------------------- partition
 * partition.hpp:44-220 */
typedef struct {
    int64_t lo, hi, w, out_act;
    int64_t* cost;   /* [N] */
} unit_t;

#define DP_INF (INT64_MAX / 4)

/* partition_units, partition.hpp:112-185; writes unit ranges (1-based). */
static void partition_units(const unit_t* units, int64_t U, int64_t N, int64_t* rlo, int64_t* rhi,
                            int64_t* t_opt_out) {
    if (U < N) { X->detail = U; raise_(E_SHAPE); }
    size_t W = (size_t)(U + 1);
    int64_t* time = (int64_t*)amalloc(sizeof(int64_t) * (size_t)(N + 1) * W);
    int64_t* wsum = (int64_t*)amalloc(sizeof(int64_t) * W);
    for (int64_t j = 1; j <= U; ++j) {
        wsum[j] = wsum[j - 1] + units[j - 1].w;
        for (int64_t n = 1; n <= N; ++n)
            time[n * W + j] = time[n * W + j - 1] + units[j - 1].cost[n - 1];
    }
#define SEG_TIME(n, k, j) (time[(n) * W + (j)] - time[(n) * W + (k)])
#define SEG_FOOT(n, k, j) \
    (2 * (wsum[j] - wsum[k]) + (N - (n) + 1) * ((k) >= 1 ? units[(k) - 1].out_act : units[(j) - 1].out_act))
    int64_t* dp = (int64_t*)amalloc(sizeof(int64_t) * (size_t)(N + 1) * W);
    for (size_t i = 0; i < (size_t)(N + 1) * W; ++i) dp[i] = DP_INF;
    dp[0] = 0;
    for (int64_t n = 1; n <= N; ++n)
        for (int64_t j = n; j <= U - (N - n); ++j)
            for (int64_t k = n - 1; k < j; ++k) {
                if (dp[(n - 1) * W + k] == DP_INF) continue;
                int64_t s = SEG_TIME(n, k, j);
                int64_t v = dp[(n - 1) * W + k] > s ? dp[(n - 1) * W + k] : s;
                if (v < dp[n * W + j]) dp[n * W + j] = v;
            }
    int64_t T_opt = dp[N * W + U];
    int64_t* g = (int64_t*)amalloc(sizeof(int64_t) * (size_t)(N + 1) * W);
    for (size_t i = 0; i < (size_t)(N + 1) * W; ++i) g[i] = DP_INF;
    g[0] = 0;
    for (int64_t n = 1; n <= N; ++n)
        for (int64_t j = n; j <= U - (N - n); ++j)
            for (int64_t k = n - 1; k < j; ++k) {
                if (g[(n - 1) * W + k] == DP_INF || SEG_TIME(n, k, j) > T_opt) continue;
                int64_t f = SEG_FOOT(n, k, j);
                int64_t v = g[(n - 1) * W + k] > f ? g[(n - 1) * W + k] : f;
                if (v < g[n * W + j]) g[n * W + j] = v;
            }
    int64_t F_opt = g[N * W + U];
    char* feas = (char*)amalloc((size_t)(N + 1) * W);
    feas[N * W + U] = 1;
    for (int64_t n = N - 1; n >= 0; --n)
        for (int64_t j = n; j <= U; ++j)
            for (int64_t j2 = j + 1; j2 <= U; ++j2) {
                if (SEG_TIME(n + 1, j, j2) > T_opt || SEG_FOOT(n + 1, j, j2) > F_opt) continue;
                if (feas[(n + 1) * W + j2]) { feas[n * W + j] = 1; break; }
            }
    int64_t cur = 0;
    for (int64_t n = 1; n <= N; ++n) {
        int64_t chosen = -1;
        for (int64_t j = cur + 1; j <= U; ++j) {
            if (SEG_TIME(n, cur, j) > T_opt || SEG_FOOT(n, cur, j) > F_opt) continue;
            if (feas[n * W + j]) { chosen = j; break; }
        }
        if (chosen < 0) raise_(E_NOMEM);   /* "partition reconstruction failed", unreachable */
        rlo[n - 1] = cur + 1;
        rhi[n - 1] = chosen;
        cur = chosen;
    }
    if (t_opt_out) *t_opt_out = T_opt;
#undef SEG_TIME
#undef SEG_FOOT
}

/* units_from_network (78-89) + partition_units + plan_from_ranges (187-200) */
static plan_t inter_layer_partition(const net_t* net, const cl_t* cl, int64_t* t_opt) {
    int64_t U = net->L, N = cl->N;
    unit_t* units = (unit_t*)amalloc(sizeof(unit_t) * (size_t)U);
    for (int64_t j = 1; j <= U; ++j) {
        units[j - 1].lo = units[j - 1].hi = j;
        units[j - 1].w = w_at(net, j);
        units[j - 1].out_act = a_at(net, j);
        units[j - 1].cost = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
        for (int64_t n = 0; n < N; ++n)
            units[j - 1].cost[n] = fp_at(net, j, cl->type[n]) + bp_at(net, j, cl->type[n]);
    }
    int64_t* rlo = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    int64_t* rhi = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    partition_units(units, U, N, rlo, rhi, t_opt);
    plan_t p = plan_new(N);
    for (int64_t n = 0; n < N; ++n) { p.lo[n] = units[rlo[n] - 1].lo; p.hi[n] = units[rhi[n] - 1].hi; }
    return p;
}

/* coarsen_by_comm (44-67) + units_from_coarse (91-107) + partition_units */
static int64_t coarse_block_count(const net_t* net, int64_t a_th) {
    int64_t K = 0;
    for (int64_t j = 1; j <= net->L; ++j)
        if (j == net->L || a_at(net, j) <= a_th) ++K;
    return K;
}

static plan_t coarse_partition(const net_t* net, const cl_t* cl, int64_t a_th, int64_t* t_opt) {
    int64_t N = cl->N, K = coarse_block_count(net, a_th);
    unit_t* units = (unit_t*)amalloc(sizeof(unit_t) * (size_t)(K > 0 ? K : 1));
    int64_t start = 1, b = 0;
    for (int64_t j = 1; j <= net->L; ++j) {
        if (!(j == net->L || a_at(net, j) <= a_th)) continue;
        unit_t* u = &units[b++];
        u->lo = start;
        u->hi = j;
        u->w = 0;
        u->cost = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
        for (int64_t i = start; i <= j; ++i) u->w += w_at(net, i);
        u->out_act = a_at(net, j);
        for (int64_t n = 0; n < N; ++n) {
            int64_t fs = 0, bs = 0;
            for (int64_t i = start; i <= j; ++i) { fs += fp_at(net, i, cl->type[n]); bs += bp_at(net, i, cl->type[n]); }
            u->cost[n] = fs + bs;
        }
        start = j + 1;
    }
    int64_t* rlo = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    int64_t* rhi = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    partition_units(units, K, N, rlo, rhi, t_opt);
    plan_t p = plan_new(N);
    for (int64_t n = 0; n < N; ++n) { p.lo[n] = units[rlo[n] - 1].lo; p.hi[n] = units[rhi[n] - 1].hi; }
    return p;
}

/* detect_comm_bottleneck, partition.hpp:228-241 (bottleneck flag only) */
static int comm_bottleneck(const plan_t* p, const net_t* net, const cl_t* cl, rat target, int64_t micro) {
    int b = 0;
    for (int64_t k = 1; k <= p->N - 1; ++k) {
        int64_t ct = link_sr_time(p, k, net, cl, micro);
        if (rgt(R(ct), target)) b = 1;
    }
    return b;
}

/* intra_layer_refine, partition.hpp:248-333 */
static rat refine_layer_cost(const net_t* net, const cl_t* cl, int64_t j, int64_t stage) {
    int32_t t = cl->type[stage];
    return R(fp_at(net, j, t) + bp_at(net, j, t));
}

static rat refine_quantize(rat x, rat t_hi, rat t_lo, rat c_from, rat c_to, rat avail) {
    if (x.d <= 1024) return x;
    rat lo = Rnd(rfloor(rmul(x, R(1024))), 1024);
    rat hi = Rnd(rceil(rmul(x, R(1024))), 1024);
    if (rge(hi, avail)) return lo;
    rat s_lo = rmax(rsub(t_hi, rmul(lo, c_from)), radd(t_lo, rmul(lo, c_to)));
    rat s_hi = rmax(rsub(t_hi, rmul(hi, c_from)), radd(t_lo, rmul(hi, c_to)));
    return rle(s_lo, s_hi) ? lo : hi;
}

static void refine_apply_move(plan_t* p, int64_t n0, int dir, rat x) {
    int64_t a = n0, b = n0 + 1;
    int shared = (p->hi[a] == p->lo[b]);
    if (dir > 0) {
        if (shared) {
            p->trail[a] = rsub(p->trail[a], x);
            p->lead[b] = radd(p->lead[b], x);
        } else {
            p->trail[a] = rsub(R(1), x);
            p->lo[b] = p->hi[a];
            p->lead[b] = x;
        }
    } else {
        if (shared) {
            p->lead[b] = rsub(p->lead[b], x);
            p->trail[a] = radd(p->trail[a], x);
        } else {
            p->lead[b] = rsub(R(1), x);
            p->hi[a] = p->lo[b];
            p->trail[a] = x;
        }
    }
}

static void intra_layer_refine(plan_t* p, const net_t* net, const cl_t* cl) {
    int64_t N = p->N;
    if (N <= 1) return;
    int changed = 1, guard = 0;
    while (changed && ++guard < 1000) {
        changed = 0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int64_t i = 0; i < N - 1; ++i) {
                int64_t n0 = (pass == 0) ? i : (N - 2 - i);
                rat t_a = stage_compute_time(p, n0, net, cl);
                rat t_b = stage_compute_time(p, n0 + 1, net, cl);
                if (req(t_a, t_b)) continue;
                int dir = rgt(t_a, t_b) ? +1 : -1;
                int64_t from = dir > 0 ? n0 : n0 + 1;
                int64_t j = dir > 0 ? p->hi[from] : p->lo[from];
                int shared = (p->hi[n0] == p->lo[n0 + 1]);
                if (dir < 0 && !shared) {
                    int64_t cur_cut = a_at(net, p->hi[n0]);
                    if (a_at(net, j) > cur_cut) continue;
                }
                rat c_from = refine_layer_cost(net, cl, j, dir > 0 ? n0 : n0 + 1);
                rat c_to = refine_layer_cost(net, cl, j, dir > 0 ? n0 + 1 : n0);
                rat t_hi = rmax(t_a, t_b), t_lo = rmin(t_a, t_b);
                rat x = rdiv(rsub(t_hi, t_lo), radd(c_from, c_to));
                rat avail = owned_fraction(p, from, j);
                if (rge(x, avail)) x = rsub(avail, Rnd(1, 1024));
                if (!rgt(x, R(0))) continue;
                x = refine_quantize(x, t_hi, t_lo, c_from, c_to, avail);
                if (!rgt(x, R(0)) || rge(x, avail)) continue;
                rat nh = rsub(t_hi, rmul(x, c_from));
                rat nl = radd(t_lo, rmul(x, c_to));
                if (rge(rmax(nh, nl), t_hi)) continue;
                refine_apply_move(p, n0, dir, x);
                changed = 1;
            }
        }
    }
}

/* memory_fine_tune, partition.hpp:339-435 */
static rat overloads(const plan_t* p, const net_t* net, const cl_t* cl, int kind, int64_t M,
                     int64_t micro, rat* over) {
    est_t e = estimate(kind, p, net, cl, M, micro);
    rat total = R(0);
    for (int64_t i = 0; i < p->N; ++i) {
        rat mem = radd(e.features[i], e.weights[i]);
        rat cap = R(cl->cap[i]);
        rat ov = rgt(mem, cap) ? rsub(mem, cap) : R(0);
        over[i] = ov;
        total = radd(total, ov);
    }
    return total;
}

static rat headroom(const plan_t* p, const net_t* net, const cl_t* cl, int kind, int64_t M,
                    int64_t micro, int64_t i) {
    est_t e = estimate(kind, p, net, cl, M, micro);
    return rsub(R(cl->cap[i]), radd(e.features[i], e.weights[i]));
}

static void memory_fine_tune(plan_t* p, const net_t* net, const cl_t* cl, int kind, int64_t M,
                             int64_t micro) {
    int64_t N = p->N;
    rat* over = (rat*)amalloc(sizeof(rat) * (size_t)N);
    rat* over2 = (rat*)amalloc(sizeof(rat) * (size_t)N);
    if (req(overloads(p, net, cl, kind, M, micro, over), R(0))) return;
    for (int64_t n = 0; n < N - 1; ++n) {
        int64_t a = n, b = n + 1;
        if (p->hi[a] != p->lo[b]) continue;
        if (rge(p->trail[a], p->lead[b])) {
            p->trail[a] = R(1);
            p->lo[b] = p->hi[a] + 1;
            p->lead[b] = R(1);
        } else {
            p->lead[b] = R(1);
            p->hi[a] = p->hi[a] - 1;
            p->trail[a] = R(1);
        }
    }
    rat total = overloads(p, net, cl, kind, M, micro, over);
    int guard = 0;
    plan_t saved = plan_new(N);
    while (rgt(total, R(0))) {
        if (++guard > 8 * (int)(N * net->L + 4)) raise_(E_INF_NOCONV);
        int64_t worst = 0;
        for (int64_t i = 1; i < N; ++i)
            if (rgt(over[i], over[worst])) worst = i;
        int64_t cn[2];
        int cd[2], nc = 0;
        if (worst > 0) { cn[nc] = worst - 1; cd[nc] = -1; ++nc; }
        if (worst < N - 1) { cn[nc] = worst + 1; cd[nc] = +1; ++nc; }
        if (nc == 2) {
            rat hr = headroom(p, net, cl, kind, M, micro, worst + 1);
            rat hl = headroom(p, net, cl, kind, M, micro, worst - 1);
            if (rgt(hr, hl)) {
                int64_t tn = cn[0]; cn[0] = cn[1]; cn[1] = tn;
                int td = cd[0]; cd[0] = cd[1]; cd[1] = td;
            }
        }
        int moved = 0;
        for (int relax = 0; relax < 2 && !moved; ++relax) {
            for (int c = 0; c < nc; ++c) {
                if (p->lo[worst] == p->hi[worst]) continue;
                plan_copy(&saved, p);
                if (cd[c] < 0) {
                    p->lo[worst] += 1;
                    p->hi[cn[c]] += 1;
                } else {
                    p->hi[worst] -= 1;
                    p->lo[cn[c]] -= 1;
                }
                rat total2 = overloads(p, net, cl, kind, M, micro, over2);
                int ok = rlt(total2, total);
                if (ok && !relax) {
                    rat target = max_stage_compute_time(p, net, cl);
                    ok = !comm_bottleneck(p, net, cl, target, micro);
                }
                if (ok) {
                    memcpy(over, over2, sizeof(rat) * (size_t)N);
                    total = total2;
                    moved = 1;
                    break;
                }
                plan_copy(p, &saved);
            }
        }
        if (!moved) raise_(E_INF_FINETUNE);
    }
}

/* balance_partition, partition.hpp:441-474 */
static plan_t balance_partition(const net_t* net, const cl_t* cl, int kind, int64_t M, int64_t micro) {
    int64_t N = cl->N;
    if (N == 1) {
        plan_t p = plan_new(1);
        p.lo[0] = 1;
        p.hi[0] = net->L;
        memory_fine_tune(&p, net, cl, kind, M, micro);
        return p;
    }
    plan_t p = inter_layer_partition(net, cl, NULL);
    rat target = max_stage_compute_time(&p, net, cl);
    if (comm_bottleneck(&p, net, cl, target, micro)) {
        int64_t min_bw = cl->bw[0];
        for (int64_t k = 1; k < N - 1; ++k)
            if (cl->bw[k] < min_bw) min_bw = cl->bw[k];
        int64_t a_th = rfloor(rdiv(rmul(R(min_bw), target), R(micro)));
        int64_t K = coarse_block_count(net, a_th);
        if (K < N) { X->detail = K; raise_(E_INF_COARSEN); }
        plan_t c = coarse_partition(net, cl, a_th, NULL);
        memory_fine_tune(&c, net, cl, kind, M, micro);
        return c;
    }
    intra_layer_refine(&p, net, cl);
    est_t e = estimate(kind, &p, net, cl, M, micro);
    if (!memory_feasible(&e, N)) memory_fine_tune(&p, net, cl, kind, M, micro);
    return p;
}

/* ---------------------------------------------------------------- simulator
 * simulator.hpp:57-274 */
typedef struct { int64_t pos, sub; int type; int64_t stage, m; } op_t;

static int op_cmp(const void* va, const void* vb) {   /* simulator.hpp:119-125 */
    const op_t* x = (const op_t*)va;
    const op_t* y = (const op_t*)vb;
    if (x->pos != y->pos) return x->pos < y->pos ? -1 : 1;
    if (x->sub != y->sub) return x->sub < y->sub ? -1 : 1;
    if (x->type != y->type) return x->type < y->type ? -1 : 1;
    if (x->stage != y->stage) return x->stage < y->stage ? -1 : 1;
    if (x->m != y->m) return x->m < y->m ? -1 : 1;
    return 0;
}

typedef struct { int64_t t_num, t_den; int d; } hw_pt;

static rat simulate_chain(int kind, int64_t N, const rat* F, const rat* B, const int64_t* SR,
                          const int64_t* act, const rat* w, int64_t M) {
    if (M < 1) invalid(0, 0);
    int async = (kind == BP_KIND_1F1B_AS || kind == BP_KIND_FBP_AS);
    int64_t* warm = (int64_t*)amalloc(sizeof(int64_t) * (size_t)(N + 1));
    for (int64_t s = 1; s <= N; ++s) {
        int64_t d = warmup_depth(kind, N, s);
        warm[s] = M < d ? M : d;
    }
#define POSF(m, s) ((m) <= warm[s] ? (m) - 1 : 2 * (m) - warm[s] - 1)
    size_t n_ops = (size_t)(2 * N * M + (async ? 0 : 2 * (N - 1) * M));
    op_t* ops = (op_t*)amalloc(sizeof(op_t) * (n_ops ? n_ops : 1));
    size_t o = 0;
    for (int64_t s = 1; s <= N; ++s)
        for (int64_t m = 1; m <= M; ++m) {
            int64_t pb = warm[s] + 2 * (m - 1), last_f = POSF(M, s);
            if (pb > last_f) pb = last_f + (m - (M - warm[s]));
            op_t f = {POSF(m, s), 2 * s, 0, s, m};
            op_t b = {pb, 2 * (N + 1 - s), 1, s, m};
            ops[o++] = f;
            ops[o++] = b;
        }
    if (!async)
        for (int64_t k = 1; k <= N - 1; ++k)
            for (int64_t m = 1; m <= M; ++m) {
                int64_t pb = warm[k + 1] + 2 * (m - 1), last_f = POSF(M, k + 1);
                if (pb > last_f) pb = last_f + (m - (M - warm[k + 1]));
                op_t tf = {POSF(m, k), 2 * k + 1, 2, k, m};
                op_t tb = {pb, 2 * (N - k) + 1, 3, k, m};
                ops[o++] = tf;
                ops[o++] = tb;
            }
    qsort(ops, o, sizeof(op_t), op_cmp);
#undef POSF
    size_t NM = (size_t)(N * M), LM = (size_t)((N > 1 ? N - 1 : 1) * M);
    rat* startF = (rat*)amalloc(sizeof(rat) * NM);
    rat* endF = (rat*)amalloc(sizeof(rat) * NM);
    rat* startB = (rat*)amalloc(sizeof(rat) * NM);
    rat* endB = (rat*)amalloc(sizeof(rat) * NM);
    rat* sFs = (rat*)amalloc(sizeof(rat) * LM);
    rat* sFe = (rat*)amalloc(sizeof(rat) * LM);
    rat* sBs = (rat*)amalloc(sizeof(rat) * LM);
    rat* sBe = (rat*)amalloc(sizeof(rat) * LM);
    rat* free_ = (rat*)amalloc(sizeof(rat) * (size_t)(N + 1));
    for (size_t i = 0; i < NM; ++i) startF[i] = endF[i] = startB[i] = endB[i] = R(0);
    for (size_t i = 0; i < LM; ++i) sFs[i] = sFe[i] = sBs[i] = sBe[i] = R(0);
    for (int64_t s = 0; s <= N; ++s) free_[s] = R(0);
#define IDX(m, s) ((size_t)(((s) - 1) * M + ((m) - 1)))
#define LIDX(m, k) ((size_t)(((k) - 1) * M + ((m) - 1)))
    for (size_t i = 0; i < o; ++i) {
        int64_t m = ops[i].m, s = ops[i].stage;
        if (ops[i].type == 0) {
            rat ready = free_[s];
            if (s > 1) {
                rat arr = async ? endF[IDX(m, s - 1)] : sFe[LIDX(m, s - 1)];
                if (rgt(arr, ready)) ready = arr;
            }
            startF[IDX(m, s)] = ready;
            endF[IDX(m, s)] = radd(ready, F[s - 1]);
            free_[s] = endF[IDX(m, s)];
        } else if (ops[i].type == 1) {
            rat ready = free_[s];
            if (rgt(endF[IDX(m, s)], ready)) ready = endF[IDX(m, s)];
            if (s < N) {
                rat arr = async ? endB[IDX(m, s + 1)] : sBe[LIDX(m, s)];
                if (rgt(arr, ready)) ready = arr;
            }
            startB[IDX(m, s)] = ready;
            endB[IDX(m, s)] = radd(ready, B[s - 1]);
            free_[s] = endB[IDX(m, s)];
        } else if (ops[i].type == 2) {
            rat ready = endF[IDX(m, s)];
            sFs[LIDX(m, s)] = ready;
            sFe[LIDX(m, s)] = radd(ready, R(SR[s - 1]));
        } else {
            rat ready = endB[IDX(m, s + 1)];
            sBs[LIDX(m, s)] = ready;
            sBe[LIDX(m, s)] = radd(ready, R(SR[s - 1]));
        }
    }
    rat makespan = R(0);
    for (int64_t s = 1; s <= N; ++s)
        if (rgt(free_[s], makespan)) makespan = free_[s];
    if (!async)
        for (int64_t k = 1; k <= N - 1; ++k) {
            if (rgt(sFe[LIDX(M, k)], makespan)) makespan = sFe[LIDX(M, k)];
            if (rgt(sBe[LIDX(M, k)], makespan)) makespan = sBe[LIDX(M, k)];
        }
    /* Event emission (182-216) adds 0 = Rat(0) * makespan to every start/end
     * and sorts: no new values, so no observable effect on explore(). */
    (void)rmul(R(0), makespan);
    /* Feature high-water (219-238): peak in-flight count times a, via the
     * reference's sweep over (FP start, BP end) points. */
    hw_pt* pts = (hw_pt*)amalloc(sizeof(hw_pt) * (size_t)(2 * M));
    for (int64_t s = 1; s <= N; ++s) {
        int64_t cur = 0, peak = 0;
        /* sort (time, delta) with frees before allocations at equal time */
        int64_t np = 0;
        for (int64_t m = 1; m <= M; ++m) {
            hw_pt a = {startF[IDX(m, s)].n, startF[IDX(m, s)].d, +1};
            hw_pt b = {endB[IDX(m, s)].n, endB[IDX(m, s)].d, -1};
            pts[np++] = a;
            pts[np++] = b;
        }
        for (int64_t i = 1; i < np; ++i) {      /* insertion sort, stable enough for counting */
            hw_pt v = pts[i];
            int64_t k = i - 1;
            while (k >= 0) {
                rat tk = {pts[k].t_num, pts[k].t_den}, tv = {v.t_num, v.t_den};
                int gt = rlt(tv, tk) || (req(tv, tk) && v.d < pts[k].d);
                if (!gt) break;
                pts[k + 1] = pts[k];
                --k;
            }
            pts[k + 1] = v;
        }
        for (int64_t i = 0; i < np; ++i) {
            cur += pts[i].d;
            if (cur > peak) peak = cur;
        }
        (void)rmul(R(peak), R(act[s - 1]));
        (void)rmul(R(2), w[s - 1]);
    }
    for (int64_t k = 1; k <= N - 1; ++k) {
        if (!req(makespan, R(0))) (void)rdiv(R(M * SR[k - 1]), makespan);
    }
#undef IDX
#undef LIDX
    return makespan;
}

/* simulate (264-274) = validate_plan + chain_instance (248-262) + simulate_chain */
static rat simulate(int kind, const plan_t* p, const net_t* net, const cl_t* cl, int64_t M, int64_t micro) {
    validate_plan(p, net);
    int64_t N = p->N;
    rat* F = (rat*)amalloc(sizeof(rat) * (size_t)N);
    rat* B = (rat*)amalloc(sizeof(rat) * (size_t)N);
    rat* W = (rat*)amalloc(sizeof(rat) * (size_t)N);
    int64_t* A = (int64_t*)amalloc(sizeof(int64_t) * (size_t)N);
    int64_t* S = (int64_t*)amalloc(sizeof(int64_t) * (size_t)(N > 1 ? N - 1 : 1));
    for (int64_t i = 1; i <= N; ++i) {
        F[i - 1] = stage_fp_time(p, i - 1, net, cl);
        B[i - 1] = stage_bp_time(p, i - 1, net, cl);
        A[i - 1] = stage_activation_bytes(p, i, net) * micro;
        W[i - 1] = stage_weight_bytes(p, i - 1, net);
    }
    for (int64_t k = 1; k <= N - 1; ++k) S[k - 1] = link_sr_time(p, k, net, cl, micro);
    return simulate_chain(kind, N, F, B, S, A, W, M);
}

/* ---------------------------------------------------------------- explore
 * explorer.hpp:17-155 */
static int kinds_of(int mode, int* k) {
    if (mode == BP_MODE_ASYNC) { k[0] = BP_KIND_1F1B_AS; k[1] = BP_KIND_FBP_AS; }
    else { k[0] = BP_KIND_1F1B_SNO; k[1] = BP_KIND_1F1B_SO; }
    return 2;
}

static int64_t n_base(const bp_query* q) {
    if (q->n_m > 0 && q->m_list) return q->n_m;
    int64_t c = 0;
    for (int64_t m = 1; m <= q->mini_batch; ++m)
        if (q->mini_batch % m == 0) ++c;
    return c;
}

static int64_t base_at(const bp_query* q, int64_t i) {
    if (q->n_m > 0 && q->m_list) return q->m_list[i];
    int64_t c = 0;
    for (int64_t m = 1; m <= q->mini_batch; ++m)
        if (q->mini_batch % m == 0 && c++ == i) return m;
    return -1;
}

/* validate_pair + the mini-batch / explicit-list checks (explorer.hpp:82-83, 32-35) */
static int query_schema_ok(const net_t* net, const cl_t* cl, const bp_query* q) {
    if (net->L < 1 || cl->N < 1) return 0;
    for (int64_t j = 0; j < net->L; ++j) {
        int anyf = 0, anyb = 0;
        for (int32_t t = 0; t < net->T; ++t) {
            int64_t f = net->fp[(size_t)t * net->L + j], b = net->bp[(size_t)t * net->L + j];
            if (f < 0 || b < 0) return 0;
            anyf |= f != 0;
            anyb |= b != 0;
        }
        if (!anyf || !anyb) return 0;
        if (net->w[j] < 0 || net->a[j] < 0) return 0;
    }
    for (int64_t k = 0; k < cl->N - 1; ++k)
        if (cl->bw[k] <= 0) return 0;
    for (int64_t i = 0; i < cl->N; ++i) {
        if (cl->cap[i] <= 0) return 0;
        for (int k = 0; k < 4; ++k)
            if (cl->minm[i * 4 + k] < 1) return 0;
        int32_t t = cl->type[i];
        if (t < 0 || t >= net->T) return 0;
        for (int64_t j = 0; j < net->L; ++j)
            if (net->fp[(size_t)t * net->L + j] == 0 || net->bp[(size_t)t * net->L + j] == 0) return 0;
    }
    if (q->mini_batch < 1) return 0;
    if (q->n_m > 0 && q->m_list)
        for (int i = 0; i < q->n_m; ++i)
            if (q->m_list[i] < 1 || q->mini_batch % q->m_list[i] != 0) return 0;
    return 1;
}

typedef struct {
    int idx;
    rat makespan, peak, maxbw;
    int64_t M;
    int kind;
} ranked_t;

static int ranked_less(const ranked_t* a, const ranked_t* b) {   /* explorer.hpp:142-152 */
    if (!req(a->makespan, b->makespan)) return rlt(a->makespan, b->makespan);
    if (!req(a->peak, b->peak)) return rlt(a->peak, b->peak);
    if (!req(a->maxbw, b->maxbw)) return rlt(a->maxbw, b->maxbw);
    if (a->M != b->M) return a->M < b->M;
    return a->kind < b->kind;
}

static int status_of(int code) {
    switch (code) {
        case E_OVERFLOW: return BP_C_ERR_OVERFLOW;
        case E_DOMAIN: return BP_C_ERR_DOMAIN;
        case E_INVALID_PLAN: return BP_C_ERR_INVALID_PLAN;
        case E_INF_COARSEN: return BP_C_REJ_COARSEN;
        case E_INF_FINETUNE: return BP_C_REJ_FINETUNE;
        case E_INF_NOCONV: return BP_C_REJ_FINETUNE_NOCONV;
        case E_SHAPE: return BP_C_REJ_SHAPE;
        case E_UB: return BP_C_REF_UB;
        default: return BP_C_ERR_DOMAIN;
    }
}

/* One candidate: explorer.hpp:104-131. */
static void eval_candidate(const net_t* net, const cl_t* cl, int kind, int64_t M, int64_t micro,
                           bp_candidate* c, bp_stage* st) {
    exc_t e;
    memset(&e, 0, sizeof(e));
    exc_t* saved = X;
    X = &e;
    int code = setjmp(e.jb);
    if (code) {
        c->status = status_of(code);
        c->detail = e.detail;
        c->detail2 = e.detail2;
        if (code == E_INVALID_PLAN) c->aux = BR(e.aux);
        afree_all(&e);
        X = saved;
        return;
    }
    plan_t p = balance_partition(net, cl, kind, M, micro);
    est_t es = estimate(kind, &p, net, cl, M, micro);
    if (!memory_feasible(&es, p.N)) {
        c->status = BP_C_REJ_MEM_POST;
        afree_all(&e);
        X = saved;
        return;
    }
    rat mk = simulate(kind, &p, net, cl, M, micro);
    rat peak = R(0), maxbw = R(0);
    for (int64_t i = 0; i < p.N; ++i) {
        rat mem = radd(es.features[i], es.weights[i]);
        if (rgt(mem, peak)) peak = mem;
    }
    for (int64_t k = 0; k < p.N - 1; ++k)
        if (rgt(es.bw[k], maxbw)) maxbw = es.bw[k];
    c->status = BP_C_OK;
    c->makespan = BR(mk);
    c->est_minibatch = BR(es.minibatch);
    c->bubble = BR(es.bubble);
    c->peak_memory = BR(peak);
    c->max_bw_demand = BR(maxbw);
    c->heuristic = es.heuristic;
    c->plan_fractional = 0;
    for (int64_t i = 0; i < p.N; ++i) {
        if (!req(p.lead[i], R(1)) || !req(p.trail[i], R(1))) c->plan_fractional = 1;
        if (!st) continue;
        st[i].lo = p.lo[i];
        st[i].hi = p.hi[i];
        st[i].lead = BR(p.lead[i]);
        st[i].trail = BR(p.trail[i]);
        st[i].features = BR(es.features[i]);
        st[i].weights = BR(es.weights[i]);
        st[i].bw_demand = i + 1 < p.N ? BR(es.bw[i]) : (bp_rat){0, 1};
    }
    afree_all(&e);
    X = saved;
}

static int is_escaping(int st) {
    return st == BP_C_ERR_OVERFLOW || st == BP_C_ERR_INVALID_PLAN || st == BP_C_ERR_DOMAIN ||
           st == BP_C_REF_UB;
}

static int q_status_of(int cst) {
    switch (cst) {
        case BP_C_ERR_OVERFLOW: return BP_Q_OVERFLOW;
        case BP_C_ERR_INVALID_PLAN: return BP_Q_INVALID_PLAN;
        case BP_C_ERR_DOMAIN: return BP_Q_DOMAIN;
        default: return BP_Q_REF_UB;
    }
}

static void explore_one(const bp_network* nets, const bp_cluster* cls, const bp_query* q,
                        bp_query_result* r, bp_candidate* cand, bp_stage* stages) {
    memset(r, 0, sizeof(*r));
    r->best = -1;
    r->first_error = -1;
    const bp_network* bn = &nets[q->network];
    const bp_cluster* bc = &cls[q->cluster];
    net_t net = {bn->n_layers, bn->n_types, bn->fp_us, bn->bp_us, bn->weight_bytes, bn->out_act_bytes};
    cl_t cl = {q->n_stages > 0 ? q->n_stages : bc->n_accels, bc->exec_mode, bc->type_id,
               bc->mem_capacity, bc->min_micro, bc->link_bw};
    if (!query_schema_ok(&net, &cl, q)) { r->status = BP_Q_SCHEMA; return; }
    int kinds[2];
    int nk = kinds_of(cl.mode, kinds);
    int64_t nb = n_base(q);
    r->n_candidates = (int32_t)(nk * nb);
    bp_candidate local;
    ranked_t* rk = (ranked_t*)calloc((size_t)(nk * nb + 1), sizeof(ranked_t));
    int nr = 0;
    for (int ki = 0; ki < nk; ++ki) {
        int64_t min_micro = 1;                               /* candidate_Ms 42-47 */
        for (int64_t i = 0; i < cl.N; ++i)
            if (cl.minm[i * 4 + kinds[ki]] > min_micro) min_micro = cl.minm[i * 4 + kinds[ki]];
        for (int64_t mi = 0; mi < nb; ++mi) {
            int64_t idx = ki * nb + mi;
            bp_candidate* c = cand ? &cand[q->cand_offset + idx] : &local;
            memset(c, 0, sizeof(*c));
            c->kind = kinds[ki];
            c->M = base_at(q, mi);
            c->micro = q->mini_batch / c->M;
            c->rank = -1;
            c->n_stages = (int32_t)cl.N;
            if (!(q->mini_batch / c->M >= min_micro)) { c->status = BP_C_REJ_MIN_MICRO; continue; }
            eval_candidate(&net, &cl, c->kind, c->M, c->micro, c,
                           stages ? stages + q->stage_offset + idx * cl.N : NULL);
            if (is_escaping(c->status) && r->first_error < 0) {
                r->first_error = (int32_t)idx;
                r->status = q_status_of(c->status);
            }
            if (c->status == BP_C_OK) {
                ranked_t* t = &rk[nr++];
                t->idx = (int)idx;
                t->makespan = RB(c->makespan);
                t->peak = RB(c->peak_memory);
                t->maxbw = RB(c->max_bw_demand);
                t->M = c->M;
                t->kind = c->kind;
            }
        }
    }
    if (r->first_error >= 0) { free(rk); return; }
    if (nr == 0) { r->status = BP_Q_NO_FEASIBLE; free(rk); return; }
    for (int i = 1; i < nr; ++i) {                  /* stable insertion sort */
        ranked_t v = rk[i];
        int k = i - 1;
        while (k >= 0 && ranked_less(&v, &rk[k])) { rk[k + 1] = rk[k]; --k; }
        rk[k + 1] = v;
    }
    r->status = BP_Q_OK;
    r->n_ranked = nr;
    r->best = rk[0].idx;
    if (cand)
        for (int i = 0; i < nr; ++i) cand[q->cand_offset + rk[i].idx].rank = i;
    r->best_kind = rk[0].kind;
    r->best_M = rk[0].M;
    r->best_micro = q->mini_batch / rk[0].M;
    r->best_makespan = BR(rk[0].makespan);
    r->best_peak_memory = BR(rk[0].peak);
    r->best_max_bw = BR(rk[0].maxbw);
    free(rk);
}

/* ---------------------------------------------------------------- exports */
int bpo_abi_version(void) { return BP_ABI_VERSION; }

int bpo_explore_batch(const bp_network* nets, int n_nets, const bp_cluster* cls, int n_cls,
                      const bp_query* q, int nq, bp_query_result* res, bp_candidate* cand,
                      bp_stage* stages) {
    if (!nets || !cls || !q || !res || n_nets < 1 || n_cls < 1) return BP_BAD_INPUT;
    for (int i = 0; i < nq; ++i) {
        if (q[i].network < 0 || q[i].network >= n_nets || q[i].cluster < 0 || q[i].cluster >= n_cls)
            return BP_BAD_INPUT;
        explore_one(nets, cls, &q[i], &res[i], cand, stages);
    }
    return BP_OK;
}

int bpo_partition(const bp_network* bn, const bp_cluster* bc, int n_stages, int64_t a_th,
                  int use_coarse, int64_t* lo, int64_t* hi, int64_t* t_opt) {
    exc_t e;
    memset(&e, 0, sizeof(e));
    exc_t* saved = X;
    X = &e;
    int code = setjmp(e.jb);
    if (code) {
        afree_all(&e);
        X = saved;
        return code == E_SHAPE ? BP_C_REJ_SHAPE : status_of(code);
    }
    net_t net = {bn->n_layers, bn->n_types, bn->fp_us, bn->bp_us, bn->weight_bytes, bn->out_act_bytes};
    cl_t cl = {n_stages > 0 ? n_stages : bc->n_accels, bc->exec_mode, bc->type_id, bc->mem_capacity,
               bc->min_micro, bc->link_bw};
    plan_t p = use_coarse ? coarse_partition(&net, &cl, a_th, t_opt) : inter_layer_partition(&net, &cl, t_opt);
    for (int64_t n = 0; n < p.N; ++n) { lo[n] = p.lo[n]; hi[n] = p.hi[n]; }
    afree_all(&e);
    X = saved;
    return BP_C_OK;
}

int bpo_simulate_chain(int kind, int n, const bp_rat* F, const bp_rat* B, const int64_t* SR,
                       const int64_t* a, const bp_rat* w, int64_t M, bp_rat* makespan) {
    exc_t e;
    memset(&e, 0, sizeof(e));
    exc_t* saved = X;
    X = &e;
    int code = setjmp(e.jb);
    if (code) {
        afree_all(&e);
        X = saved;
        return status_of(code);
    }
    rat* f = (rat*)amalloc(sizeof(rat) * (size_t)n);
    rat* b = (rat*)amalloc(sizeof(rat) * (size_t)n);
    rat* ww = (rat*)amalloc(sizeof(rat) * (size_t)n);
    for (int i = 0; i < n; ++i) { f[i] = RB(F[i]); b[i] = RB(B[i]); ww[i] = RB(w[i]); }
    *makespan = BR(simulate_chain(kind, n, f, b, SR, a, ww, M));
    afree_all(&e);
    X = saved;
    return BP_C_OK;
}

static int closed_form(int which, int kind, int64_t M, int64_t N, bp_rat F, bp_rat B, bp_rat SR,
                       bp_rat* out) {
    exc_t e;
    memset(&e, 0, sizeof(e));
    exc_t* saved = X;
    X = &e;
    int code = setjmp(e.jb);
    if (code) {
        afree_all(&e);
        X = saved;
        return status_of(code);
    }
    rat r = which ? bubble_fraction(kind, M, N, RB(F), RB(B), RB(SR))
                  : minibatch_time(kind, M, N, RB(F), RB(B), RB(SR));
    *out = BR(r);
    afree_all(&e);
    X = saved;
    return BP_C_OK;
}

int bpo_minibatch_time(int kind, int64_t M, int64_t N, bp_rat F, bp_rat B, bp_rat SR, bp_rat* out) {
    return closed_form(0, kind, M, N, F, B, SR, out);
}
int bpo_bubble_fraction(int kind, int64_t M, int64_t N, bp_rat F, bp_rat B, bp_rat SR, bp_rat* out) {
    return closed_form(1, kind, M, N, F, B, SR, out);
}
