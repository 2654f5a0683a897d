// rat.cuh -- exact rationals on the device with bapipe::Rat semantics.
//
// bapipe::Rat (rational.hpp:14-110) stores a reduced int64 num/den (den > 0);
// every + - * / computes the exact 128-bit result, reduces it by the gcd, and
// throws std::overflow_error when the REDUCED value does not fit int64
// (from128, lines 83-95).  Only values matter for results, and the overflow
// predicate depends only on the reduced value, so any exact algorithm that
// produces the same reduced value reproduces the reference bit for bit.  We
// use the classic gcd-splitting forms (Knuth 4.5.1) so the common cases need
// one 64-bit binary gcd and no 128-bit division.
//
// Errors do not throw: the first error is latched into an Err word and the
// caller stops at its next check (exception emulation, first-error-wins).
#pragma once
#include <math.h>
#include <stdint.h>

// The emulation code is __host__ __device__ so tests/emu can run it on the
// CPU against the oracle; the product runs it only inside the kernels.
#ifdef __CUDACC__
#define BPK_HD __host__ __device__ __forceinline__
#define BPK_HDNI static __host__ __device__ __noinline__
#else
#define BPK_HD inline
#define BPK_HDNI static inline
#endif

// find-first-set (1-based, 0 for 0) on both sides
#ifdef __CUDACC__
__host__ __device__ __forceinline__ int bpk_ffs64(long long x) {
#ifdef __CUDA_ARCH__
    return __ffsll(x);
#else
    return __builtin_ffsll(x);
#endif
}
#else
inline int bpk_ffs64(long long x) { return __builtin_ffsll(x); }
#endif

namespace bpk {

// host-only operation counters for the test emulator (tests/emu, BPK_OPSTATS)
#if defined(BPK_OPSTATS) && !defined(__CUDA_ARCH__)
extern unsigned long long bpk_opstats[32];
#define BPK_COUNT(i) (++bpk_opstats[i])
#else
#define BPK_COUNT(i) ((void)0)
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;

// Candidate-level error codes (map 1:1 onto BP_C_* in bapipe_b200.h).
enum : uint32_t {
    ERR_NONE = 0,
    ERR_OVERFLOW = 7,      // BP_C_ERR_OVERFLOW
    ERR_INVALID_PLAN = 8,  // BP_C_ERR_INVALID_PLAN
    ERR_DOMAIN = 9,        // BP_C_ERR_DOMAIN
    ERR_UB = 10            // BP_C_REF_UB
};

struct Err {
    uint32_t code;
    BPK_HD void set(uint32_t c) {
        if (code == ERR_NONE) code = c;
    }
    BPK_HD bool bad() const { return code != ERR_NONE; }
};

struct Rat {
    int64_t n, d;
};

BPK_HD Rat R(int64_t v) { return Rat{v, 1}; }

// Out-of-line Rat operations return their error by value: an Err passed by
// reference to a non-inlined function has to live in local memory, and every
// error test in the caller's loops then became a local-memory load.  NAME_body
// is the operation, inlined into the out-of-line NAME_v (where its Err is a
// register); NAME is the inline wrapper applying the first-error-wins latch.
struct RatE {
    Rat r;
    uint32_t err;
};

// ---- integer helpers ----------------------------------------------------
// GPUs have no native 64-bit divide; the helpers below keep the common cases
// (operands below 2^32, exact quotients) off the generic software routines.
// 32-bit find-first-set on the device (BREV + FLO): the 64-bit __ffsll it
// replaces was ~15% of the exact simulators' instructions through gcd_u32
BPK_HD int ctz32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __ffs((int)x) - 1;
#else
    return __builtin_ffs((int)x) - 1;
#endif
}

BPK_HD uint32_t gcd_u32(uint32_t u, uint32_t v) {
    if (u == 0) return v;
    if (v == 0) return u;
    // a power of two on either side (the 1/1024-quantized fractions of
    // refine make these common): the gcd is the lowest set bit of u | v
    const uint32_t o = u | v;
    BPK_COUNT(0);
    if ((u & (u - 1)) == 0 || (v & (v - 1)) == 0) return o & (0u - o);
    BPK_COUNT(1);
    int shift = ctz32(u | v);
    u >>= ctz32(u);
    do {
        BPK_COUNT(2);
        v >>= ctz32(v);
        uint32_t lo = u < v ? u : v, hi = u < v ? v : u;
        u = lo;
        v = hi - lo;
    } while (v != 0);
    return u << shift;
}

BPK_HD uint64_t umod64(uint64_t a, uint64_t b) {
    if (((a | b) >> 32) == 0) return (uint32_t)a % (uint32_t)b;
    return a % b;
}

// x mod m for a 32-bit m without the 64-bit software remainder: a quotient
// estimate from a double reciprocal (off by at most ~2^13), one exact
// correction in double (|r| < 2^53), then integer fix-ups.  The result is
// exact whatever the reciprocal's rounding, so host and device agree.
BPK_HD uint32_t umod_u64_u32(uint64_t x, uint32_t m) {
    if ((m & (m - 1)) == 0) return m == 0 ? 0 : (uint32_t)x & (m - 1);
    if ((x >> 32) == 0) return (uint32_t)x % m;
#ifdef __CUDA_ARCH__
    const double rm = __drcp_rn((double)m);
#else
    const double rm = 1.0 / (double)m;
#endif
    const uint64_t q = (uint64_t)((double)x * rm);
    int64_t r = (int64_t)(x - q * (uint64_t)m);
    r -= (int64_t)((double)r * rm) * (int64_t)m;
    // the double quotient is within one of r / m (|r| < 2^44), so r is now in
    // (-2m, 2m): predicated fix-ups instead of loops
    if (r < 0) r += m;
    if (r < 0) r += m;
    if (r >= (int64_t)m) r -= m;
    return (uint32_t)r;
}

// out of line: inlined at its ~20 call sites it dominated the kernels' code
// size (instruction-cache misses were the top stall in refine and prune)
BPK_HDNI uint64_t gcd_u64_wide(uint64_t u, uint64_t v) {
    if (u == 0) return v;
    if (v == 0) return u;
    const uint64_t o = u | v;
    BPK_COUNT(3);
    if ((u & (u - 1)) == 0 || (v & (v - 1)) == 0) return o & (0ull - o);   // see gcd_u32
    if (u < v) { uint64_t t = u; u = v; v = t; }
    BPK_COUNT(4);
    if ((v >> 32) == 0) {              // one Euclid step brings both below 2^32
        const uint32_t r = umod_u64_u32(u, (uint32_t)v);
        return r == 0 ? v : gcd_u32((uint32_t)v, r);
    }
    BPK_COUNT(5);
    int shift = bpk_ffs64((long long)(u | v)) - 1;
    u >>= (bpk_ffs64((long long)u) - 1);
    do {
        BPK_COUNT(6);
        v >>= (bpk_ffs64((long long)v) - 1);
        uint64_t lo = u < v ? u : v, hi = u < v ? v : u;
        u = lo;
        v = hi - lo;
    } while (v != 0);
    return u << shift;
}

// the common case (both below 2^32) inline, the wide one out of line
BPK_HD uint64_t gcd_u64(uint64_t u, uint64_t v) {
    if (((u | v) >> 32) == 0) return gcd_u32((uint32_t)u, (uint32_t)v);
    return gcd_u64_wide(u, v);
}

// a / g for g dividing a exactly: shift out the twos, multiply by the
// inverse of the odd part modulo 2^64 (Newton: 3 -> 6 -> 12 -> 24 -> 48 -> 96 bits).
BPK_HD uint64_t udiv_exact64(uint64_t a, uint64_t g) {
    if (g == 1) return a;
    if (((a | g) >> 32) == 0) return (uint32_t)a / (uint32_t)g;
    BPK_COUNT(7);
    int tz = bpk_ffs64((long long)g) - 1;
    a >>= tz;
    g >>= tz;
    uint64_t x = (3 * g) ^ 2;
    x *= 2 - g * x;
    x *= 2 - g * x;
    x *= 2 - g * x;
    x *= 2 - g * x;
    return a * x;
}

BPK_HD int64_t sdiv_exact64(int64_t a, uint64_t g) {
    return a < 0 ? -(int64_t)udiv_exact64((uint64_t)0 - (uint64_t)a, g) : (int64_t)udiv_exact64((uint64_t)a, g);
}

BPK_HD int ctz128(u128 x) {
    uint64_t lo = (uint64_t)x;
    if (lo) return bpk_ffs64((long long)lo) - 1;
    return 64 + bpk_ffs64((long long)(uint64_t)(x >> 64)) - 1;
}

BPK_HDNI u128 gcd_u128(u128 u, u128 v) {
    BPK_COUNT(9);
    if (u == 0) return v;
    if (v == 0) return u;
    if ((u >> 64) == 0 && (v >> 64) == 0) return gcd_u64((uint64_t)u, (uint64_t)v);
    int shift = ctz128(u | v);
    u >>= ctz128(u);
    do {
        v >>= ctz128(v);
        if (u > v) { u128 t = u; u = v; v = t; }
        v -= u;
        if ((u >> 64) == 0 && (v >> 64) == 0) {
            u = gcd_u64((uint64_t)u, (uint64_t)v);
            v = 0;
        }
    } while (v != 0);
    return u << shift;
}

BPK_HD u128 uabs128(i128 x) { return x < 0 ? (u128)(-x) : (u128)x; }

// from128 (rational.hpp:83-95): reduce an exact 128-bit fraction, check fit.
BPK_HD Rat from128_body(i128 n, i128 d, Err& e) {
    if (d == 0) { e.set(ERR_DOMAIN); return Rat{0, 1}; }
    if (d < 0) { n = -n; d = -d; }
    u128 g = gcd_u128(uabs128(n), (u128)d);
    if (g > 1) { n /= (i128)g; d /= (i128)g; }
    if (n > (i128)INT64_MAX || n < (i128)INT64_MIN || d > (i128)INT64_MAX) {
        e.set(ERR_OVERFLOW);
        return Rat{0, 1};
    }
    return Rat{(int64_t)n, (int64_t)d};
}

BPK_HDNI RatE from128_v(i128 n, i128 d) {
    Err e{ERR_NONE};
    const Rat r = from128_body(n, d, e);
    return RatE{r, e.code};
}
BPK_HD Rat from128(i128 n, i128 d, Err& e) {
    const RatE x = from128_v(n, d);
    if (x.err) e.set(x.err);
    return x.r;
}

// A 128-bit value already known to be reduced: only the range check.
BPK_HD Rat fit128(i128 n, i128 d, Err& e) {
    if (n > (i128)INT64_MAX || n < (i128)INT64_MIN || d > (i128)INT64_MAX) {
        e.set(ERR_OVERFLOW);
        return Rat{0, 1};
    }
    return Rat{(int64_t)n, (int64_t)d};
}

BPK_HD uint64_t uabs64(int64_t x) {
    return x < 0 ? (uint64_t)0 - (uint64_t)x : (uint64_t)x;
}

// Rat(n, d) constructor -> normalize() (rational.hpp:18, 100-106).
BPK_HD Rat rat_nd_body(int64_t n, int64_t d, Err& e) {
    if (d == 0) { e.set(ERR_DOMAIN); return Rat{0, 1}; }
    if (d < 0) { n = -n; d = -d; }
    uint64_t g = gcd_u64(uabs64(n), (uint64_t)d);
    if (g > 1) { n = sdiv_exact64(n, g); d = (int64_t)udiv_exact64((uint64_t)d, g); }
    return Rat{n, d};
}

BPK_HDNI RatE rat_nd_v(int64_t n, int64_t d) {
    Err e{ERR_NONE};
    const Rat r = rat_nd_body(n, d, e);
    return RatE{r, e.code};
}
BPK_HD Rat rat_nd(int64_t n, int64_t d, Err& e) {
    const RatE x = rat_nd_v(n, d);
    if (x.err) e.set(x.err);
    return x.r;
}

BPK_HD bool fits64(i128 x) { return x <= (i128)INT64_MAX && x >= (i128)INT64_MIN; }

// Inverse of an odd m modulo 2^32 (Newton: 5 -> 10 -> 20 -> 40 correct bits)
// and its lift to 2^64 (one more step).
BPK_HD uint32_t inv32_odd(uint32_t m) {
    uint32_t x = (3 * m) ^ 2;
    x *= 2 - m * x;
    x *= 2 - m * x;
    x *= 2 - m * x;
    return x;
}
BPK_HD uint64_t inv64_lift(uint32_t m, uint32_t x32) {
    uint64_t x = x32;
    return x * (2 - (uint64_t)m * x);
}


// a + s*b with s = +1 / -1 (operator+ / operator-), Knuth 4.5.1: with
// g = gcd(a.d, b.d), t = a.n*(b.d/g) + b.n*(a.d/g) and g2 = gcd(t, g) the
// reduced result is (t/g2) / ((a.d/g)*(b.d/g2)).
// Out of line on purpose: inlining every Rat operation into the refine and
// simulator loops produced ~1 MB of SASS and the kernels stalled on
// instruction fetch (ncu: "no_instruction" 17.5 cycles per issue).

BPK_HD Rat rat_addsub_general(Rat a, Rat b, int s, Err& e);

BPK_HD Rat rat_addsub_body(Rat a, Rat b, int s, Err& e) {
    BPK_COUNT(11);
    i128 bn = s > 0 ? (i128)b.n : -(i128)b.n;
    if (a.d == 1 && b.d == 1) return fit128((i128)a.n + bn, 1, e);
    if (a.d == 1) return fit128((i128)a.n * b.d + bn, b.d, e);        // gcd(num, b.d) = 1
    if (b.d == 1) return fit128((i128)bn * a.d + a.n, a.d, e);
    if (((uint64_t)(a.d | b.d) >> 32) == 0 && b.n != INT64_MIN) {
        // Hot path (the simulator's and refine's common case): 32-bit
        // denominators and a 64-bit t.  Exact quotients come from inverses
        // mod 2^32 / 2^64 and t mod g from umod_u64_u32, so no 64-bit
        // software division runs.
        const uint32_t da = (uint32_t)a.d, db = (uint32_t)b.d;
        const int64_t bs = s > 0 ? b.n : -b.n;
        const uint32_t g = gcd_u32(da, db);
        if (g == 1) return fit128((i128)a.n * db + (i128)bs * da, (i128)((uint64_t)da * db), e);
        const int tz = ctz32(g);
        const uint32_t ig = inv32_odd(g >> tz);
        const uint32_t ad = (da >> tz) * ig, bd = (db >> tz) * ig;   // da / g, db / g
        const i128 t = (i128)a.n * bd + (i128)bs * ad;
        if (t == 0) return Rat{0, 1};
        if (fits64(t)) {
            const int64_t tt = (int64_t)t;
            const uint64_t ut = uabs64(tt);
            const uint32_t tm = umod_u64_u32(ut, g);
            const uint32_t g2 = tm == 0 ? g : gcd_u32(tm, g);
            const int tz2 = ctz32(g2);
            const uint32_t i2 = inv32_odd(g2 >> tz2);
            const uint64_t q = (ut >> tz2) * inv64_lift(g2 >> tz2, i2);      // |t| / g2
            const uint64_t den = (uint64_t)ad * (uint32_t)((db >> tz2) * i2);  // (da/g) * (db/g2)
            if (q > (tt < 0 ? (uint64_t)1 << 63 : (uint64_t)INT64_MAX) || den > (uint64_t)INT64_MAX) {
                e.set(ERR_OVERFLOW);
                return Rat{0, 1};
            }
            return Rat{tt < 0 ? (int64_t)((uint64_t)0 - q) : (int64_t)q, (int64_t)den};
        }
    }
    return rat_addsub_general(a, b, s, e);
}

// 64-bit denominators or a 128-bit t: kept out of the hot function so the
// kernels' instruction stream stays small.
BPK_HD Rat rat_addsub_general_body(Rat a, Rat b, int s, Err& e) {
    BPK_COUNT(8);
    i128 bn = s > 0 ? (i128)b.n : -(i128)b.n;
    uint64_t g = gcd_u64((uint64_t)a.d, (uint64_t)b.d);
    if (g == 1) return fit128((i128)a.n * b.d + bn * a.d, (i128)a.d * b.d, e);
    int64_t ad = (int64_t)udiv_exact64((uint64_t)a.d, g), bd = (int64_t)udiv_exact64((uint64_t)b.d, g);
    i128 t = (i128)a.n * bd + bn * ad;
    if (t == 0) return Rat{0, 1};
    const bool small = fits64(t);
    uint64_t tm = small ? umod64(uabs64((int64_t)t), g) : (uint64_t)(uabs128(t) % (u128)g);
    uint64_t g2 = tm == 0 ? g : gcd_u64(tm, g);
    i128 num = small ? (i128)sdiv_exact64((int64_t)t, g2) : t / (i128)g2;
    i128 den = (i128)ad * (i128)udiv_exact64((uint64_t)b.d, g2);
    return fit128(num, den, e);
}

BPK_HDNI RatE rat_addsub_general_v(Rat a, Rat b, int s) {
    Err e{ERR_NONE};
    const Rat r = rat_addsub_general_body(a, b, s, e);
    return RatE{r, e.code};
}
BPK_HD Rat rat_addsub_general(Rat a, Rat b, int s, Err& e) {
    const RatE x = rat_addsub_general_v(a, b, s);
    if (x.err) e.set(x.err);
    return x.r;
}

BPK_HDNI RatE rat_addsub_v(Rat a, Rat b, int s) {
    Err e{ERR_NONE};
    const Rat r = rat_addsub_body(a, b, s, e);
    return RatE{r, e.code};
}
BPK_HD Rat rat_addsub(Rat a, Rat b, int s, Err& e) {
    const RatE x = rat_addsub_v(a, b, s);
    if (x.err) e.set(x.err);
    return x.r;
}

BPK_HD Rat rat_add(Rat a, Rat b, Err& e) {
    if (a.d == 1 && b.d == 1) return fit128((i128)a.n + b.n, 1, e);
    return rat_addsub(a, b, +1, e);
}
BPK_HD Rat rat_sub(Rat a, Rat b, Err& e) {
    if (a.d == 1 && b.d == 1) return fit128((i128)a.n - b.n, 1, e);
    return rat_addsub(a, b, -1, e);
}

// operator* (rational.hpp:33-35).
BPK_HD Rat rat_mul_nl_body(Rat a, Rat b, Err& e) {
    BPK_COUNT(10);
    if (a.n == 0 || b.n == 0) return Rat{0, 1};
    if (a.d == 1 && b.d == 1) return fit128((i128)a.n * b.n, 1, e);
    uint64_t g1 = (b.d == 1) ? 1 : gcd_u64(uabs64(a.n), (uint64_t)b.d);
    uint64_t g2 = (a.d == 1) ? 1 : gcd_u64(uabs64(b.n), (uint64_t)a.d);
    int64_t an = sdiv_exact64(a.n, g1);
    int64_t bd = (int64_t)udiv_exact64((uint64_t)b.d, g1);
    int64_t bn = sdiv_exact64(b.n, g2);
    int64_t ad = (int64_t)udiv_exact64((uint64_t)a.d, g2);
    return fit128((i128)an * bn, (i128)ad * bd, e);
}

BPK_HDNI RatE rat_mul_nl_v(Rat a, Rat b) {
    Err e{ERR_NONE};
    const Rat r = rat_mul_nl_body(a, b, e);
    return RatE{r, e.code};
}
BPK_HD Rat rat_mul_nl(Rat a, Rat b, Err& e) {
    const RatE x = rat_mul_nl_v(a, b);
    if (x.err) e.set(x.err);
    return x.r;
}

// operator/ (rational.hpp:36-39): b == 0 -> domain_error.
BPK_HD Rat rat_mul(Rat a, Rat b, Err& e) {
    if (a.d == 1 && b.d == 1) return fit128((i128)a.n * b.n, 1, e);
    return rat_mul_nl(a, b, e);
}

BPK_HD Rat rat_div_body(Rat a, Rat b, Err& e) {
    if (b.n == 0) { e.set(ERR_DOMAIN); return Rat{0, 1}; }
    // a / b = a * (b.d / b.n); keep the sign on the numerator.
    if (b.n == INT64_MIN) return from128((i128)a.n * b.d, (i128)a.d * b.n, e);
    Rat inv = b.n < 0 ? Rat{-b.d, -b.n} : Rat{b.d, b.n};
    return rat_mul(a, inv, e);
}

BPK_HDNI RatE rat_div_v(Rat a, Rat b) {
    Err e{ERR_NONE};
    const Rat r = rat_div_body(a, b, e);
    return RatE{r, e.code};
}
BPK_HD Rat rat_div(Rat a, Rat b, Err& e) {
    const RatE x = rat_div_v(a, b);
    if (x.err) e.set(x.err);
    return x.r;
}

// Comparisons cross-multiply in 128 bits and never throw (lines 47-56).
BPK_HD bool rat_eq(Rat a, Rat b) { return a.n == b.n && a.d == b.d; }
BPK_HD bool rat_lt(Rat a, Rat b) {
    if (a.d == b.d) return a.n < b.n;
    // the cross products in double decide unless they are within a few ulps
    // of each other (each carries a relative error below 2^-51); otherwise
    // the exact 128-bit products do
    const double x = (double)a.n * (double)b.d, y = (double)b.n * (double)a.d;
    const double m = 0x1p-48 * fmax(fabs(x), fabs(y));
    if (x < y - m) return true;
    if (x > y + m) return false;
    return (i128)a.n * b.d < (i128)b.n * a.d;
}
BPK_HD bool rat_gt(Rat a, Rat b) { return rat_lt(b, a); }
BPK_HD bool rat_le(Rat a, Rat b) { return !rat_lt(b, a); }
BPK_HD bool rat_ge(Rat a, Rat b) { return !rat_lt(a, b); }
BPK_HD Rat rat_max(Rat a, Rat b) { return rat_lt(a, b) ? b : a; }   // std::max
BPK_HD Rat rat_min(Rat a, Rat b) { return rat_lt(b, a) ? b : a; }   // std::min

BPK_HD int64_t rat_floor(Rat a) {   // 59-63
    int64_t q = a.n / a.d;
    if (a.n % a.d != 0 && a.n < 0) --q;
    return q;
}
BPK_HD int64_t rat_ceil(Rat a) {    // 64-68
    int64_t q = a.n / a.d;
    if (a.n % a.d != 0 && a.n > 0) ++q;
    return q;
}

BPK_HD int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace bpk
