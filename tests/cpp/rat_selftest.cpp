// rat_selftest.cpp -- host build of csrc/rat.cuh (the same code the kernels
// run): every fast path of rat_addsub / umod_u64_u32 / inv32_odd against a
// plain __int128 restatement of rational.hpp's from128 (reduce by gcd, throw
// when the reduced value leaves int64).  Prints "ok <n>" or the first failure.
#include <cstdio>
#include <cstdlib>

#include "../../paper_2012_12544_b200/csrc/rat.cuh"

using namespace bpk;

namespace {

struct Ref {
    bool ovf;
    int64_t n, d;
};

unsigned __int128 ugcd(unsigned __int128 a, unsigned __int128 b) {
    while (b) {
        unsigned __int128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

Ref ref_from128(__int128 n, __int128 d) {   // rational.hpp:83-95
    if (d < 0) { n = -n; d = -d; }
    unsigned __int128 g = ugcd(n < 0 ? (unsigned __int128)(-n) : (unsigned __int128)n, (unsigned __int128)d);
    if (g > 1) { n /= (__int128)g; d /= (__int128)g; }
    if (n > (__int128)INT64_MAX || n < (__int128)INT64_MIN || d > (__int128)INT64_MAX) return {true, 0, 1};
    return {false, (int64_t)n, (int64_t)d};
}

uint64_t st = 0x2012125440ull;
uint64_t rnd() {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return st;
}

int64_t pick_den() {
    switch (rnd() % 6) {
        case 0: return 1 + (int64_t)(rnd() % 1024);
        case 1: return 1 + (int64_t)(rnd() % ((uint64_t)1 << 32));
        case 2: return (int64_t)(1024 * (1 + rnd() % 4096));
        case 3: return (int64_t)((1 + rnd() % 65536) * (1 + rnd() % 65536));
        case 4: return 1 + (int64_t)(rnd() >> 2);
        default: return (int64_t)(((uint64_t)1 << 32) - 1 - rnd() % 3);
    }
}

int64_t pick_num(int64_t d) {
    switch (rnd() % 5) {
        case 0: return (int64_t)(rnd() % 100000);
        case 1: return (int64_t)(rnd() >> 1) * ((rnd() & 1) ? 1 : -1);
        case 2: return (int64_t)(rnd() % ((uint64_t)1 << 40)) * ((rnd() & 1) ? 1 : -1);
        case 3: return d * (int64_t)(rnd() % 1000) + (int64_t)(rnd() % (uint64_t)d);
        default: return (rnd() & 1) ? INT64_MAX - (int64_t)(rnd() % 4) : INT64_MIN + (int64_t)(rnd() % 4);
    }
}

Rat reduced(int64_t n, int64_t d) {
    Err e{ERR_NONE};
    return rat_nd(n, d, e);
}

}  // namespace

int main(int argc, char** argv) {
    const long iters = argc > 1 ? atol(argv[1]) : 2000000;
    for (long it = 0; it < iters; ++it) {
        // umod_u64_u32
        {
            uint64_t x = rnd() >> (rnd() % 40);
            uint32_t m = (uint32_t)(rnd() >> (32 + rnd() % 32));
            if (m == 0) m = 1;
            if (umod_u64_u32(x, m) != x % m) {
                printf("umod fail x=%llu m=%u\n", (unsigned long long)x, m);
                return 1;
            }
            const uint64_t gu = rnd() >> (rnd() % 64), gv = rnd() >> (rnd() % 64);
            if (gcd_u64(gu, gv) != (uint64_t)ugcd(gu, gv)) {
                printf("gcd fail %llu %llu\n", (unsigned long long)gu, (unsigned long long)gv);
                return 1;
            }
            uint32_t o = (uint32_t)rnd() | 1u;
            if (o * inv32_odd(o) != 1u || (uint64_t)o * inv64_lift(o, inv32_odd(o)) != 1ull) {
                printf("inverse fail %u\n", o);
                return 1;
            }
        }
        int64_t ad = pick_den(), bd = pick_den();
        Rat a = reduced(pick_num(ad), ad), b = reduced(pick_num(bd), bd);
        for (int s = -1; s <= 1; s += 2) {
            Err e{ERR_NONE};
            Rat r = rat_addsub(a, b, s, e);
            __int128 bn = s > 0 ? (__int128)b.n : -(__int128)b.n;
            Ref w = ref_from128((__int128)a.n * b.d + bn * a.d, (__int128)a.d * b.d);
            if (w.ovf != e.bad() || (!w.ovf && (w.n != r.n || w.d != r.d))) {
                printf("addsub fail s=%d a=%lld/%lld b=%lld/%lld got %s %lld/%lld want %s %lld/%lld\n", s,
                       (long long)a.n, (long long)a.d, (long long)b.n, (long long)b.d, e.bad() ? "ovf" : "ok",
                       (long long)r.n, (long long)r.d, w.ovf ? "ovf" : "ok", (long long)w.n, (long long)w.d);
                return 1;
            }
        }
    }
    printf("ok %ld\n", iters);
    return 0;
}
