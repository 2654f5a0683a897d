// tests/cpp/rat_latency_bench.cu -- TOOL (not collected by pytest): latency in
// cycles of the slim refine walk's arithmetic primitives (csrc/refine_fast.cuh)
// on one GPU thread, each as a dependent chain (the walk is one thread's
// serial chain, so latency, not throughput, is what a step costs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tests/cpp/rat_latency_bench.cu -o /tmp/rlb && /tmp/rlb
#include <cstdio>

#include "../../paper_2012_12544_b200/csrc/refine_fast.cuh"

using namespace bpk;

constexpr int ITERS = 2000;

__global__ void kbench(long long* out, int64_t seed) {
    if (threadIdx.x) return;
    long long c0, c1;
    int k = 0;
    // 0: rf_add_small, power-of-two b
    {
        Rat a{(seed % 1000) + 12345, 3 * 512}, b{(seed & 7) + 1, 1024};
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { a = rf_add_small(a, b, (i & 1) ? 1 : -1); a.d &= 0x7fffffff; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += a.n;
    }
    // 1: rf_mul_int
    {
        Rat x{(seed & 1023) | 1, 1024};
        int64_t c = 177 + (seed & 3);
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { Rat y = rf_mul_int(x, c); c = (y.n & 0x3ff) + 100; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += c;
    }
    // 2: stage_time_safe
    {
        Rat t{(seed & 0xfffff) * 512 + 1, 512}, l{3, 1024}, r{5, 1024};
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { bool s = stage_time_safe(t, l, r); t.n += s ? 1 : 2; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += t.n;
    }
    // 3: gcd_u32 on power-of-two denominators
    {
        uint32_t a = 512 << (seed & 1), b = 1024;
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { uint32_t g = gcd_u32(a, b); a = (g << 1) | (a & 0x400); b = 1024 + (g & 1); b &= ~1u; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += a;
    }
    // 4: gcd_u32 on 2^9 * small odd
    {
        uint32_t a = 512 * 139, b = 512 * 21 + (uint32_t)(seed & 0);
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { uint32_t g = gcd_u32(a, b); a = 512 * 139 + (g & 0x10000); }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += a;
    }
    // 5: gcd_mod, odd m ~ 2^8 (64-bit a)
    {
        uint64_t a = 123456789012ull + seed;
        uint32_t m = 255;
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { uint32_t g = gcd_mod(a, m); a += g; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += (long long)a;
    }
    // 6: rf_div32 non-power-of-two (out-of-line divide)
    {
        uint32_t a = 3 * 7 * 11 * 13 * 1000, g = 21 + (uint32_t)(seed & 0);
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { uint32_t q = rf_div32(a, g); a = q * 21 + (a & 0); }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += a;
    }
    // 7: rf_lt (128-bit cross products)
    {
        Rat a{(int64_t)(seed | 1) << 30, 3 * 1024}, b{77777777, 1 << 20};
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { bool lt = rf_lt(a, b); a.n += lt ? 1 : 3; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += a.n;
    }
    // 8: umod_u64_u32 (64-bit a, odd m)
    {
        uint64_t a = 987654321098ull + seed;
        uint32_t m = 1234567;
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { uint32_t r = umod_u64_u32(a, m); a += r | 1; }
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += (long long)a;
    }
    // 9: 64-bit multiply chain
    {
        uint64_t a = 3 + seed;
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) a = a * 0x9e3779b97f4a7c15ull + 1;
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += (long long)a;
    }
    // 11: ctz via __ffs (BREV + FLO)
    {
        uint32_t a = 0x1000u | (uint32_t)(seed & 0);
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { int z = __ffs(a) - 1; a = (1u << ((z + 1) & 15)) | 0x10000u; }
        c1 = clock64();
        out[11] = (c1 - c0) / ITERS;
        out[16] += a;
    }
    // 12: ctz via __popc((x & -x) - 1)
    {
        uint32_t a = 0x1000u | (uint32_t)(seed & 0);
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { int z = __popc((a & (0u - a)) - 1); a = (1u << ((z + 1) & 15)) | 0x10000u; }
        c1 = clock64();
        out[12] = (c1 - c0) / ITERS;
        out[16] += a;
    }
    // 13: baseline of 11/12 (the same chain with a constant shift)
    {
        uint32_t a = 0x1000u | (uint32_t)(seed & 0);
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { int z = (int)(a & 7); a = (1u << ((z + 1) & 15)) | 0x10000u; }
        c1 = clock64();
        out[13] = (c1 - c0) / ITERS;
        out[16] += a;
    }
    // 14: float estimate of a small quotient (I2F.S64, MUFU.RCP, F2I.S64)
    {
        int64_t num = ((int64_t)1 << 50) + seed, den = ((int64_t)1 << 42) + 12345;
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) { int64_t k = (int64_t)((float)num * __frcp_rn((float)den)); num += k & 1; }
        c1 = clock64();
        out[14] = (c1 - c0) / ITERS;
        out[16] += num;
    }
    // 10: 32-bit add chain (loop overhead + 1 op)
    {
        uint32_t a = (uint32_t)seed;
        c0 = clock64();
        for (int i = 0; i < ITERS; ++i) a = a * 3 + 1;
        c1 = clock64();
        out[k++] = (c1 - c0) / ITERS;
        out[16] += a;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 32 * sizeof(long long));
    cudaMemset(d, 0, 32 * sizeof(long long));
    kbench<<<1, 32>>>(d, 1);
    long long h[32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"rf_add_small (pow2 b)", "rf_mul_int", "stage_time_safe", "gcd_u32 pow2",
                           "gcd_u32 2^9*odd", "gcd_mod odd m", "rf_div32 odd", "rf_lt", "umod_u64_u32",
                           "64-bit mul chain", "32-bit mad chain", "ctz via ffs", "ctz via popc",
                           "(chain baseline)", "float quotient"};
    for (int k = 0; k < 15; ++k) printf("%-24s %6lld cycles\n", names[k], h[k]);
    return 0;
}
