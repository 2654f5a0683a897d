// tests/cpp/refine_walk_bench.cu -- TOOL (not collected by pytest): the slim
// refine walk (csrc/refine_fast.cuh) of one query on one GPU thread, with its
// inputs in shared memory exactly as k_refine_fast stages them, timed with
// clock64 per step section.  Input: a dump of the walk's inputs written by the
// test emulator (BPEMU_DUMP_REFINE=<query>, tests/emu/emu.cpp), e.g.
// tests/cpp/refine_q18895.bin = C5 query 18895 (N = 64, L = 128, 3,255
// boundary steps, the sweep's longest walk).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRF_PROF \
//        -I include tests/cpp/refine_walk_bench.cu -o /tmp/rwb && /tmp/rwb tests/cpp/refine_q18895.bin
#include <cstdio>
#include <vector>

#include "../../paper_2012_12544_b200/csrc/refine_fast.cuh"

using namespace bpk;

__global__ void kwalk(const int32_t* in, int L, int T, int N, const Rat* t0, int64_t* stats, long long* prof,
                      int reps) {
    extern __shared__ __align__(16) unsigned char sm[];
    Rat* t = reinterpret_cast<Rat*>(sm);
    Rat* lead = t + N;
    Rat* trail = lead + N;
    int32_t* cost = reinterpret_cast<int32_t*>(trail + N);
    int32_t* act = cost + T * L;
    int32_t* type = act + L;
    int32_t* lo = type + N;
    int32_t* hi = lo + N;
    uint8_t* memo = reinterpret_cast<uint8_t*>(hi + N);
    if (threadIdx.x) return;
    long long total = 0;
    for (int r = 0; r < reps; ++r) {
        for (int k = 0; k < T * L + L + N; ++k) cost[k] = in[k];
        for (int s = 0; s < N; ++s) {
            lo[s] = in[T * L + L + N + s];
            hi[s] = in[T * L + L + 2 * N + s];
            t[s] = t0[s];
            lead[s] = R(1);
            trail[s] = R(1);
        }
        FastRefine q{cost, act, type, L, N, lo, hi, lead, trail, t, memo};
        const long long c0 = clock64();
        const int res = refine_fast_walk(q, stats, prof + 8 * r);
        total += clock64() - c0;
        stats[3] = res;
    }
    stats[4] = total / reps;
}

int main(int argc, char** argv) {
    FILE* f = fopen(argc > 1 ? argv[1] : "tests/cpp/refine_q18895.bin", "rb");
    if (!f) return 1;
    int32_t h[3];
    if (fread(h, 4, 3, f) != 3) return 1;
    const int L = h[0], T = h[1], N = h[2];
    std::vector<int32_t> in(T * L + L + 3 * N);
    if (fread(in.data(), 4, in.size(), f) != in.size()) return 1;
    std::vector<Rat> t(N);
    if (fread(t.data(), sizeof(Rat), N, f) != (size_t)N) return 1;
    fclose(f);
    int32_t* din;
    Rat* dt;
    int64_t* dst;
    long long* dprof;
    const int reps = 3;
    cudaMalloc(&din, in.size() * 4);
    cudaMalloc(&dt, N * sizeof(Rat));
    cudaMalloc(&dst, 8 * 8);
    cudaMalloc(&dprof, 8 * 8 * reps);
    cudaMemset(dprof, 0, 8 * 8 * reps);
    cudaMemcpy(din, in.data(), in.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, t.data(), N * sizeof(Rat), cudaMemcpyHostToDevice);
    const size_t smem = 3 * N * sizeof(Rat) + (T * L + L + 3 * N) * 4 + N + 64;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kwalk<<<1, 32, smem>>>(din, L, T, N, dt, dst, dprof, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int64_t st[8];
    long long prof[8 * reps];
    cudaMemcpy(st, dst, sizeof st, cudaMemcpyDeviceToHost);
    cudaMemcpy(prof, dprof, sizeof prof, cudaMemcpyDeviceToHost);
    printf("L %d T %d N %d: result %lld, iterations %lld, steps %lld, moves %lld\n", L, T, N, (long long)st[3],
           (long long)st[0], (long long)st[1], (long long)st[2]);
    printf("walk: %lld cycles (%.1f per evaluated step), %d reps in %.3f ms\n", (long long)st[4],
           (double)st[4] / st[1], reps, ms);
    const char* names[8] = {"compare", "layer+avail", "x", "quantize", "accept", "commit", "-", "loop/skip"};
    for (int k = 0; k < 8; ++k)
        printf("  %-12s %10lld cycles  %7.1f per step\n", names[k], prof[8 * (reps - 1) + k],
               (double)prof[8 * (reps - 1) + k] / st[1]);
    return 0;
}
