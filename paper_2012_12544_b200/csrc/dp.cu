// dp.cu -- K2 minmax_dp: exact min-max contiguous partition (partition.hpp:112-185).
//
// One thread block per DP instance (a query's whole-layer partition, or one
// comm-coarsened partition per distinct a_th).  The recurrences are the
// reference's, on the same integers:
//   pass 1   dp[n][j] = min_k max(dp[n-1][k], seg(n,k,j))           T_opt = dp[N][U]
//   pass 2   g[n][j]  = min_{seg<=T_opt} max(g[n-1][k], foot(n,k,j)) F_opt = g[N][U]
//   feas     suffix feasibility under (T_opt, F_opt), then the earliest-cut greedy
// Transitions that provably cannot change a value are skipped, so the
// results are bit-identical while the work drops from N*U^2 to ~U^2:
//   * pass 1 scans k downward from j-1 and stops once seg(k,j) >= the best
//     value so far (every further k has a larger seg) or seg > T_ub, where
//     T_ub is the min-max value of an explicit equal-count partition
//     (dp values above T_ub cannot lie on an optimal path);
//   * pass 2 stops once seg > T_opt (the reference `continue`s on those) or
//     once 2*(W[j]-W[k]) >= best (foot only grows as k decreases);
//   * feas stops at seg > T_opt, or (k >= 1) once foot > F_opt.
// Rows live in shared memory; the block's threads split each row's j range
// and the feasibility rows are packed into bits with warp ballots.
#include "batch.cuh"
#include "kernels.h"

namespace bpk {

#define DP_INF (INT64_MAX / 4)
constexpr int DP_THREADS = 256;

struct DPSmem {
    int64_t* C;      // [T_slots][U+1] cost prefix per type slot
    int64_t* W;      // [U+1]
    int64_t* A;      // [U+1] out_act of unit j (A[0] unused)
    int64_t* r0;     // [U+1] rolling rows
    int64_t* r1;
    uint32_t* feas;  // [(N+1)][words]
    int32_t* pos;    // [U+1] layer index of unit boundary j
    int32_t* fwd;    // [N+1] band upper bounds
    int32_t* bwd;    // [N+1] band lower bounds
};

__device__ __forceinline__ int64_t dmax(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t dmin(int64_t a, int64_t b) { return a < b ? a : b; }

// Row bands under a threshold T (warp 0: forward, warp 1: backward).
//   fwd[n]: farthest unit boundary n stages can reach with every segment
//           <= T; bwd[n]: earliest boundary from which stages n+1..N can cover
//           the rest with segments <= T.
// Stages may take zero units in this relaxation, so fwd bounds the reachable
// set from above and bwd the completable set from below, on heterogeneous
// chains too.  A state (n, j) outside [bwd[n], fwd[n]] lies on no partition
// with all segments <= T, so pass 1 (T = T_ub >= T_opt) and pass 2 / feas
// (T = T_opt) may skip it without changing dp[N][U], g[N][U] or any feas bit
// the reconstruction reads.  Each greedy step is a 32-ary search (C is
// increasing along units): ceil(log32 U) ballot rounds per stage.
__device__ void dp_bands(const DPSmem& S, const ChainView& c, int N, int U, int64_t T, int warp, int lane) {
    const unsigned FULL = 0xffffffffu;
    if (warp == 0) {
        int cur = 0;
        if (lane == 0) S.fwd[0] = 0;
        for (int n = 1; n <= N; ++n) {
            const int64_t* C = S.C + (size_t)c.type[n - 1] * (U + 1);
            const int64_t target = C[cur] + T;
            int a = cur, b = U - (N - n);          // answer in [a, b], C[a] <= target
            if (b < a) b = a;
            while (a < b) {
                const int step = (b - a + 31) / 32;
                const int j = a + (lane + 1) * step;
                const unsigned m = __ballot_sync(FULL, j <= b && C[j] <= target);
                if (m == 0) {
                    b = a + step - 1;
                } else {
                    a += (32 - __clz(m)) * step;
                    b = min(b, a + step - 1);
                }
            }
            cur = a;
            if (lane == 0) S.fwd[n] = cur;
        }
    } else if (warp == 1) {
        int cur = U;
        if (lane == 0) S.bwd[N] = U;
        for (int n = N; n >= 1; --n) {
            const int64_t* C = S.C + (size_t)c.type[n - 1] * (U + 1);
            const int64_t target = C[cur] - T;
            int a = n - 1, b = cur;                // answer in [a, b], C[b] >= target
            if (a > b) a = b;
            while (a < b) {
                const int step = (b - a + 31) / 32;
                const int k = b - (lane + 1) * step;
                const unsigned m = __ballot_sync(FULL, k >= a && C[k] >= target);
                if (m == 0) {
                    a = b - step + 1;
                } else {
                    b -= (32 - __clz(m)) * step;
                    a = max(a, b - step + 1);
                }
            }
            cur = b;
            if (lane == 0) S.bwd[n - 1] = cur;
        }
    }
}

__global__ void __launch_bounds__(DP_THREADS) k_partition(BatchDev B, int which, int max_units, int max_N, int T_slots) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int64_t s_red[DP_THREADS / 32];
    __shared__ int32_t s_U;
    __shared__ int64_t s_T, s_F;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_items = B.dp_count[which];
    // items are handed out dynamically after each block's first (their sizes
    // differ by orders of magnitude; the list is heaviest first)
    __shared__ int s_next;
    auto next_item = [&]() {
        __syncthreads();
        if (tid == 0) s_next = (int)gridDim.x + atomicAdd(&B.dp_count[2 + which], 1);
        __syncthreads();
        return s_next;
    };
    for (int it = blockIdx.x; it < n_items; it = next_item()) {
        DPItem item = B.dp_items[(which == 0 ? 0 : B.nq) + it];
        if (which == 0 && B.qrep[item.q] != item.q) continue;   // shared: k_dedup_copy_dp
        const QDesc Q = B.q[item.q];
        NetView v = net_view(B.P, Q.net);
        ChainView c = chain_view(B.P, Q.cl, Q.N);
        const int N = Q.N;
        const int64_t L = v.L;
        // ---- units: boundaries pos[0..U] (pos[0] = 0, pos[U] = L)
        DPSmem S;
        {
            unsigned char* p = smem_raw;
            S.C = (int64_t*)p; p += (size_t)T_slots * (max_units + 1) * 8;
            S.W = (int64_t*)p; p += (size_t)(max_units + 1) * 8;
            S.A = (int64_t*)p; p += (size_t)(max_units + 1) * 8;
            S.r0 = (int64_t*)p; p += (size_t)(max_units + 1) * 8;
            S.r1 = (int64_t*)p; p += (size_t)(max_units + 1) * 8;
            S.pos = (int32_t*)p; p += (size_t)(max_units + 1) * 4;
            p = (unsigned char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
            S.feas = (uint32_t*)p;
            p += (size_t)(max_N + 1) * (((size_t)max_units + 1 + 31) / 32) * 4;
            S.fwd = (int32_t*)p;
            S.bwd = S.fwd + (max_N + 1);
        }
        if (item.a_th < 0) {
            for (int64_t j = tid; j <= L; j += DP_THREADS) S.pos[j] = (int32_t)j;
            if (tid == 0) s_U = (int32_t)L;
        } else {
            // coarsen_by_comm (44-67): cut after layer j iff a_j <= a_th or j == L.
            // Block-wide stream compaction over the layers in chunks.
            if (tid == 0) { S.pos[0] = 0; s_U = 0; }
            __syncthreads();
            for (int64_t base = 0; base < L; base += DP_THREADS) {
                int64_t j = base + tid + 1;   // 1-based layer
                bool cut = (j <= L) && (j == L || v.a[j - 1] <= item.a_th);
                unsigned bal = __ballot_sync(0xffffffffu, cut);
                if (lane == 0) s_red[warp] = __popc(bal);
                __syncthreads();
                int before = 0;
                for (int w = 0; w < warp; ++w) before += (int)s_red[w];
                int total = 0;
                for (int w = 0; w < DP_THREADS / 32; ++w) total += (int)s_red[w];
                int off = s_U + before + __popc(bal & ((1u << lane) - 1u));
                if (cut) S.pos[off + 1] = (int32_t)j;
                __syncthreads();
                if (tid == 0) s_U += total;
                __syncthreads();
            }
        }
        __syncthreads();
        const int U = s_U;
        // ---- type slots: the chain uses types c.type[0..N-1]; slot = index
        // among the first distinct occurrences (at most T_slots).
        // Cost prefix C[slot][j] = Pc_type[pos[j]]; W, A likewise.
        // (T_slots = number of types in the network; slot = type id.)
        for (int t = 0; t < T_slots && t < v.T; ++t)
            for (int j = tid; j <= U; j += DP_THREADS)
                S.C[(size_t)t * (U + 1) + j] = v.Pc[(int64_t)t * (L + 1) + S.pos[j]];
        for (int j = tid; j <= U; j += DP_THREADS) {
            S.W[j] = v.Pw[S.pos[j]];
            S.A[j] = j >= 1 ? v.a[S.pos[j] - 1] : 0;
        }
        __syncthreads();
        auto Cn = [&](int n) -> const int64_t* { return S.C + (size_t)c.type[n - 1] * (U + 1); };
        if (U < N) {   // InfeasibleShape (115-117)
            if (tid == 0) {
                if (item.a_th < 0) { B.qs[item.q].dp_shape = 1; }
            }
            __syncthreads();
            continue;
        }
        // ---- T_ub: equal-count split (a valid partition) -> upper bound on T_opt
        int64_t my = 0;
        for (int n = 1 + tid; n <= N; n += DP_THREADS) {
            int64_t k = ((int64_t)(n - 1) * U) / N, j = ((int64_t)n * U) / N;
            const int64_t* C = Cn(n);
            my = dmax(my, C[j] - C[k]);
        }
        for (int o = 16; o > 0; o >>= 1) my = dmax(my, __shfl_xor_sync(0xffffffffu, my, o));
        if (lane == 0) s_red[warp] = my;
        __syncthreads();
        int64_t T_ub = 0;
        for (int w = 0; w < DP_THREADS / 32; ++w) T_ub = dmax(T_ub, s_red[w]);
        __syncthreads();
        unsigned long long work = 0;
        dp_bands(S, c, N, U, T_ub, warp, lane);
        __syncthreads();
        // ---- pass 1
        int64_t* prev = S.r0;
        int64_t* cur = S.r1;
        for (int j = tid; j <= U; j += DP_THREADS) prev[j] = (j == 0) ? 0 : DP_INF;
        __syncthreads();
        for (int n = 1; n <= N; ++n) {
            const int64_t* C = Cn(n);
            const int jlo = max(n, S.bwd[n]), jhi = min(U - (N - n), S.fwd[n]);
            for (int j = tid; j <= U; j += DP_THREADS) {
                int64_t best = DP_INF;
                if (j >= jlo && j <= jhi) {
                    const int64_t cj = C[j];
                    for (int k = j - 1; k >= n - 1; --k) {
                        int64_t s = cj - C[k];
                        if (s > T_ub || s >= best) break;
                        int64_t v2 = dmax(prev[k], s);
                        best = dmin(best, v2);
                        ++work;
                    }
                    if (best > T_ub) best = DP_INF;
                }
                cur[j] = best;
            }
            __syncthreads();
            int64_t* t = prev; prev = cur; cur = t;
        }
        if (tid == 0) s_T = prev[U];
        __syncthreads();
        const int64_t T_opt = s_T;
        dp_bands(S, c, N, U, T_opt, warp, lane);
        // ---- pass 2
        for (int j = tid; j <= U; j += DP_THREADS) prev[j] = (j == 0) ? 0 : DP_INF;
        __syncthreads();
        for (int n = 1; n <= N; ++n) {
            const int64_t* C = Cn(n);
            const int64_t cN = (int64_t)(N - n + 1);
            const int jlo = max(n, S.bwd[n]), jhi = min(U - (N - n), S.fwd[n]);
            for (int j = tid; j <= U; j += DP_THREADS) {
                int64_t best = DP_INF;
                if (j >= jlo && j <= jhi) {
                    const int64_t cj = C[j], wj = S.W[j];
                    for (int k = j - 1; k >= n - 1; --k) {
                        if (cj - C[k] > T_opt) break;
                        int64_t w2 = 2 * (wj - S.W[k]);
                        if (w2 >= best) break;
                        ++work;
                        int64_t gp = prev[k];
                        if (gp == DP_INF) continue;
                        int64_t foot = w2 + cN * (k >= 1 ? S.A[k] : S.A[j]);
                        best = dmin(best, dmax(gp, foot));
                    }
                }
                cur[j] = best;
            }
            __syncthreads();
            int64_t* t = prev; prev = cur; cur = t;
        }
        if (tid == 0) s_F = prev[U];
        __syncthreads();
        const int64_t F_opt = s_F;
        // ---- feasibility suffix table (162-170), bit rows
        const int words = (U + 1 + 31) / 32;
        for (int w = tid; w < words * (N + 1); w += DP_THREADS) S.feas[w] = 0;
        __syncthreads();
        if (tid == 0) S.feas[(size_t)N * words + (U >> 5)] |= 1u << (U & 31);
        __syncthreads();
        for (int n = N - 1; n >= 0; --n) {
            const int64_t* C = Cn(n + 1);
            const int64_t cN = (int64_t)(N - n);
            const uint32_t* nxt = S.feas + (size_t)(n + 1) * words;
            const int jlo = max(n, S.bwd[n]), jhi = min(U, S.fwd[n]);
            for (int base = warp * 32; base <= U; base += DP_THREADS) {
                int j = base + lane;
                bool f = false;
                if (j >= jlo && j <= jhi) {
                    const int64_t cj = C[j], wj = S.W[j];
                    for (int j2 = j + 1; j2 <= U; ++j2) {
                        if (C[j2] - cj > T_opt) break;
                        ++work;
                        int64_t foot = 2 * (S.W[j2] - wj) + cN * (j >= 1 ? S.A[j] : S.A[j2]);
                        if (foot > F_opt) {
                            if (j >= 1) break;
                            continue;
                        }
                        if ((nxt[j2 >> 5] >> (j2 & 31)) & 1u) { f = true; break; }
                    }
                }
                unsigned bal = __ballot_sync(0xffffffffu, f);
                if (lane == 0 && base <= U) S.feas[(size_t)n * words + (base >> 5)] = bal;
            }
            __syncthreads();
        }
        // ---- earliest-cut greedy reconstruction (172-184), one warp
        if (warp == 0) {
            int curj = 0;
            int64_t target = 0;
            bool failed = false;
            for (int n = 1; n <= N && !failed; ++n) {
                const int64_t* C = Cn(n);
                const int64_t cN = (int64_t)(N - n + 1);
                const uint32_t* fr = S.feas + (size_t)n * words;
                int chosen = -1;
                for (int base = curj + 1; base <= U; base += 32) {
                    int j = base + lane;
                    bool in_t = false, ok = false;
                    if (j <= U) {
                        int64_t s = C[j] - C[curj];
                        in_t = s <= T_opt;
                        if (in_t) {
                            int64_t foot = 2 * (S.W[j] - S.W[curj]) + cN * (curj >= 1 ? S.A[curj] : S.A[j]);
                            ok = foot <= F_opt && ((fr[j >> 5] >> (j & 31)) & 1u);
                        }
                    }
                    unsigned bo = __ballot_sync(0xffffffffu, ok);
                    if (bo) { chosen = base + __ffs(bo) - 1; break; }
                    unsigned bt = __ballot_sync(0xffffffffu, in_t);
                    if (bt != 0xffffffffu) break;   // seg grows with j: nothing further fits
                }
                if (chosen < 0) { failed = true; break; }
                target = dmax(target, C[chosen] - C[curj]);
                if (lane == 0) {
                    if (item.a_th < 0) {
                        B.qlo[Q.qstage_off + n - 1] = S.pos[curj] + 1;
                        B.qhi[Q.qstage_off + n - 1] = S.pos[chosen];
                    } else {
                        // the coarse plan goes to both kinds' candidate slots
                        for (int k = 0; k < 2; ++k) {
                            int64_t local = (int64_t)k * Q.nbase + item.mslot;
                            int64_t o = Q.stage_off + local * N + (n - 1);
                            B.clo[o] = S.pos[curj] + 1;
                            B.chi[o] = S.pos[chosen];
                        }
                    }
                }
                curj = chosen;
            }
            if (lane == 0) {
                if (item.a_th < 0) {
                    B.qs[item.q].target = failed ? -1 : target;
                } else {
                    B.ms[Q.mslot_off + item.mslot].coarse_ok = failed ? 0 : 1;
                }
            }
        }
        // instrumentation: transitions performed
        for (int o = 16; o > 0; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
        if (lane == 0) atomicAdd(&B.work[which], work);
        __syncthreads();
    }
}

void launch_partition(const BatchDev& B, int which, int grid, int max_units, int max_N, int T_slots,
                      cudaStream_t st) {
    size_t bytes = partition_smem_bytes(max_units, max_N, T_slots);
    k_partition<<<grid, DP_THREADS, bytes, st>>>(B, which, max_units, max_N, T_slots);
}

cudaError_t partition_attributes_init(int optin_bytes) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, k_partition);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_partition, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin_bytes - (int)a.sharedSizeBytes);
}

// Layout of k_partition's dynamic shared memory (must match DPSmem above).
size_t partition_smem_bytes(int max_units, int max_N, int T_slots) {
    size_t words = ((size_t)max_units + 1 + 31) / 32;
    size_t b = (size_t)(max_units + 1) * 8 * (size_t)(T_slots + 4) + (size_t)(max_units + 1) * 4;
    b = (b + 15) & ~(size_t)15;
    return b + (size_t)(max_N + 1) * words * 4 + 2 * (size_t)(max_N + 1) * 4;
}

}  // namespace bpk
