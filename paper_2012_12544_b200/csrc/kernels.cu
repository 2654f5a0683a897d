// kernels.cu -- the explore() pipeline kernels other than the DP.
//
//   k_cost_prefix  K1  per-network prefix sums of fp, bp, fp+bp (per type) and
//                      w, block-wide scans over the SoA layer tables staged
//                      in shared memory (replaces units_from_network's and
//                      stage_*_time's per-call sums, partition.hpp:78-131,
//                      plan.hpp:90-132)
//   k_setup        K0  candidate records, thread per query
//   k_bottleneck   K1b comm-bottleneck test, a_th, coarse block count; queues
//                      the coarse DP items (thread per query)
//   k_refine       K3a intra_layer_refine, thread per query
//   k_prune        K3b balance_partition branches + estimate + memory
//                      fine-tune, thread per candidate
//   k_sim          K4  schedule simulation, thread per candidate
//   k_rank         K5  ranking / query outcome, thread per query
//   k_best             argmin of the per-query bests (multi-GPU exchange record)
#include "kernels.h"
#include "phases.cuh"

namespace bpk {

constexpr int SCAN_THREADS = 1024;

// Block-wide inclusive scan of one int64 per thread.
__device__ __forceinline__ int64_t block_scan(int64_t x, int64_t* warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < (int)(blockDim.x >> 5)) warp_tot[lane] = t;
    }
    __syncthreads();
    int64_t r = x + (warp > 0 ? warp_tot[warp - 1] : 0);
    __syncthreads();
    return r;
}

// One block per (network, table) with table = 0..T-1 (fp/bp/fp+bp of type t)
// or T (weights).  Layers are streamed through shared memory in tiles of
// SCAN_THREADS with coalesced loads; the running carry crosses tiles.
__global__ void __launch_bounds__(SCAN_THREADS) k_cost_prefix(const NetDesc* nets, const int64_t* fp,
                                                              const int64_t* bp, const int64_t* w, int64_t* Pfp,
                                                              int64_t* Pbp, int64_t* Pc, int64_t* Pw) {
    __shared__ int64_t tot[32];
    __shared__ int64_t tile_f[SCAN_THREADS], tile_b[SCAN_THREADS];
    const NetDesc d = nets[blockIdx.x];
    const int table = blockIdx.y;
    if (table > d.T) return;
    const int64_t L = d.L;
    int64_t carry_f = 0, carry_b = 0;
    if (table < d.T) {
        const int64_t* f = fp + d.off_typed + (int64_t)table * L;
        const int64_t* b = bp + d.off_typed + (int64_t)table * L;
        int64_t* of = Pfp + d.off_tpref + (int64_t)table * (L + 1);
        int64_t* ob = Pbp + d.off_tpref + (int64_t)table * (L + 1);
        int64_t* oc = Pc + d.off_tpref + (int64_t)table * (L + 1);
        if (threadIdx.x == 0) { of[0] = 0; ob[0] = 0; oc[0] = 0; }
        for (int64_t base = 0; base < L; base += SCAN_THREADS) {
            int64_t j = base + threadIdx.x;
            tile_f[threadIdx.x] = j < L ? f[j] : 0;
            tile_b[threadIdx.x] = j < L ? b[j] : 0;
            __syncthreads();
            int64_t sf = block_scan(tile_f[threadIdx.x], tot) + carry_f;
            int64_t sb = block_scan(tile_b[threadIdx.x], tot) + carry_b;
            if (j < L) { of[j + 1] = sf; ob[j + 1] = sb; oc[j + 1] = sf + sb; }
            if (threadIdx.x == SCAN_THREADS - 1) { tile_f[0] = sf; tile_b[0] = sb; }
            __syncthreads();
            carry_f = tile_f[0];
            carry_b = tile_b[0];
            __syncthreads();
        }
    } else {
        const int64_t* ww = w + d.off_layer;
        int64_t* ow = Pw + d.off_pref;
        if (threadIdx.x == 0) ow[0] = 0;
        for (int64_t base = 0; base < L; base += SCAN_THREADS) {
            int64_t j = base + threadIdx.x;
            tile_f[threadIdx.x] = j < L ? ww[j] : 0;
            __syncthreads();
            int64_t s = block_scan(tile_f[threadIdx.x], tot) + carry_f;
            if (j < L) ow[j + 1] = s;
            if (threadIdx.x == SCAN_THREADS - 1) tile_f[0] = s;
            __syncthreads();
            carry_f = tile_f[0];
            __syncthreads();
        }
    }
}

__global__ void k_setup(BatchDev B) {
    int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi < B.nq) setup_query(B, qi);
}

__global__ void k_bottleneck(BatchDev B) {
    int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= B.nq) return;
    const QDesc Q = B.q[qi];
    for (int m = 0; m < Q.nbase; ++m) {
        if (bottleneck_slot(B, qi, m)) {
            int idx = atomicAdd(&B.dp_count[1], 1);
            B.dp_items[B.nq + idx] = DPItem{qi, m, B.ms[Q.mslot_off + m].a_th};
        }
    }
}

// Queries / candidates are visited in the host's scheduling order
// (host_prep.hpp) so that the lanes of a warp run similar work.
__global__ void k_refine(BatchDev B) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < B.nq) refine_query(B, B.qorder[i]);
}

__global__ void k_prune(BatchDev B) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < B.ncand) prune_candidate(B, B.cperm[i]);
}

__global__ void k_rank(BatchDev B) {
    int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi < B.nq) rank_query(B, qi);
}

// Deterministic argmin over the batch's query bests (makespan, peak memory,
// max bandwidth demand, M, kind -- explorer.hpp:144-151 -- then query id).
__device__ __forceinline__ bool best_less(const bp_best_record& a, const bp_best_record& b) {
    if (a.valid != b.valid) return a.valid > b.valid;
    if (!a.valid) return a.query_id < b.query_id;
    Rat am{a.makespan.num, a.makespan.den}, bm{b.makespan.num, b.makespan.den};
    if (!rat_eq(am, bm)) return rat_lt(am, bm);
    Rat ap{a.peak_memory.num, a.peak_memory.den}, bpm{b.peak_memory.num, b.peak_memory.den};
    if (!rat_eq(ap, bpm)) return rat_lt(ap, bpm);
    Rat aw{a.max_bw.num, a.max_bw.den}, bw{b.max_bw.num, b.max_bw.den};
    if (!rat_eq(aw, bw)) return rat_lt(aw, bw);
    if (a.M != b.M) return a.M < b.M;
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.query_id < b.query_id;
}

constexpr int BEST_THREADS = 256;

__global__ void __launch_bounds__(BEST_THREADS) k_best(BatchDev B, bp_best_record* out, int64_t query_base,
                                                       const int64_t* query_ids) {
    __shared__ bp_best_record sh[BEST_THREADS];
    bp_best_record mine{};
    mine.valid = 0;
    mine.query_id = INT64_MAX;
    for (int qi = threadIdx.x; qi < B.nq; qi += blockDim.x) {
        const bp_query_result& r = B.res[qi];
        bp_best_record x{};
        x.valid = r.status == BP_Q_OK ? 1 : 0;
        x.query_id = query_ids ? query_ids[qi] : query_base + qi;
        if (x.valid) {
            x.makespan = r.best_makespan;
            x.peak_memory = r.best_peak_memory;
            x.max_bw = r.best_max_bw;
            x.M = r.best_M;
            x.kind = r.best_kind;
        }
        if (best_less(x, mine)) mine = x;
    }
    sh[threadIdx.x] = mine;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s && best_less(sh[threadIdx.x + s], sh[threadIdx.x])) sh[threadIdx.x] = sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

static inline int blocks(int64_t n, int t) { return (int)((n + t - 1) / t); }

void launch_cost_prefix(const NetDesc* nets, int n_nets, const int64_t* fp, const int64_t* bp, const int64_t* w,
                        int64_t* Pfp, int64_t* Pbp, int64_t* Pc, int64_t* Pw, cudaStream_t st, int max_T) {
    dim3 grid(n_nets, max_T + 1);
    k_cost_prefix<<<grid, SCAN_THREADS, 0, st>>>(nets, fp, bp, w, Pfp, Pbp, Pc, Pw);
}

void launch_setup(const BatchDev& B, cudaStream_t st) {
    if (B.nq) k_setup<<<blocks(B.nq, 128), 128, 0, st>>>(B);
}
void launch_bottleneck(const BatchDev& B, cudaStream_t st) {
    if (B.nq) k_bottleneck<<<blocks(B.nq, 128), 128, 0, st>>>(B);
}
void launch_refine(const BatchDev& B, cudaStream_t st) {
    if (B.nq) k_refine<<<blocks(B.nq, 64), 64, 0, st>>>(B);
}
void launch_prune(const BatchDev& B, cudaStream_t st) {
    if (B.ncand) k_prune<<<blocks(B.ncand, 128), 128, 0, st>>>(B);
}
void launch_rank(const BatchDev& B, cudaStream_t st) {
    if (B.nq) k_rank<<<blocks(B.nq, 128), 128, 0, st>>>(B);
}
void launch_best(const BatchDev& B, bp_best_record* out, int64_t query_base, const int64_t* query_ids,
                 cudaStream_t st) {
    k_best<<<1, BEST_THREADS, 0, st>>>(B, out, query_base, query_ids);
}

}  // namespace bpk
