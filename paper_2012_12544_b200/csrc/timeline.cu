// timeline.cu -- kernels and host entry for one plan's full-timeline
// simulate and estimate (timeline.cuh).  Not on the
// sweep path: one plan per call, so the walk is one thread (it is a serial
// recurrence) and the per-stage sorts and high-water marks are one thread per
// stage.
#include <cuda_runtime.h>

#include <vector>

#include "kernels.h"
#include "timeline.cuh"

namespace bpk {

namespace {

__device__ void tl_bind(TlArgs& A, const Pools& P, int net, int cl, int clusterN) {
    A.v = net_view(P, net);
    A.c = chain_view(P, cl, A.N < clusterN ? A.N : clusterN);
}

__global__ void k_tl_walk(TlArgs A, Pools P, int net, int cl, bp_timeline_result* res) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    tl_bind(A, P, net, cl, A.clusterN);
    bp_timeline_result r{};
    r.status = BP_C_OK;
    if (tl_chain(A, r)) tl_walk(A, r);
    *res = r;
}

__global__ void k_tl_stages(TlArgs A, Pools P, int net, int cl, bp_timeline_result* res, TlPoint* pts,
                            TlPoint* tmp, Rat* hw, Rat* ws, Rat* busy) {
    if (res->status != BP_C_OK) return;
    tl_bind(A, P, net, cl, A.clusterN);
    const int s = blockIdx.x * blockDim.x + threadIdx.x + 1;
    uint32_t code = 0;
    if (s <= A.N) code = tl_stage(A, s, pts + (int64_t)(s - 1) * 2 * A.M, tmp + (int64_t)(s - 1) * 2 * A.M, hw, ws);
    if (s == 1 && !code) code = tl_busy(A, busy);
    // every error these can raise is an overflow: the first one decides
    if (code) atomicCAS(&res->status, (int32_t)BP_C_OK, (int32_t)code);
}

__global__ void k_tl_estimate(TlArgs A, Pools P, int net, int cl, bp_estimate_result* res, bp_stage* st,
                              int32_t* inf, Rat* scr, int64_t* scr64) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    tl_bind(A, P, net, cl, A.clusterN);
    bp_estimate_result r{};
    tl_estimate(A, r, st, inf, scr, scr64);
    *res = r;
}

// one device allocation carved into arrays
struct Carve {
    std::vector<size_t> off;
    size_t end = 0;
    template <class T>
    size_t take(size_t n) {
        size_t o = end;
        end += ((n ? n : 1) * sizeof(T) + 255) & ~(size_t)255;
        return o;
    }
};

template <class T>
T* at(void* base, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

cudaError_t upload_plan(const bp_plan_request& q, void* base, size_t olo, size_t ohi, size_t old, size_t otr) {
    const size_t N = (size_t)q.n_stages;
    cudaError_t e = cudaMemcpy(at<int32_t>(base, olo), q.lo, N * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(at<int32_t>(base, ohi), q.hi, N * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(at<bp_rat>(base, old), q.lead, N * sizeof(bp_rat), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(at<bp_rat>(base, otr), q.trail, N * sizeof(bp_rat), cudaMemcpyHostToDevice);
    return e;
}

}  // namespace

cudaError_t timeline_simulate(const Pools& P, int clusterN, const bp_plan_request& q, bp_timeline_result* res,
                              bp_event* events, int64_t cap, bp_rat* highwater, bp_rat* wstatic, bp_rat* busy,
                              int64_t* h2d, int64_t* d2h) {
    const int N = q.n_stages;
    const int64_t M = q.M > 0 ? q.M : 0, mini = q.mini_batches > 0 ? q.mini_batches : 0;
    const size_t NM = (size_t)N * (size_t)M, LM = (size_t)(N > 1 ? N - 1 : 0) * (size_t)M;
    const size_t nev = (size_t)mini * (2 * NM + 4 * LM);
    Carve C;
    const size_t olo = C.take<int32_t>(N), ohi = C.take<int32_t>(N), old = C.take<Rat>(N), otr = C.take<Rat>(N);
    const size_t oF = C.take<Rat>(N), oB = C.take<Rat>(N), oW = C.take<Rat>(N), oa = C.take<int64_t>(N),
                 oSR = C.take<int64_t>(N);
    const size_t osF = C.take<Rat>(NM), oeF = C.take<Rat>(NM), osB = C.take<Rat>(NM), oeB = C.take<Rat>(NM);
    const size_t otFs = C.take<Rat>(LM), otFe = C.take<Rat>(LM), otBs = C.take<Rat>(LM), otBe = C.take<Rat>(LM);
    const size_t omk = C.take<Rat>(1), ooff = C.take<int64_t>((size_t)N + 1);
    const size_t oev = C.take<bp_event>(nev), oevt = C.take<bp_event>(nev);
    const size_t opt = C.take<TlPoint>(2 * NM), opt2 = C.take<TlPoint>(2 * NM);
    const size_t ohw = C.take<Rat>(N), ows = C.take<Rat>(N), obusy = C.take<Rat>(N), ores = C.take<bp_timeline_result>(1);
    void* base = nullptr;
    cudaError_t e = cudaMalloc(&base, C.end);
    if (e != cudaSuccess) return e;
    e = upload_plan(q, base, olo, ohi, old, otr);
    *h2d += (int64_t)N * (8 + 2 * (int64_t)sizeof(bp_rat));
    TlArgs A{};
    A.N = N;
    A.kind = q.kind;
    A.clusterN = clusterN;
    A.M = q.M;
    A.micro = q.micro;
    A.mini = mini;
    A.lo = at<int32_t>(base, olo);
    A.hi = at<int32_t>(base, ohi);
    A.lead = at<Rat>(base, old);
    A.trail = at<Rat>(base, otr);
    A.F = at<Rat>(base, oF);
    A.B = at<Rat>(base, oB);
    A.W = at<Rat>(base, oW);
    A.a = at<int64_t>(base, oa);
    A.SR = at<int64_t>(base, oSR);
    A.sF = at<Rat>(base, osF);
    A.eF = at<Rat>(base, oeF);
    A.sB = at<Rat>(base, osB);
    A.eB = at<Rat>(base, oeB);
    A.tFs = at<Rat>(base, otFs);
    A.tFe = at<Rat>(base, otFe);
    A.tBs = at<Rat>(base, otBs);
    A.tBe = at<Rat>(base, otBe);
    A.makespan1 = at<Rat>(base, omk);
    A.ev = at<bp_event>(base, oev);
    A.ev_tmp = at<bp_event>(base, oevt);
    A.off = at<int64_t>(base, ooff);
    bp_timeline_result* dres = at<bp_timeline_result>(base, ores);
    if (e == cudaSuccess) {
        k_tl_walk<<<1, 1>>>(A, P, q.network, q.cluster, dres);
        k_tl_stages<<<(N + 63) / 64 > 0 ? (N + 63) / 64 : 1, 64>>>(A, P, q.network, q.cluster, dres,
                                                                     at<TlPoint>(base, opt), at<TlPoint>(base, opt2),
                                                                     at<Rat>(base, ohw), at<Rat>(base, ows),
                                                                     at<Rat>(base, obusy));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(res, dres, sizeof(*res), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && res->status == BP_C_OK) {
        const int64_t n = res->n_events < cap ? res->n_events : cap;
        if (events && n > 0) e = cudaMemcpy(events, at<bp_event>(base, oev), (size_t)n * sizeof(bp_event),
                                            cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && highwater)
            e = cudaMemcpy(highwater, at<Rat>(base, ohw), (size_t)N * sizeof(Rat), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && wstatic)
            e = cudaMemcpy(wstatic, at<Rat>(base, ows), (size_t)N * sizeof(Rat), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && busy && N > 1)
            e = cudaMemcpy(busy, at<Rat>(base, obusy), (size_t)(N - 1) * sizeof(Rat), cudaMemcpyDeviceToHost);
        *d2h += n * (int64_t)sizeof(bp_event) + (3 * (int64_t)N) * (int64_t)sizeof(Rat);
    }
    cudaFree(base);
    return e;
}

cudaError_t timeline_estimate(const Pools& P, int clusterN, const bp_plan_request& q, bp_estimate_result* res,
                              bp_stage* stages, int32_t* infeasible, int64_t* h2d, int64_t* d2h) {
    const int N = q.n_stages;
    Carve C;
    const size_t olo = C.take<int32_t>(N), ohi = C.take<int32_t>(N), old = C.take<Rat>(N), otr = C.take<Rat>(N);
    const size_t oscr = C.take<Rat>(7 * (size_t)N), oscr64 = C.take<int64_t>(2 * (size_t)N);
    const size_t ost = C.take<bp_stage>(N), oinf = C.take<int32_t>(N), ores = C.take<bp_estimate_result>(1);
    void* base = nullptr;
    cudaError_t e = cudaMalloc(&base, C.end);
    if (e != cudaSuccess) return e;
    e = upload_plan(q, base, olo, ohi, old, otr);
    *h2d += (int64_t)N * (8 + 2 * (int64_t)sizeof(bp_rat));
    TlArgs A{};
    A.N = N;
    A.kind = q.kind;
    A.clusterN = clusterN;
    A.M = q.M;
    A.micro = q.micro;
    A.mini = 1;
    A.lo = at<int32_t>(base, olo);
    A.hi = at<int32_t>(base, ohi);
    A.lead = at<Rat>(base, old);
    A.trail = at<Rat>(base, otr);
    bp_estimate_result* dres = at<bp_estimate_result>(base, ores);
    if (e == cudaSuccess) {
        k_tl_estimate<<<1, 1>>>(A, P, q.network, q.cluster, dres, at<bp_stage>(base, ost), at<int32_t>(base, oinf),
                                at<Rat>(base, oscr), at<int64_t>(base, oscr64));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(res, dres, sizeof(*res), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && res->status == BP_C_OK) {
        if (stages) e = cudaMemcpy(stages, at<bp_stage>(base, ost), (size_t)N * sizeof(bp_stage), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && infeasible)
            e = cudaMemcpy(infeasible, at<int32_t>(base, oinf), (size_t)N * 4, cudaMemcpyDeviceToHost);
        *d2h += (int64_t)N * (int64_t)(sizeof(bp_stage) + 4);
    }
    cudaFree(base);
    return e;
}

}  // namespace bpk
