// api.cu -- host implementation of the C ABI in include/bapipe_b200.h.
//
// The boundary replaces bapipe::explore (explorer.hpp:80-155) for batches of
// queries.  Host work is limited to validation and layout (host_prep.hpp);
// every candidate evaluation runs in the sm_100a kernels (kernels.cu, dp.cu).
// There is no CPU fallback: without a usable device, bp_create returns NULL.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "host_prep.hpp"
#include "kernels.h"

using namespace bpk;

namespace {

thread_local std::string g_err;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    bool ensure(size_t bytes) {
        if (bytes <= cap) return true;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return false;
        cap = bytes;
        return true;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct HostPinned {
    void* p = nullptr;
    size_t cap = 0;
    bool ensure(size_t bytes) {
        if (bytes <= cap) return true;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return false;
        cap = bytes;
        return true;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

struct KStat {
    double ms = 0;
    int64_t launches = 0;
    double work = 0;
};

// Bump layout of one contiguous allocation.
struct Layout {
    size_t off = 0;
    template <class T>
    size_t take(size_t n) {
        size_t o = off;
        off += ((n * sizeof(T)) + 255) & ~(size_t)255;
        return o;
    }
};

}  // namespace

struct bp_batch {
    HostBatch hb;
    BatchDev dev{};
    DevBuf mem;
    HostPinned stage_in;
    size_t in_off = 0, in_bytes = 0;
    size_t cand_off = 0, stage_off = 0, res_off = 0;
    bool details = false;
    int nq = 0;
    int dp_grid = 0, dp_max_units = 0;
    int refine_grid = 0;       // slim refine kernel: persistent grid, 0 = not used
    int refine_warps = 1;      // its walking warps per block
    size_t refine_bytes = 0;   // its dynamic shared memory
    uint64_t gen = 0;          // bp_ctx::gen at prepare: the device tables it points at
    // this batch's own side stream and fork / join events (concurrent batches
    // of one context must not share them)
    cudaStream_t side = nullptr, lane = nullptr;
    cudaStream_t rstream = nullptr;   // the refine walks, at the device's greatest priority
    cudaGraphExec_t gexec = nullptr;  // run_graph: the captured kernel sequence
    std::vector<char> gkey;           // ... and the launch inputs it was captured with
    int64_t glaunches = 0;            // own kernels per replay
    bool graph_failed = false;
    cudaEvent_t gfork = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, done = nullptr, rjoin = nullptr;
    int prio = 0;              // priority of this batch's own streams (split parts)
    // BP_OPT_SPLIT: the batch runs as two parts on two streams (see split_prepare)
    std::vector<bp_batch*> parts;
    std::vector<std::vector<int32_t>> part_q;      // parent query index of each part query
    DevBuf part_ids;                               // device: parent query index per part query (parts concatenated)
    DevBuf part_best;                              // device: one bp_best_record per part
    DevBuf res_all;                                // device: the parts' query results in the caller's order
    DevBuf part_woff;                              // device: (candidate, stage) offset in the caller's layout per part query
    DevBuf cand_all, stage_all;                    // device: the parts' candidate / stage records in the caller's layout
    std::vector<int64_t> part_ids_host;
};

struct bp_ctx {
    int device = 0;
    int sm_count = 148;
    std::string err;
    int64_t launches = 0;
    int64_t h2d = 0, d2h = 0;
    HostNets hn;
    HostCls hc;
    bool have_nets = false, have_cls = false;
    uint64_t gen = 0;        // bumped by every bp_set_networks / bp_set_clusters
    DevBuf nets_mem, cls_mem;
    HostPinned stage_tables;   // pinned staging of the network tables
    HostPinned stage_cls;      // ... and of the cluster tables
    // table uploads run on their own stream and end with tables_ev: the set_*
    // calls return without waiting, and every consumer of the device tables
    // (a batch run, a timeline call) orders itself after the event
    cudaStream_t tstream = nullptr;
    cudaEvent_t tables_ev = nullptr;
    cudaEvent_t nets_ev = nullptr, cls_ev = nullptr;   // each staging buffer's last copy
    // batch runs enqueued since the last table upload (an event on each
    // caller stream): an upload's copies wait for them on the device, so
    // that no run in flight reads a table while it is overwritten
    std::vector<cudaEvent_t> runs;
    cudaEvent_t tl_base = nullptr;   // diagnostics (BP_TIMELINE): recorded at each profiled run's start
    Pools P{};
    int max_T = 1;
    size_t smem_optin = 227 * 1024;   // cudaDeviceProp::sharedMemPerBlockOptin
    bool prof = false;
    bool dedup = true;       // BP_OPT_DEDUP
    bool plan_only = false;  // BP_OPT_PLAN_ONLY
    bool prune_lb = false;   // BP_OPT_PRUNE_LB
    int split = 4;           // BP_OPT_SPLIT: parts per large batch (0 = off)
    std::map<std::string, KStat> stats;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> event_pool;
    bp_batch* cached = nullptr;
    bool stats_accumulate = false;   // fetching the parts of a split batch: work counters add up
};

namespace {

int fail(bp_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    g_err = msg;
    return code;
}

int cuda_fail(bp_ctx* c, cudaError_t e, const char* where) {
    return fail(c, BP_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

cudaEvent_t get_event(bp_ctx* c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void note_run(bp_ctx* c, cudaStream_t st);
void tables_wait_runs(bp_ctx* c);

// Launch wrapper: counts launches, brackets them with events when profiling.
template <class F>
void timed(bp_ctx* c, const char* name, cudaStream_t st, F&& f, int n_kernels = 1) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->prof) {
        a = get_event(c);
        b = get_event(c);
        cudaEventRecord(a, st);
    }
    f();
    c->launches += n_kernels;
    if (c->prof) {
        cudaEventRecord(b, st);
        c->pending.push_back({name, {a, b}});
    }
}

// Phase spans (several launches, possibly on both streams) for the profile:
// an event on the main stream before the phase and one after its join.
cudaEvent_t phase_begin(bp_ctx* c, cudaStream_t st) {
    if (!c->prof) return nullptr;
    cudaEvent_t a = get_event(c);
    cudaEventRecord(a, st);
    return a;
}
void phase_end(bp_ctx* c, const char* name, cudaStream_t st, cudaEvent_t a) {
    if (!a) return;
    cudaEvent_t b = get_event(c);
    cudaEventRecord(b, st);
    c->pending.push_back({name, {a, b}});
}

void collect(bp_ctx* c) {
    refine_trace_collect();
    // BP_TIMELINE=<file>: append every span's start / end (ms from the first
    // span's start) -- the launch timeline of a profiled run (tests/timeline_probe.py)
    static const char* tl = getenv("BP_TIMELINE");
    if (tl && !c->pending.empty()) {
        if (FILE* f = fopen(tl, "a")) {
            cudaEvent_t base = c->tl_base ? c->tl_base : c->pending.front().second.first;
            cudaEventSynchronize(c->pending.back().second.second);
            for (auto& p : c->pending) {
                float a = 0, b = 0;
                cudaEventSynchronize(p.second.second);
                cudaEventElapsedTime(&a, base, p.second.first);
                cudaEventElapsedTime(&b, base, p.second.second);
                fprintf(f, "%s %.4f %.4f\n", p.first.c_str(), a, b);
            }
            fprintf(f, "--\n");
            fclose(f);
        }
    }
    for (auto& p : c->pending) {
        float ms = 0;
        cudaEventSynchronize(p.second.second);
        cudaEventElapsedTime(&ms, p.second.first, p.second.second);
        KStat& k = c->stats[p.first];
        k.ms += ms;
        k.launches += 1;
        c->event_pool.push_back(p.second.first);
        c->event_pool.push_back(p.second.second);
    }
    c->pending.clear();
}

void note_run(bp_ctx* c, cudaStream_t st) {
    cudaEvent_t ev = get_event(c);
    cudaEventRecord(ev, st);
    c->runs.push_back(ev);
    if (c->runs.size() > 64) {   // drop the finished ones
        std::vector<cudaEvent_t> keep;
        for (cudaEvent_t e : c->runs) {
            if (cudaEventQuery(e) == cudaSuccess) c->event_pool.push_back(e);
            else keep.push_back(e);
        }
        c->runs.swap(keep);
    }
}

void tables_wait_runs(bp_ctx* c) {
    for (cudaEvent_t e : c->runs) {
        cudaStreamWaitEvent(c->tstream, e, 0);
        c->event_pool.push_back(e);   // the wait is bound at this call: the event may be reused
    }
    c->runs.clear();
}

template <class T>
T* dptr(void* base, size_t off) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + off);
}

int upload_networks(bp_ctx* c) {
    HostNets& H = c->hn;
    Layout L;
    size_t o_desc = L.take<NetDesc>(H.desc.size());
    size_t o_fp = L.take<int64_t>(H.fp.size());
    size_t o_bp = L.take<int64_t>(H.bp.size());
    size_t o_w = L.take<int64_t>(H.w.size());
    size_t o_a = L.take<int64_t>(H.a.size());
    size_t o_as = L.take<int64_t>(H.asort.size());
    size_t o_Pfp = L.take<int64_t>(H.n_tpref);
    size_t o_Pbp = L.take<int64_t>(H.n_tpref);
    size_t o_Pc = L.take<int64_t>(H.n_tpref);
    size_t o_Pw = L.take<int64_t>(H.n_pref);
    size_t o_tok = L.take<uint8_t>(H.type_ok.size());
    if (!c->nets_mem.ensure(L.off)) return fail(c, BP_OUT_OF_MEMORY, "cudaMalloc(networks)");
    // the previous network upload's copies have read the staging buffer
    cudaEventSynchronize(c->nets_ev);
    if (!c->stage_tables.ensure(L.off)) return fail(c, BP_OUT_OF_MEMORY, "cudaHostAlloc(tables)");
    void* b = c->nets_mem.p;
    // through pinned staging, laid out as on the device: the tables are
    // staged in 256 KB pieces on the host pool, then copied in two DMAs (the
    // prefix tables between them are the device's own, k_cost_prefix)
    char* stg = static_cast<char*>(c->stage_tables.p);
    struct Piece { size_t off; const void* src; size_t bytes; };
    const Piece tabs[] = {{o_desc, H.desc.data(), H.desc.size() * sizeof(NetDesc)}, {o_fp, H.fp.data(), H.fp.size() * 8},
                          {o_bp, H.bp.data(), H.bp.size() * 8},   {o_w, H.w.data(), H.w.size() * 8},
                          {o_a, H.a.data(), H.a.size() * 8},      {o_as, H.asort.data(), H.asort.size() * 8},
                          {o_tok, H.type_ok.data(), H.type_ok.size()}};
    std::vector<Piece> pieces;
    const size_t PIECE = 256 * 1024;
    for (const Piece& t : tabs) {
        c->h2d += (int64_t)t.bytes;
        for (size_t a = 0; a < t.bytes; a += PIECE)
            pieces.push_back({t.off + a, static_cast<const char*>(t.src) + a, std::min(PIECE, t.bytes - a)});
    }
    host_parallel_for((int)pieces.size(), [&](int k) { std::memcpy(stg + pieces[k].off, pieces[k].src, pieces[k].bytes); });
    cudaError_t e = cudaMemcpyAsync(b, stg, o_Pfp, cudaMemcpyHostToDevice, c->tstream);
    if (e == cudaSuccess && H.type_ok.size())
        e = cudaMemcpyAsync(dptr<char>(b, o_tok), stg + o_tok, H.type_ok.size(), cudaMemcpyHostToDevice, c->tstream);
    if (e == cudaSuccess) e = cudaEventRecord(c->nets_ev, c->tstream);
    if (e != cudaSuccess) return cuda_fail(c, e, "upload networks");
    Pools& P = c->P;
    P.nets = dptr<NetDesc>(b, o_desc);
    P.fp = dptr<int64_t>(b, o_fp);
    P.bp = dptr<int64_t>(b, o_bp);
    P.w = dptr<int64_t>(b, o_w);
    P.a = dptr<int64_t>(b, o_a);
    P.asort = dptr<int64_t>(b, o_as);
    P.Pfp = dptr<int64_t>(b, o_Pfp);
    P.Pbp = dptr<int64_t>(b, o_Pbp);
    P.Pc = dptr<int64_t>(b, o_Pc);
    P.Pw = dptr<int64_t>(b, o_Pw);
    P.type_ok = dptr<uint8_t>(b, o_tok);
    c->max_T = std::max(1, H.max_T);
    // K1 cost_prefix on the device
    if (!H.desc.empty()) {
        timed(c, "cost_prefix", c->tstream, [&] {
            launch_cost_prefix(P.nets, (int)H.desc.size(), P.fp, P.bp, P.w, const_cast<int64_t*>(P.Pfp),
                               const_cast<int64_t*>(P.Pbp), const_cast<int64_t*>(P.Pc), const_cast<int64_t*>(P.Pw),
                               c->tstream, c->max_T);
        });
    }
    e = cudaEventRecord(c->tables_ev, c->tstream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "cost_prefix");
    if (c->prof) {
        cudaStreamSynchronize(c->tstream);
        collect(c);
    }
    return BP_OK;
}

int upload_clusters(bp_ctx* c) {
    HostCls& H = c->hc;
    Layout L;
    size_t o_desc = L.take<ClDesc>(H.desc.size());
    size_t o_t = L.take<int32_t>(H.ctype.size());
    size_t o_cap = L.take<int64_t>(H.cap.size());
    size_t o_mm = L.take<int64_t>(H.minm.size());
    size_t o_bw = L.take<int64_t>(H.bw.size());
    if (!c->cls_mem.ensure(L.off)) return fail(c, BP_OUT_OF_MEMORY, "cudaMalloc(clusters)");
    cudaEventSynchronize(c->cls_ev);   // the previous cluster upload has read the staging buffer
    if (!c->stage_cls.ensure(L.off)) return fail(c, BP_OUT_OF_MEMORY, "cudaHostAlloc(tables)");
    void* b = c->cls_mem.p;
    auto up = [&](size_t off, const void* src, size_t bytes) {
        c->h2d += (int64_t)bytes;
        if (!bytes) return cudaSuccess;
        std::memcpy(static_cast<char*>(c->stage_cls.p) + off, src, bytes);
        return cudaMemcpyAsync(dptr<char>(b, off), static_cast<char*>(c->stage_cls.p) + off, bytes,
                               cudaMemcpyHostToDevice, c->tstream);
    };
    cudaError_t e = up(o_desc, H.desc.data(), H.desc.size() * sizeof(ClDesc));
    if (e == cudaSuccess) e = up(o_t, H.ctype.data(), H.ctype.size() * 4);
    if (e == cudaSuccess) e = up(o_cap, H.cap.data(), H.cap.size() * 8);
    if (e == cudaSuccess) e = up(o_mm, H.minm.data(), H.minm.size() * 8);
    if (e == cudaSuccess) e = up(o_bw, H.bw.data(), H.bw.size() * 8);
    if (e == cudaSuccess) e = cudaEventRecord(c->cls_ev, c->tstream);
    if (e == cudaSuccess) e = cudaEventRecord(c->tables_ev, c->tstream);
    if (e != cudaSuccess) return cuda_fail(c, e, "upload clusters");
    c->P.cls = dptr<ClDesc>(b, o_desc);
    c->P.ctype = dptr<int32_t>(b, o_t);
    c->P.cap = dptr<int64_t>(b, o_cap);
    c->P.minm = dptr<int64_t>(b, o_mm);
    c->P.bw = dptr<int64_t>(b, o_bw);
    return BP_OK;
}

// Host prep + device layout + H2D of the batch's inputs (on stream st).
int prepare_built(bp_ctx* c, bp_batch* B, int nq, int details, cudaStream_t st);

int prepare(bp_ctx* c, bp_batch* B, const bp_query* q, int nq, int details, cudaStream_t st) {
    if (!c->have_nets || !c->have_cls) return fail(c, BP_BAD_INPUT, "networks/clusters not set");
    std::string err;
    static const bool timing = getenv("BP_HOST_TIMING") != nullptr;   // diagnostics (stderr)
    const auto t0 = std::chrono::steady_clock::now();
    if (!build_batch(q, nq, c->hn, c->hc, B->hb, err)) return fail(c, BP_BAD_INPUT, err);
    const auto t1 = std::chrono::steady_clock::now();
    const HostBatch& hb = B->hb;
    for (int i = 0; i < nq; ++i)
        if (q[i].cand_offset != hb.q[i].cand_off || q[i].stage_offset != hb.q[i].stage_off)
            return fail(c, BP_BAD_INPUT, "query offsets differ from bp_layout(); call bp_layout first");
    const auto t2 = std::chrono::steady_clock::now();
    if (timing)
        fprintf(stderr, "prepare: build_batch %.2f ms, offset check %.2f ms\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
    return prepare_built(c, B, nq, details, st);
}

// The device layout, arena and pinned staging of a batch whose host build
// (B->hb) is done.
int prepare_built(bp_ctx* c, bp_batch* B, int nq, int details, cudaStream_t) {
    static const bool timing = getenv("BP_HOST_TIMING") != nullptr;
    const HostBatch& hb = B->hb;
    const auto t2 = std::chrono::steady_clock::now();
    // candidate and stage-slot indices are int32 in the kernels' work lists
    if (hb.ncand >= INT32_MAX || hb.nstage >= ((int64_t)1 << 40))
        return fail(c, BP_BAD_INPUT, "batch too large (" + std::to_string(hb.ncand) +
                                         " candidates; at most 2^31 - 1 per batch: split it)");
    B->nq = nq;
    B->gen = c->gen;
    B->details = details != 0;
    const size_t nqs = (size_t)nq, nc = (size_t)hb.ncand, ns = (size_t)hb.nstage, nqst = (size_t)hb.nqstage,
                 nms = (size_t)hb.nmslot;
    Layout L;
    // inputs (one H2D copy): QDesc, Mpool, dp_count
    size_t o_q = L.take<QDesc>(nqs);
    size_t o_M = L.take<int64_t>(hb.Mpool.size());
    size_t o_cnt = L.take<int32_t>(4);
    size_t in_end = L.off;
    // DP items and the scheduling orders (built on the device, k_sched_*)
    size_t o_items = L.take<DPItem>(nqs + nms);
    size_t o_qord = L.take<int32_t>(nqs);
    size_t o_cperm = L.take<int32_t>(nc);
    const size_t otemp_bytes = sched_temp_bytes(std::max(1, nq));
    size_t o_okey = L.take<unsigned long long>(nqs), o_okey2 = L.take<unsigned long long>(nqs);
    size_t o_oval = L.take<int32_t>(nqs), o_ocnt = L.take<int32_t>(nqs), o_ocoff = L.take<int32_t>(nqs),
           o_owfl = L.take<int32_t>(nqs), o_owoff = L.take<int32_t>(nqs), o_otemp = L.take<char>(otemp_bytes);
    // outputs
    size_t o_res = L.take<bp_query_result>(nqs);
    size_t o_cand = L.take<bp_candidate>(nc);
    size_t o_st = L.take<bp_stage>(details ? ns : 0);
    // state
    size_t o_qs = L.take<QState>(nqs), o_ms = L.take<MState>(nms), o_cs = L.take<CState>(nc);
    size_t o_qlo = L.take<int32_t>(nqst), o_qhi = L.take<int32_t>(nqst);
    size_t o_ql = L.take<Rat>(nqst), o_qt = L.take<Rat>(nqst), o_qF = L.take<Rat>(nqst), o_qB = L.take<Rat>(nqst),
           o_qW = L.take<Rat>(nqst), o_qT = L.take<Rat>(nqst);
    size_t o_qd = L.take<uint8_t>(nqst);
    size_t o_clo = L.take<int32_t>(ns), o_chi = L.take<int32_t>(ns);
    size_t o_sF = L.take<Rat>(ns), o_sB = L.take<Rat>(ns), o_sW = L.take<Rat>(ns), o_sM = L.take<Rat>(ns),
           o_sM0 = L.take<Rat>(ns);
    size_t o_sA = L.take<int64_t>(ns), o_sSR = L.take<int64_t>(ns);
    size_t o_sim = L.take<char>(sim_exact_state_bytes(c->sm_count, std::max(1, hb.max_N)));
    size_t o_xkey = L.take<int32_t>(nc), o_xsorted = L.take<int32_t>(nc), o_xhist = L.take<int32_t>(XBUCKETS + 1);
    size_t o_cq = L.take<int32_t>(nc), o_co = L.take<int32_t>(nc);
    size_t o_work = L.take<unsigned long long>(WORK_SLOTS);
    int32_t dtab = 1;
    while (dtab < 2 * std::max(1, nq)) dtab <<= 1;
    size_t o_qrep = L.take<int32_t>(nqs), o_dkey = L.take<unsigned long long>((size_t)dtab),
           o_drep = L.take<int32_t>((size_t)dtab);
    int32_t stab = 1;
    while (stab < 2 * std::max<int64_t>(1, hb.ncand)) stab <<= 1;
    size_t o_skey = L.take<unsigned long long>((size_t)stab), o_srep = L.take<int32_t>((size_t)stab);
    size_t o_rlist = L.take<int32_t>(2 * nqs), o_rcount = L.take<int32_t>(4);
    size_t o_plist = L.take<int32_t>(nc), o_pctr = L.take<int32_t>(3);
    size_t o_qseed = L.take<unsigned long long>(nqs), o_qinc = L.take<bp_rat>(nqs);
    size_t o_pkey = L.take<unsigned long long>((size_t)stab), o_pbest = L.take<unsigned long long>((size_t)stab);
    int32_t ctab = 1;
    while (ctab < 2 * std::max<int64_t>(1, (int64_t)nms)) ctab <<= 1;
    size_t o_ckey = L.take<unsigned long long>((size_t)ctab), o_crep = L.take<int32_t>((size_t)ctab);
    size_t o_slist = L.take<int32_t>((size_t)SIM_CLASSES * nc), o_scnt = L.take<int32_t>(2 * SIM_CLASSES);   // counts, then hand-out counters
    size_t o_ftmp = L.take<int32_t>(nc);
    const auto t3 = std::chrono::steady_clock::now();
    if (!B->mem.ensure(L.off + 256)) return fail(c, BP_OUT_OF_MEMORY, "cudaMalloc(batch)");
    if (timing)
        fprintf(stderr, "prepare: layout %.2f ms, device arena %.2f ms (%zu MB)\n",
                std::chrono::duration<double, std::milli>(t3 - t2).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t3).count(),
                L.off >> 20);
    void* b = B->mem.p;
    // stage the inputs in pinned memory and copy once
    if (!B->stage_in.ensure(in_end)) return fail(c, BP_OUT_OF_MEMORY, "cudaHostAlloc");
    char* h = (char*)B->stage_in.p;
    {   // in chunks on the host pool (the records were just written by its workers)
        const size_t CH = 8192;
        const QDesc* src = hb.q.data();
        host_parallel_for((int)((nqs + CH - 1) / CH), [&](int k) {
            const size_t a = (size_t)k * CH, n = std::min(CH, nqs - a);
            std::memcpy(h + o_q + a * sizeof(QDesc), src + a, n * sizeof(QDesc));
        });
    }
    if (!hb.Mpool.empty()) std::memcpy(h + o_M, hb.Mpool.data(), hb.Mpool.size() * 8);
    int32_t cnt[4] = {0, 0, 0, 0};   // [0] is set by k_sched_scatter, [1] by k_coarse_queue
    std::memcpy(h + o_cnt, cnt, sizeof(cnt));
    B->in_off = 0;
    B->in_bytes = in_end;
    B->res_off = o_res;
    B->cand_off = o_cand;
    B->stage_off = o_st;
    BatchDev& D = B->dev;
    D = BatchDev{};
    D.P = c->P;
    D.nq = nq;
    D.ncand = hb.ncand;
    D.q = dptr<QDesc>(b, o_q);
    D.Mpool = dptr<int64_t>(b, o_M);
    D.qs = dptr<QState>(b, o_qs);
    D.ms = dptr<MState>(b, o_ms);
    D.cs = dptr<CState>(b, o_cs);
    D.cand = dptr<bp_candidate>(b, o_cand);
    D.stages = details ? dptr<bp_stage>(b, o_st) : nullptr;
    D.res = dptr<bp_query_result>(b, o_res);
    D.qlo = dptr<int32_t>(b, o_qlo);
    D.qhi = dptr<int32_t>(b, o_qhi);
    D.qlead = dptr<Rat>(b, o_ql);
    D.qtrail = dptr<Rat>(b, o_qt);
    D.qF = dptr<Rat>(b, o_qF);
    D.qB = dptr<Rat>(b, o_qB);
    D.qW = dptr<Rat>(b, o_qW);
    D.qT = dptr<Rat>(b, o_qT);
    D.qdirty = dptr<uint8_t>(b, o_qd);
    D.clo = dptr<int32_t>(b, o_clo);
    D.chi = dptr<int32_t>(b, o_chi);
    D.sF = dptr<Rat>(b, o_sF);
    D.sB = dptr<Rat>(b, o_sB);
    D.sW = dptr<Rat>(b, o_sW);
    D.sMem = dptr<Rat>(b, o_sM);
    D.sMem0 = dptr<Rat>(b, o_sM0);
    D.sA = dptr<int64_t>(b, o_sA);
    D.sSR = dptr<int64_t>(b, o_sSR);
    D.simbuf = dptr<Rat>(b, o_sim);
    D.xkey = dptr<int32_t>(b, o_xkey);
    D.xsorted = dptr<int32_t>(b, o_xsorted);
    D.xhist = dptr<int32_t>(b, o_xhist);
    D.max_N = std::max(1, hb.max_N);
    D.max_nbase = std::max(1, hb.max_nbase);
    D.cq = dptr<int32_t>(b, o_cq);
    D.corder = dptr<int32_t>(b, o_co);
    D.dp_items = dptr<DPItem>(b, o_items);
    D.dp_count = dptr<int32_t>(b, o_cnt);
    D.work = dptr<unsigned long long>(b, o_work);
    D.qrep = dptr<int32_t>(b, o_qrep);
    D.dkey = dptr<unsigned long long>(b, o_dkey);
    D.drep = dptr<int32_t>(b, o_drep);
    D.dmask = dtab - 1;
    D.skey = dptr<unsigned long long>(b, o_skey);
    D.srep = dptr<int32_t>(b, o_srep);
    D.smask = stab - 1;
    D.ckey = dptr<unsigned long long>(b, o_ckey);
    D.crep = dptr<int32_t>(b, o_crep);
    D.cmask = ctab - 1;
    D.rlist = dptr<int32_t>(b, o_rlist);
    D.rcount = dptr<int32_t>(b, o_rcount);
    D.plist = dptr<int32_t>(b, o_plist);
    D.qseed = dptr<unsigned long long>(b, o_qseed);
    D.qinc = dptr<bp_rat>(b, o_qinc);
    D.pctr = dptr<int32_t>(b, o_pctr);
    D.pkey = dptr<unsigned long long>(b, o_pkey);
    D.pbest = dptr<unsigned long long>(b, o_pbest);
    D.pmask = stab - 1;
    D.qorder = dptr<int32_t>(b, o_qord);
    D.cperm = dptr<int32_t>(b, o_cperm);
    D.okey = dptr<unsigned long long>(b, o_okey);
    D.okey2 = dptr<unsigned long long>(b, o_okey2);
    D.oval = dptr<int32_t>(b, o_oval);
    D.ocnt = dptr<int32_t>(b, o_ocnt);
    D.ocoff = dptr<int32_t>(b, o_ocoff);
    D.owfl = dptr<int32_t>(b, o_owfl);
    D.owoff = dptr<int32_t>(b, o_owoff);
    D.otemp = dptr<char>(b, o_otemp);
    D.otemp_bytes = otemp_bytes;
    D.sim_list = dptr<int32_t>(b, o_slist);
    D.sim_count = dptr<int32_t>(b, o_scnt);
    D.flow_tmp = dptr<int32_t>(b, o_ftmp);
    D.details = details ? 1 : 0;
    // DP launch geometry: blocks resident per SM bounded by shared memory
    int max_units = std::max(1, c->hn.max_L);
    size_t smem = partition_smem_bytes(max_units, std::max(1, hb.max_N), c->max_T);
    if (smem > c->smem_optin)
        return fail(c, BP_BAD_INPUT, "network too large for the shared-memory DP (L=" + std::to_string(max_units) + ")");
    int per_sm = (int)std::max<size_t>(1, (size_t)(200 * 1024) / (smem + 1024));
    if (per_sm > 8) per_sm = 8;
    B->dp_grid = c->sm_count * per_sm;
    B->dp_max_units = max_units;
    B->refine_grid = refine_setup(std::max(1, hb.max_N), max_units, c->max_T, &B->refine_bytes, &B->refine_warps);
    return BP_OK;
}

int upload_inputs(bp_ctx* c, bp_batch* B, cudaStream_t st) {
    cudaError_t e = cudaMemcpyAsync(B->mem.p, B->stage_in.p, B->in_bytes, cudaMemcpyHostToDevice, st);
    c->h2d += (int64_t)B->in_bytes;
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D batch inputs");
    return BP_OK;
}

// the batch's own side and refine streams and their fork / join events
void ensure_streams(bp_batch* B) {
    if (B->side) return;
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&B->side, cudaStreamNonBlocking, B->prio);
    cudaStreamCreateWithPriority(&B->rstream, cudaStreamNonBlocking, greatest);
    if (!B->fork) cudaEventCreateWithFlags(&B->fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&B->join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&B->rjoin, cudaEventDisableTiming);
}

void set_run_flags(bp_ctx* c, BatchDev& D) {
    D.dedup = c->dedup ? 1 : 0;
    D.plan_only = c->plan_only ? 1 : 0;
    D.prune_lb = c->prune_lb && !c->plan_only ? 1 : 0;
}

int run(bp_ctx* c, bp_batch* B, cudaStream_t st) {
    BatchDev& D = B->dev;
    const HostBatch& hb = B->hb;
    set_run_flags(c, D);
    cudaError_t e;
    e = cudaMemsetAsync(D.cand, 0, (size_t)hb.ncand * sizeof(bp_candidate), st);
    if (e == cudaSuccess && D.stages) e = cudaMemsetAsync(D.stages, 0, (size_t)hb.nstage * sizeof(bp_stage), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(D.dp_count + 1, 0, 3 * sizeof(int32_t), st);   // [1], hand-out [2..3]
    if (e == cudaSuccess) e = cudaMemsetAsync(D.work, 0, WORK_SLOTS * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(c, e, "memset");
    const int T = c->max_T, maxN = std::max(1, hb.max_N);
    timed(c, "setup", st, [&] { launch_setup(D, st); });
    timed(c, "dedup", st, [&] { launch_dedup(D, st); }, 2);
    // 3 own kernels (+ CUB's radix sort / scans, library code, not counted);
    // after dedup: the DP item list holds class representatives only
    timed(c, "sched", st, [&] { launch_sched(D, st); }, 3);
    if (!hb.whole_items.empty()) {
        timed(c, "minmax_dp", st, [&] {
            launch_partition(D, 0, std::min<int>(B->dp_grid, (int)hb.whole_items.size()), B->dp_max_units, maxN, T,
                             st);
        });
        timed(c, "dedup_copy", st, [&] { launch_dedup_copy_dp(D, st); });
    }
    timed(c, "bottleneck", st, [&] { launch_bottleneck(D, st); }, 2);
    // fork: coarse DPs (side stream) || refine (main stream); both only read
    // the whole-layer DP results and write disjoint state
    ensure_streams(B);
    launch_prune_reset(D, st);
    cudaEvent_t ph = phase_begin(c, st);
    const bool general_refine = refine_region_bytes(maxN) > 200 * 1024 || !D.dedup;
    timed(c, "refine_list", st, [&] { launch_refine_list(D, B->refine_grid, st); }, general_refine ? 0 : 1);
    // fork: refine (its own stream at the greatest priority: the walks are
    // the step's critical path, and their blocks must reach the SMs before
    // the coarse DPs' or another part's fill them) || the coarse DPs (side
    // stream); both only read the whole-layer DP results and write disjoint state
    cudaEventRecord(B->fork, st);
    cudaStreamWaitEvent(B->rstream, B->fork, 0);
    cudaStreamWaitEvent(B->side, B->fork, 0);
    const int refine_launches = general_refine || !B->refine_grid ? 1 : 2;
    timed(c, "refine", B->rstream, [&] {
        launch_refine(D, c->sm_count, B->refine_grid, B->refine_warps, B->refine_bytes, B->dp_max_units, T,
                      B->rstream);
    }, refine_launches);
    timed(c, "dedup_copy", B->rstream, [&] { launch_dedup_copy_refine(D, B->rstream); });
    cudaEventRecord(B->rjoin, B->rstream);
    if (hb.nmslot > 0) {
        timed(c, "minmax_dp_coarse", B->side,
              [&] { launch_partition(D, 1, B->dp_grid, B->dp_max_units, maxN, T, B->side); });
        timed(c, "dedup_copy", B->side, [&] { launch_coarse_copy(D, B->side); });
    }
    cudaEventRecord(B->join, B->side);
    cudaStreamWaitEvent(st, B->rjoin, 0);
    cudaStreamWaitEvent(st, B->join, 0);
    // (pruning the coarse-path candidates on the side stream while refine runs,
    // launch_prune(D, 0, side), was measured no faster overall: refine's
    // single-lane walks slow down by as much as the overlap saves; running
    // the coarse DPs before refine instead of beside it was ~1 ms slower)
    phase_end(c, "phase_refine", st, ph);   // coarse DP beside refine, up to the join
    ph = phase_begin(c, st);
    timed(c, "prune_list", st, [&] { launch_prune(D, -1, st, 1); }, 2);
    timed(c, "prune", st, [&] { launch_prune(D, -1, st, 2); });
    timed(c, "prune_members", st, [&] { launch_prune(D, -1, st, 4); });
    timed(c, "prune_members_full", st, [&] { launch_prune(D, -1, st, 8); });
    if (D.plan_only) {   // `bapipe plan`: no simulation
        timed(c, "plan_finish", st, [&] { launch_plan_finish(D, st); });
        timed(c, "rank", st, [&] { launch_rank(D, st); });
        e = cudaGetLastError();
        return e == cudaSuccess ? BP_OK : cuda_fail(c, e, "kernel launch");
    }
    phase_end(c, "phase_prune", st, ph);
    ph = phase_begin(c, st);
    timed(c, "sim_prep", st, [&] { launch_sim_prep(D, st); }, 4);
    if (D.prune_lb) {   // BP_OPT_PRUNE_LB round 1: bounds, one seed per query
        timed(c, "lb_prune", st, [&] {
            launch_lb_bound(D, st);
            launch_lb_round1(D, st);
        }, 2);
    }
    static const char* fast_names[8] = {"sim_fast_g2", "sim_fast_g4", "sim_fast_g8", "sim_fast_g16",
                                        "sim_fast_g32", "sim_fast_g32s2", "sim_fast_g32s4", "sim_fast_g32s8"};
    // the simulator classes are independent: the two exact ones on the side
    // stream overlap the fast classes and the N <= 32 dataflow kernel, so
    // their latency tails overlap instead of adding up
    cudaEventRecord(B->fork, st);
    cudaStreamWaitEvent(B->side, B->fork, 0);
    timed(c, "sim_flow64", B->side, [&] { launch_sim_flow(D, 1, c->sm_count, B->side); });
    timed(c, "sim_exact", B->side, [&] { launch_sim_exact(D, c->sm_count, B->side); }, 4);
    cudaEventRecord(B->join, B->side);
    // the long dataflow kernel first, the short scaled-integer classes after
    // it: the phase ends on short kernels (LPT over the launches)
    timed(c, "sim_flow32", st, [&] { launch_sim_flow(D, 0, c->sm_count, st); });
    for (int k = 0; k < 8; ++k) timed(c, fast_names[k], st, [&] { launch_sim_fast(D, k, c->sm_count, st); });
    cudaStreamWaitEvent(st, B->join, 0);
    timed(c, "sim_share", st, [&] { launch_sim_share(D, st); });
    if (D.prune_lb) {   // round 2: the candidates whose bound does not exceed their query's best
        timed(c, "lb_prune", st, [&] { launch_lb_round2(D, st); }, 2);
        for (int k = 0; k < 8; ++k) timed(c, fast_names[k], st, [&] { launch_sim_fast(D, k, c->sm_count, st); });
        timed(c, "lb_prune", st, [&] { launch_lb_finish(D, st); });
    }
    phase_end(c, "phase_sims", st, ph);
    timed(c, "rank", st, [&] { launch_rank(D, st); });
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "kernel launch");
    return BP_OK;
}

// A batch's kernel sequence as a CUDA graph: captured on the first run (on
// the batch's own lane stream, with its side and refine streams forked and
// joined inside), replayed by every later run whose launch inputs are the
// same -- the device tables and arena (BatchDev, by value in every kernel
// node), and the host-side sizes run() decides launches on.  One graph launch
// replaces ~45 kernel launches: the parts of a split batch start together,
// and bp_explore_batch's second part is not held back by the first part's
// launch calls.  Profiling runs launch kernel by kernel (events per launch).
struct GraphKey {
    BatchDev dev;
    int64_t whole_items, nmslot;
    int refine_grid, refine_warps, dp_grid, dp_max_units, max_T, sm_count;
    size_t refine_bytes;
};

GraphKey graph_key(bp_ctx* c, bp_batch* B) {
    GraphKey k;
    std::memset(&k, 0, sizeof(k));
    std::memcpy(&k.dev, &B->dev, sizeof(BatchDev));
    k.whole_items = (int64_t)B->hb.whole_items.size();
    k.nmslot = B->hb.nmslot;
    k.refine_grid = B->refine_grid;
    k.refine_warps = B->refine_warps;
    k.refine_bytes = B->refine_bytes;
    k.dp_grid = B->dp_grid;
    k.dp_max_units = B->dp_max_units;
    k.max_T = c->max_T;
    k.sm_count = c->sm_count;
    return k;
}

int run_graph(bp_ctx* c, bp_batch* B, cudaStream_t st) {
    static const bool off = getenv("BP_NO_GRAPHS") != nullptr;
    cudaStreamWaitEvent(st, c->tables_ev, 0);   // the device tables are uploaded
    if (c->prof || off || B->graph_failed) return run(c, B, st);
    set_run_flags(c, B->dev);
    ensure_streams(B);
    if (!B->lane) {
        cudaStreamCreateWithPriority(&B->lane, cudaStreamNonBlocking, B->prio);
        cudaEventCreateWithFlags(&B->done, cudaEventDisableTiming);
    }
    if (!B->gfork) cudaEventCreateWithFlags(&B->gfork, cudaEventDisableTiming);
    cudaStream_t lane = B->lane;
    const GraphKey key = graph_key(c, B);
    if (!B->gexec || std::memcmp(&key, B->gkey.data(), sizeof(key)) != 0) {
        if (B->gexec) cudaGraphExecDestroy(B->gexec);
        B->gexec = nullptr;
        const int64_t l0 = c->launches;
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamBeginCapture(lane, cudaStreamCaptureModeThreadLocal);
        int rc = e == cudaSuccess ? run(c, B, lane) : BP_CUDA_ERROR;
        const cudaError_t e2 = e == cudaSuccess ? cudaStreamEndCapture(lane, &g) : e;
        if (rc != BP_OK || e2 != cudaSuccess || cudaGraphInstantiate(&B->gexec, g, 0) != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            B->gexec = nullptr;
            cudaGetLastError();
            c->launches = l0;
            B->graph_failed = true;   // launch this batch kernel by kernel from now on
            return run(c, B, st);
        }
        cudaGraphDestroy(g);
        B->glaunches = c->launches - l0;
        c->launches = l0;
        B->gkey.assign((const char*)&key, (const char*)&key + sizeof(key));
    }
    if (st != lane) {
        cudaEventRecord(B->gfork, st);
        cudaStreamWaitEvent(lane, B->gfork, 0);
    }
    cudaError_t e = cudaGraphLaunch(B->gexec, lane);
    if (e != cudaSuccess) return cuda_fail(c, e, "graph launch");
    c->launches += B->glaunches;
    if (st != lane) {
        cudaEventRecord(B->done, lane);
        cudaStreamWaitEvent(st, B->done, 0);
    }
    return BP_OK;
}

int fetch(bp_ctx* c, bp_batch* B, bp_query_result* res, bp_candidate* cand, bp_stage* stages, cudaStream_t st) {
    const HostBatch& hb = B->hb;
    cudaError_t e = cudaSuccess;
    if (res) e = cudaMemcpyAsync(res, B->dev.res, (size_t)B->nq * sizeof(bp_query_result), cudaMemcpyDeviceToHost, st);
    if (res) c->d2h += (int64_t)B->nq * (int64_t)sizeof(bp_query_result);
    if (cand) c->d2h += hb.ncand * (int64_t)sizeof(bp_candidate);
    if (stages && B->dev.stages) c->d2h += hb.nstage * (int64_t)sizeof(bp_stage);
    if (e == cudaSuccess && cand && hb.ncand)
        e = cudaMemcpyAsync(cand, B->dev.cand, (size_t)hb.ncand * sizeof(bp_candidate), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && stages && B->dev.stages && hb.nstage)
        e = cudaMemcpyAsync(stages, B->dev.stages, (size_t)hb.nstage * sizeof(bp_stage), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(c, e, "fetch");
    if (c->prof) {
        // algorithmic work of the most recent run (per launch, not summed):
        // DP transitions of each partition launch, simulated events per class
        unsigned long long work[WORK_SLOTS];
        static const char* names[SIM_CLASSES] = {"sim_fast_g2", "sim_fast_g4", "sim_fast_g8", "sim_fast_g16",
                                                 "sim_fast_g32", "sim_fast_g32s2", "sim_fast_g32s4",
                                                 "sim_fast_g32s8", "sim_exact", "sim_flow32", "sim_flow64"};
        if (cudaMemcpy(work, B->dev.work, sizeof(work), cudaMemcpyDeviceToHost) == cudaSuccess) {
            // a split batch's parts add up (the critical paths take the maximum)
            auto put = [&](const char* k, unsigned long long v, bool is_max = false) {
                double& w = c->stats[k].work;
                w = !c->stats_accumulate ? (double)v : is_max ? std::max(w, (double)v) : w + (double)v;
            };
            put("minmax_dp", work[WORK_DP_WHOLE]);
            put("minmax_dp_coarse", work[WORK_DP_COARSE]);
            put("refine", work[WORK_REFINE]);
            put("refine_critical_path", work[WORK_REFINE_MAX], true);
            put("prune", work[WORK_PRUNE]);
            put("refine_moves", work[WORK_REFINE_MOVES]);
            put("refine_exact_steps", work[WORK_REFINE_EXACT]);
            put("prune_trials", work[WORK_PRUNE_TRIALS]);
            put("prune_critical_path", work[WORK_PRUNE_MAX], true);
            for (int k = 0; k < SIM_CLASSES; ++k) put(names[k], work[WORK_SIM_EVENTS + k]);
        }
        collect(c);
    }
    return BP_OK;
}


// ---- BP_OPT_SPLIT: a large batch runs as two parts, concurrently.
// The queries with the batch's largest stage count carry the longest
// intra_layer_refine walks (a serial chain per query: the refine launch lasts
// as long as its longest walk, with most SMs idle) and the largest
// simulations; run as their own batch on a second stream, the other queries'
// refine, prune and simulate phases overlap that walk.  Each part is a
// complete batch (its own dedup tables, lists and arena); results are
// identical to one batch (no result depends on the sharing, see
// BP_OPT_DEDUP), and the parts' outputs are scattered back into the caller's
// layout at fetch.
constexpr int SPLIT_MIN_QUERIES = 4096, SPLIT_MIN_PART = 512;

bool split_groups(const bp_ctx* c, const bp_query* q, int nq, std::vector<std::vector<int32_t>>& groups) {
    groups.clear();
    if (!c->split || c->plan_only || nq < SPLIT_MIN_QUERIES) return false;
    std::vector<int> n(nq);
    for (int i = 0; i < nq; ++i) {
        // a query the host build would reject: no split, so that the one-batch
        // path reports it with its own index
        if (q[i].cluster < 0 || q[i].cluster >= (int)c->hc.desc.size() || q[i].network < 0 ||
            q[i].network >= (int)c->hn.desc.size() || q[i].n_stages < 0 ||
            q[i].n_stages > c->hc.desc[q[i].cluster].N || (q[i].n_m > 0 && !q[i].m_list))
            return false;
        n[i] = q[i].n_stages > 0 ? q[i].n_stages : c->hc.desc[q[i].cluster].N;
    }
    // parts by stage count, largest first: the largest N, then (three parts)
    // the next largest, then the rest; a part too small to pay is merged into
    // the rest
    const int want = c->split;
    std::vector<int> levels;   // the stage counts that get their own part
    {
        std::vector<int> sorted(n);
        std::sort(sorted.begin(), sorted.end(), std::greater<int>());
        sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
        for (int v : sorted) {
            if ((int)levels.size() + 1 >= want) break;
            const int cnt = (int)std::count(n.begin(), n.end(), v);
            if (cnt < SPLIT_MIN_PART) break;
            levels.push_back(v);
        }
    }
    if (levels.empty()) return false;
    groups.assign(levels.size() + 1, {});
    for (int i = 0; i < nq; ++i) {
        size_t k = 0;
        while (k < levels.size() && n[i] != levels[k]) ++k;
        groups[k].push_back(i);
    }
    while (groups.size() > 1 && (int)groups.back().size() < SPLIT_MIN_PART) {
        // the rest is too small: fold it into the last level's part
        std::vector<int32_t> r = std::move(groups.back());
        groups.pop_back();
        if (groups.size() == 1) return false;
        groups.back().insert(groups.back().end(), r.begin(), r.end());
        std::sort(groups.back().begin(), groups.back().end());
    }
    return groups.size() >= 2;
}

// A part's streams: the first part (the largest stage count: the longest
// refine walks and simulations, the step's critical chain) at the highest
// priority, so that its kernels take the SMs first whenever they are ready and
// the other part's fill the gaps (its refine phase, its prune tail).
void make_part_lane(bp_batch* p, size_t k, size_t nparts) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);   // lo = least (0), hi = greatest (negative)
    p->prio = nparts <= 1 ? hi : hi + (int)((int64_t)(lo - hi) * (int64_t)k / (int64_t)(nparts - 1));
    cudaStreamCreateWithPriority(&p->lane, cudaStreamNonBlocking, p->prio);
    cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming);
}

// eager (bp_explore_batch): each part is uploaded and launched on its own
// stream as soon as its host build is done, so the first part's kernels (the
// long refine walks) run while the host builds the second.  *ran tells the
// caller that the batch ran.
int prepare_any(bp_ctx* c, bp_batch* B, const bp_query* q, int nq, int details, cudaStream_t st,
                bool eager = false, bool* ran = nullptr) {
    if (ran) *ran = false;
    std::vector<std::vector<int32_t>> groups;
    if (!split_groups(c, q, nq, groups)) {
        for (bp_batch* p : B->parts) bp_batch_free(c, p);
        B->parts.clear();
        return prepare(c, B, q, nq, details, st);
    }
    if (!c->have_nets || !c->have_cls) return fail(c, BP_BAD_INPUT, "networks/clusters not set");
    B->nq = nq;
    B->gen = c->gen;
    B->details = details != 0;
    while (B->parts.size() > groups.size()) {
        bp_batch_free(c, B->parts.back());
        B->parts.pop_back();
    }
    while (B->parts.size() < groups.size()) B->parts.push_back(new bp_batch());
    B->part_q = std::move(groups);
    B->part_ids_host.clear();
    if (eager) {
        if (!B->fork) cudaEventCreateWithFlags(&B->fork, cudaEventDisableTiming);
        cudaEventRecord(B->fork, st);
    }
    std::string err;
    static const bool timing = getenv("BP_HOST_TIMING") != nullptr;   // diagnostics (stderr)
    const auto t0 = std::chrono::steady_clock::now();
    auto since = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    for (size_t k = 0; k < B->parts.size(); ++k) {
        // the part's host build, on its own queries (its own dense layout)
        const std::vector<int32_t>& idx = B->part_q[k];
        const int32_t* ix = idx.data();
        bp_batch* p = B->parts[k];
        if (!build_batch_at([q, ix](int j) -> const bp_query& { return q[ix[j]]; }, (int)idx.size(), c->hn, c->hc,
                            p->hb, err))
            return fail(c, BP_BAD_INPUT, err);
        const double tb = since();
        int rc = prepare_built(c, p, (int)idx.size(), details, st);
        if (rc != BP_OK) return rc;
        if (timing) fprintf(stderr, "split part %zu (%zu queries): built %.2f ms, prepared %.2f ms\n", k, idx.size(), tb, since());
        if (eager) {
            if (!p->lane) make_part_lane(p, k, B->parts.size());
            cudaStreamWaitEvent(p->lane, B->fork, 0);
            if ((rc = upload_inputs(c, p, p->lane)) != BP_OK || (rc = run_graph(c, p, p->lane)) != BP_OK) return rc;
            cudaEventRecord(p->done, p->lane);
            cudaStreamWaitEvent(st, p->done, 0);
            if (timing) fprintf(stderr, "split part %zu launched %.2f ms\n", k, since());
        }
    }
    if (eager) note_run(c, st);
    for (size_t k = 0; k < B->parts.size(); ++k)
        for (int32_t i : B->part_q[k]) B->part_ids_host.push_back(i);
    // the whole batch's layout, in the caller's query order, from the parts'
    // builds: the caller's offsets must be bp_layout's, and fetch scatters
    // the parts' records to them
    HostBatch& hb = B->hb;
    hb.q.resize(nq);
    for (size_t k = 0; k < B->parts.size(); ++k)
        for (size_t j = 0; j < B->part_q[k].size(); ++j) hb.q[B->part_q[k][j]] = B->parts[k]->hb.q[j];
    hb.ncand = hb.nstage = 0;
    for (int i = 0; i < nq; ++i) {
        QDesc& d = hb.q[i];
        d.cand_off = hb.ncand;
        d.stage_off = hb.nstage;
        hb.ncand += 2 * (int64_t)d.nbase;
        hb.nstage += 2 * (int64_t)d.nbase * d.N;
        if (q[i].cand_offset != d.cand_off || q[i].stage_offset != d.stage_off)
            return fail(c, BP_BAD_INPUT, "query offsets differ from bp_layout(); call bp_layout first");
    }
    // per part query (parts concatenated): its parent index, then the offsets
    // of its candidate and stage records in the caller's layout
    const size_t npq = B->part_ids_host.size(), idb = npq * sizeof(int64_t);
    if (!B->part_ids.ensure(idb) || !B->part_woff.ensure(2 * idb) ||
        !B->part_best.ensure(B->parts.size() * sizeof(bp_best_record)) || !B->stage_in.ensure(3 * idb))
        return fail(c, BP_OUT_OF_MEMORY, "cudaMalloc(split)");
    std::memcpy(B->stage_in.p, B->part_ids_host.data(), idb);
    int64_t* wo = reinterpret_cast<int64_t*>(static_cast<char*>(B->stage_in.p) + idb);
    for (size_t j = 0; j < npq; ++j) {
        const QDesc& d = hb.q[B->part_ids_host[j]];
        wo[2 * j] = d.cand_off;
        wo[2 * j + 1] = d.stage_off;
    }
    B->in_bytes = 3 * idb;   // upload_any copies them with the parts' inputs
    if (eager) {
        cudaError_t e = cudaMemcpyAsync(B->part_ids.p, B->stage_in.p, idb, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(B->part_woff.p, wo, 2 * idb, cudaMemcpyHostToDevice, st);
        c->h2d += (int64_t)(3 * idb);
        if (e != cudaSuccess) return cuda_fail(c, e, "H2D split ids");
        if (ran) *ran = true;
    }
    return BP_OK;
}

int upload_any(bp_ctx* c, bp_batch* B, cudaStream_t st) {
    if (B->parts.empty()) return upload_inputs(c, B, st);
    const size_t idb = B->in_bytes / 3;
    cudaError_t e = cudaMemcpyAsync(B->part_ids.p, B->stage_in.p, idb, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(B->part_woff.p, static_cast<char*>(B->stage_in.p) + idb, 2 * idb, cudaMemcpyHostToDevice, st);
    c->h2d += (int64_t)B->in_bytes;
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D split ids");
    for (bp_batch* p : B->parts)
        if (const int rc = upload_inputs(c, p, st); rc != BP_OK) return rc;
    return BP_OK;
}

int run_any(bp_ctx* c, bp_batch* B, cudaStream_t st) {
    if (B->parts.empty()) {
        const int rc = run_graph(c, B, st);
        if (rc == BP_OK) note_run(c, st);
        return rc;
    }
    if (!B->fork) cudaEventCreateWithFlags(&B->fork, cudaEventDisableTiming);
    cudaEventRecord(B->fork, st);
    for (size_t k = 0; k < B->parts.size(); ++k) {
        bp_batch* p = B->parts[k];
        if (!p->lane) make_part_lane(p, k, B->parts.size());
        cudaStreamWaitEvent(p->lane, B->fork, 0);
        if (const int rc = run_graph(c, p, p->lane); rc != BP_OK) return rc;
        cudaEventRecord(p->done, p->lane);
        cudaStreamWaitEvent(st, p->done, 0);
    }
    note_run(c, st);
    return BP_OK;
}

int fetch_any(bp_ctx* c, bp_batch* B, bp_query_result* res, bp_candidate* cand, bp_stage* stages, cudaStream_t st) {
    if (B->parts.empty()) return fetch(c, B, res, cand, stages, st);
    // query results: scattered into the caller's order on the device (part_ids),
    // then one D2H straight into the caller's buffer
    if (res) {
        const size_t bytes = (size_t)B->nq * sizeof(bp_query_result);
        if (!B->res_all.ensure(bytes)) return fail(c, BP_OUT_OF_MEMORY, "cudaMalloc(split results)");
        const int64_t* ids = (const int64_t*)B->part_ids.p;
        for (size_t k = 0; k < B->parts.size(); ++k) {
            launch_scatter_results(B->parts[k]->dev.res, B->parts[k]->nq, ids, (bp_query_result*)B->res_all.p, st);
            ids += B->part_q[k].size();
        }
        c->launches += (int64_t)B->parts.size();
        const cudaError_t e = cudaMemcpyAsync(res, B->res_all.p, bytes, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return cuda_fail(c, e, "fetch");
        c->d2h += (int64_t)bytes;
    }
    // candidate / stage records (details): scattered on the device into the
    // caller's layout (part_woff), then one D2H each
    const HostBatch& wh = B->hb;
    const bool want_st = stages && B->details;
    if (cand || want_st) {
        if ((cand && !B->cand_all.ensure((size_t)wh.ncand * sizeof(bp_candidate))) ||
            (want_st && !B->stage_all.ensure((size_t)wh.nstage * sizeof(bp_stage))))
            return fail(c, BP_OUT_OF_MEMORY, "cudaMalloc(split records)");
        const int64_t* wo = (const int64_t*)B->part_woff.p;
        for (size_t k = 0; k < B->parts.size(); ++k) {
            launch_scatter_records(B->parts[k]->dev, wo, cand ? (bp_candidate*)B->cand_all.p : nullptr,
                                   want_st ? (bp_stage*)B->stage_all.p : nullptr, st);
            wo += 2 * B->part_q[k].size();
        }
        c->launches += (int64_t)B->parts.size();
        cudaError_t e = cudaSuccess;
        if (cand && wh.ncand)
            e = cudaMemcpyAsync(cand, B->cand_all.p, (size_t)wh.ncand * sizeof(bp_candidate), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && want_st && wh.nstage)
            e = cudaMemcpyAsync(stages, B->stage_all.p, (size_t)wh.nstage * sizeof(bp_stage), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return cuda_fail(c, e, "fetch");
        if (cand) c->d2h += wh.ncand * (int64_t)sizeof(bp_candidate);
        if (want_st) c->d2h += wh.nstage * (int64_t)sizeof(bp_stage);
    }
    // each part's fetch: waits, and collects its profile
    c->stats_accumulate = false;
    for (size_t k = 0; k < B->parts.size(); ++k) {
        const int rc = fetch(c, B->parts[k], nullptr, nullptr, nullptr, st);
        c->stats_accumulate = true;
        if (rc != BP_OK) { c->stats_accumulate = false; return rc; }
    }
    c->stats_accumulate = false;
    return BP_OK;
}

int best_any(bp_ctx* c, bp_batch* B, void* dev_out, int64_t query_base, cudaStream_t st) {
    if (B->parts.empty()) {
        timed(c, "best", st, [&] { launch_best(B->dev, (bp_best_record*)dev_out, query_base, nullptr, st); });
    } else {
        const int64_t* ids = (const int64_t*)B->part_ids.p;
        bp_best_record* recs = (bp_best_record*)B->part_best.p;
        timed(c, "best", st, [&] {
            for (size_t k = 0; k < B->parts.size(); ++k) {
                launch_best(B->parts[k]->dev, recs + k, query_base, ids, st);
                ids += B->part_q[k].size();
            }
            launch_best_merge(recs, (int)B->parts.size(), (bp_best_record*)dev_out, st);
        }, (int)B->parts.size() + 1);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BP_OK : cuda_fail(c, e, "best");
}

}  // namespace

extern "C" {

int bp_abi_version(void) { return BP_ABI_VERSION; }

const char* bp_last_error(const bp_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

bp_ctx* bp_create(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        g_err = std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "count = 0");
        return nullptr;
    }
    if (device < 0 || device >= n) {
        g_err = "device index out of range";
        return nullptr;
    }
    cudaDeviceProp prop;
    if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        g_err = "cannot use device";
        return nullptr;
    }
    if (prop.major < 10) {
        g_err = "libbapipe_b200 is built for sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                std::to_string(prop.minor);
        return nullptr;
    }
    // the kernels with large dynamic shared memory may use up to the opt-in
    // limit on this device (a per-device function attribute, set once here:
    // lowering it per batch would race with other contexts' launches)
    if (const cudaError_t ke = kernel_attributes_init((int)prop.sharedMemPerBlockOptin); ke != cudaSuccess) {
        g_err = std::string("cannot set kernel attributes: ") + cudaGetErrorString(ke);
        return nullptr;
    }
    refine_trace_collect();   // diagnostics (BP_REFINE_TRACE): allocates the trace buffer
    bp_ctx* c = new (std::nothrow) bp_ctx();
    if (!c) return nullptr;
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->tstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->tables_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->nets_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->cls_ev, cudaEventDisableTiming) != cudaSuccess) {
        g_err = "cannot create the table upload stream";
        delete c;
        return nullptr;
    }
    c->smem_optin = (size_t)prop.sharedMemPerBlockOptin;
    return c;
}

void bp_destroy(bp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->cached) bp_batch_free(c, c->cached);
    c->nets_mem.release();
    c->cls_mem.release();
    c->stage_tables.release();
    c->stage_cls.release();
    if (c->tstream) cudaStreamDestroy(c->tstream);
    for (cudaEvent_t ev : {c->tables_ev, c->nets_ev, c->cls_ev, c->tl_base})
        if (ev) cudaEventDestroy(ev);
    for (auto e : c->event_pool) cudaEventDestroy(e);
    delete c;
}

int bp_set_networks(bp_ctx* c, const bp_network* nets, int n) {
    if (!c || (!nets && n > 0) || n < 0) return fail(c, BP_BAD_INPUT, "bad arguments");
    try {
        cudaSetDevice(c->device);
        std::string err;
        static const bool timing = getenv("BP_HOST_TIMING") != nullptr;   // diagnostics (stderr)
        const auto t0 = std::chrono::steady_clock::now();
        // batches prepared before this call point at the old tables: they are
        // refused from now on (bp_batch_*: generation check), and whatever
        // run is still in flight finishes before the upload overwrites a table
        // (the upload waits for the runs on the device, tables_wait_runs)
        ++c->gen;
        c->have_nets = false;
        tables_wait_runs(c);
        if (!build_nets(nets, n, c->hn, err, false)) return fail(c, BP_BAD_INPUT, err);
        const auto t1 = std::chrono::steady_clock::now();
        int rc = upload_networks(c);
        c->have_nets = rc == BP_OK;
        if (timing) {
            const auto t2 = std::chrono::steady_clock::now();
            fprintf(stderr, "bp_set_networks: build %.2f ms, upload + prefix %.2f ms\n",
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count());
        }
        return rc;
    } catch (const std::bad_alloc&) {
        return fail(c, BP_OUT_OF_MEMORY, "host allocation failed");
    }
}

int bp_set_clusters(bp_ctx* c, const bp_cluster* cls, int n) {
    if (!c || (!cls && n > 0) || n < 0) return fail(c, BP_BAD_INPUT, "bad arguments");
    try {
        cudaSetDevice(c->device);
        std::string err;
        ++c->gen;
        c->have_cls = false;
        tables_wait_runs(c);
        if (!build_clusters(cls, n, c->hc, err)) return fail(c, BP_BAD_INPUT, err);
        int rc = upload_clusters(c);
        c->have_cls = rc == BP_OK;
        return rc;
    } catch (const std::bad_alloc&) {
        return fail(c, BP_OUT_OF_MEMORY, "host allocation failed");
    }
}

int bp_layout(bp_ctx* c, bp_query* q, int nq, int64_t* total_candidates, int64_t* total_stages) {
    if (!c || (!q && nq > 0) || nq < 0) return fail(c, BP_BAD_INPUT, "bad arguments");
    try {
        HostBatch hb;
        std::string err;
        if (!build_batch(q, nq, c->hn, c->hc, hb, err)) return fail(c, BP_BAD_INPUT, err);
        for (int i = 0; i < nq; ++i) {
            q[i].cand_offset = hb.q[i].cand_off;
            q[i].stage_offset = hb.q[i].stage_off;
        }
        if (total_candidates) *total_candidates = hb.ncand;
        if (total_stages) *total_stages = hb.nstage;
        return BP_OK;
    } catch (const std::bad_alloc&) {
        return fail(c, BP_OUT_OF_MEMORY, "host allocation failed");
    }
}

bp_batch* bp_batch_prepare(bp_ctx* c, const bp_query* q, int nq, int want_details, void* stream) {
    if (!c || (!q && nq > 0) || nq < 0) { fail(c, BP_BAD_INPUT, "bad arguments"); return nullptr; }
    try {
        cudaSetDevice(c->device);
        bp_batch* B = new bp_batch();
        cudaStream_t st = (cudaStream_t)stream;
        if (prepare_any(c, B, q, nq, want_details, st) != BP_OK || upload_any(c, B, st) != BP_OK) {
            bp_batch_free(c, B);
            return nullptr;
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) {
            bp_batch_free(c, B);
            fail(c, BP_CUDA_ERROR, "prepare sync");
            return nullptr;
        }
        return B;
    } catch (const std::bad_alloc&) {
        fail(c, BP_OUT_OF_MEMORY, "host allocation failed");
        return nullptr;
    }
}

static bool stale(const bp_ctx* c, const bp_batch* B) { return B->gen != c->gen; }
static const char* STALE = "batch prepared before the last bp_set_networks / bp_set_clusters: prepare it again";

static void mark_run_start(bp_ctx* c, cudaStream_t st) {
    if (!c->prof) return;
    if (!c->tl_base) cudaEventCreate(&c->tl_base);
    cudaEventRecord(c->tl_base, st);
}

int bp_batch_run(bp_ctx* c, bp_batch* B, void* stream) {
    if (!c || !B) return fail(c, BP_BAD_INPUT, "bad arguments");
    if (stale(c, B)) return fail(c, BP_BAD_INPUT, STALE);
    cudaSetDevice(c->device);
    mark_run_start(c, (cudaStream_t)stream);
    return run_any(c, B, (cudaStream_t)stream);
}

int bp_batch_fetch(bp_ctx* c, bp_batch* B, bp_query_result* res, bp_candidate* cand, bp_stage* stages,
                   void* stream) {
    if (!c || !B) return fail(c, BP_BAD_INPUT, "bad arguments");
    if (stale(c, B)) return fail(c, BP_BAD_INPUT, STALE);
    cudaSetDevice(c->device);
    return fetch_any(c, B, res, cand, stages, (cudaStream_t)stream);
}

int bp_batch_best(bp_ctx* c, bp_batch* B, void* dev_out, int64_t query_base, void* stream) {
    if (!c || !B || !dev_out) return fail(c, BP_BAD_INPUT, "bad arguments");
    if (stale(c, B)) return fail(c, BP_BAD_INPUT, STALE);
    cudaSetDevice(c->device);
    return best_any(c, B, dev_out, query_base, (cudaStream_t)stream);
}

void bp_batch_free(bp_ctx* c, bp_batch* B) {
    if (!B) return;
    if (c) cudaSetDevice(c->device);
    for (bp_batch* p : B->parts) bp_batch_free(c, p);
    B->mem.release();
    B->stage_in.release();
    B->part_ids.release();
    B->part_best.release();
    B->res_all.release();
    B->part_woff.release();
    B->cand_all.release();
    B->stage_all.release();
    if (B->side) cudaStreamDestroy(B->side);
    if (B->rstream) cudaStreamDestroy(B->rstream);
    if (B->lane) cudaStreamDestroy(B->lane);
    if (B->gexec) cudaGraphExecDestroy(B->gexec);
    for (cudaEvent_t ev : {B->fork, B->join, B->done, B->rjoin, B->gfork})
        if (ev) cudaEventDestroy(ev);
    delete B;
}

int bp_explore_batch(bp_ctx* c, const bp_query* q, int nq, bp_query_result* res, bp_candidate* cand,
                     bp_stage* stages, void* stream) {
    if (!c || (!q && nq > 0) || nq < 0 || !res) return fail(c, BP_BAD_INPUT, "bad arguments");
    try {
        cudaSetDevice(c->device);
        cudaStream_t st = (cudaStream_t)stream;
        if (!c->cached) c->cached = new bp_batch();
        bp_batch* B = c->cached;
        static const bool timing = getenv("BP_HOST_TIMING") != nullptr;   // diagnostics (stderr)
        auto now = [] { return std::chrono::steady_clock::now(); };
        const auto t0 = now();
        cudaEvent_t te0 = nullptr, te1 = nullptr;   // diagnostics: the call's span on the caller's stream
        if (timing) {
            cudaEventCreate(&te0);
            cudaEventCreate(&te1);
            cudaEventRecord(te0, st);
        }
        bool ran = false;
        mark_run_start(c, st);
        int rc = prepare_any(c, B, q, nq, stages != nullptr, st, true, &ran);
        const auto t1 = now();
        if (rc == BP_OK && !ran) rc = upload_any(c, B, st);
        if (rc == BP_OK && !ran) rc = run_any(c, B, st);
        const auto t2 = now();
        if (rc == BP_OK) rc = fetch_any(c, B, res, cand, stages, st);
        if (timing) {
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            cudaEventRecord(te1, st);
            cudaEventSynchronize(te1);
            float dev = 0;
            cudaEventElapsedTime(&dev, te0, te1);
            fprintf(stderr, "bp_explore_batch: prepare %.2f ms, launch %.2f ms, wait+fetch %.2f ms; caller-stream span %.2f ms\n",
                    ms(t0, t1), ms(t1, t2), ms(t2, now()), dev);
            cudaEventDestroy(te0);
            cudaEventDestroy(te1);
        }
        return rc;
    } catch (const std::bad_alloc&) {
        return fail(c, BP_OUT_OF_MEMORY, "host allocation failed");
    }
}

int64_t bp_launch_count(const bp_ctx* c) { return c ? c->launches : 0; }

int bp_set_profiling(bp_ctx* c, int enable) {
    if (!c) return BP_BAD_INPUT;
    c->prof = enable != 0;
    if (enable) c->stats.clear();
    return BP_OK;
}

int bp_set_option(bp_ctx* c, int option, int64_t value) {
    if (!c) return BP_BAD_INPUT;
    switch (option) {
        case BP_OPT_DEDUP: c->dedup = value != 0; return BP_OK;
        case BP_OPT_PLAN_ONLY: c->plan_only = value != 0; return BP_OK;
        case BP_OPT_PRUNE_LB: c->prune_lb = value != 0; return BP_OK;
        case BP_OPT_SPLIT: c->split = value <= 0 ? 0 : value == 1 ? 4 : (int)std::min<int64_t>(value, 8); return BP_OK;
        default: return fail(c, BP_BAD_INPUT, "unknown option " + std::to_string(option));
    }
}

static int plan_request_ok(bp_ctx* c, const bp_plan_request* q) {
    if (!c || !q) return fail(c, BP_BAD_INPUT, "null argument");
    if (!c->have_nets || !c->have_cls) return fail(c, BP_BAD_INPUT, "bp_set_networks / bp_set_clusters first");
    if (q->network < 0 || q->network >= (int)c->hn.desc.size() || q->cluster < 0 ||
        q->cluster >= (int)c->hc.desc.size())
        return fail(c, BP_BAD_INPUT, "network / cluster index out of range");
    if (q->n_stages < 1 || !q->lo || !q->hi || !q->lead || !q->trail)
        return fail(c, BP_BAD_INPUT, "plan with no stages");
    if (q->kind < 0 || q->kind > 3) return fail(c, BP_BAD_INPUT, "unknown schedule kind");
    for (int s = 0; s < q->n_stages; ++s)
        if (q->lead[s].den <= 0 || q->trail[s].den <= 0) return fail(c, BP_BAD_INPUT, "fraction with den <= 0");
    return BP_OK;
}

int bp_simulate_plan(bp_ctx* c, const bp_plan_request* q, bp_timeline_result* res, bp_event* events, int64_t cap,
                     bp_rat* highwater, bp_rat* weight_static, bp_rat* busy) {
    int rc = plan_request_ok(c, q);
    if (rc != BP_OK) return rc;
    if (!res) return fail(c, BP_BAD_INPUT, "null result");
    if (q->mini_batches < 1) return fail(c, BP_BAD_INPUT, "mini_batches >= 1 required");
    cudaEventSynchronize(c->tables_ev);
    const cudaError_t e = timeline_simulate(c->P, c->hc.desc[(size_t)q->cluster].N, *q, res, events, cap, highwater,
                                            weight_static, busy, &c->h2d, &c->d2h);
    c->launches += 2;
    if (e != cudaSuccess) return cuda_fail(c, e, "bp_simulate_plan");
    if (res->status == BP_C_OK && res->n_events > cap && events) return fail(c, BP_BAD_INPUT, "event capacity too small");
    return BP_OK;
}

int bp_estimate_plan(bp_ctx* c, const bp_plan_request* q, bp_estimate_result* res, bp_stage* stages,
                     int32_t* mem_infeasible) {
    int rc = plan_request_ok(c, q);
    if (rc != BP_OK) return rc;
    if (!res) return fail(c, BP_BAD_INPUT, "null result");
    if (q->n_stages > c->hc.desc[(size_t)q->cluster].N)
        return fail(c, BP_BAD_INPUT, "plan longer than the cluster");
    cudaEventSynchronize(c->tables_ev);
    const cudaError_t e = timeline_estimate(c->P, c->hc.desc[(size_t)q->cluster].N, *q, res, stages, mem_infeasible,
                                            &c->h2d, &c->d2h);
    c->launches += 1;
    if (e != cudaSuccess) return cuda_fail(c, e, "bp_estimate_plan");
    return BP_OK;
}

int bp_kernel_stats(const bp_ctx* c, char* names48, double* ms, int64_t* launches, double* work, int cap) {
    if (!c) return 0;
    int i = 0;
    for (auto& kv : c->stats) {
        if (i >= cap) break;
        if (names48) {
            std::memset(names48 + 48 * i, 0, 48);
            std::strncpy(names48 + 48 * i, kv.first.c_str(), 47);
        }
        if (ms) ms[i] = kv.second.ms;
        if (launches) launches[i] = kv.second.launches;
        if (work) work[i] = kv.second.work;
        ++i;
    }
    return i;
}

int bp_transfer_stats(const bp_ctx* c, int64_t* h2d, int64_t* d2h) {
    if (!c) return BP_BAD_INPUT;
    if (h2d) *h2d = c->h2d;
    if (d2h) *d2h = c->d2h;
    return BP_OK;
}

int bp_best_less(const bp_best_record* a, const bp_best_record* b) {
    if (a->valid != b->valid) return a->valid > b->valid;
    if (!a->valid) return a->query_id < b->query_id;
    auto lt = [](bp_rat x, bp_rat y) { return (__int128)x.num * y.den < (__int128)y.num * x.den; };
    auto eq = [](bp_rat x, bp_rat y) { return x.num == y.num && x.den == y.den; };
    if (!eq(a->makespan, b->makespan)) return lt(a->makespan, b->makespan);
    if (!eq(a->peak_memory, b->peak_memory)) return lt(a->peak_memory, b->peak_memory);
    if (!eq(a->max_bw, b->max_bw)) return lt(a->max_bw, b->max_bw);
    if (a->M != b->M) return a->M < b->M;
    if (a->kind != b->kind) return a->kind < b->kind;
    return a->query_id < b->query_id;
}

}  // extern "C"
