// tests/emu/emu.cpp -- TEST HARNESS (never the product): runs the product's
// per-thread phase code (csrc/phases.cuh, compiled for the host) on the CPU,
// with a sequential mirror of the k_partition DP, behind the oracle-style
// batch entry point.  It lets tests/test_emu.py check the exact-emulation
// logic against the reference without a GPU; the product itself only ever
// runs these phases inside CUDA kernels (libbapipe_b200.so).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2012_12544_b200/csrc/host_prep.hpp"
#include "../../paper_2012_12544_b200/csrc/phases.cuh"
#include "../../paper_2012_12544_b200/csrc/refine_fast.cuh"
#include "../../paper_2012_12544_b200/csrc/timeline.cuh"

using namespace bpk;

#ifdef BPK_OPSTATS
unsigned long long bpk::bpk_opstats[32];
#endif

namespace {

const int64_t INF = INT64_MAX / 4;

// Mirror of k_refine_fast (csrc/kernels.cu): the slim walk in its regime,
// else the general refine (k_refine_smem).  BPEMU_NOFAST=1: general only;
// BPEMU_FAST_CHECK=1: run both and abort on any difference.  Returns 1 when
// the slim walk finished the query.
int emu_refine(const BatchDev& B, int qi) {
    if (!refine_wanted(B, qi)) return 0;
    static const bool nofast = getenv("BPEMU_NOFAST") && atoi(getenv("BPEMU_NOFAST"));
    static const bool check = getenv("BPEMU_FAST_CHECK") && atoi(getenv("BPEMU_FAST_CHECK"));
    if (nofast) { refine_query(B, qi); return 0; }
    const QDesc Q = B.q[qi];
    const NetView v = net_view(B.P, Q.net);
    const ChainView c = chain_view(B.P, Q.cl, Q.N);
    const int N = Q.N, L = (int)v.L, T = v.T;
    const int64_t o = Q.qstage_off;
    std::vector<int32_t> cost((size_t)T * L), act(L), type(N), lo(N), hi(N);
    std::vector<Rat> lead(N, R(1)), trail(N, R(1)), t(N);
    std::vector<uint8_t> memo(N);
    bool bad = false;
    for (int k = 0; k < T * L; ++k) {
        const int64_t x = v.fp[k] + v.bp[k];
        bad |= x < 0 || x >= (1 << 19);
        cost[k] = (int32_t)x;
    }
    for (int j = 0; j < L; ++j) {
        bad |= v.a[j] < 0 || v.a[j] > INT32_MAX;
        act[j] = (int32_t)v.a[j];
    }
    for (int s = 0; s < N; ++s) {
        lo[s] = B.qlo[o + s];
        hi[s] = B.qhi[o + s];
        type[s] = c.type[s];
        const int64_t x = stage_sum_whole(lo[s], hi[s], v.Pfp + (int64_t)type[s] * (v.L + 1)) +
                          stage_sum_whole(lo[s], hi[s], v.Pbp + (int64_t)type[s] * (v.L + 1));
        bad |= x < 0 || x >= (1 << 20);
        t[s] = R(x);
    }
    if (getenv("BPEMU_DUMP_REFINE") && atoi(getenv("BPEMU_DUMP_REFINE")) == qi) {
        // the slim walk's inputs of one query (tests/cpp/refine_walk_bench.cu)
        FILE* f = fopen(getenv("BPEMU_DUMP_FILE") ? getenv("BPEMU_DUMP_FILE") : "/tmp/refine_query.bin", "wb");
        int32_t hdr[3] = {L, T, N};
        fwrite(hdr, 4, 3, f);
        fwrite(cost.data(), 4, cost.size(), f);
        fwrite(act.data(), 4, act.size(), f);
        fwrite(type.data(), 4, N, f);
        fwrite(lo.data(), 4, N, f);
        fwrite(hi.data(), 4, N, f);
        fwrite(t.data(), sizeof(Rat), N, f);
        fclose(f);
    }
    int64_t st[4] = {0, 0, 0, 0};
    int r = RF_BAIL;
    if (!bad) {
        FastRefine f{cost.data(), act.data(), type.data(), L, N, lo.data(), hi.data(), lead.data(), trail.data(),
                     t.data(), memo.data()};
        r = refine_fast_walk(f, st);
    }
    if (r == RF_BAIL) { refine_query(B, qi); return 0; }
    if (check) {
        refine_query(B, qi);
        const QState& qs = B.qs[qi];
        bool same = qs.refine_iters == st[0] && qs.refine_evals == st[1] && qs.refine_moves == st[2];
        for (int s = 0; s < N; ++s)
            same = same && B.qlo[o + s] == lo[s] && B.qhi[o + s] == hi[s] && B.qlead[o + s].n == lead[s].n &&
                   B.qlead[o + s].d == lead[s].d && B.qtrail[o + s].n == trail[s].n && B.qtrail[o + s].d == trail[s].d;
        if (!same) {
            fprintf(stderr, "emu: slim refine differs from the general refine on query %d (N %d L %d)\n", qi, N, L);
            abort();
        }
        // the general walk already committed; restore the DP plan is not needed
        return 1;
    }
    refine_commit(B, qi, v, c, lo.data(), hi.data(), lead.data(), trail.data(), st, true, Err{ERR_NONE});
    return 1;
}

// Sequential mirror of k_partition (csrc/dp.cu): same windows, same order.
void host_partition(const BatchDev& B, const DPItem& item, uint64_t& work) {
    const QDesc Q = B.q[item.q];
    NetView v = net_view(B.P, Q.net);
    ChainView c = chain_view(B.P, Q.cl, Q.N);
    const int N = Q.N;
    const int64_t L = v.L;
    std::vector<int32_t> pos;
    pos.push_back(0);
    for (int64_t j = 1; j <= L; ++j)
        if (item.a_th < 0 || j == L || v.a[j - 1] <= item.a_th) pos.push_back((int32_t)j);
    const int U = (int)pos.size() - 1;
    if (U < N) {
        if (item.a_th < 0) B.qs[item.q].dp_shape = 1;
        return;
    }
    std::vector<int64_t> C((size_t)v.T * (U + 1)), W(U + 1), A(U + 1);
    for (int t = 0; t < v.T; ++t)
        for (int j = 0; j <= U; ++j) C[(size_t)t * (U + 1) + j] = v.Pc[(int64_t)t * (L + 1) + pos[j]];
    for (int j = 0; j <= U; ++j) {
        W[j] = v.Pw[pos[j]];
        A[j] = j >= 1 ? v.a[pos[j] - 1] : 0;
    }
    auto Cn = [&](int n) { return &C[(size_t)c.type[n - 1] * (U + 1)]; };
    int64_t T_ub = 0;
    for (int n = 1; n <= N; ++n) {
        int64_t k = ((int64_t)(n - 1) * U) / N, j = ((int64_t)n * U) / N;
        T_ub = std::max(T_ub, Cn(n)[j] - Cn(n)[k]);
    }
    // bands (mirror of dp_bands in csrc/dp.cu): row n can only matter for
    // j in [bwd[n], fwd[n]] -- fwd = farthest greedy reach of n stages, bwd =
    // earliest start from which stages n+1..N can cover the rest -- under T.
    // Stages may take zero units in this relaxation, which makes fwd an upper
    // bound of the reachable set's maximum and bwd a lower bound of the
    // completable set's minimum even on heterogeneous chains.
    std::vector<int> fwd(N + 1), bwd(N + 1);
    auto bands = [&](int64_t T) {
        int cur = 0;
        fwd[0] = 0;
        for (int n = 1; n <= N; ++n) {
            const int64_t* Cc = Cn(n);
            int hi = U - (N - n), j = cur;
            while (j < hi && Cc[j + 1] - Cc[cur] <= T) ++j;
            cur = std::max(j, cur);
            fwd[n] = cur;
        }
        cur = U;
        bwd[N] = U;
        for (int n = N; n >= 1; --n) {
            const int64_t* Cc = Cn(n);
            int lo = n - 1, k = cur;
            while (k > lo && Cc[cur] - Cc[k - 1] <= T) --k;
            cur = k;
            bwd[n - 1] = cur;
        }
    };
    bands(T_ub);
    std::vector<int64_t> prev(U + 1), cur(U + 1);
    for (int j = 0; j <= U; ++j) prev[j] = j == 0 ? 0 : INF;
    for (int n = 1; n <= N; ++n) {
        const int64_t* Cc = Cn(n);
        for (int j = 0; j <= U; ++j) {
            int64_t best = INF;
            if (j >= n && j <= U - (N - n) && j >= bwd[n] && j <= fwd[n]) {
                for (int k = j - 1; k >= n - 1; --k) {
                    int64_t s = Cc[j] - Cc[k];
                    if (s > T_ub || s >= best) break;
                    best = std::min(best, std::max(prev[k], s));
                    ++work;
                }
                if (best > T_ub) best = INF;
            }
            cur[j] = best;
        }
        std::swap(prev, cur);
    }
    const int64_t T_opt = prev[U];
    bands(T_opt);
    for (int j = 0; j <= U; ++j) prev[j] = j == 0 ? 0 : INF;
    for (int n = 1; n <= N; ++n) {
        const int64_t* Cc = Cn(n);
        const int64_t cN = N - n + 1;
        for (int j = 0; j <= U; ++j) {
            int64_t best = INF;
            if (j >= n && j <= U - (N - n) && j >= bwd[n] && j <= fwd[n]) {
                for (int k = j - 1; k >= n - 1; --k) {
                    if (Cc[j] - Cc[k] > T_opt) break;
                    int64_t w2 = 2 * (W[j] - W[k]);
                    if (w2 >= best) break;
                    ++work;
                    if (prev[k] == INF) continue;
                    int64_t foot = w2 + cN * (k >= 1 ? A[k] : A[j]);
                    best = std::min(best, std::max(prev[k], foot));
                }
            }
            cur[j] = best;
        }
        std::swap(prev, cur);
    }
    const int64_t F_opt = prev[U];
    std::vector<std::vector<char>> feas(N + 1, std::vector<char>(U + 1, 0));
    feas[N][U] = 1;
    for (int n = N - 1; n >= 0; --n) {
        const int64_t* Cc = Cn(n + 1);
        const int64_t cN = N - n;
        for (int j = std::max(n, bwd[n]); j <= U && j <= fwd[n]; ++j) {
            for (int j2 = j + 1; j2 <= U; ++j2) {
                if (Cc[j2] - Cc[j] > T_opt) break;
                ++work;
                int64_t foot = 2 * (W[j2] - W[j]) + cN * (j >= 1 ? A[j] : A[j2]);
                if (foot > F_opt) {
                    if (j >= 1) break;
                    continue;
                }
                if (feas[n + 1][j2]) { feas[n][j] = 1; break; }
            }
        }
    }
    int curj = 0;
    int64_t target = 0;
    for (int n = 1; n <= N; ++n) {
        const int64_t* Cc = Cn(n);
        const int64_t cN = N - n + 1;
        int chosen = -1;
        for (int j = curj + 1; j <= U; ++j) {
            if (Cc[j] - Cc[curj] > T_opt) break;
            int64_t foot = 2 * (W[j] - W[curj]) + cN * (curj >= 1 ? A[curj] : A[j]);
            if (foot > F_opt) continue;
            if (feas[n][j]) { chosen = j; break; }
        }
        if (chosen < 0) {
            if (item.a_th < 0) B.qs[item.q].target = -1;
            return;
        }
        target = std::max(target, Cc[chosen] - Cc[curj]);
        if (item.a_th < 0) {
            B.qlo[Q.qstage_off + n - 1] = pos[curj] + 1;
            B.qhi[Q.qstage_off + n - 1] = pos[chosen];
        } else {
            for (int k = 0; k < 2; ++k) {
                int64_t o = Q.stage_off + ((int64_t)k * Q.nbase + item.mslot) * N + (n - 1);
                B.clo[o] = pos[curj] + 1;
                B.chi[o] = pos[chosen];
            }
        }
        curj = chosen;
    }
    if (item.a_th < 0) B.qs[item.q].target = target;
    else B.ms[Q.mslot_off + item.mslot].coarse_ok = 1;
}

template <class T>
T* vec(std::vector<T>& v, size_t n) {
    v.assign(n ? n : 1, T{});
    return v.data();
}

}  // namespace

static int g_plan_only = 0;   // BP_OPT_PLAN_ONLY

static Pools host_pools(const HostNets& HN, const HostCls& HC) {
    Pools P{};
    P.nets = HN.desc.data();
    P.cls = HC.desc.data();
    P.fp = HN.fp.data();
    P.bp = HN.bp.data();
    P.w = HN.w.data();
    P.a = HN.a.data();
    P.asort = HN.asort.data();
    P.Pfp = HN.Pfp.data();
    P.Pbp = HN.Pbp.data();
    P.Pc = HN.Pc.data();
    P.Pw = HN.Pw.data();
    P.type_ok = HN.type_ok.data();
    P.ctype = HC.ctype.data();
    P.cap = HC.cap.data();
    P.minm = HC.minm.data();
    P.bw = HC.bw.data();
    return P;
}

extern "C" void bpemu_set_plan_only(int v) { g_plan_only = v; }

// bp_simulate_plan / bp_estimate_plan replayed on the host (timeline.cuh)
extern "C" int bpemu_plan(const bp_network* nets, int n_nets, const bp_cluster* cls, int n_cls,
                          const bp_plan_request* q, bp_timeline_result* tres, bp_event* events, int64_t cap,
                          bp_rat* hw, bp_rat* ws, bp_rat* busy, bp_estimate_result* eres, bp_stage* st, int32_t* inf) {
    std::string err;
    HostNets HN;
    HostCls HC;
    if (!build_nets(nets, n_nets, HN, err, true) || !build_clusters(cls, n_cls, HC, err)) return BP_BAD_INPUT;
    const Pools P = host_pools(HN, HC);
    const int N = q->n_stages, clusterN = HC.desc[(size_t)q->cluster].N;
    TlArgs A{};
    A.v = net_view(P, q->network);
    A.c = chain_view(P, q->cluster, N < clusterN ? N : clusterN);
    A.N = N;
    A.kind = q->kind;
    A.clusterN = clusterN;
    A.M = q->M;
    A.micro = q->micro;
    A.mini = q->mini_batches;
    A.lo = q->lo;
    A.hi = q->hi;
    A.lead = reinterpret_cast<const Rat*>(q->lead);
    A.trail = reinterpret_cast<const Rat*>(q->trail);
    std::vector<Rat> F(N), Bv(N), W(N);
    std::vector<int64_t> a(N), SR(N), off(N + 1);
    if (eres) {   // estimate
        std::vector<Rat> scr(7 * (size_t)N);
        std::vector<int64_t> scr64(2 * (size_t)N);
        *eres = bp_estimate_result{};
        tl_estimate(A, *eres, st, inf, scr.data(), scr64.data());
        return BP_OK;
    }
    const int64_t M = q->M > 0 ? q->M : 0, mini = q->mini_batches;
    const size_t NM = (size_t)N * M, LM = (size_t)(N > 1 ? N - 1 : 0) * M;
    const size_t nev = (size_t)mini * (2 * NM + 4 * LM);
    std::vector<Rat> sF(NM + 1), eF(NM + 1), sB(NM + 1), eB(NM + 1), tFs(LM + 1), tFe(LM + 1), tBs(LM + 1),
        tBe(LM + 1), mk(1);
    std::vector<bp_event> ev(nev + 1), evt(nev + 1);
    std::vector<TlPoint> pts(2 * M + 1), tmp(2 * M + 1);
    std::vector<Rat> hwv(N), wsv(N), busyv(N);
    A.F = F.data();
    A.B = Bv.data();
    A.W = W.data();
    A.a = a.data();
    A.SR = SR.data();
    A.sF = sF.data();
    A.eF = eF.data();
    A.sB = sB.data();
    A.eB = eB.data();
    A.tFs = tFs.data();
    A.tFe = tFe.data();
    A.tBs = tBs.data();
    A.tBe = tBe.data();
    A.makespan1 = mk.data();
    A.ev = ev.data();
    A.ev_tmp = evt.data();
    A.off = off.data();
    bp_timeline_result r{};
    r.status = BP_C_OK;
    if (tl_chain(A, r) && tl_walk(A, r)) {
        uint32_t code = 0;
        for (int s = 1; s <= N && !code; ++s) code = tl_stage(A, s, pts.data(), tmp.data(), hwv.data(), wsv.data());
        if (!code) code = tl_busy(A, busyv.data());
        if (code) r.status = (int32_t)code;
    }
    *tres = r;
    if (r.status == BP_C_OK) {
        for (int64_t i = 0; i < r.n_events && i < cap; ++i) events[i] = ev[(size_t)i];
        for (int s = 0; s < N; ++s) {
            hw[s] = bp_rat{hwv[s].n, hwv[s].d};
            ws[s] = bp_rat{wsv[s].n, wsv[s].d};
            if (s + 1 < N) busy[s] = bp_rat{busyv[s].n, busyv[s].d};
        }
    }
    return BP_OK;
}

extern "C" int bpemu_explore_batch(const bp_network* nets, int n_nets, const bp_cluster* cls, int n_cls,
                                   const bp_query* qs, int nq, bp_query_result* res, bp_candidate* cand,
                                   bp_stage* stages, uint64_t* dp_work) {
    std::string err;
    HostNets HN;
    HostCls HC;
    HostBatch HB;
    if (!build_nets(nets, n_nets, HN, err, true) || !build_clusters(cls, n_cls, HC, err) ||
        !build_batch(qs, nq, HN, HC, HB, err))
        return BP_BAD_INPUT;
    for (int i = 0; i < nq; ++i)
        if (qs[i].cand_offset != HB.q[i].cand_off || qs[i].stage_offset != HB.q[i].stage_off) return BP_BAD_INPUT;
    BatchDev B{};
    B.plan_only = g_plan_only;
    B.P.nets = HN.desc.data();
    B.P.cls = HC.desc.data();
    B.P.fp = HN.fp.data();
    B.P.bp = HN.bp.data();
    B.P.w = HN.w.data();
    B.P.a = HN.a.data();
    B.P.asort = HN.asort.data();
    B.P.Pfp = HN.Pfp.data();
    B.P.Pbp = HN.Pbp.data();
    B.P.Pc = HN.Pc.data();
    B.P.Pw = HN.Pw.data();
    B.P.type_ok = HN.type_ok.data();
    B.P.ctype = HC.ctype.data();
    B.P.cap = HC.cap.data();
    B.P.minm = HC.minm.data();
    B.P.bw = HC.bw.data();
    B.nq = nq;
    B.ncand = HB.ncand;
    B.q = HB.q.data();
    B.Mpool = HB.Mpool.data();
    std::vector<QState> vqs;
    std::vector<MState> vms;
    std::vector<CState> vcs;
    std::vector<bp_candidate> vcand;
    std::vector<bp_stage> vst;
    std::vector<bp_query_result> vres;
    std::vector<int32_t> vqlo, vqhi, vclo, vchi, vcq, vco;
    std::vector<Rat> vql, vqt, vqF, vqB, vqW, vqT, vsF, vsB, vsW, vsM, vsim;
    std::vector<uint8_t> vqd;
    std::vector<int64_t> vsA, vsSR;
    B.qs = vec(vqs, nq);
    B.ms = vec(vms, HB.nmslot);
    B.cs = vec(vcs, HB.ncand);
    B.cand = vec(vcand, HB.ncand);
    B.details = stages != nullptr;
    B.stages = stages ? vec(vst, HB.nstage) : nullptr;
    B.res = vec(vres, nq);
    B.qlo = vec(vqlo, HB.nqstage);
    B.qhi = vec(vqhi, HB.nqstage);
    B.qlead = vec(vql, HB.nqstage);
    B.qtrail = vec(vqt, HB.nqstage);
    B.qF = vec(vqF, HB.nqstage);
    B.qB = vec(vqB, HB.nqstage);
    B.qW = vec(vqW, HB.nqstage);
    B.qT = vec(vqT, HB.nqstage);
    B.qdirty = vec(vqd, HB.nqstage);
    B.clo = vec(vclo, HB.nstage);
    B.chi = vec(vchi, HB.nstage);
    B.sF = vec(vsF, HB.nstage);
    B.sB = vec(vsB, HB.nstage);
    B.sW = vec(vsW, HB.nstage);
    B.sMem = vec(vsM, HB.nstage);
    B.sA = vec(vsA, HB.nstage);
    B.sSR = vec(vsSR, HB.nstage);
    B.simbuf = vec(vsim, 9 * HB.nstage);
    B.cq = vec(vcq, HB.ncand);
    B.corder = vec(vco, HB.ncand);
    uint64_t work = 0;
    for (int i = 0; i < nq; ++i) setup_query(B, i);
    for (const DPItem& it : HB.whole_items) host_partition(B, it, work);
    for (int i = 0; i < nq; ++i)
        for (int m = 0; m < HB.q[i].nbase; ++m)
            if (bottleneck_slot(B, i, m)) host_partition(B, DPItem{i, m, B.ms[HB.q[i].mslot_off + m].a_th}, work);
    int64_t r_it = 0, r_ev = 0, r_mv = 0, r_ex = 0, r_q = 0, r_max = 0, r_fast = 0;
    for (int i = 0; i < nq; ++i) {
        r_fast += emu_refine(B, i);
        if (B.qs[i].refined) {
            ++r_q;
            r_it += B.qs[i].refine_iters;
            r_ev += B.qs[i].refine_evals;
            r_mv += B.qs[i].refine_moves;
            r_ex += B.qs[i].refine_exact;
            r_max = std::max<int64_t>(r_max, B.qs[i].refine_evals);
        }
    }
    if (getenv("BPEMU_STATS"))
        fprintf(stderr, "emu refine: queries %lld (slim %lld) iterations %lld evaluated steps %lld (max %lld) moves %lld exact %lld\n",
                (long long)r_q, (long long)r_fast, (long long)r_it, (long long)r_ev, (long long)r_max, (long long)r_mv,
                (long long)r_ex);
#ifdef BPK_OPSTATS
    if (getenv("BPEMU_STATS")) {
        fprintf(stderr, "opstats");
        for (int k = 0; k < 32; ++k) fprintf(stderr, " %llu", bpk_opstats[k]);
        fprintf(stderr, "\n");
    }
#endif
    if (getenv("BPEMU_REFINE_ONLY")) {
        for (int i = 0; i < nq; ++i)
            if (B.qs[i].refined) fprintf(stderr, "q %d N %d L %lld evals %lld moves %lld\n", i, HB.q[i].N,
                                         (long long)net_view(B.P, HB.q[i].net).L, (long long)B.qs[i].refine_evals,
                                         (long long)B.qs[i].refine_moves);
        return 0;
    }
    for (int64_t c = 0; c < HB.ncand; ++c) prune_candidate(B, c);
    if (B.plan_only) {   // `bapipe plan`: no simulation (k_plan_finish)
        for (int64_t c = 0; c < HB.ncand; ++c)
            if (B.cs[c].sim_ready && B.cand[c].status == C_PENDING) {
                B.cand[c].status = BP_C_OK;
                B.cand[c].makespan = bp_rat{0, 1};
            }
        for (int i = 0; i < nq; ++i) rank_query(B, i);
        if (stages) for (int64_t i = 0; i < HB.nstage; ++i) stages[i] = B.stages[i];
        for (int64_t i = 0; i < HB.ncand; ++i) cand[i] = B.cand[i];
        for (int i = 0; i < nq; ++i) res[i] = B.res[i];
        return 0;
    }
    int64_t exact_n = 0, exact_ovf = 0, fast_n = 0;
    const size_t mn = (size_t)std::max(1, HB.max_N);
    std::vector<Rat> s_fr(mn), s_pf(mn), s_pb(mn), s_f(mn), s_b(mn);
    std::vector<int64_t> s_sr(mn), s_a(mn);
    SimState S{s_fr.data(), s_pf.data(), s_pb.data(), s_f.data(), s_b.data(), s_sr.data(), s_a.data(), 1};
    for (int64_t c = 0; c < HB.ncand; ++c) {
        int cls = sim_classify(B, c);
        if (cls < 0) continue;
#ifdef BPK_OPSTATS
        unsigned long long before[32];
        for (int k = 0; k < 32; ++k) before[k] = bpk_opstats[k];
#endif
        sim_exact(B, c, S);
        if (getenv("BPEMU_DUMP_SIM") && cls >= SIM_EXACT) {
            // the exact simulator's inputs (stage F / B, link SR) of exact-class candidates
            static FILE* df = fopen(getenv("BPEMU_DUMP_SIM"), "w");
            const bp_candidate& cd = B.cand[c];
            fprintf(df, "C %lld %d %lld %d %d", (long long)c, cd.n_stages, (long long)cd.M, cd.kind, cd.status);
            for (int s = 0; s < cd.n_stages; ++s)
                fprintf(df, " %lld %lld %lld %lld %lld", (long long)S.dF(s).n, (long long)S.dF(s).d,
                        (long long)S.dB(s).n, (long long)S.dB(s).d, (long long)S.sr(s));
            fprintf(df, "\n");
        }
#ifdef BPK_OPSTATS
        if (cls < SIM_EXACT)   // count the exact-class candidates' Rat work only
            for (int k = 0; k < 32; ++k) bpk_opstats[k] = before[k];
#endif
        if (cls == SIM_EXACT) {
            ++exact_n;
            exact_ovf += B.cand[c].status == BP_C_ERR_OVERFLOW;
            if (getenv("BPEMU_STATS") && atoi(getenv("BPEMU_STATS")) > 1)
                fprintf(stderr, "exact N=%d M=%lld kind=%d status=%d D=%lld\n", B.cand[c].n_stages,
                        (long long)B.cand[c].M, B.cand[c].kind, B.cand[c].status, (long long)B.cs[c].D);
        } else {
            ++fast_n;
        }
    }
    if (getenv("BPEMU_STATS"))
        fprintf(stderr, "emu sim: fast %lld exact %lld (overflow %lld)\n", (long long)fast_n, (long long)exact_n,
                (long long)exact_ovf);
#ifdef BPK_OPSTATS
    if (getenv("BPEMU_STATS")) {
        fprintf(stderr, "opstats after sims");
        for (int k = 0; k < 32; ++k) fprintf(stderr, " %llu", bpk_opstats[k]);
        fprintf(stderr, "\n");
    }
#endif
    for (int i = 0; i < nq; ++i) rank_query(B, i);
    std::memcpy(res, B.res, sizeof(bp_query_result) * (size_t)nq);
    if (cand) std::memcpy(cand, B.cand, sizeof(bp_candidate) * (size_t)HB.ncand);
    if (stages) std::memcpy(stages, B.stages, sizeof(bp_stage) * (size_t)HB.nstage);
    if (dp_work) *dp_work = work;
    return BP_OK;
}
