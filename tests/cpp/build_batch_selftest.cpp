// The host batch build in chunks on the worker pool (host_prep.hpp
// build_batch_at) against the same build as one serial chunk: every query
// record (offsets, validation, its M list), the DP work items and the
// totals must agree, and a failing query must be reported with the same
// index and message.  Random networks, clusters and queries (some invalid:
// missing types, bad M lists, mini-batch 0), 40,000 queries per trial so that
// several chunks of 8,192 are joined.  Usage: build_batch_selftest [trials].
#include <cstdio>
#include <cstdlib>
#include <random>

#include "host_prep.hpp"

using namespace bpk;

struct World {
    std::vector<std::vector<int64_t>> fp, bp, w, a;
    std::vector<bp_network> nets;
    std::vector<std::vector<int32_t>> types;
    std::vector<std::vector<int64_t>> cap, minm, bw;
    std::vector<bp_cluster> cls;
    std::vector<std::vector<int64_t>> mlists;
    std::vector<bp_query> q;
};

static void make(World& W, std::mt19937_64& g, int nq) {
    auto U = [&](int64_t lo, int64_t hi) { return std::uniform_int_distribution<int64_t>(lo, hi)(g); };
    const int nn = (int)U(1, 6), nc = (int)U(1, 6);
    W.fp.resize(nn); W.bp.resize(nn); W.w.resize(nn); W.a.resize(nn); W.nets.resize(nn);
    for (int i = 0; i < nn; ++i) {
        const int L = (int)U(1, 40), T = (int)U(1, 3);
        W.fp[i].resize((size_t)T * L); W.bp[i].resize((size_t)T * L); W.w[i].resize(L); W.a[i].resize(L);
        for (auto& x : W.fp[i]) x = U(0, 9) == 0 ? 0 : U(1, 100);   // 0: no time for that type
        for (auto& x : W.bp[i]) x = U(1, 100);
        for (auto& x : W.w[i]) x = U(0, 1000);
        for (auto& x : W.a[i]) x = U(0, 1000);
        W.nets[i] = bp_network{L, T, W.fp[i].data(), W.bp[i].data(), W.w[i].data(), W.a[i].data()};
    }
    W.types.resize(nc); W.cap.resize(nc); W.minm.resize(nc); W.bw.resize(nc); W.cls.resize(nc);
    for (int i = 0; i < nc; ++i) {
        const int n = (int)U(1, 12);
        W.types[i].resize(n); W.cap[i].resize(n); W.minm[i].assign((size_t)4 * n, 1); W.bw[i].resize(std::max(1, n - 1));
        for (auto& t : W.types[i]) t = (int32_t)U(0, 2);
        for (auto& c : W.cap[i]) c = U(1, 1 << 20);
        for (auto& b : W.bw[i]) b = U(1, 100);
        W.cls[i] = bp_cluster{n, (int32_t)U(0, 1), W.types[i].data(), W.cap[i].data(), W.minm[i].data(), W.bw[i].data()};
    }
    W.mlists.resize(8);
    for (auto& m : W.mlists) {
        m.resize((size_t)U(1, 5));
        for (auto& x : m) x = U(0, 8);   // 0: an invalid micro-batch count
    }
    W.q.resize(nq);
    for (int i = 0; i < nq; ++i) {
        bp_query& b = W.q[i];
        b = bp_query{};
        b.network = (int32_t)U(0, nn - 1);
        b.cluster = (int32_t)U(0, nc - 1);
        b.n_stages = (int32_t)U(0, W.cls[b.cluster].n_accels);
        b.mini_batch = U(0, 12) == 0 ? 0 : (int64_t)(U(0, 1) ? 128 : U(1, 64));
        if (U(0, 4) == 0) {
            const auto& m = W.mlists[(size_t)U(0, 7)];
            b.n_m = (int32_t)m.size();
            b.m_list = m.data();
        }
    }
}

static int compare(const HostBatch& A, const HostBatch& B, int nq) {
    if (A.ncand != B.ncand || A.nstage != B.nstage || A.nqstage != B.nqstage || A.nmslot != B.nmslot ||
        A.max_units != B.max_units || A.max_N != B.max_N || A.max_nbase != B.max_nbase)
        return 1;
    for (int i = 0; i < nq; ++i) {
        const QDesc &x = A.q[i], &y = B.q[i];
        if (x.net != y.net || x.cl != y.cl || x.N != y.N || x.nbase != y.nbase || x.mini != y.mini ||
            x.cand_off != y.cand_off || x.stage_off != y.stage_off || x.qstage_off != y.qstage_off ||
            x.mslot_off != y.mslot_off || x.schema_ok != y.schema_ok)
            return 2;
        for (int k = 0; k < x.nbase; ++k)
            if (A.Mpool[(size_t)(x.m_off + k)] != B.Mpool[(size_t)(y.m_off + k)]) return 3;
    }
    if (A.whole_items.size() != B.whole_items.size()) return 4;
    for (size_t k = 0; k < A.whole_items.size(); ++k)
        if (A.whole_items[k].q != B.whole_items[k].q) return 5;
    return 0;
}

int main(int argc, char** argv) {
    const int trials = argc > 1 ? atoi(argv[1]) : 20;
    std::mt19937_64 g(0x2012125440ull);
    for (int t = 0; t < trials; ++t) {
        World W;
        const int nq = 40000;
        make(W, g, nq);
        HostNets HN;
        HostCls HC;
        std::string err;
        if (!build_nets(W.nets.data(), (int)W.nets.size(), HN, err, false) ||
            !build_clusters(W.cls.data(), (int)W.cls.size(), HC, err)) {
            printf("tables: %s\n", err.c_str());
            return 1;
        }
        HostBatch A, B;
        std::string ea, eb;
        const bool ra = build_batch(W.q.data(), nq, HN, HC, A, ea);
        const bool rb = build_batch(W.q.data(), nq, HN, HC, B, eb, 1 << 30);
        if (ra != rb || !ra) {
            printf("trial %d: build results %d %d (%s | %s)\n", t, ra, rb, ea.c_str(), eb.c_str());
            return 1;
        }
        if (const int c = compare(A, B, nq)) {
            printf("trial %d: chunked build differs (%d)\n", t, c);
            return 1;
        }
        // an out-of-range query late in the batch: the same first error
        const int bad = (int)(g() % nq), bad2 = bad + (int)(g() % (nq - bad));
        W.q[bad2].network = -1;
        W.q[bad].cluster = (int32_t)W.cls.size();
        const bool fa = build_batch(W.q.data(), nq, HN, HC, A, ea);
        const bool fb = build_batch(W.q.data(), nq, HN, HC, B, eb, 1 << 30);
        if (fa || fb || ea != eb) {
            printf("trial %d: errors differ (%s | %s)\n", t, ea.c_str(), eb.c_str());
            return 1;
        }
    }
    printf("ok %d trials\n", trials);
    return 0;
}
