// host_prep.hpp -- host-side preparation of networks, clusters and query
// batches (plain C++; shared by api.cu and the tests/emu harness).
//
//   * validation mirrors validate_network / validate_cluster / validate_pair
//     (profiles.hpp:83-132) plus explore()'s mini-batch and candidate_Ms
//     checks (explorer.hpp:82-83, 26-49) and resolves to a per-query flag;
//   * K1 cost_prefix tables (prefix sums per accelerator type) are built on
//     the host at upload time for the CPU harness and on the device
//     (cost_prefix kernel) for the product;
//   * the batch layout assigns each query its candidate / stage / M-slot
//     ranges (dense, in query order, the same rule as bp_layout()).
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <pthread.h>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "batch.cuh"

namespace bpk {

struct HostNets {
    std::vector<NetDesc> desc;
    std::vector<int64_t> fp, bp, w, a, asort, Pfp, Pbp, Pc, Pw;
    std::vector<uint8_t> type_ok;
    int max_L = 0, max_T = 0;
    // lengths of the prefix tables (Pw; Pfp / Pbp / Pc): the device builds
    // them (k_cost_prefix); the host arrays are filled only when asked
    size_t n_pref = 0, n_tpref = 0;
};

struct HostCls {
    std::vector<ClDesc> desc;
    std::vector<int32_t> ctype;
    std::vector<int32_t> pmax;   // host only: prefix maximum of ctype per cluster (build_batch's type check)
    std::vector<int64_t> cap, minm, bw;
    int max_N = 0;
};

// Run f(i) for i in [0, n) on up to 8 host threads (serially when n is small).
// A persistent pool of host worker threads (created on first use, never
// destroyed): host_parallel_for hands out the indices [0, n) to the workers
// and the calling thread.  Dispatch is a condition-variable wake-up (tens of
// microseconds), not a thread creation per call.
class HostPool {
  public:
    static HostPool& get() {
        // leaked on purpose (no teardown order at exit); a forked child has
        // none of the parent's workers, so it starts a pool of its own
        static std::once_flag once;
        std::call_once(once, [] { pthread_atfork(nullptr, nullptr, [] { slot() = nullptr; }); });
        HostPool*& p = slot();
        if (!p) p = new HostPool();
        return *p;
    }
    int workers() const { return (int)th_.size(); }
    template <class F>
    void run(int n, F& f) {
        std::lock_guard<std::mutex> call(call_);   // one parallel region at a time
        std::atomic<int> next{0};
        auto body = [&] {
            for (int i; (i = next.fetch_add(1)) < n;) f(i);
        };
        {
            std::lock_guard<std::mutex> l(m_);
            job_ = body;
            busy_ = (int)th_.size();
            ++gen_;
        }
        cv_.notify_all();
        body();
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return busy_ == 0; });
        job_ = nullptr;
    }

  private:
    static HostPool*& slot() {
        static HostPool* p = nullptr;
        return p;
    }
    HostPool() {
        const int hw = (int)std::thread::hardware_concurrency();
        const int n = std::max(0, std::min(7, hw - 1));
        for (int t = 0; t < n; ++t)
            th_.emplace_back([this] {
                uint64_t seen = 0;
                for (;;) {
                    std::function<void()> job;
                    {
                        std::unique_lock<std::mutex> l(m_);
                        cv_.wait(l, [&] { return gen_ != seen; });
                        seen = gen_;
                        job = job_;
                    }
                    if (job) job();
                    std::lock_guard<std::mutex> l(m_);
                    if (--busy_ == 0) done_.notify_one();
                }
            });
        for (auto& t : th_) t.detach();
    }
    std::vector<std::thread> th_;
    std::mutex m_, call_;
    std::condition_variable cv_, done_;
    std::function<void()> job_;
    uint64_t gen_ = 0;
    int busy_ = 0;
};

template <class F>
inline void host_parallel_for(int n, F&& f) {
    if (n <= 1 || HostPool::get().workers() == 0) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    HostPool::get().run(n, f);
}

// One network's tables into its slices of H (layout already in H.desc[i]):
// schema flags, the SoA copies, the sorted activations, the magnitude check
// and, when asked, the host prefix tables.  Returns 0, 2 (weight sum beyond
// 2^62) or 3 (time sum beyond 2^62).
inline int fill_net(const bp_network& b, HostNets& H, NetDesc& d, bool prefix) {
    const int64_t LIM = (int64_t)1 << 62;
    const int64_t L = b.n_layers;
    const int T = b.n_types;
    bool valid = L >= 1;
    uint8_t* tok = H.type_ok.data() + d.off_tflag;
    for (int t = 0; t < T; ++t) tok[t] = 1;
    for (int64_t j = 0; j < L; ++j) {
        bool anyf = false, anyb = false;
        for (int t = 0; t < T; ++t) {
            int64_t f = b.fp_us[(size_t)t * L + j], bb = b.bp_us[(size_t)t * L + j];
            if (f < 0 || bb < 0) valid = false;          // present but < 1
            anyf |= f != 0;
            anyb |= bb != 0;
            if (f == 0 || bb == 0) tok[t] = 0;
        }
        if (!anyf || !anyb) valid = false;                // maps must be non-empty
        if (b.weight_bytes[j] < 0 || b.out_act_bytes[j] < 0) valid = false;
    }
    d.valid = valid ? 1 : 0;
    if (!valid)
        for (int t = 0; t < T; ++t) tok[t] = 0;
    std::copy(b.fp_us, b.fp_us + (size_t)T * L, H.fp.data() + d.off_typed);
    std::copy(b.bp_us, b.bp_us + (size_t)T * L, H.bp.data() + d.off_typed);
    std::copy(b.weight_bytes, b.weight_bytes + L, H.w.data() + d.off_layer);
    std::copy(b.out_act_bytes, b.out_act_bytes + L, H.a.data() + d.off_layer);
    int64_t* as = H.asort.data() + d.off_layer;   // the L-1 cut activations, sorted, then a 0
    if (L > 0) {
        std::copy(b.out_act_bytes, b.out_act_bytes + (L - 1), as);
        std::sort(as, as + (L - 1));
        as[L - 1] = 0;
    }
    // the magnitude check on the (clamped, non-decreasing) prefix sums:
    // their totals bound every partial sum.  The tables themselves are built
    // on the device (k_cost_prefix); the host copy only when asked (the test
    // emulator).
    int64_t sw = 0;
    for (int64_t j = 0; j < L; ++j) {
        sw += std::max<int64_t>(b.weight_bytes[j], 0);
        if (sw >= LIM) return 2;
    }
    for (int t = 0; t < T; ++t) {
        int64_t sf = 0, sb = 0;
        for (int64_t j = 0; j < L; ++j) {
            sf += std::max<int64_t>(b.fp_us[(size_t)t * L + j], 0);
            sb += std::max<int64_t>(b.bp_us[(size_t)t * L + j], 0);
            if (sf + sb >= LIM) return 3;
        }
    }
    if (prefix) {
        int64_t* Pw = H.Pw.data() + d.off_pref;
        sw = 0;
        Pw[0] = 0;
        for (int64_t j = 0; j < L; ++j) Pw[j + 1] = (sw += std::max<int64_t>(b.weight_bytes[j], 0));
        for (int t = 0; t < T; ++t) {
            int64_t* Pf = H.Pfp.data() + d.off_tpref + (size_t)t * (L + 1);
            int64_t* Pb = H.Pbp.data() + d.off_tpref + (size_t)t * (L + 1);
            int64_t* Pc = H.Pc.data() + d.off_tpref + (size_t)t * (L + 1);
            int64_t sf = 0, sb = 0;
            Pf[0] = Pb[0] = Pc[0] = 0;
            for (int64_t j = 0; j < L; ++j) {
                sf += std::max<int64_t>(b.fp_us[(size_t)t * L + j], 0);
                sb += std::max<int64_t>(b.bp_us[(size_t)t * L + j], 0);
                Pf[j + 1] = sf;
                Pb[j + 1] = sb;
                Pc[j + 1] = sf + sb;
            }
        }
    }
    return 0;
}

inline bool build_nets(const bp_network* nets, int n, HostNets& H, std::string& err, bool prefix) {
    // pass 1: argument checks and the layout (offsets of every network's
    // slices); pass 2, over networks in parallel: the tables themselves.
    // Errors are reported for the first failing network, as a serial pass
    // would (a network's magnitude error before a later one's bad arrays).
    H.desc.assign((size_t)std::max(n, 0), NetDesc{});
    H.max_L = H.max_T = 0;
    size_t nl = 0, ntl = 0, np = 0, ntp = 0, nf = 0;
    int m = n;   // networks [0, m) have well-formed arguments
    for (int i = 0; i < n; ++i) {
        const bp_network& b = nets[i];
        if (b.n_layers < 0 || b.n_types < 1 ||
            (b.n_layers > 0 && (!b.fp_us || !b.bp_us || !b.weight_bytes || !b.out_act_bytes))) {
            m = i;
            break;
        }
        NetDesc& d = H.desc[(size_t)i];
        d.L = b.n_layers;
        d.T = b.n_types;
        d.off_layer = (int64_t)nl;
        d.off_typed = (int64_t)ntl;
        d.off_pref = (int64_t)np;
        d.off_tpref = (int64_t)ntp;
        d.off_tflag = (int64_t)nf;
        nl += (size_t)b.n_layers;
        ntl += (size_t)b.n_types * (size_t)b.n_layers;
        np += (size_t)b.n_layers + 1;
        ntp += (size_t)b.n_types * ((size_t)b.n_layers + 1);
        nf += (size_t)b.n_types;
        H.max_L = std::max<int>(H.max_L, b.n_layers);
        H.max_T = std::max<int>(H.max_T, b.n_types);
    }
    // (the vectors keep their capacity across calls: a sweep re-uploads its
    // tables every step, with no fresh pages to fault in)
    H.fp.resize(ntl);
    H.bp.resize(ntl);
    H.w.resize(nl);
    H.a.resize(nl);
    H.asort.resize(nl);
    H.type_ok.resize(nf);
    H.n_pref = np;
    H.n_tpref = ntp;
    H.Pw.resize(prefix ? np : 0);
    H.Pfp.resize(prefix ? ntp : 0);
    H.Pbp.resize(prefix ? ntp : 0);
    H.Pc.resize(prefix ? ntp : 0);
    std::vector<int> status((size_t)m, 0);
    host_parallel_for(m, [&](int i) { status[(size_t)i] = fill_net(nets[i], H, H.desc[(size_t)i], prefix); });
    for (int i = 0; i < m; ++i)
        if (status[(size_t)i]) {
            err = "network " + std::to_string(i) + (status[(size_t)i] == 2 ? ": weight sum beyond 2^62"
                                                                           : ": time sum beyond 2^62");
            return false;
        }
    if (m < n) {
        err = "network " + std::to_string(m) + ": bad array arguments";
        return false;
    }
    return true;
}

inline bool build_clusters(const bp_cluster* cls, int n, HostCls& H, std::string& err) {
    H = HostCls();
    for (int i = 0; i < n; ++i) {
        const bp_cluster& c = cls[i];
        if (c.n_accels < 1 || !c.type_id || !c.mem_capacity || !c.min_micro || (c.n_accels > 1 && !c.link_bw) ||
            (c.exec_mode != 0 && c.exec_mode != 1)) {
            err = "cluster " + std::to_string(i) + ": bad arguments";
            return false;
        }
        ClDesc d{};
        d.N = c.n_accels;
        d.mode = c.exec_mode;
        d.off_acc = (int64_t)H.ctype.size();
        d.off_link = (int64_t)H.bw.size();
        d.first_bad_acc = c.n_accels;
        d.first_bad_link = c.n_accels - 1;
        for (int k = 0; k < c.n_accels; ++k) {
            H.ctype.push_back(c.type_id[k]);
            H.pmax.push_back(k == 0 ? c.type_id[k] : std::max(H.pmax.back(), c.type_id[k]));
            H.cap.push_back(c.mem_capacity[k]);
            bool bad = c.mem_capacity[k] <= 0 || c.type_id[k] < 0;
            for (int q = 0; q < 4; ++q) {
                H.minm.push_back(c.min_micro[(size_t)k * 4 + q]);
                if (c.min_micro[(size_t)k * 4 + q] < 1) bad = true;
            }
            if (bad && d.first_bad_acc == c.n_accels) d.first_bad_acc = k;
        }
        for (int k = 0; k + 1 < c.n_accels; ++k) {
            H.bw.push_back(c.link_bw[k]);
            if (c.link_bw[k] <= 0 && d.first_bad_link == c.n_accels - 1) d.first_bad_link = k;
        }
        H.bw.push_back(1);   // keep every cluster's link slice non-empty
        H.desc.push_back(d);
        H.max_N = std::max(H.max_N, c.n_accels);
    }
    return true;
}

struct HostBatch {
    std::vector<QDesc> q;
    std::vector<int64_t> Mpool;
    std::vector<DPItem> whole_items;   // in query order (the device sorts its own copy)
    int64_t ncand = 0, nstage = 0, nqstage = 0, nmslot = 0;
    int max_units = 0, max_N = 0, max_nbase = 0;
};

// One chunk of the batch build: queries [i0, i1) into HB.q with offsets
// relative to the chunk and M lists in the chunk's own pool (the chunks are
// joined by build_batch_at).
struct BuildChunk {
    std::vector<int64_t> mpool;
    std::vector<DPItem> items;
    int64_t ncand = 0, nstage = 0, nqstage = 0, nmslot = 0;
    int max_units = 0, max_N = 0, max_nbase = 0;
    int err_i = -1;
    std::string err;
};

template <class QAt>
inline void build_chunk(QAt& qat, int i0, int i1, const HostNets& HN, const HostCls& HC,
                        const std::vector<int32_t>& first_bad_type, QDesc* qd, BuildChunk& ch) {
    ch.mpool.clear();
    ch.items.clear();
    ch.ncand = ch.nstage = ch.nqstage = ch.nmslot = 0;
    ch.max_units = ch.max_N = ch.max_nbase = 0;
    ch.err_i = -1;
    std::unordered_map<int64_t, std::pair<int64_t, int>> divisors;   // mini -> (offset, count)
    int64_t last_mini = -1;
    std::pair<int64_t, int> last_div{0, 0};
    auto fail_at = [&](int i, const char* what) {
        ch.err_i = i;
        ch.err = "query " + std::to_string(i) + what;
    };
    for (int i = i0; i < i1; ++i) {
        const bp_query& b = qat(i);
        if (b.network < 0 || b.network >= (int)HN.desc.size() || b.cluster < 0 || b.cluster >= (int)HC.desc.size()) {
            fail_at(i, ": network/cluster index out of range");
            return;
        }
        const NetDesc& nd = HN.desc[b.network];
        const ClDesc& cd = HC.desc[b.cluster];
        int N = b.n_stages > 0 ? b.n_stages : cd.N;
        if (N > cd.N || b.n_stages < 0) {
            fail_at(i, ": n_stages exceeds the cluster");
            return;
        }
        QDesc Q{};
        Q.net = b.network;
        Q.cl = b.cluster;
        Q.N = N;
        Q.mini = b.mini_batch;
        bool ok = nd.valid && N <= cd.first_bad_acc && N - 1 <= cd.first_bad_link && b.mini_batch >= 1;
        const bool types_ok = N < 1 || HC.pmax[cd.off_acc + N - 1] < first_bad_type[b.network];
        for (int k = 0; k < N && ok && !types_ok; ++k) {
            int32_t t = HC.ctype[cd.off_acc + k];
            if (t >= nd.T || !HN.type_ok[nd.off_tflag + t]) ok = false;
        }
        if (b.n_m > 0) {
            if (!b.m_list) {
                fail_at(i, ": m_list is NULL");
                return;
            }
            Q.m_off = (int64_t)ch.mpool.size();
            Q.nbase = b.n_m;
            for (int k = 0; k < b.n_m; ++k) {
                int64_t m = b.m_list[k];
                if (m < 1 || (b.mini_batch >= 1 && b.mini_batch % m != 0)) ok = false;
                ch.mpool.push_back(m < 1 ? 1 : m);
            }
        } else if (b.mini_batch >= 1 && b.mini_batch == last_mini) {   // sweeps repeat one mini-batch size
            Q.m_off = last_div.first;
            Q.nbase = last_div.second;
        } else if (b.mini_batch >= 1) {
            auto it = divisors.find(b.mini_batch);
            if (it == divisors.end()) {
                int64_t off = (int64_t)ch.mpool.size();
                std::vector<int64_t> small, large;
                for (int64_t d = 1; d * d <= b.mini_batch; ++d)
                    if (b.mini_batch % d == 0) {
                        small.push_back(d);
                        if (d != b.mini_batch / d) large.push_back(b.mini_batch / d);
                    }
                for (auto x : small) ch.mpool.push_back(x);
                for (auto r = large.rbegin(); r != large.rend(); ++r) ch.mpool.push_back(*r);
                it = divisors.emplace(b.mini_batch, std::make_pair(off, (int)(small.size() + large.size()))).first;
            }
            Q.m_off = it->second.first;
            Q.nbase = it->second.second;
            last_mini = b.mini_batch;
            last_div = it->second;
        }
        Q.schema_ok = ok ? 1 : 0;   // nbase kept: the output layout counts the slots
        Q.cand_off = ch.ncand;
        Q.stage_off = ch.nstage;
        Q.qstage_off = ch.nqstage;
        Q.mslot_off = ch.nmslot;
        ch.ncand += 2 * (int64_t)Q.nbase;
        ch.nstage += 2 * (int64_t)Q.nbase * N;
        ch.nqstage += N;
        ch.nmslot += Q.nbase;
        ch.max_N = std::max(ch.max_N, N);
        ch.max_nbase = std::max(ch.max_nbase, Q.nbase);
        if (ok && N >= 2) {
            ch.items.push_back(DPItem{i, -1, -1});
            ch.max_units = std::max(ch.max_units, nd.L);
        }
        qd[i] = Q;
    }
}

// qat(i): the batch's i-th query (a split part reads the caller's array
// through its index list, without a gathered copy).  Large batches are built
// in chunks on the host pool (their QDesc writes are the cost), then joined:
// the same records as one serial pass (offsets are prefix sums in query
// order; the M lists live in per-chunk runs of Mpool), and the first failing
// query's error.
template <class QAt>
inline bool build_batch_at(QAt&& qat, int nq, const HostNets& HN, const HostCls& HC, HostBatch& HB,
                           std::string& err, int chunk = 8192) {
    // reuse the vectors' capacity across calls (a sweep is re-prepared per step)
    HB.q.resize(nq);
    // per network, the smallest type id without a profile: a chain prefix
    // whose largest type id is below it passes validate_pair's type check
    // at once (otherwise the per-accelerator loop decides)
    std::vector<int32_t> first_bad_type(HN.desc.size());
    for (size_t n = 0; n < HN.desc.size(); ++n) {
        int32_t t = 0;
        while (t < HN.desc[n].T && HN.type_ok[HN.desc[n].off_tflag + t]) ++t;
        first_bad_type[n] = t;
    }
    const int CHUNK = std::max(1, chunk);
    const int nch = std::max(1, (int)(((int64_t)nq + CHUNK - 1) / CHUNK));
    // (the calling thread's chunk records, reached through a plain pointer:
    // a thread_local named inside the lambda would be each worker's own)
    static thread_local std::vector<BuildChunk> chunk_store;
    if ((int)chunk_store.size() < nch) chunk_store.resize(nch);
    BuildChunk* const chunks = chunk_store.data();
    QDesc* qd = HB.q.data();
    host_parallel_for(nch, [&](int k) {
        build_chunk(qat, k * CHUNK, (int)std::min<int64_t>(nq, (int64_t)(k + 1) * CHUNK), HN, HC, first_bad_type, qd,
                    chunks[k]);
    });
    for (int k = 0; k < nch; ++k)
        if (chunks[k].err_i >= 0) {
            err = chunks[k].err;
            return false;
        }
    // join: chunk bases, then every query's offsets
    std::vector<int64_t> bc(nch), bs(nch), bq(nch), bm(nch), bp(nch);
    HB.Mpool.clear();
    HB.whole_items.clear();
    HB.ncand = HB.nstage = HB.nqstage = HB.nmslot = 0;
    HB.max_units = HB.max_N = HB.max_nbase = 0;
    for (int k = 0; k < nch; ++k) {
        const BuildChunk& ch = chunks[k];
        bc[k] = HB.ncand;
        bs[k] = HB.nstage;
        bq[k] = HB.nqstage;
        bm[k] = HB.nmslot;
        bp[k] = (int64_t)HB.Mpool.size();
        HB.ncand += ch.ncand;
        HB.nstage += ch.nstage;
        HB.nqstage += ch.nqstage;
        HB.nmslot += ch.nmslot;
        HB.max_units = std::max(HB.max_units, ch.max_units);
        HB.max_N = std::max(HB.max_N, ch.max_N);
        HB.max_nbase = std::max(HB.max_nbase, ch.max_nbase);
        HB.Mpool.insert(HB.Mpool.end(), ch.mpool.begin(), ch.mpool.end());
        HB.whole_items.insert(HB.whole_items.end(), ch.items.begin(), ch.items.end());
    }
    if (nch > 1)
        host_parallel_for(nch - 1, [&](int k1) {
            const int k = k1 + 1;
            for (int i = k * CHUNK, e = (int)std::min<int64_t>(nq, (int64_t)(k + 1) * CHUNK); i < e; ++i) {
                QDesc& Q = qd[i];
                Q.cand_off += bc[k];
                Q.stage_off += bs[k];
                Q.qstage_off += bq[k];
                Q.mslot_off += bm[k];
                if (Q.nbase > 0) Q.m_off += bp[k];
            }
        });
    // The scheduling orders (queries by stage count, layers, network and
    // chain type signature; candidates following their query; whole-layer DP
    // items heaviest first) are built on the device (kernels.cu, k_sched_*):
    // results do not depend on them.
    return true;
}

inline bool build_batch(const bp_query* qs, int nq, const HostNets& HN, const HostCls& HC, HostBatch& HB,
                        std::string& err, int chunk = 8192) {
    return build_batch_at([qs](int i) -> const bp_query& { return qs[i]; }, nq, HN, HC, HB, err, chunk);
}

}  // namespace bpk
