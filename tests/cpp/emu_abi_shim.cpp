// emu_abi_shim.cpp -- TEST HARNESS ONLY.  Implements the subset of the
// include/bapipe_b200.h entry points that include/bapipe_b200/explorer.hpp
// calls, over the CPU replay in tests/emu/emu.cpp, so that the C++ drop-in's
// host logic (type-id flattening, result rebuilding, exception mapping) is
// checked on machines without a GPU.  Linked statically into a test
// executable; never part of libbapipe_b200.so, which has no CPU path.
#include <string>
#include <vector>

#include "../emu/emu.cpp"

struct bp_ctx {
    std::vector<bp_network> nets;
    std::vector<bp_cluster> cls;
    HostNets hn;
    HostCls hc;
    std::string err;
};

static std::string g_err = "ok";

extern "C" {
bp_ctx* bp_create(int) { return new bp_ctx(); }
void bp_destroy(bp_ctx* c) { delete c; }
const char* bp_last_error(const bp_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }
int bp_abi_version(void) { return BP_ABI_VERSION; }

// The pointers stay owned by the caller until bp_explore_batch returns, which
// is how explorer.hpp uses them.
int bp_set_networks(bp_ctx* c, const bp_network* n, int k) {
    c->nets.assign(n, n + k);
    return build_nets(n, k, c->hn, c->err, true) ? BP_OK : BP_BAD_INPUT;
}
int bp_set_clusters(bp_ctx* c, const bp_cluster* cl, int k) {
    c->cls.assign(cl, cl + k);
    return build_clusters(cl, k, c->hc, c->err) ? BP_OK : BP_BAD_INPUT;
}
int bp_layout(bp_ctx* c, bp_query* q, int nq, int64_t* tc, int64_t* ts) {
    HostBatch hb;
    if (!build_batch(q, nq, c->hn, c->hc, hb, c->err)) return BP_BAD_INPUT;
    for (int i = 0; i < nq; ++i) {
        q[i].cand_offset = hb.q[i].cand_off;
        q[i].stage_offset = hb.q[i].stage_off;
    }
    *tc = hb.ncand;
    *ts = hb.nstage;
    return BP_OK;
}
int bp_set_option(bp_ctx*, int option, int64_t value) {
    if (option == BP_OPT_PLAN_ONLY) bpemu_set_plan_only(value != 0);
    return option == BP_OPT_DEDUP || option == BP_OPT_PLAN_ONLY ? BP_OK : BP_BAD_INPUT;
}
int bp_simulate_plan(bp_ctx* c, const bp_plan_request* q, bp_timeline_result* res, bp_event* events, int64_t cap,
                     bp_rat* hw, bp_rat* ws, bp_rat* busy) {
    return bpemu_plan(c->nets.data(), (int)c->nets.size(), c->cls.data(), (int)c->cls.size(), q, res, events, cap,
                      hw, ws, busy, nullptr, nullptr, nullptr);
}
int bp_estimate_plan(bp_ctx* c, const bp_plan_request* q, bp_estimate_result* res, bp_stage* st, int32_t* inf) {
    return bpemu_plan(c->nets.data(), (int)c->nets.size(), c->cls.data(), (int)c->cls.size(), q, nullptr, nullptr,
                      0, nullptr, nullptr, nullptr, res, st, inf);
}
int bp_explore_batch(bp_ctx* c, const bp_query* q, int nq, bp_query_result* res, bp_candidate* cand,
                     bp_stage* stages, void*) {
    uint64_t work = 0;
    return bpemu_explore_batch(c->nets.data(), (int)c->nets.size(), c->cls.data(), (int)c->cls.size(), q, nq, res,
                               cand, stages, &work);
}
}
