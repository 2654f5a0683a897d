"""Parity of the CUDA product (libbapipe_b200.so, sm_100a) with the reference.

Every test calls through the C ABI.  Bit-exact on every output record: cut
points, fractions, schedule kind, M, ranked order, rejection reasons, exact
rational makespan / estimate / memory / bandwidth values, and the query
outcome (including the reference's overflow_error / InvalidPlan escapes and
its undefined-behaviour cases, which must be reported, not computed).
"""
import os

import numpy as np
import pytest
import scenarios
from conftest import ROOT, assert_same

from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.problem import BEST_DTYPE, RESULT_DTYPE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    from paper_2012_12544_b200.runtime import Explorer
    e = Explorer(0)
    yield e
    e.close()


@pytest.fixture(scope="module")
def c5(ex):
    p = W.config_c5()
    res, cand, _ = ex.explore(p, details=False)
    return p, res


@pytest.mark.parametrize("name", [n for n, _ in scenarios.SCENARIOS])
def test_product_matches_reference_fixtures(ex, golden, name):
    p = scenarios.build(name)
    res, cand, st = ex.explore(p, details=True)
    g = golden[name]
    assert_same(res, g["res"], name + "/res")
    assert_same(cand, g["cand"], name + "/cand")
    if "stages" in g:
        assert_same(st, g["stages"], name + "/stages")


@pytest.mark.parametrize("seed", [31, 32, 33])
def test_product_matches_oracle_on_random_batches(ex, port, seed):
    p = W.random_problem(seed, n_queries=120, max_L=40, max_N=16, cap_range=(500, 80000), bw_range=(1, 800),
                         act_max=3000)
    for x, y, part in zip(ex.explore(p), port.explore(p), ("res", "cand", "stages")):
        assert_same(x, y, f"seed {seed} {part}")


def test_full_c5_sweep_matches_reference(c5):
    """All 65,536 queries of the 2^20-candidate sweep against the reference's
    own explore() run on the full sweep (tests/golden/make_c5_full.py)."""
    path = os.path.join(ROOT, "tests", "golden", "c5_full_ref.npz")
    if not os.path.exists(path):
        pytest.skip("c5_full_ref.npz not generated")
    p, res = c5
    want = np.load(path)["res"].view(RESULT_DTYPE)
    assert np.array_equal(res["status"], want["status"])
    ok = want["status"] == 0
    for f in ("best_kind", "best_M", "best_micro", "best_makespan", "best_peak_memory", "best_max_bw"):
        assert res[f][ok].tobytes() == want[f][ok].tobytes(), f


def test_full_c5_sweep_properties(ex, c5):
    """Size-independent properties at full size: determinism, the split
    (device-resident) API agrees with the host API, every ranked list is
    sorted by the reference's 5 keys, and the device best-record reduction
    matches its host mirror."""
    p, res = c5
    res2, _, _ = ex.explore(p, details=False)
    assert res.tobytes() == res2.tobytes()
    b = ex.prepare(p, details=False)
    ex.run(b)
    res3, _, _ = ex.fetch(b, p)
    assert res.tobytes() == res3.tobytes()
    import torch

    from paper_2012_12544_b200.sweep import best_record_from_results
    rec = torch.zeros(BEST_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ex.best(b, rec.data_ptr())
    torch.cuda.synchronize()
    sub = np.arange(0, p.queries.size)
    want = best_record_from_results(res, sub)
    assert rec.cpu().numpy().tobytes() == want.tobytes()
    ex.free(b)


def test_dedup_off_is_identical(ex, c5):
    """BP_OPT_DEDUP only shares work: with it off every query / candidate is
    evaluated on its own and every output byte is the same (full sweep:
    per-query records; a sample: candidate and stage records too)."""
    p, res = c5
    s = scenarios.c5_sample(61)
    on = ex.explore(s, details=True)
    ex.dedup(False)
    try:
        off_full, _, _ = ex.explore(p, details=False)
        off = ex.explore(s, details=True)
    finally:
        ex.dedup(True)
    assert res.tobytes() == off_full.tobytes()
    for x, y, part in zip(on, off, ("res", "cand", "stages")):
        assert_same(x, y, "dedup on/off " + part)


def test_ranked_lists_sorted_on_c5_sample(ex):
    from fractions import Fraction as Fr
    p = scenarios.c5_sample(257)
    res, cand, _ = ex.explore(p, details=True)
    for qi in range(p.queries.size):
        lo = int(p.queries["cand_offset"][qi])
        cs = cand[lo:lo + int(p.n_candidates[qi])]
        ranked = sorted([c for c in cs if c["rank"] >= 0], key=lambda c: c["rank"])
        keys = [(Fr(int(c["makespan"]["num"]), int(c["makespan"]["den"])),
                 Fr(int(c["peak_memory"]["num"]), int(c["peak_memory"]["den"])),
                 Fr(int(c["max_bw_demand"]["num"]), int(c["max_bw_demand"]["den"])), int(c["M"]), int(c["kind"]))
                for c in ranked]
        assert keys == sorted(keys)
        assert (res[qi]["status"] == 0) == bool(ranked)


def test_plan_only_matches_explore(ex):
    """BP_OPT_PLAN_ONLY (`bapipe plan`: balance_partition + estimate, no
    min-micro filter, no simulation) agrees with the full explore on every
    candidate both evaluate: the same plan, estimate and prune-phase outcome;
    candidates explore drops at simulate() are feasible plans here."""
    import ctypes as C
    from paper_2012_12544_b200 import abi
    sim_phase = {0, 7, 8, 9}                     # OK, or an error raised by simulate()
    for p in (scenarios.c5_sample(61), W.random_problem(3, n_queries=80, max_L=30, max_N=12,
                                                          cap_range=(1000, 60000), bw_range=(1, 500),
                                                          act_max=3000)):
        _, full, full_st = ex.explore(p, details=True)
        assert ex.lib.bp_set_option(ex.ctx, abi.BP_OPT_PLAN_ONLY, 1) == 0
        try:
            _, po, po_st = ex.explore(p, details=True)
        finally:
            ex.lib.bp_set_option(ex.ctx, abi.BP_OPT_PLAN_ONLY, 0)
        n_ok = 0
        for qi in range(p.queries.size):
            lo = int(p.queries["cand_offset"][qi])
            N = int(p.queries["n_stages"][qi]) or p.clusters[int(p.queries["cluster"][qi])].N
            so = int(p.queries["stage_offset"][qi])
            for i in range(lo, lo + int(p.n_candidates[qi])):
                f, g = full[i], po[i]
                if f["status"] == 1:                 # min-micro: not evaluated by explore
                    continue
                if f["status"] in sim_phase and g["status"] == 0:
                    if f["status"] == 0:
                        n_ok += 1
                        for k in ("est_minibatch", "bubble", "heuristic", "peak_memory", "max_bw_demand"):
                            assert f[k].tobytes() == g[k].tobytes(), (qi, i, k)
                        s0 = so + (i - lo) * N
                        assert full_st[s0:s0 + N].tobytes() == po_st[s0:s0 + N].tobytes(), (qi, i)
                    continue
                assert f["status"] == g["status"] and f["detail"] == g["detail"], (qi, i, f, g)
        assert n_ok > 0


def test_graph_replay_equals_launch_by_launch(ex):
    """A prepared batch runs as a CUDA graph (captured on its first run,
    replayed after); a profiled run launches kernel by kernel.  Same records,
    same own-kernel count, on a split-size C5 sample (two parts) and on a
    small batch; and a replay after the inputs changed (same sizes: the graph
    is reused) gives the new inputs' results."""
    for p in (W.subset(W.config_c5(models=8), np.arange(4096)), scenarios.c5_sample(257)):
        b = ex.prepare(p, details=True)
        outs, counts = [], []
        for prof in (False, False, True):
            ex.profiling(prof)
            n0 = ex.launches()
            ex.run(b)
            counts.append(ex.launches() - n0)
            outs.append(ex.fetch(b, p, details=True))
        ex.profiling(False)
        ex.free(b)
        assert counts[0] == counts[1] == counts[2]
        for o in outs[1:]:
            for x, y, part in zip(outs[0], o, ("res", "cand", "stages")):
                assert_same(x, y, "graph replay " + part)
    # same sizes, other queries: 8 models' worth of the sweep, two different model ranges
    a = W.config_c5(models=8)
    z = W.config_c5(models=8, model_base=40)
    want = ex.explore(z, details=False)[0]
    got_a = ex.explore(a, details=False)[0]
    got_z = ex.explore(z, details=False)[0]
    assert got_z.tobytes() == want.tobytes()
    assert got_a.tobytes() != got_z.tobytes()


def test_pinned_outputs_equal_pageable(ex):
    """bp_explore_batch into page-locked caller buffers (bench.py's e2e legs):
    the records equal those of pageable buffers, on a split-size C5 sample,
    twice in a row (buffers reused).  (Writing each part's records straight
    into the page-locked buffers from the scatter kernels, zero-copy, was
    measured: no gain for the query records, 2x slower for the candidate
    records -- fine-grained PCIe writes.)"""
    p = W.subset(W.config_c5(models=8), np.arange(4096))
    want = ex.explore(p, details="candidates")
    out = p.alloc_outputs("candidates", pinned=True)
    for _ in range(2):
        out[0][:] = np.zeros(1, dtype=out[0].dtype)
        out[1][:] = np.zeros(1, dtype=out[1].dtype)
        got = ex.explore(p, details="candidates", out=out)
        assert got[0].tobytes() == want[0].tobytes()
        assert got[1].tobytes() == want[1].tobytes()
