"""Full-scale parity: every one of the 2^20 C5 candidates against the reference.

tests/golden/c5_cand_ref.npz holds, for every candidate of the full C5 sweep,
a 64-bit digest of its bp_candidate record and its per-stage bp_stage records
as the reference itself produced them (oracle/_ref: bapipe::explore() for the
ranking, then the per-(kind, M) replay of explorer.hpp:96-132;
tests/golden/make_c5_cand.py), plus every query's bp_query_result.  The CUDA
product must reproduce every digest:

  * the whole sweep as one batch, batch dedup on and off;
  * the sweep cut into 8 shards, run as separate batches, both class-aligned
    (the multi-GPU strong-scaling split, workloads.shard_classes) and by the
    per-query LPT split (workloads.shard_queries), which cuts dedup classes;
  * five copies of the sweep in one batch (5 x 2^20 > 2^22 candidates: the
    batch-level indices of the prune representative and every work list)
    give five copies of the 1x records.

The two queries where the reference has undefined behaviour (memory
fine-tune's collapse emptying a stage, reported as REF_UB) are compared too:
their records are the product's REF_UB report and the reference harness's.
"""
import os

import numpy as np
import pytest
from conftest import ROOT
from digest import candidate_digests

from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.problem import RESULT_DTYPE

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden", "c5_cand_ref.npz")


@pytest.fixture(scope="module")
def gold():
    if not os.path.exists(GOLD):
        pytest.skip("c5_cand_ref.npz not generated")
    z = np.load(GOLD)
    return {"digest": z["digest"], "status": z["status"], "res": z["res"].view(RESULT_DTYPE)}


@pytest.fixture(scope="module")
def ex():
    from paper_2012_12544_b200.runtime import Explorer
    e = Explorer(0)
    yield e
    e.close()


@pytest.fixture(scope="module")
def c5():
    return W.config_c5()


def check(got_digest, want_digest, status, what):
    bad = np.nonzero(got_digest != want_digest)[0]
    assert bad.size == 0, (f"{what}: {bad.size} of {want_digest.size} candidates differ from the reference; "
                           f"first {bad[:8].tolist()} (reference status {status[bad[:8]].tolist()})")


def global_candidates(p, idx):
    """Global candidate indices (in p's layout) of the queries idx, in order."""
    q = p.queries
    return np.concatenate([np.arange(q["cand_offset"][i], q["cand_offset"][i] + p.n_candidates[i]) for i in idx])


@pytest.mark.parametrize("dedup,split", [(True, True), (False, True), (True, False), (True, 2)],
                         ids=["dedup_split", "no_dedup", "one_batch", "two_parts"])
def test_c5_every_candidate_matches_reference(ex, c5, gold, dedup, split):
    """BP_OPT_SPLIT on (the default: the N = 64, 32 and 24 queries and the rest
    run as four concurrent parts), off, and two parts (N = 64 and the rest);
    batch dedup on and off."""
    ex.dedup(dedup)
    ex.split(split)
    try:
        res, cand, st = ex.explore(c5, details=True)
    finally:
        ex.dedup(True)
        ex.split(True)
    assert res.tobytes() == gold["res"].tobytes(), "per-query records differ"
    check(candidate_digests(c5, cand, st), gold["digest"], gold["status"], "C5 one batch")


@pytest.mark.parametrize("how", ["class", "lpt"])
def test_c5_shards_match_reference(ex, c5, gold, how):
    shards = W.shard_classes(c5, 8) if how == "class" else W.shard_queries(
        [c5.networks[i].L for i in c5.queries["network"]], c5.queries["n_stages"], 8)
    assert sorted(np.concatenate(shards).tolist()) == list(range(c5.queries.size))
    got = np.zeros_like(gold["digest"])
    for idx in shards:
        s = W.subset(c5, idx)
        res, cand, st = ex.explore(s, details=True)
        assert res.tobytes() == gold["res"][idx].tobytes(), f"{how} shard: per-query records differ"
        got[global_candidates(c5, idx)] = candidate_digests(s, cand, st)
    check(got, gold["digest"], gold["status"], f"C5 in 8 {how} shards")


def test_c5_five_copies_in_one_batch(ex, c5):
    one_res, one_cand, _ = ex.explore(c5, details="candidates")
    five = W.subset(c5, np.tile(np.arange(c5.queries.size), 5))
    assert five.total_candidates == 5 * c5.total_candidates > (1 << 22)
    res, cand, _ = ex.explore(five, details="candidates")
    for k in range(5):
        assert res[k * c5.queries.size:(k + 1) * c5.queries.size].tobytes() == one_res.tobytes(), k
        c = cand[k * c5.total_candidates:(k + 1) * c5.total_candidates]
        if c.tobytes() != one_cand.tobytes():
            bad = np.nonzero((c.view(np.uint8).reshape(c.size, -1) !=
                              one_cand.view(np.uint8).reshape(c.size, -1)).any(axis=1))[0]
            raise AssertionError(f"copy {k}: {bad.size} candidate records differ from the 1x batch, "
                                 f"first {bad[:5].tolist()}")


def test_c5_lower_bound_pruning_keeps_every_query_result(ex, c5, gold):
    """BP_OPT_PRUNE_LB: the full sweep's per-query records are
    the reference's; every skipped candidate is feasible in the unpruned run
    with a makespan above its query's best."""
    from fractions import Fraction as Fr

    from paper_2012_12544_b200.abi import BP_C_PRUNED_LB
    ex.prune_lb(True)
    try:
        res, cand, _ = ex.explore(c5, details="candidates")
    finally:
        ex.prune_lb(False)
    assert res.tobytes() == gold["res"].tobytes()
    pruned = np.nonzero(cand["status"] == BP_C_PRUNED_LB)[0]
    assert pruned.size > 0
    _, full, _ = ex.explore(c5, details="candidates")
    keep = cand["status"] != BP_C_PRUNED_LB
    assert cand[keep]["status"].tobytes() == full[keep]["status"].tobytes()
    assert cand[keep]["makespan"].tobytes() == full[keep]["makespan"].tobytes()
    assert np.all(full["status"][pruned] == 0)
    qi = np.searchsorted(c5.queries["cand_offset"], pruned, side="right") - 1
    ok = res["status"][qi] == 0          # queries that escaped an error report no best
    pruned, qi = pruned[ok], qi[ok]
    for i, q in zip(pruned[:: max(1, pruned.size // 4000)], qi[:: max(1, pruned.size // 4000)]):
        b = res[q]["best_makespan"]
        m = full[i]["makespan"]
        assert Fr(int(m["num"]), int(m["den"])) > Fr(int(b["num"]), int(b["den"]))
