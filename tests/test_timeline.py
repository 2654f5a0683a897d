"""One plan's full-timeline simulate and estimate (
timeline.cuh / bp_simulate_plan / bp_estimate_plan) against the reference's
own simulate() (simulator.hpp:264-274: every event, makespan, feature
high-water, static weights, link busy fractions) and estimate()
(cost_models.hpp:124-166), field by field, on random plans: fractional
boundaries, broken plans (validate_plan's codes), stage-count mismatches,
two mini-batches, and huge co-prime denominators that overflow.
  * CPU: the kernel code replayed on the host (tests/emu);
  * GPU: libbapipe_b200.so."""
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import timeline_util as T  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402


def problems():
    yield "rand", W.random_problem(7, n_queries=40, max_L=24, max_N=8, cap_range=(1000, 60000), bw_range=(1, 500),
                                   act_max=3000)
    yield "heavy", W.random_problem(107, n_queries=20, max_L=40, max_N=16, cap_range=(1000, 60000),
                                    bw_range=(1, 50), act_max=100000)


def compare(impl_cls, count):
    if not os.path.exists(os.path.join(T.ROOT, "oracle", "_ref", "libbapipe_ref.so")):
        pytest.skip("oracle/_ref not built")
    stats = {"ok": 0, "invalid": 0, "overflow": 0, "other": 0}
    codes = set()
    for name, p in problems():
        ref, impl = T.Ref(p), impl_cls(p)
        for i, (q, _buf) in enumerate(T.cases(p, seed={"rand": 11, "heavy": 23}[name], count=count)):
            want, got = ref.simulate(q), impl.simulate(q)
            assert got == want, (name, i, {k: (got.get(k), want.get(k)) for k in want if got.get(k) != want.get(k)})
            st = want["status"]
            if st == 8:
                codes.add(want["invalid"][0])
            stats["ok" if st == 0 else "invalid" if st == 8 else "overflow" if st == 7 else "other"] += 1
            if st == 0:
                want_e, got_e = ref.estimate(q), impl.estimate(q)
                assert got_e == want_e, (name, i, got_e, want_e)
    # the random plans must exercise every outcome
    print("timeline outcomes", stats, "invalid codes", sorted(codes))
    assert stats["ok"] > 0 and stats["invalid"] > 0 and stats["overflow"] > 0, stats
    assert {1, 2, 4, 8, 9, 10}.issubset(codes), codes   # range, fraction, gap, coverage, stage count, M


def test_timeline_emulator_matches_reference():
    compare(T.Emu, 60)


@pytest.mark.gpu
def test_timeline_b200_matches_reference():
    compare(T.Product, 60)
