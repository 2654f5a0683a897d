"""The reference's acceptance gate (proj/tests/acceptance.cpp) run against the
CUDA product, for the criteria its public entry points expose:

* c1 (acceptance.cpp:41-80): the simulated makespan of a balanced chain
  equals the closed-form mini-batch time (cost_models.hpp:50-63), 1f1b-so
  gated on SR <= min(F, B) (a lower bound otherwise), and the pinned values
  AS = FBP = 300, SNO = 324, SO = 308 of balanced(3, 10, 20, 2) at M = 8;
* c4 (183-236): the simulated per-stage feature high-water equals
  min(M, warm-up depth) * a (the clamped law) everywhere;
* c5 (239-289): SO <= SNO where the overlap assumption holds, async <= both
  sync kinds when SR > 0;
* c6 (291-343): the explorer picks 1f1b-sno / 1f1b-so / fbp-as in the three
  constructed scenarios.

Every simulation is bp_simulate_plan on the device (balanced chains: one
layer per stage, fp = F, bp = B, activation a = SR over 1-byte/us links at
micro-batch 1, so link_sr = SR exactly); c6 is bp_explore_batch.  The seeded
grids are this file's own (numpy), as wide as the reference's.
"""
from fractions import Fraction

import numpy as np
import pytest

import timeline_util as T
from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.abi import MODE_ASYNC, MODE_SYNC
from paper_2012_12544_b200.problem import Cluster, Problem

pytestmark = pytest.mark.gpu
AS, FBP, SNO, SO = 0, 1, 2, 3


@pytest.fixture(scope="module")
def ex():
    from paper_2012_12544_b200.runtime import Explorer
    e = Explorer(0)
    yield e
    e.close()


def minibatch_time(kind, M, N, F, B, SR):   # cost_models.hpp:50-63
    base = (M + N - 1) * (F + B)
    if kind == SNO:
        return base + (N + M - 2 - -(-(M - 1) // N)) * 2 * SR
    if kind == SO:
        return base + (N - 1) * 2 * SR
    return base


def warmup_depth(kind, N, i):   # schedule_kind.hpp: doubled warm-up for fbp-as / 1f1b-so
    return (N - i + 1) * (2 if kind in (FBP, SO) else 1)


class Balanced:
    """One problem holding balanced chains: network (F, B, a) with N layers,
    an async and a sync cluster of N accelerators, 1-byte/us links."""

    def __init__(self, ex):
        self.ex, self.p, self.nets, self.cls = ex, Problem(name="balanced"), {}, {}

    def net(self, N, F, B, a):
        k = (N, F, B, a)
        if k not in self.nets:
            self.nets[k] = self.p.add_network(W.uniform_network(N, F, B, 0, a))
        return self.nets[k]

    def cluster(self, N, mode):
        k = (N, mode)
        if k not in self.cls:
            self.cls[k] = self.p.add_cluster(Cluster(mode, [0] * N, [1 << 40] * N, [1] * (N - 1)))
        return self.cls[k]

    def prepare(self, cases):
        for N, F, B, SR, _ in cases:
            self.net(N, F, B, SR)
            self.cluster(N, MODE_ASYNC)
            self.cluster(N, MODE_SYNC)
        self.p.set_queries([0], 0, 0, 1)
        self.ex.load(self.p, force=True)

    def simulate(self, kind, N, F, B, SR, M):
        plan = (list(range(1, N + 1)), list(range(1, N + 1)), [(1, 1)] * N, [(1, 1)] * N)
        mode = MODE_ASYNC if kind in (AS, FBP) else MODE_SYNC
        q, keep = T.request(self.net(N, F, B, SR), self.cluster(N, mode), kind, N, M, 1, 1, plan)
        res, ev, hw, ws, busy = self.ex.plan_call(q, "simulate", T.capacity(q))
        assert res.status == 0, (kind, N, F, B, SR, M, res.status)
        return Fraction(res.makespan.num, res.makespan.den), [Fraction(h.num, h.den) for h in hw[:N]]


def grid(seed, count):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(1, 9)), int(rng.integers(1, 51)), int(rng.integers(1, 51)), int(rng.integers(0, 11)),
             int(rng.integers(1, 17))) for _ in range(count)]


def test_c1_makespan_equals_closed_form(ex):
    cases = grid(1, 600) + [(3, 10, 20, 2, 8)]
    b = Balanced(ex)
    b.prepare(cases)
    exact = 0
    for N, F, B, SR, M in cases:
        for k in (AS, FBP, SNO, SO):
            sim = b.simulate(k, N, F, B, SR, M)[0]
            form = minibatch_time(k, M, N, F, B, SR)
            if k != SO or SR <= min(F, B):
                exact += 1
                assert sim == form, (k, N, F, B, SR, M, sim, form)
            else:
                assert sim >= form, (k, N, F, B, SR, M, sim, form)
    assert exact >= 2000
    assert [b.simulate(k, 3, 10, 20, 2, 8)[0] for k in (AS, FBP, SNO, SO)] == [300, 300, 324, 308]


def test_c4_feature_highwater_clamped_law(ex):
    cases = [c for c in grid(4, 300) if c[3] > 0]
    b = Balanced(ex)
    b.prepare(cases)
    for N, F, B, a, M in cases:
        for k in (AS, FBP, SNO, SO):
            hw = b.simulate(k, N, F, B, a, M)[1]
            for i in range(1, N + 1):
                # stage i holds the activation entering it (stage 1: its own output, simulator.hpp:248-262)
                assert hw[i - 1] == min(M, warmup_depth(k, N, i)) * a, (k, N, M, i, hw[i - 1])


def test_c5_schedule_orderings(ex):
    cases = grid(5, 400)
    b = Balanced(ex)
    b.prepare(cases)
    for N, F, B, SR, M in cases:
        so, sno = b.simulate(SO, N, F, B, SR, M)[0], b.simulate(SNO, N, F, B, SR, M)[0]
        asy = b.simulate(AS, N, F, B, SR, M)[0]
        assert minibatch_time(SO, M, N, F, B, SR) <= minibatch_time(SNO, M, N, F, B, SR)
        if SR <= min(F, B):
            assert so <= sno, (N, F, B, SR, M)
        if SR > 0:
            assert asy <= sno and asy <= so, (N, F, B, SR, M)


def test_c6_explorer_scenarios(ex):
    p = Problem(name="c6")
    p.add_network(W.uniform_network(3, 10, 20, 100, 50))
    p.add_cluster(Cluster(MODE_SYNC, [0] * 3, [400, 1000000, 1000000], [50, 50]))      # memory-tight sync
    p.add_cluster(Cluster(MODE_SYNC, [0] * 3, [1000000] * 3, [50, 50]))                 # abundant sync
    mm = np.ones((3, 4), dtype=np.int64)
    mm[:, AS] = 4                                                                         # 1f1b-as floor
    p.add_cluster(Cluster(MODE_ASYNC, [0] * 3, [600] * 3, [50, 50], mm))                 # tight async
    p.set_queries([0, 0, 0], [0, 1, 2], 0, [4, 4, 8], m_lists=[[4], [4], None])
    res, _, _ = ex.explore(p, details=False)
    assert res["status"].tolist() == [0, 0, 0]
    assert res["best_kind"].tolist() == [SNO, SO, FBP]
    assert int(res["best_M"][2]) == 8
