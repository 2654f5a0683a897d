"""The oracle (oracle/bapipe_oracle.c) pinned to the reference.

(a) the reference's own golden vectors restated from proj/tests/*.cpp;
(b) the compiled reference (oracle/_ref) on the golden scenarios and on
    seeded random batches.
"""
from fractions import Fraction as Fr
from itertools import combinations

import numpy as np
import pytest
import scenarios
from conftest import assert_same

from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.abi import KIND_1F1B_AS, KIND_1F1B_SNO, KIND_1F1B_SO, KIND_FBP_AS

KINDS = (KIND_1F1B_AS, KIND_FBP_AS, KIND_1F1B_SNO, KIND_1F1B_SO)


def test_mt19937_64_matches_std():
    # std::mt19937_64 default seed 5489: 10000th output (C++ standard [rand.predef])
    assert int(W.MT19937_64(5489).draw(10000)[-1]) == 9981545732273789042


# ---- cost_models.hpp closed forms: test_cost_models.cpp:9-49
def test_minibatch_time_closed_forms(port):
    want = {KIND_1F1B_AS: 300, KIND_FBP_AS: 300, KIND_1F1B_SNO: 324, KIND_1F1B_SO: 308}
    for k, v in want.items():
        assert port.closed_form("minibatch", k, 8, 3, 10, 20, 2) == (0, Fr(v))


def test_bubble_fractions(port):
    assert port.closed_form("bubble", KIND_1F1B_AS, 8, 3, 10, 20, 2)[1] == Fr(2, 10)
    assert port.closed_form("bubble", KIND_FBP_AS, 8, 3, 10, 20, 2)[1] == Fr(1, 5)
    assert port.closed_form("bubble", KIND_1F1B_SNO, 8, 3, 10, 20, 2)[1] == Fr(2 * 34 + 4 * 4, 324)
    assert port.closed_form("bubble", KIND_1F1B_SO, 8, 3, 10, 20, 2)[1] == Fr(2 * 34, 308)
    for k in KINDS:
        assert port.closed_form("bubble", k, 4, 1, 10, 20, 2)[1] == 0
    # the documented SNO non-monotonicity counterexample (46-49)
    assert port.closed_form("bubble", KIND_1F1B_SNO, 12, 2, 13, 29, 4)[1] == Fr(5, 33)
    assert port.closed_form("bubble", KIND_1F1B_SNO, 13, 2, 13, 29, 4)[1] == Fr(7, 46)


# ---- simulator.hpp: test_simulator.cpp:34-129
def test_simulate_chain_pinned(port):
    assert port.simulate_chain(KIND_1F1B_AS, [10, 10], [10, 10], [0], 2) == (0, 60)
    assert port.simulate_chain(KIND_1F1B_SNO, [7], [11], [], 5) == (0, 90)
    for k, v in ((KIND_1F1B_AS, 300), (KIND_FBP_AS, 300), (KIND_1F1B_SNO, 324), (KIND_1F1B_SO, 308)):
        assert port.simulate_chain(k, [10] * 3, [20] * 3, [2, 2], 8) == (0, v)
    assert port.simulate_chain(KIND_1F1B_SNO, [10, 10], [20, 20], [5], 1) == (0, 70)
    assert port.simulate_chain(KIND_1F1B_AS, [10, 10], [20, 20], [5], 1) == (0, 60)
    assert port.simulate_chain(KIND_1F1B_AS, [Fr(21, 2), 10], [10, 10], [0], 1)[1].denominator == 2


def test_simulator_matches_closed_forms_on_balanced_grid(port):
    """acceptance.cpp criterion 1 (seeded grid, SO gated on SR <= min(F, B))."""
    rng = np.random.default_rng(1)
    for _ in range(150):
        M, N = int(rng.integers(1, 17)), int(rng.integers(1, 9))
        F, B, SR = int(rng.integers(1, 51)), int(rng.integers(1, 51)), int(rng.integers(0, 11))
        for k in KINDS:
            sim = port.simulate_chain(k, [F] * N, [B] * N, [SR] * (N - 1), M)[1]
            form = port.closed_form("minibatch", k, M, N, F, B, SR)[1]
            if k != KIND_1F1B_SO or SR <= min(F, B):
                assert sim == form
            else:
                assert sim >= form


# ---- partition_units vs exhaustive enumeration: test_partitioner.cpp:68-96
def brute_minmax(net, types):
    L, N = net.L, len(types)
    c = net.fp + net.bp
    best = None
    for cuts in combinations(range(1, L), N - 1):
        b = (0,) + cuts + (L,)
        worst = max(int(c[types[n], b[n]:b[n + 1]].sum()) for n in range(N))
        best = worst if best is None else min(best, worst)
    return best


def test_partition_matches_exhaustive_enumeration(port):
    rng = np.random.default_rng(20240817)
    for _ in range(200):
        N = int(rng.integers(1, 5))
        L = N + int(rng.integers(0, 13 - N))
        net = W.Network(rng.integers(1, 51, size=(2, L)), rng.integers(1, 51, size=(2, L)),
                        rng.integers(0, 1000, size=L), rng.integers(0, 1000, size=L))
        types = [int(t) for t in (rng.integers(0, 2, size=N) if rng.random() < 0.5 else np.zeros(N, int))]
        cl = W.Cluster(0, types, [10**9] * N, [10**6] * (N - 1))
        st, lo, hi, t_opt = port.partition(net, cl)
        assert st == 0
        assert lo[0] == 1 and hi[-1] == L and all(lo[1:] == hi[:-1] + 1)
        got = max(int((net.fp + net.bp)[types[n], lo[n] - 1:hi[n]].sum()) for n in range(N))
        assert got == t_opt == brute_minmax(net, types)


def test_partition_rejects_more_stages_than_layers(port):
    st, *_ = port.partition(W.uniform_network(2, 10, 10, 0, 0), W.Cluster(0, [0, 0, 0], [10**9] * 3, [10**6] * 2))
    assert st == 5   # BP_C_REJ_SHAPE (InfeasibleShape, partition.hpp:115-117)


# ---- the whole explore() path against the reference's own outputs
@pytest.mark.parametrize("name", [n for n, _ in scenarios.SCENARIOS])
def test_oracle_matches_reference_fixtures(port, golden, name):
    p = scenarios.build(name)
    res, cand, st = port.explore(p, details=True)
    g = golden[name]
    assert_same(res, g["res"], name + "/res")
    assert_same(cand, g["cand"], name + "/cand")
    if "stages" in g:
        assert_same(st, g["stages"], name + "/stages")


def test_reference_scenarios_readable(golden):
    """Spot-check the fixtures against the reference unit tests' own numbers."""
    from paper_2012_12544_b200.problem import CAND_DTYPE  # noqa: F401
    r = golden["explorer_abundant_so"]
    assert r["res"][0]["best_kind"] == KIND_1F1B_SO
    assert (r["res"][0]["best_makespan"]["num"], r["res"][0]["best_makespan"]["den"]) == (184, 1)
    sno = [c for c in r["cand"] if c["kind"] == KIND_1F1B_SNO][0]
    assert int(sno["makespan"]["num"]) == 188                                        # test_explorer.cpp:79-94
    assert golden["explorer_memory_tight_sno"]["res"][0]["best_kind"] == KIND_1F1B_SNO   # 60-77
    assert golden["explorer_m1_tie_sno"]["res"][0]["best_kind"] == KIND_1F1B_SNO        # 96-106
    a = golden["explorer_async_fbp"]
    assert (a["res"][0]["best_kind"], a["res"][0]["best_M"], a["res"][0]["best_micro"]) == (KIND_FBP_AS, 8, 1)
    as_st = [int(c["status"]) for c in a["cand"] if c["kind"] == KIND_1F1B_AS]
    assert as_st.count(1) == 2 and as_st.count(3) == 2                                  # 108-132
    assert golden["explorer_all_rejected"]["res"][0]["status"] == 1                     # NoFeasiblePlan 161-172
    st = golden["refine_31_2"]["stages"]
    assert st[0]["trail"]["den"] == 20 or st[1]["lead"]["den"] == 20                    # 9/20 split -> 31/2 each
    assert golden["partition_comm_coarse"]["stages"][0]["hi"] == 2                      # test_partitioner.cpp:279
    assert golden["partition_comm_infeasible"]["res"][0]["status"] == 1                 # 283-285


def test_oracle_matches_live_reference_on_random_batches(port, ref):
    for seed in (11, 12):
        p = W.random_problem(seed, n_queries=80)
        a = port.explore(p, details=True)
        b = ref.explore(p, details=True)
        for x, y, part in zip(a, b, ("res", "cand", "stages")):
            assert_same(x, y, f"seed {seed} {part}")
