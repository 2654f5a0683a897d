"""TEST HARNESS for the one-plan entry points (bp_simulate_plan /
bp_estimate_plan): random plans, the three
implementations behind one call shape -- the product (runtime.Explorer), the
host replay of the same kernel code (tests/emu) and the reference itself
(oracle/_ref, simulator.hpp:264-274 / cost_models.hpp:124-166) -- and a
field-by-field comparison of their outputs."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests", "emu"))

from paper_2012_12544_b200 import abi  # noqa: E402

KIND_SYNC = (2, 3)
KIND_ASYNC = (0, 1)


def random_plan(rng, L, N, den_max=64, big=False):
    """A plan of N stages over L layers: random cuts, some boundaries shared
    with complementary fractions; occasionally broken on purpose (the
    reference's validate_plan then decides).  big: huge co-prime
    denominators, to drive the exact Rat paths into overflow."""
    lo, hi, lead, trail = [], [], [], []
    cuts = sorted(rng.choice(np.arange(1, L), size=min(N - 1, L - 1), replace=False).tolist()) if L > 1 else []
    while len(cuts) < N - 1:
        cuts.append(cuts[-1] if cuts else 1)
    start = 1
    bounds = []
    for k in range(N):
        end = cuts[k] if k < N - 1 else L
        bounds.append([start, max(end, start)])
        start = end + 1
    for k in range(N):
        lo.append(bounds[k][0])
        hi.append(bounds[k][1])
        lead.append((1, 1))
        trail.append((1, 1))
    for k in range(N - 1):   # share the boundary layer of stages k, k+1
        if rng.random() < 0.6 and hi[k] < L and lo[k + 1] <= hi[k + 1]:
            d = int(rng.integers(1000003, 2000003)) if big else int(rng.integers(2, den_max + 1))
            n = int(rng.integers(1, d))
            g = np.gcd(n, d)
            lo[k + 1] = hi[k]
            trail[k] = (n // g, d // g)
            lead[k + 1] = ((d - n) // g, d // g)
    if rng.random() < 0.15:   # break something
        k = int(rng.integers(0, N))
        what = int(rng.integers(0, 5))
        if what == 0:
            hi[k] = L + 1
        elif what == 1:
            trail[k] = (3, 2)
        elif what == 2:
            lead[k] = (1, 3)
        elif what == 3 and k + 1 < N:       # a gap: not contiguous
            lo[k + 1] = hi[k] + 2
        elif k + 1 < N and lo[k + 1] == hi[k]:   # shared layer, fractions not summing to 1
            lead[k + 1] = (1, 7) if lead[k + 1] != (1, 7) else (2, 7)
    return lo, hi, lead, trail


def request(net, cl, kind, n_stages, M, micro, mini, plan):
    lo, hi, lead, trail = plan
    n = len(lo)
    buf = ((C.c_int32 * n)(*lo), (C.c_int32 * n)(*hi), (abi.bp_rat * n)(*[abi.bp_rat(a, b) for a, b in lead]),
           (abi.bp_rat * n)(*[abi.bp_rat(a, b) for a, b in trail]))
    q = abi.bp_plan_request(network=net, cluster=cl, kind=kind, n_stages=n, M=M, micro=micro, mini_batches=mini,
                            lo=buf[0], hi=buf[1], lead=buf[2], trail=buf[3])
    return q, buf


def capacity(q):
    n, M = q.n_stages, max(q.M, 0)
    return q.mini_batches * (2 * n * M + 4 * (n - 1) * M)


def _rat(r):
    return (r.num, r.den)


def sim_record(res, ev, hw, ws, busy, n):
    out = {"status": res.status}
    if res.status == 8:
        out["invalid"] = (res.detail, res.detail2, _rat(res.aux) if res.detail == 8 else None)
    if res.status == 0:
        out["makespan"] = _rat(res.makespan)
        out["events"] = [(e.stage, e.kind, e.micro_batch, _rat(e.start), _rat(e.end)) for e in ev[:res.n_events]]
        out["highwater"] = [_rat(x) for x in hw[:n]]
        out["wstatic"] = [_rat(x) for x in ws[:n]]
        out["busy"] = [_rat(x) for x in busy[:max(n - 1, 0)]]
    return out


def est_record(res, st, inf, n):
    out = {"status": res.status}
    if res.status == 0:
        out["est"] = (res.heuristic, _rat(res.minibatch_time), _rat(res.bubble_fraction))
        out["stages"] = [(_rat(s.features), _rat(s.weights), _rat(s.bw_demand), int(f)) for s, f in zip(st[:n], inf)]
    return out


class Ref:
    """oracle/_ref: the reference's simulate() / estimate()."""

    def __init__(self, problem):
        from pyoracle import REF_SO
        self.lib = C.CDLL(REF_SO)
        self.nets, self.cls = problem.c_networks(), problem.c_clusters()
        self.nn, self.nc = len(problem.networks), len(problem.clusters)

    def simulate(self, q):
        cap = capacity(q)
        res = abi.bp_timeline_result()
        ev = (abi.bp_event * max(cap, 1))()
        n = q.n_stages
        hw, ws, busy = (abi.bp_rat * n)(), (abi.bp_rat * n)(), (abi.bp_rat * max(n - 1, 1))()
        rc = self.lib.bpref_simulate_plan(self.nets, self.nn, self.cls, self.nc, C.byref(q), C.byref(res), ev,
                                          C.c_int64(cap), hw, ws, busy)
        assert rc == 0
        return sim_record(res, ev, hw, ws, busy, n)

    def estimate(self, q):
        n = q.n_stages
        res = abi.bp_estimate_result()
        st = (abi.bp_stage * n)()
        inf = (C.c_int32 * n)()
        rc = self.lib.bpref_estimate_plan(self.nets, self.nn, self.cls, self.nc, C.byref(q), C.byref(res), st, inf)
        assert rc == 0
        return est_record(res, st, inf, n)


class Emu:
    """tests/emu: the kernel code replayed on the host."""

    def __init__(self, problem):
        import pyemu
        if not os.path.exists(pyemu.SO):
            pyemu.build()
        self.lib = C.CDLL(pyemu.SO)
        self.nets, self.cls = problem.c_networks(), problem.c_clusters()
        self.nn, self.nc = len(problem.networks), len(problem.clusters)

    def simulate(self, q):
        cap = capacity(q)
        res = abi.bp_timeline_result()
        ev = (abi.bp_event * max(cap, 1))()
        n = q.n_stages
        hw, ws, busy = (abi.bp_rat * n)(), (abi.bp_rat * n)(), (abi.bp_rat * max(n - 1, 1))()
        rc = self.lib.bpemu_plan(self.nets, self.nn, self.cls, self.nc, C.byref(q), C.byref(res), ev,
                                 C.c_int64(cap), hw, ws, busy, None, None, None)
        assert rc == 0
        return sim_record(res, ev, hw, ws, busy, n)

    def estimate(self, q):
        n = q.n_stages
        res = abi.bp_estimate_result()
        st = (abi.bp_stage * n)()
        inf = (C.c_int32 * n)()
        rc = self.lib.bpemu_plan(self.nets, self.nn, self.cls, self.nc, C.byref(q), None, None, C.c_int64(0), None,
                                 None, None, C.byref(res), st, inf)
        assert rc == 0
        return est_record(res, st, inf, n)


class Product:
    """libbapipe_b200.so on the GPU."""

    def __init__(self, problem):
        from paper_2012_12544_b200.runtime import Explorer
        self.ex = Explorer(0)
        self.ex.load(problem)

    def simulate(self, q):
        res, ev, hw, ws, busy = self.ex.plan_call(q, "simulate", capacity(q))
        return sim_record(res, ev, hw, ws, busy, q.n_stages)

    def estimate(self, q):
        res, st, inf = self.ex.plan_call(q, "estimate")
        return est_record(res, st, inf, q.n_stages)


def cases(problem, seed, count, big_every=5):
    """(request, buffers) for random plans over the problem's queries."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        qi = int(rng.integers(0, problem.queries.size))
        q = problem.queries[qi]
        net, cl = int(q["network"]), int(q["cluster"])
        cls = problem.clusters[cl]
        N = cls.N   # the whole cluster: simulate() checks the plan against it
        L = problem.networks[net].L
        kinds = KIND_ASYNC if cls.mode == 1 else KIND_SYNC
        kind = int(kinds[int(rng.integers(0, 2))])
        M = int(rng.integers(1, 9)) if rng.random() > 0.04 else 0   # M < 1: InvalidPlan("M >= 1 required")
        micro = int(rng.integers(1, 5))
        mini = 1 if rng.random() < 0.8 else 2
        n_plan = N - 1 if (N > 1 and rng.random() < 0.05) else N   # a valid plan, wrong stage count
        plan = random_plan(rng, L, n_plan, big=(i % big_every == big_every - 1))
        out.append(request(net, cl, kind, N, M, micro, mini, plan))
    return out
