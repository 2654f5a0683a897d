"""TEST INFRASTRUCTURE: Python loaders for the CPU checkers.

  RefOracle     oracle/_ref/libbapipe_ref.so  -- the reference itself
  PortOracle    oracle/_build/libbapipe_oracle.so -- the C restatement

Both run a `paper_2012_12544_b200.problem.Problem` and return numpy result
arrays with the product ABI's layout.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2012_12544_b200 import abi
from paper_2012_12544_b200.problem import Problem, ptr

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libbapipe_ref.so")
REF_FAST_SO = os.path.join(HERE, "_ref", "libbapipe_ref_fast.so")   # -O3 -march=native, timing only
PORT_SO = os.path.join(HERE, "_build", "libbapipe_oracle.so")


def build(ref=True):
    """Compile the checkers (ref needs /root/reference; skipped if absent)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available():
    return os.path.exists(REF_SO)


def port_available():
    return os.path.exists(PORT_SO)


class _Base:
    def _common(self, p: Problem):
        return p.c_networks(), p.c_clusters()


class RefOracle(_Base):
    kind = "reference"

    def __init__(self, fast=False):
        """fast: the timing build (no bounds checks, so no REF_UB detection);
        falls back to the checking build when it is absent."""
        so = REF_FAST_SO if fast and os.path.exists(REF_FAST_SO) else REF_SO
        if not os.path.exists(so):
            raise RuntimeError(f"{so} not built (make -C oracle ref)")
        self.lib = C.CDLL(so)
        self.build = "-O3 -march=native" if so == REF_FAST_SO else "-O3 -D_GLIBCXX_ASSERTIONS"
        vp = C.c_void_p
        self.lib.bpref_explore_batch.restype = C.c_int
        self.lib.bpref_explore_batch.argtypes = [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, C.c_int]
        self.lib.bpref_explore_timed.restype = C.c_int
        self.lib.bpref_explore_timed.argtypes = [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int]

    def explore(self, p: Problem, details=True, threads=1):
        nets, cls = self._common(p)
        res, cand, st = p.alloc_outputs(details)
        rc = self.lib.bpref_explore_batch(C.cast(nets, C.c_void_p), len(p.networks), C.cast(cls, C.c_void_p),
                                          len(p.clusters), p.queries.ctypes.data, p.queries.size,
                                          res.ctypes.data, None if cand is None else cand.ctypes.data,
                                          None if st is None else st.ctypes.data, threads)
        assert rc == 0, rc
        return res, cand, st

    def explore_timed(self, p: Problem, threads=1, query_index=None):
        """explore() only (no replay), on `threads` host threads."""
        nets, cls = self._common(p)
        q = p.queries if query_index is None else np.ascontiguousarray(p.queries[query_index])
        res = np.zeros(q.size, dtype=p.alloc_outputs(False)[0].dtype)
        rc = self.lib.bpref_explore_timed(C.cast(nets, C.c_void_p), len(p.networks), C.cast(cls, C.c_void_p),
                                          len(p.clusters), q.ctypes.data, q.size, res.ctypes.data, threads)
        assert rc == 0, rc
        return res


class PortOracle(_Base):
    kind = "port"

    def __init__(self):
        if not os.path.exists(PORT_SO):
            raise RuntimeError(f"{PORT_SO} not built (make -C oracle oracle)")
        self.lib = C.CDLL(PORT_SO)
        vp = C.c_void_p
        L = self.lib
        L.bpo_explore_batch.restype = C.c_int
        L.bpo_explore_batch.argtypes = [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp]
        L.bpo_partition.restype = C.c_int
        L.bpo_partition.argtypes = [vp, vp, C.c_int, C.c_int64, C.c_int, vp, vp, vp]
        L.bpo_simulate_chain.restype = C.c_int
        L.bpo_simulate_chain.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_int64, vp]
        for n in ("bpo_minibatch_time", "bpo_bubble_fraction"):
            f = getattr(L, n)
            f.restype = C.c_int
            f.argtypes = [C.c_int, C.c_int64, C.c_int64, abi.bp_rat, abi.bp_rat, abi.bp_rat,
                          C.POINTER(abi.bp_rat)]

    def explore(self, p: Problem, details=True, threads=1):
        nets, cls = self._common(p)
        res, cand, st = p.alloc_outputs(details)
        rc = self.lib.bpo_explore_batch(C.cast(nets, C.c_void_p), len(p.networks), C.cast(cls, C.c_void_p),
                                        len(p.clusters), p.queries.ctypes.data, p.queries.size,
                                        res.ctypes.data, None if cand is None else cand.ctypes.data,
                                        None if st is None else st.ctypes.data)
        assert rc == 0, rc
        return res, cand, st

    def partition(self, net, cl, n_stages=0, a_th=-1):
        """inter_layer_partition (or the coarse overload when a_th >= 0)."""
        N = n_stages or cl.N
        lo = np.zeros(N, dtype=np.int64)
        hi = np.zeros(N, dtype=np.int64)
        t = np.zeros(1, dtype=np.int64)
        p = Problem()
        p.add_network(net)
        p.add_cluster(cl)
        nets, cls = p.c_networks(), p.c_clusters()
        st = self.lib.bpo_partition(C.cast(nets, C.c_void_p), C.cast(cls, C.c_void_p), N, max(a_th, 0),
                                    1 if a_th >= 0 else 0, lo.ctypes.data, hi.ctypes.data, t.ctypes.data)
        return st, lo, hi, int(t[0])

    def simulate_chain(self, kind, F, B, SR, M, a=None, w=None):
        from fractions import Fraction
        n = len(F)
        RA = np.dtype([("num", "<i8"), ("den", "<i8")])
        f = np.array([(Fraction(x).numerator, Fraction(x).denominator) for x in F], dtype=RA)
        b = np.array([(Fraction(x).numerator, Fraction(x).denominator) for x in B], dtype=RA)
        ww = np.array([(Fraction(x).numerator, Fraction(x).denominator) for x in (w or [0] * n)], dtype=RA)
        sr = np.asarray(list(SR) + [0], dtype=np.int64)
        aa = np.asarray(a or [0] * n, dtype=np.int64)
        out = np.zeros(1, dtype=RA)
        st = self.lib.bpo_simulate_chain(kind, n, f.ctypes.data, b.ctypes.data, sr.ctypes.data, aa.ctypes.data,
                                         ww.ctypes.data, M, out.ctypes.data)
        return st, Fraction(int(out[0]["num"]), int(out[0]["den"])) if st == 0 else None

    def closed_form(self, which, kind, M, N, F, B, SR):
        from fractions import Fraction

        def br(x):
            x = Fraction(x)
            return abi.bp_rat(x.numerator, x.denominator)
        out = abi.bp_rat()
        f = self.lib.bpo_bubble_fraction if which == "bubble" else self.lib.bpo_minibatch_time
        st = f(kind, M, N, br(F), br(B), br(SR), C.byref(out))
        return st, Fraction(out.num, out.den) if st == 0 else None
