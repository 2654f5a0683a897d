"""Batch of explore() queries as structure-of-arrays numpy buffers.

`Problem` owns the network tables, cluster tables and the query array in the
exact memory layout of include/bapipe_b200.h, so a batch of 65,536 queries is
handed to any implementation of the ABI (the CUDA product, or the test-only
oracles) without per-query Python work.  Result buffers are numpy structured
arrays with the dtypes below (byte-identical to the C structs).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi

RAT = np.dtype([("num", "<i8"), ("den", "<i8")])
QUERY_DTYPE = np.dtype([("network", "<i4"), ("cluster", "<i4"), ("n_stages", "<i4"), ("n_m", "<i4"),
                        ("mini_batch", "<i8"), ("m_list", "<u8"), ("cand_offset", "<i8"),
                        ("stage_offset", "<i8")])
RESULT_DTYPE = np.dtype([("status", "<i4"), ("n_candidates", "<i4"), ("n_ranked", "<i4"),
                         ("best", "<i4"), ("first_error", "<i4"), ("best_kind", "<i4"),
                         ("best_M", "<i8"), ("best_micro", "<i8"), ("best_makespan", RAT),
                         ("best_peak_memory", RAT), ("best_max_bw", RAT)])
CAND_DTYPE = np.dtype([("kind", "<i4"), ("status", "<i4"), ("M", "<i8"), ("micro", "<i8"),
                       ("detail", "<i8"), ("detail2", "<i8"), ("rank", "<i4"), ("n_stages", "<i4"),
                       ("heuristic", "<i4"), ("plan_fractional", "<i4"), ("makespan", RAT),
                       ("est_minibatch", RAT), ("bubble", RAT), ("peak_memory", RAT),
                       ("max_bw_demand", RAT), ("aux", RAT)])
STAGE_DTYPE = np.dtype([("lo", "<i8"), ("hi", "<i8"), ("lead", RAT), ("trail", RAT),
                        ("features", RAT), ("weights", RAT), ("bw_demand", RAT)])
BEST_DTYPE = np.dtype([("makespan", RAT), ("peak_memory", RAT), ("max_bw", RAT), ("M", "<i8"),
                       ("kind", "<i4"), ("valid", "<i4"), ("query_id", "<i8"), ("pad", "<i8")])

assert QUERY_DTYPE.itemsize == C.sizeof(abi.bp_query)
assert RESULT_DTYPE.itemsize == C.sizeof(abi.bp_query_result)
assert CAND_DTYPE.itemsize == C.sizeof(abi.bp_candidate)
assert STAGE_DTYPE.itemsize == C.sizeof(abi.bp_stage)
assert BEST_DTYPE.itemsize == C.sizeof(abi.bp_best_record)


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


@dataclass
class Network:
    """NetworkProfile (profiles.hpp:46-51) as SoA.  fp/bp are [n_types, L];
    0 marks a missing accelerator type."""
    fp: np.ndarray
    bp: np.ndarray
    w: np.ndarray
    a: np.ndarray
    name: str = "net"

    def __post_init__(self):
        self.fp = _i64(np.atleast_2d(self.fp))
        self.bp = _i64(np.atleast_2d(self.bp))
        self.w = _i64(self.w)
        self.a = _i64(self.a)
        assert self.fp.shape == self.bp.shape and self.fp.shape[1] == self.w.size == self.a.size

    @property
    def L(self):
        return self.w.size

    @property
    def T(self):
        return self.fp.shape[0]


@dataclass
class Cluster:
    """ClusterSpec (profiles.hpp:67-73) as SoA; min_micro is [N, 4]."""
    mode: int
    types: np.ndarray
    cap: np.ndarray
    bw: np.ndarray
    min_micro: np.ndarray | None = None

    def __post_init__(self):
        self.types = np.ascontiguousarray(np.asarray(self.types, dtype=np.int32))
        self.cap = _i64(self.cap)
        self.bw = _i64(self.bw)
        n = self.types.size
        if self.min_micro is None:
            self.min_micro = np.ones((n, 4), dtype=np.int64)
        self.min_micro = _i64(self.min_micro).reshape(n, 4)

    @property
    def N(self):
        return self.types.size


@dataclass
class Problem:
    networks: list = field(default_factory=list)
    clusters: list = field(default_factory=list)
    queries: np.ndarray | None = None
    m_lists: list = field(default_factory=list)    # keeps explicit M lists alive
    name: str = ""

    # -- building ------------------------------------------------------------
    def add_network(self, net: Network) -> int:
        self.networks.append(net)
        return len(self.networks) - 1

    def add_cluster(self, cl: Cluster) -> int:
        self.clusters.append(cl)
        return len(self.clusters) - 1

    def set_queries(self, network, cluster, n_stages, mini_batch, m_lists=None):
        network = np.asarray(network, dtype=np.int32).ravel()
        nq = network.size
        q = np.zeros(nq, dtype=QUERY_DTYPE)
        q["network"] = network
        q["cluster"] = np.broadcast_to(np.asarray(cluster, dtype=np.int32), (nq,))
        q["n_stages"] = np.broadcast_to(np.asarray(n_stages, dtype=np.int32), (nq,))
        q["mini_batch"] = np.broadcast_to(np.asarray(mini_batch, dtype=np.int64), (nq,))
        self.m_lists = []
        if m_lists is not None:
            for i, ml in enumerate(m_lists):
                if ml is None:
                    continue
                arr = _i64(ml)
                self.m_lists.append(arr)
                q["n_m"][i] = arr.size
                q["m_list"][i] = arr.ctypes.data
        self.queries = q
        self.layout()
        return q

    def n_stages_of(self, i):
        q = self.queries[i]
        return int(q["n_stages"]) if q["n_stages"] > 0 else self.clusters[int(q["cluster"])].N

    def layout(self):
        """Dense cand_offset / stage_offset (same rule as bp_layout)."""
        q = self.queries
        nb = np.empty(q.size, dtype=np.int64)
        cache = {}
        for i in range(q.size):
            if q["n_m"][i] > 0:
                nb[i] = q["n_m"][i]
            else:
                mb = int(q["mini_batch"][i])
                if mb not in cache:
                    cache[mb] = sum(1 for m in range(1, mb + 1) if mb % m == 0) if mb >= 1 else 0
                nb[i] = cache[mb]
        ncand = 2 * nb
        nst = np.where(q["n_stages"] > 0, q["n_stages"],
                       np.array([c.N for c in self.clusters], dtype=np.int64)[q["cluster"]])
        q["cand_offset"] = np.concatenate([[0], np.cumsum(ncand)[:-1]])
        q["stage_offset"] = np.concatenate([[0], np.cumsum(ncand * nst)[:-1]])
        self.total_candidates = int(ncand.sum())
        self.total_stages = int((ncand * nst).sum())
        self.n_candidates = ncand

    # -- ctypes views ----------------------------------------------------------
    def _cached(self, name, arrays, build):
        """ctypes descriptor arrays hold raw pointers into the numpy arrays:
        rebuild them only when an array object was replaced (e.g. by pin())."""
        c = getattr(self, name, None)
        if c is not None and len(c[0]) == len(arrays) and all(x is y for x, y in zip(c[0], arrays)):
            return c[1]
        out = build()
        setattr(self, name, (arrays, out))
        return out

    def c_networks(self):
        arrays = [x for n in self.networks for x in (n.fp, n.bp, n.w, n.a)]
        return self._cached("_c_nets", arrays, self._build_c_networks)

    def c_clusters(self):
        arrays = [x for c in self.clusters for x in (c.types, c.cap, c.bw, c.min_micro)]
        return self._cached("_c_cls", arrays, self._build_c_clusters)

    def _build_c_networks(self):
        arr = (abi.bp_network * len(self.networks))()
        for i, n in enumerate(self.networks):
            arr[i].n_layers = n.L
            arr[i].n_types = n.T
            arr[i].fp_us = n.fp.ctypes.data_as(abi.P64)
            arr[i].bp_us = n.bp.ctypes.data_as(abi.P64)
            arr[i].weight_bytes = n.w.ctypes.data_as(abi.P64)
            arr[i].out_act_bytes = n.a.ctypes.data_as(abi.P64)
        return arr

    def _build_c_clusters(self):
        arr = (abi.bp_cluster * len(self.clusters))()
        for i, c in enumerate(self.clusters):
            arr[i].n_accels = c.N
            arr[i].exec_mode = c.mode
            arr[i].type_id = c.types.ctypes.data_as(abi.P32)
            arr[i].mem_capacity = c.cap.ctypes.data_as(abi.P64)
            arr[i].min_micro = c.min_micro.ctypes.data_as(abi.P64)
            arr[i].link_bw = (c.bw.ctypes.data_as(abi.P64) if c.bw.size else
                              C.cast(C.c_void_p(0), abi.P64))
        return arr

    def c_queries(self):
        return self.queries.ctypes.data_as(C.POINTER(abi.bp_query))

    def pin(self):
        """Move every host array into page-locked memory (torch pinned
        buffers) so host<->device copies run at full PCIe/NVLink-C2C rate."""
        import torch

        def pinned(a):
            if a.dtype.names is None:
                t = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), pin_memory=True)
                out = t.numpy()
            else:
                t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
                out = t.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
            out[...] = a
            self._pinned.append(t)
            return out

        self._pinned = []
        for n in self.networks:
            n.fp, n.bp, n.w, n.a = pinned(n.fp), pinned(n.bp), pinned(n.w), pinned(n.a)
        for c in self.clusters:
            c.types, c.cap, c.bw, c.min_micro = pinned(c.types), pinned(c.cap), pinned(c.bw), pinned(c.min_micro)
        ml = [pinned(m) for m in self.m_lists]
        q = pinned(self.queries)
        j = 0
        for i in range(q.size):
            if q["n_m"][i] > 0:
                q["m_list"][i] = ml[j].ctypes.data
                j += 1
        self.m_lists, self.queries = ml, q
        return self

    def alloc_outputs(self, details=True, pinned=False):
        """details: True = query, candidate and stage records; "candidates" =
        query and candidate records (no per-stage plans); False = query
        records only."""
        if pinned:   # page-locked host buffers (kept alive on the problem), for reuse across calls
            import torch

            def buf(n, dt, name):
                t = torch.empty(max(1, n) * dt.itemsize, dtype=torch.uint8, pin_memory=True)
                setattr(self, name, t)
                return t.numpy().view(dt)[:n]
            res = buf(self.queries.size, RESULT_DTYPE, "_pinned_res")
            cand = buf(self.total_candidates, CAND_DTYPE, "_pinned_cand") if details else None
            st = (buf(self.total_stages, STAGE_DTYPE, "_pinned_st")
                  if details and details != "candidates" else None)
            return res, cand, st
        res = np.zeros(self.queries.size, dtype=RESULT_DTYPE)
        cand = np.zeros(self.total_candidates, dtype=CAND_DTYPE) if details else None
        st = np.zeros(self.total_stages, dtype=STAGE_DTYPE) if details and details != "candidates" else None
        return res, cand, st


def ptr(a, ctype):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))
