"""Python handle on the CUDA product library (libbapipe_b200.so).

`Explorer` owns one bp_ctx on one device.  It is plumbing for tests and the
benchmark: every candidate evaluation happens in the sm_100a kernels behind
the C ABI.  There is no CPU fallback -- constructing an Explorer without a
usable B200 raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .problem import BEST_DTYPE, Problem


class Explorer:
    def __init__(self, device: int = 0):
        self.lib = abi.product_library()
        self.ctx = self.lib.bp_create(device)
        if not self.ctx:
            raise RuntimeError("bp_create failed: " + self.lib.bp_last_error(None).decode())
        self._loaded = None

    def close(self):
        if self.ctx:
            self.lib.bp_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != abi.BP_OK:
            raise RuntimeError(f"{what}: rc={rc}: {self.lib.bp_last_error(self.ctx).decode()}")

    def load(self, p: Problem, force=False):
        """Upload p's network and cluster tables (skipped if already loaded)."""
        if self._loaded is p and not force:
            return
        nets, cls = p.c_networks(), p.c_clusters()
        self._check(self.lib.bp_set_networks(self.ctx, nets, len(p.networks)), "bp_set_networks")
        self._check(self.lib.bp_set_clusters(self.ctx, cls, len(p.clusters)), "bp_set_clusters")
        self._keep = (nets, cls)
        self._loaded = p

    def explore(self, p: Problem, details=True, stream=None, out=None):
        """explore() for every query of p: host buffers in, host buffers out.
        out: (res, cand, st) from p.alloc_outputs (e.g. pinned, reused across
        calls) instead of fresh arrays."""
        self.load(p)
        res, cand, st = out if out is not None else p.alloc_outputs(details)
        rc = self.lib.bp_explore_batch(self.ctx, p.c_queries(), p.queries.size,
                                       res.ctypes.data_as(C.POINTER(abi.bp_query_result)),
                                       None if cand is None else cand.ctypes.data_as(C.POINTER(abi.bp_candidate)),
                                       None if st is None else st.ctypes.data_as(C.POINTER(abi.bp_stage)),
                                       stream)
        self._check(rc, "bp_explore_batch")
        return res, cand, st

    # -- split form (device-resident timing) ---------------------------------
    def prepare(self, p: Problem, details=False, stream=None):
        self.load(p)
        b = self.lib.bp_batch_prepare(self.ctx, p.c_queries(), p.queries.size, 1 if details else 0, stream)
        if not b:
            raise RuntimeError("bp_batch_prepare: " + self.lib.bp_last_error(self.ctx).decode())
        return b

    def run(self, batch, stream=None):
        self._check(self.lib.bp_batch_run(self.ctx, batch, stream), "bp_batch_run")

    def fetch(self, batch, p: Problem, details=False, stream=None):
        res, cand, st = p.alloc_outputs(details)
        self._check(self.lib.bp_batch_fetch(self.ctx, batch, res.ctypes.data_as(C.POINTER(abi.bp_query_result)),
                                            None if cand is None else cand.ctypes.data_as(C.POINTER(abi.bp_candidate)),
                                            None if st is None else st.ctypes.data_as(C.POINTER(abi.bp_stage)),
                                            stream), "bp_batch_fetch")
        return res, cand, st

    def best(self, batch, dev_ptr: int, query_base=0, stream=None):
        self._check(self.lib.bp_batch_best(self.ctx, batch, C.c_void_p(dev_ptr), query_base, stream), "bp_batch_best")

    def free(self, batch):
        self.lib.bp_batch_free(self.ctx, batch)

    # -- instrumentation -----------------------------------------------------
    def launches(self) -> int:
        return int(self.lib.bp_launch_count(self.ctx))

    def transfers(self):
        h, d = C.c_int64(0), C.c_int64(0)
        self.lib.bp_transfer_stats(self.ctx, C.byref(h), C.byref(d))
        return h.value, d.value

    def profiling(self, on=True):
        self.lib.bp_set_profiling(self.ctx, 1 if on else 0)

    def dedup(self, on=True):
        """BP_OPT_DEDUP: share identical subproblems within a batch (default
        on; results are identical either way)."""
        rc = self.lib.bp_set_option(self.ctx, abi.BP_OPT_DEDUP, 1 if on else 0)
        if rc != 0:
            raise RuntimeError(self.lib.bp_last_error(self.ctx).decode())

    def prune_lb(self, on=True):
        """BP_OPT_PRUNE_LB: skip simulating scaled-integer candidates whose
        makespan lower bound exceeds their query's best (per-query results
        identical; skipped candidates get BP_C_PRUNED_LB)."""
        rc = self.lib.bp_set_option(self.ctx, abi.BP_OPT_PRUNE_LB, 1 if on else 0)
        if rc != 0:
            raise RuntimeError(self.lib.bp_last_error(self.ctx).decode())

    def split(self, on=True):
        """BP_OPT_SPLIT: run large batches as concurrent parts by stage count
        (default on: up to four parts; an int k >= 2 asks for up to k;
        results are identical either way)."""
        value = (1 if on else 0) if isinstance(on, bool) else int(on)
        rc = self.lib.bp_set_option(self.ctx, abi.BP_OPT_SPLIT, value)
        if rc != 0:
            raise RuntimeError(self.lib.bp_last_error(self.ctx).decode())

    def plan_call(self, req, which, cap=0):
        """bp_simulate_plan (which='simulate') or bp_estimate_plan on a
        bp_plan_request for this context's loaded problem.  Returns the raw
        result records (see tests/timeline_util.py)."""
        n = req.n_stages
        if which == "simulate":
            res = abi.bp_timeline_result()
            ev = (abi.bp_event * max(cap, 1))()
            hw, ws, busy = (abi.bp_rat * n)(), (abi.bp_rat * n)(), (abi.bp_rat * max(n - 1, 1))()
            self._check(self.lib.bp_simulate_plan(self.ctx, C.byref(req), C.byref(res), ev, cap, hw, ws, busy),
                        "bp_simulate_plan")
            return res, ev, hw, ws, busy
        res = abi.bp_estimate_result()
        st = (abi.bp_stage * n)()
        inf = (C.c_int32 * n)()
        self._check(self.lib.bp_estimate_plan(self.ctx, C.byref(req), C.byref(res), st, inf), "bp_estimate_plan")
        return res, st, inf

    def kernel_stats(self):
        cap = 64
        names = C.create_string_buffer(48 * cap)
        ms = (C.c_double * cap)()
        launches = (C.c_int64 * cap)()
        work = (C.c_double * cap)()
        n = self.lib.bp_kernel_stats(self.ctx, names, ms, launches, work, cap)
        out = {}
        for i in range(n):
            nm = names.raw[48 * i:48 * (i + 1)].split(b"\0", 1)[0].decode()
            out[nm] = {"ms": ms[i], "launches": launches[i], "work": work[i]}
        return out


def best_less(a, b) -> bool:
    """Host copy of bp_best_less (deterministic argmin order)."""
    lib = abi.product_library()
    ra, rb = abi.bp_best_record(), abi.bp_best_record()
    C.memmove(C.byref(ra), np.ascontiguousarray(a).ctypes.data, C.sizeof(ra))
    C.memmove(C.byref(rb), np.ascontiguousarray(b).ctypes.data, C.sizeof(rb))
    return bool(lib.bp_best_less(C.byref(ra), C.byref(rb)))


def empty_best(n=1):
    return np.zeros(n, dtype=BEST_DTYPE)
