"""ctypes mirror of include/bapipe_b200.h (the C ABI of the explore() path).

The structs here are byte-for-byte the ones in the header; `load_library`
opens a shared object exporting that ABI.  The product library
(`paper_2012_12544_b200/libbapipe_b200.so`, CUDA) is opened by
`product_library()`, which raises if it is missing -- there is no CPU
fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
PRODUCT_SO = os.path.join(HERE, "libbapipe_b200.so")

BP_ABI_VERSION = 1

# return codes
BP_OK, BP_BAD_INPUT, BP_CUDA_ERROR, BP_NO_DEVICE, BP_OUT_OF_MEMORY = 0, 1, 2, 3, 4
# schedule kinds (schedule_kind.hpp:15-19) and their strings (21-33)
KIND_1F1B_AS, KIND_FBP_AS, KIND_1F1B_SNO, KIND_1F1B_SO = 0, 1, 2, 3
KIND_NAMES = ("1f1b-as", "fbp-as", "1f1b-sno", "1f1b-so")
MODE_SYNC, MODE_ASYNC = 0, 1

# per-query status
Q_OK, Q_NO_FEASIBLE, Q_OVERFLOW, Q_INVALID_PLAN, Q_DOMAIN, Q_REF_UB, Q_SCHEMA = range(7)
Q_NAMES = ("ok", "no_feasible", "overflow", "invalid_plan", "domain", "ref_ub", "schema")
# per-candidate status
(C_OK, C_REJ_MIN_MICRO, C_REJ_COARSEN, C_REJ_FINETUNE, C_REJ_FINETUNE_NOCONV, C_REJ_SHAPE,
 C_REJ_MEM_POST, C_ERR_OVERFLOW, C_ERR_INVALID_PLAN, C_ERR_DOMAIN, C_REF_UB) = range(11)
C_NAMES = ("ok", "min_micro_batch", "coarsen", "finetune", "finetune_noconv", "shape",
           "mem_post", "overflow", "invalid_plan", "domain", "ref_ub")
# InvalidPlan codes
IP_RANGE, IP_FRACTION, IP_FIRST, IP_CONTIG, IP_SHARED_FULL, IP_LEAD_UNSHARED, IP_LAST, IP_COVERAGE = range(1, 9)

P64 = C.POINTER(C.c_int64)
P32 = C.POINTER(C.c_int32)


class bp_network(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("n_types", C.c_int32), ("fp_us", P64), ("bp_us", P64),
                ("weight_bytes", P64), ("out_act_bytes", P64)]


class bp_cluster(C.Structure):
    _fields_ = [("n_accels", C.c_int32), ("exec_mode", C.c_int32), ("type_id", P32),
                ("mem_capacity", P64), ("min_micro", P64), ("link_bw", P64)]


class bp_query(C.Structure):
    _fields_ = [("network", C.c_int32), ("cluster", C.c_int32), ("n_stages", C.c_int32),
                ("n_m", C.c_int32), ("mini_batch", C.c_int64), ("m_list", P64),
                ("cand_offset", C.c_int64), ("stage_offset", C.c_int64)]


class bp_rat(C.Structure):
    _fields_ = [("num", C.c_int64), ("den", C.c_int64)]


class bp_query_result(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_candidates", C.c_int32), ("n_ranked", C.c_int32),
                ("best", C.c_int32), ("first_error", C.c_int32), ("best_kind", C.c_int32),
                ("best_M", C.c_int64), ("best_micro", C.c_int64), ("best_makespan", bp_rat),
                ("best_peak_memory", bp_rat), ("best_max_bw", bp_rat)]


class bp_candidate(C.Structure):
    _fields_ = [("kind", C.c_int32), ("status", C.c_int32), ("M", C.c_int64), ("micro", C.c_int64),
                ("detail", C.c_int64), ("detail2", C.c_int64), ("rank", C.c_int32),
                ("n_stages", C.c_int32), ("heuristic", C.c_int32), ("plan_fractional", C.c_int32),
                ("makespan", bp_rat), ("est_minibatch", bp_rat), ("bubble", bp_rat),
                ("peak_memory", bp_rat), ("max_bw_demand", bp_rat), ("aux", bp_rat)]


class bp_stage(C.Structure):
    _fields_ = [("lo", C.c_int64), ("hi", C.c_int64), ("lead", bp_rat), ("trail", bp_rat),
                ("features", bp_rat), ("weights", bp_rat), ("bw_demand", bp_rat)]


class bp_best_record(C.Structure):
    _fields_ = [("makespan", bp_rat), ("peak_memory", bp_rat), ("max_bw", bp_rat),
                ("M", C.c_int64), ("kind", C.c_int32), ("valid", C.c_int32),
                ("query_id", C.c_int64), ("pad", C.c_int64)]


class bp_plan_request(C.Structure):
    _fields_ = [("network", C.c_int32), ("cluster", C.c_int32), ("kind", C.c_int32), ("n_stages", C.c_int32),
                ("M", C.c_int64), ("micro", C.c_int64), ("mini_batches", C.c_int64), ("lo", P32), ("hi", P32),
                ("lead", C.POINTER(bp_rat)), ("trail", C.POINTER(bp_rat))]


class bp_event(C.Structure):
    _fields_ = [("stage", C.c_int64), ("kind", C.c_int32), ("pad", C.c_int32), ("micro_batch", C.c_int64),
                ("start", bp_rat), ("end", bp_rat)]


class bp_timeline_result(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_int32), ("detail", C.c_int64), ("detail2", C.c_int64),
                ("aux", bp_rat), ("makespan", bp_rat), ("n_events", C.c_int64)]


class bp_estimate_result(C.Structure):
    _fields_ = [("status", C.c_int32), ("heuristic", C.c_int32), ("minibatch_time", bp_rat),
                ("bubble_fraction", bp_rat)]


assert C.sizeof(bp_query) == 48
assert C.sizeof(bp_candidate) == 152
assert C.sizeof(bp_stage) == 96
assert C.sizeof(bp_best_record) == 80
assert C.sizeof(bp_plan_request) == 72
assert C.sizeof(bp_event) == 56
assert C.sizeof(bp_timeline_result) == 64

# Every symbol include/bapipe_b200.h declares (checked by tests/test_abi.py).
PRODUCT_SYMBOLS = (
    "bp_create", "bp_destroy", "bp_last_error", "bp_abi_version", "bp_set_networks",
    "bp_set_clusters", "bp_layout", "bp_explore_batch", "bp_batch_prepare", "bp_batch_run",
    "bp_batch_fetch", "bp_batch_best", "bp_batch_free", "bp_launch_count", "bp_set_profiling",
    "bp_kernel_stats", "bp_transfer_stats", "bp_best_less", "bp_set_option", "bp_simulate_plan",
    "bp_estimate_plan",
)
BP_OPT_DEDUP = 1
BP_OPT_PLAN_ONLY = 2
BP_OPT_PRUNE_LB = 3
BP_OPT_SPLIT = 4
BP_C_PRUNED_LB = 11


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


def bind_product(lib: C.CDLL) -> C.CDLL:
    vp = C.c_void_p
    _sig(lib, "bp_create", vp, [C.c_int])
    _sig(lib, "bp_destroy", None, [vp])
    _sig(lib, "bp_last_error", C.c_char_p, [vp])
    _sig(lib, "bp_abi_version", C.c_int, [])
    _sig(lib, "bp_set_networks", C.c_int, [vp, C.POINTER(bp_network), C.c_int])
    _sig(lib, "bp_set_clusters", C.c_int, [vp, C.POINTER(bp_cluster), C.c_int])
    _sig(lib, "bp_layout", C.c_int, [vp, C.POINTER(bp_query), C.c_int, P64, P64])
    _sig(lib, "bp_explore_batch", C.c_int,
         [vp, C.POINTER(bp_query), C.c_int, C.POINTER(bp_query_result), C.POINTER(bp_candidate),
          C.POINTER(bp_stage), vp])
    _sig(lib, "bp_batch_prepare", vp, [vp, C.POINTER(bp_query), C.c_int, C.c_int, vp])
    _sig(lib, "bp_batch_run", C.c_int, [vp, vp, vp])
    _sig(lib, "bp_batch_fetch", C.c_int,
         [vp, vp, C.POINTER(bp_query_result), C.POINTER(bp_candidate), C.POINTER(bp_stage), vp])
    _sig(lib, "bp_batch_best", C.c_int, [vp, vp, vp, C.c_int64, vp])
    _sig(lib, "bp_batch_free", None, [vp, vp])
    _sig(lib, "bp_launch_count", C.c_int64, [vp])
    _sig(lib, "bp_set_profiling", C.c_int, [vp, C.c_int])
    _sig(lib, "bp_set_option", C.c_int, [vp, C.c_int, C.c_int64])
    _sig(lib, "bp_kernel_stats", C.c_int,
         [vp, C.c_char_p, C.POINTER(C.c_double), P64, C.POINTER(C.c_double), C.c_int])
    _sig(lib, "bp_transfer_stats", C.c_int, [vp, P64, P64])
    _sig(lib, "bp_best_less", C.c_int, [C.POINTER(bp_best_record), C.POINTER(bp_best_record)])
    _sig(lib, "bp_simulate_plan", C.c_int,
         [vp, C.POINTER(bp_plan_request), C.POINTER(bp_timeline_result), C.POINTER(bp_event), C.c_int64,
          C.POINTER(bp_rat), C.POINTER(bp_rat), C.POINTER(bp_rat)])
    _sig(lib, "bp_estimate_plan", C.c_int,
         [vp, C.POINTER(bp_plan_request), C.POINTER(bp_estimate_result), C.POINTER(bp_stage), P32])
    return lib


_PRODUCT = None


def product_library() -> C.CDLL:
    """Open the CUDA product library; raise if it is absent (no fallback)."""
    global _PRODUCT
    if _PRODUCT is None:
        if not os.path.exists(PRODUCT_SO):
            raise RuntimeError(
                f"{PRODUCT_SO} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the explore() path has no CPU fallback)")
        _PRODUCT = bind_product(C.CDLL(PRODUCT_SO))
        if _PRODUCT.bp_abi_version() != BP_ABI_VERSION:
            raise RuntimeError("libbapipe_b200.so ABI version mismatch")
    return _PRODUCT
