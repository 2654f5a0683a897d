"""The C ABI boundary: the product library loads and exports every symbol
include/bapipe_b200.h declares; record layouts agree with the header; without
a GPU the product refuses to run (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2012_12544_b200 import abi
from paper_2012_12544_b200.problem import BEST_DTYPE, CAND_DTYPE, QUERY_DTYPE, RESULT_DTYPE, STAGE_DTYPE

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "bapipe_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bp_[a-z_]+)\s*\(", src)))


def test_header_declarations_are_the_abi_list():
    assert declared_functions() == sorted(abi.PRODUCT_SYMBOLS)


def test_product_library_exports_every_declared_symbol():
    lib = abi.product_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.bp_abi_version() == abi.BP_ABI_VERSION


def test_record_layouts_match_header():
    assert QUERY_DTYPE.itemsize == C.sizeof(abi.bp_query) == 48
    assert RESULT_DTYPE.itemsize == C.sizeof(abi.bp_query_result)
    assert CAND_DTYPE.itemsize == C.sizeof(abi.bp_candidate) == 152
    assert STAGE_DTYPE.itemsize == C.sizeof(abi.bp_stage) == 96
    assert BEST_DTYPE.itemsize == C.sizeof(abi.bp_best_record) == 80
    for f, _ in abi.bp_candidate._fields_:
        assert getattr(abi.bp_candidate, f).offset == CAND_DTYPE.fields[f][1], f


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="a GPU is present")
def test_no_cpu_fallback_without_gpu():
    from paper_2012_12544_b200.runtime import Explorer
    with pytest.raises(RuntimeError, match="bp_create failed"):
        Explorer(0)


def test_best_record_order():
    from paper_2012_12544_b200.runtime import best_less
    a = np.zeros(1, BEST_DTYPE)[0]
    b = np.zeros(1, BEST_DTYPE)[0]
    for r, mk, q in ((a, 100, 7), (b, 100, 3)):
        r["valid"], r["makespan"]["num"], r["makespan"]["den"] = 1, mk, 1
        r["peak_memory"]["den"] = r["max_bw"]["den"] = 1
        r["M"], r["query_id"] = 4, q
    assert best_less(b, a) and not best_less(a, b)          # query id breaks a full tie
    a["makespan"]["num"] = 99
    assert best_less(a, b)                                    # makespan first (explorer.hpp:144)
    b["valid"] = 0
    assert best_less(a, b) and not best_less(b, a)            # an infeasible shard never wins
