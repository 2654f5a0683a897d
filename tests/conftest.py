import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tests", "emu")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN_NPZ = os.path.join(ROOT, "tests", "golden", "reference_fixtures.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (libbapipe_b200.so kernels); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    """Reference outputs per scenario (tests/golden/make_golden.py)."""
    from paper_2012_12544_b200.problem import CAND_DTYPE, RESULT_DTYPE, STAGE_DTYPE
    z = np.load(GOLDEN_NPZ)
    out = {}
    for key in z.files:
        name, part = key.rsplit("/", 1)
        dt = {"res": RESULT_DTYPE, "cand": CAND_DTYPE, "stages": STAGE_DTYPE}[part]
        out.setdefault(name, {})[part] = z[key].view(dt)
    return out


@pytest.fixture(scope="session")
def port():
    import pyoracle
    if not pyoracle.port_available():
        pyoracle.build(ref=False)
    return pyoracle.PortOracle()


@pytest.fixture(scope="session")
def ref():
    import pyoracle
    if not pyoracle.ref_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    return pyoracle.RefOracle()


@pytest.fixture(scope="session")
def emu():
    import pyemu
    return pyemu.Emu()


def assert_same(got, want, name):
    """Bit-exact comparison of result record arrays with a readable diff."""
    assert got.shape == want.shape, f"{name}: shape {got.shape} != {want.shape}"
    if got.tobytes() == want.tobytes():
        return
    bad = [i for i in range(got.size) if got[i].tobytes() != want[i].tobytes()]
    raise AssertionError(f"{name}: {len(bad)} records differ; first: got {got[bad[0]]} want {want[bad[0]]}")
