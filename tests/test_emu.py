"""The product's per-thread phase code (csrc/phases.cuh, model.cuh, rat.cuh),
compiled for the host by tests/emu, against the reference's outputs.

This runs the exact-emulation logic of the CUDA kernels (estimate, fine-tune,
refine, validate, exact simulator, ranking) and a sequential mirror of the
windowed DP on the CPU, so every logic change is checked here without a GPU.
The GPU tests (test_gpu_parity.py) check the kernels themselves.
"""
import numpy as np
import pytest
import scenarios
from conftest import assert_same

from paper_2012_12544_b200 import workloads as W


@pytest.mark.parametrize("name", [n for n, _ in scenarios.SCENARIOS])
def test_emu_matches_reference_fixtures(emu, golden, name):
    p = scenarios.build(name)
    res, cand, st = emu.explore(p, details=True)
    g = golden[name]
    assert_same(res, g["res"], name + "/res")
    assert_same(cand, g["cand"], name + "/cand")
    if "stages" in g:
        assert_same(st, g["stages"], name + "/stages")


@pytest.mark.parametrize("seed", [21, 22, 23, 24])
def test_emu_matches_oracle_on_heavy_random(emu, port, seed):
    p = W.random_problem(seed, n_queries=60, max_L=30, max_N=12, cap_range=(1000, 60000), bw_range=(1, 500),
                         act_max=3000)
    for x, y, part in zip(emu.explore(p), port.explore(p), ("res", "cand", "stages")):
        assert_same(x, y, f"seed {seed} {part}")


def test_windowed_dp_does_less_work_than_the_full_dp(emu):
    """The pruned DP visits far fewer transitions than N*(U-N+1)*(U-N+2)."""
    p = W.config_c4("homogeneous")
    emu.explore(p, details=False)
    U, N = 1000, 64
    full = N * (U - N + 1) * (U - N + 2)
    assert 0 < emu.last_work < full / 4
