"""bench.py's JSON line keeps the driver's contract (a small sweep: 8 models,
2 steps): the required keys, e2e with its copied bytes, the roofline and
clocks objects, a positive launch count, and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [line for line in out.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run("--models", "8", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-per-call")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline", "sweep_roofline"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac"} <= set(d["roofline"])
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "workload" in d["config"]


def test_reference_arm_line():
    d = run("--impl", "reference", "--models", "8", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference"
    if "unavailable" not in d:
        assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0 and "cpu_baseline" in d
