"""Build the product library (sm_100a) and the test-only checkers.

    python -m paper_2012_12544_b200.build          # product + oracles

The product is one shared library, paper_2012_12544_b200/libbapipe_b200.so,
compiled with nvcc for `-gencode arch=compute_100a,code=sm_100a` (B200 only)
with the system g++ as host compiler (dynamic libstdc++; see oracle/Makefile
for why the /opt/gcc wrapper is avoided).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libbapipe_b200.so")
SOURCES = ["api.cu", "kernels.cu", "dp.cu", "sim.cu", "xwave.cu", "timeline.cu"]
HEADERS = ["rat.cuh", "common.cuh", "model.cuh", "refine_fast.cuh", "batch.cuh", "phases.cuh", "kernels.h", "host_prep.hpp", "timeline.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _host_cxx():
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_product(force=False, verbose=False):
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "bapipe_b200.h")]
    if not force and not _stale(SO, deps):
        return SO
    objs = []
    jobs = []
    os.makedirs(os.path.join(CSRC, "_obj"), exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(CSRC, "_obj", src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [_nvcc(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-ccbin", _host_cxx(),
               "-I" + os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        jobs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    for j in jobs:
        out, _ = j.communicate()
        if verbose or j.returncode:
            sys.stdout.write(out)
        if j.returncode:
            raise RuntimeError("nvcc failed")
    tmp = SO + ".tmp"
    subprocess.run([_nvcc(), *ARCH, "-shared", "-Xlinker", "--no-undefined", "-ccbin", _host_cxx(), "-o", tmp, *objs], check=True)
    os.replace(tmp, SO)
    return SO


CLI = os.path.join(HERE, "bin", "bapipe")
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def build_cli(force=False):
    """The `bapipe` command-line front end (cli/bapipe.cpp), linked against
    the product library; needs nlohmann/json.hpp (shipped with the image)."""
    if not os.path.exists(os.path.join(JSON_DIR, "json.hpp")):
        return None
    src = os.path.join(HERE, "cli", "bapipe.cpp")
    deps = [src, SO] + [os.path.join(ROOT, "include", "bapipe_b200", f) for f in ("explorer.hpp", "io.hpp", "gantt.hpp")]
    if not force and not _stale(CLI, deps):
        return CLI
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    subprocess.run([_host_cxx(), "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), "-I" + JSON_DIR, "-o",
                    CLI, src, "-L" + HERE, "-lbapipe_b200", "-Wl,-rpath,$ORIGIN/.."], check=True)
    return CLI


PERCALL = os.path.join(HERE, "bin", "percall")


def build_percall(force=False):
    """bench.py's per-call latency tool (cli/percall.cpp) on the drop-in
    explore(); oracle/Makefile builds the same source against the reference."""
    if not os.path.exists(os.path.join(JSON_DIR, "json.hpp")):
        return None
    src = os.path.join(HERE, "cli", "percall.cpp")
    deps = [src, SO] + [os.path.join(ROOT, "include", "bapipe_b200", f) for f in ("explorer.hpp", "io.hpp")]
    if not force and not _stale(PERCALL, deps):
        return PERCALL
    os.makedirs(os.path.dirname(PERCALL), exist_ok=True)
    subprocess.run([_host_cxx(), "-std=c++17", "-O2", "-pthread", "-I" + os.path.join(ROOT, "include"),
                    "-I" + JSON_DIR, "-o", PERCALL, src, "-L" + HERE, "-lbapipe_b200", "-Wl,-rpath,$ORIGIN/.."],
                   check=True)
    return PERCALL


def build_oracles():
    """Test-only checkers: the C restatement always, oracle/_ref when the
    reference sources are present (dev container only)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/include"):
        targets += ["ref", "dropin", "cli", "percall"]
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")] + targets, check=True)
    emu = os.path.join(ROOT, "tests", "emu")
    if os.path.isdir(emu):
        sys.path.insert(0, emu)
        import pyemu  # noqa: E402
        if _stale(pyemu.SO, [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(emu, "emu.cpp")]):
            pyemu.build()


if __name__ == "__main__":
    build_product(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_cli(force="--force" in sys.argv)
    build_percall(force="--force" in sys.argv)
    build_oracles()
    print(SO)
