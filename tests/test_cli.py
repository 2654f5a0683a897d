"""The `bapipe` CLI (paper_2012_12544_b200/cli/bapipe.cpp; SURVEY.md 8f rows
F1, F2, F3): validate / plan / explore / simulate (full timeline, --trace,
--gantt csv/svg); JSON ingest with the reference's schema errors, canonical JSON /
table reports, the run manifest and exit codes, against the reference's own
outputs (tests/golden/make_cli_golden.py -> tests/golden/cli/expected.json).
Every case compares stdout, stderr, the exit code and the -o / --gantt files
byte for byte.
  * CPU: the CLI linked with tests/cpp/emu_abi_shim.cpp (kernel phase code
    replayed on the host);
  * GPU: the CLI linked with libbapipe_b200.so.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI_DIR = os.path.join(ROOT, "tests", "golden", "cli")
SRC = os.path.join(ROOT, "paper_2012_12544_b200", "cli", "bapipe.cpp")
PKG = os.path.join(ROOT, "paper_2012_12544_b200")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def expected():
    with open(os.path.join(CLI_DIR, "expected.json")) as f:
        return json.load(f)


def build(out, extra):
    if not os.path.exists(os.path.join(JSON_DIR, "json.hpp")):
        pytest.skip("nlohmann json.hpp not found")
    subprocess.run([CXX, "-std=c++17", "-O2", "-Wno-enum-compare", "-I" + os.path.join(ROOT, "include"),
                    "-I" + JSON_DIR, "-o", out, SRC] + extra, check=True, capture_output=True, text=True)


def check_all(exe, tmp_path):
    bad = []
    out_files = ("best_plan.json", "gantt.csv", "gantt.svg")
    for want in expected():
        for name in out_files:
            if os.path.exists(os.path.join(CLI_DIR, name)):
                os.remove(os.path.join(CLI_DIR, name))
        p = subprocess.run(["bapipe"] + want["args"], executable=exe, cwd=CLI_DIR, capture_output=True, text=True,
                           timeout=600)
        got = {"args": want["args"], "rc": p.returncode, "stdout": p.stdout, "stderr": p.stderr}
        for name in out_files:
            path = os.path.join(CLI_DIR, name)
            if os.path.exists(path):
                got["out_file" if name == "best_plan.json" else name] = open(path).read()
                os.remove(path)
        if got != want:
            diff = [k for k in want if got.get(k) != want[k]] + [k for k in got if k not in want]
            bad.append((" ".join(want["args"]), diff, got.get("stderr", "")[:200]))
    assert not bad, bad


def test_cli_matches_reference_on_emulator(tmp_path):
    exe = str(tmp_path / "bapipe")
    build(exe, [os.path.join(ROOT, "tests", "cpp", "emu_abi_shim.cpp")])
    check_all(exe, tmp_path)


def test_cli_usage_errors(tmp_path):
    exe = str(tmp_path / "bapipe")
    build(exe, [os.path.join(ROOT, "tests", "cpp", "emu_abi_shim.cpp")])
    for args in (["explore", "tri_net.json", "tri_roomy.json"],        # --minibatch required
                 ["plan", "tri_net.json", "tri_roomy.json"],            # --schedule required
                 ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_whole.json", "--schedule", "1f1b-sno"],
                 ["simulate", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-sno", "--micro", "2"],
                 ["frobnicate"], [],
                 ["explore", "tri_net.json", "tri_roomy.json", "--minibatch", "x"]):
        p = subprocess.run(["bapipe"] + args, executable=exe, cwd=CLI_DIR, capture_output=True, text=True)
        assert p.returncode == 1 and p.stdout == "", (args, p.stdout, p.stderr)


@pytest.mark.gpu
def test_cli_matches_reference_on_b200(tmp_path):
    so = os.path.join(PKG, "libbapipe_b200.so")
    assert os.path.exists(so), "libbapipe_b200.so not built"
    exe = str(tmp_path / "bapipe")
    build(exe, ["-L" + PKG, "-lbapipe_b200", "-Wl,-rpath," + PKG])
    check_all(exe, tmp_path)
