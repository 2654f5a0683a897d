"""The C++ drop-in boundary (include/bapipe_b200/explorer.hpp).

tests/cpp/dropin_scenarios.cpp runs every explore() case of the reference's
tests/test_explorer.cpp, its error paths and 80 seeded heterogeneous chains
(40 near the int64 limits, where Rat: overflow escapes), and prints every field
of each ExplorationResult or the exception type + what().  The same source
compiled against the reference headers produced tests/golden/dropin_expected.txt
(tests/golden/make_dropin_expected.sh); here it is compiled against the
drop-in header and must print the identical text:
  * CPU: linked with tests/cpp/emu_abi_shim.cpp (the kernels' phase code
    replayed on the host) -- checks the header's host logic;
  * GPU: linked with libbapipe_b200.so -- the product path on the B200.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
GOLDEN = os.path.join(ROOT, "tests", "golden", "dropin_expected.txt")
PKG = os.path.join(ROOT, "paper_2012_12544_b200")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _build(out, extra):
    cmd = [CXX, "-std=c++17", "-O2", "-Wall", "-Wno-enum-compare", "-I" + os.path.join(ROOT, "include"), "-o", out,
           os.path.join(CPP, "dropin_scenarios.cpp")] + extra
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def _run(exe):
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return p.stdout


def _diff(got, want):
    g, w = got.splitlines(), want.splitlines()
    for i, (a, b) in enumerate(zip(g, w)):
        if a != b:
            return f"line {i + 1}:\n  got  {a[:300]}\n  want {b[:300]}"
    return f"length {len(g)} != {len(w)}"


def test_header_is_self_contained(tmp_path):
    src = tmp_path / "inc.cpp"
    src.write_text('#include "bapipe_b200/explorer.hpp"\nint main() { return 0; }\n')
    subprocess.run([CXX, "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                    str(src)], check=True)


def test_schema_errors_raise_before_any_device_work(tmp_path):
    """Validation (profiles.hpp:83-132, explorer.hpp:82-89) runs in the header:
    it throws the reference's exception and message without touching the ABI."""
    src = tmp_path / "schema.cpp"
    src.write_text(r'''
#include "bapipe_b200/explorer.hpp"
#include <cstdio>
using namespace bapipe_b200;
int main() {
    ClusterSpec cl;
    cl.accelerators.push_back({"g0", "gpu", 100, {}});
    NetworkProfile net = synth_uniform_network(2, 1, 1, 1, 1, {"fpga"});
    try { validate_pair(net, cl); } catch (const SchemaError& e) { std::puts(e.what()); }
    TrainingConfig cfg; cfg.mini_batch_size = 6; cfg.micro_batch_candidates = std::vector<std::int64_t>{4};
    try { candidate_Ms(cfg, cl, ScheduleKind::OneFOneB_SO); } catch (const SchemaError& e) { std::puts(e.what()); }
    return 0;
}''')
    exe = str(tmp_path / "schema")
    subprocess.run([CXX, "-std=c++17", "-I" + os.path.join(ROOT, "include"), "-o", exe, str(src)], check=True)
    out = _run(exe).splitlines()
    assert out == ["schema error: layer 0 ('layer0') lacks times for accelerator type 'gpu'",
                   "schema error: micro-batch candidate 4 does not divide mini-batch 6"]


def test_dropin_matches_reference_on_emulator(tmp_path):
    exe = str(tmp_path / "dropin_emu")
    _build(exe, [os.path.join(CPP, "emu_abi_shim.cpp")])
    got, want = _run(exe), open(GOLDEN).read()
    assert got == want, _diff(got, want)


def test_golden_regenerates_from_reference():
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_scenarios_ref")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_scenarios_ref not built (make -C oracle dropin)")
    got, want = _run(exe), open(GOLDEN).read()
    assert got == want, _diff(got, want)


REF_INC = "/root/reference/proj/include"
JSON_DIR = os.path.join(ROOT, "oracle", "_ref", "vendor")


def test_interop_with_reference_types(tmp_path):
    """include/bapipe_b200/interop.hpp: reference-typed inputs and results
    (explore_as) agree with bapipe::explore on every scenario."""
    if not (os.path.isdir(REF_INC) and os.path.exists(os.path.join(JSON_DIR, "json.hpp"))):
        pytest.skip("reference headers not present (dev container only)")
    exe = str(tmp_path / "interop")
    subprocess.run([CXX, "-std=c++20", "-O2", "-Wno-enum-compare", "-I" + os.path.join(ROOT, "include"),
                    "-I" + REF_INC, "-I" + JSON_DIR, "-o", exe, os.path.join(CPP, "interop_check.cpp"),
                    os.path.join(CPP, "emu_abi_shim.cpp")], check=True, capture_output=True, text=True)
    out = _run(exe)
    assert out.strip().endswith("0 mismatches"), out[-3000:]


@pytest.mark.gpu
def test_dropin_matches_reference_on_b200(tmp_path):
    so = os.path.join(PKG, "libbapipe_b200.so")
    assert os.path.exists(so), "libbapipe_b200.so not built (python -c 'import __graft_entry__ as g; g.build()')"
    exe = str(tmp_path / "dropin_gpu")
    _build(exe, ["-L" + PKG, "-lbapipe_b200", "-Wl,-rpath," + PKG])
    got, want = _run(exe), open(GOLDEN).read()
    assert got == want, _diff(got, want)
