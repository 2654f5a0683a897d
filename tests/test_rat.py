"""csrc/rat.cuh on the host: every fast path of the exact-rational kernels'
arithmetic against an __int128 restatement of rational.hpp:83-95
(tests/cpp/rat_selftest.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def test_rat_arithmetic_matches_int128_reference(tmp_path):
    exe = str(tmp_path / "ratst")
    subprocess.run([CXX, "-std=c++17", "-O2", "-o", exe, os.path.join(ROOT, "tests", "cpp", "rat_selftest.cpp")],
                   check=True)
    out = subprocess.run([exe, "1000000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("ok"), out.stdout + out.stderr
