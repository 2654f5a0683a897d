"""Host preparation (csrc/host_prep.hpp, plain C++): the batch build in
chunks on the worker pool equals the one-chunk build on random batches of
40,000 queries (records, M lists, DP items, totals, first error)
(tests/cpp/build_batch_selftest.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def test_chunked_batch_build_equals_serial(tmp_path):
    exe = str(tmp_path / "bbst")
    subprocess.run([CXX, "-std=c++17", "-O2", "-pthread", "-Wno-enum-compare", "-I" + os.path.join(ROOT, "include"),
                    "-I" + os.path.join(ROOT, "paper_2012_12544_b200", "csrc"), "-x", "c++",
                    os.path.join(ROOT, "tests", "cpp", "build_batch_selftest.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe, "8"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("ok"), out.stdout + out.stderr
