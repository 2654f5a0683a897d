"""B200-native drop-in for BaPipe's explore() candidate-evaluation path.

The product is the CUDA shared library libbapipe_b200.so behind the C ABI in
include/bapipe_b200.h; this package holds its sources (csrc/), the ctypes
binding (abi.py), batch marshalling (problem.py), synthetic workloads
(workloads.py) and the Python mirror of the reference interface
(explorer.py).
"""
from . import abi, problem, workloads  # noqa: F401
