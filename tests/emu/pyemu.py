"""TEST HARNESS loader for tests/emu/emu.cpp (CPU replay of the product's
per-thread phase code; never used by the product)."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libbapipe_emu.so")
ROOT = os.path.dirname(os.path.dirname(HERE))


def build():
    os.makedirs(os.path.join(HERE, "_build"), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O2", "-fPIC", "-shared", "-Wno-enum-compare",
                    "-I" + os.path.join(ROOT, "include"), "-o", SO, os.path.join(HERE, "emu.cpp")], check=True)


class Emu:
    kind = "emu"

    def __init__(self):
        if not os.path.exists(SO):
            build()
        self.lib = C.CDLL(SO)
        vp = C.c_void_p
        self.lib.bpemu_explore_batch.restype = C.c_int
        self.lib.bpemu_explore_batch.argtypes = [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp]

    def explore(self, p, details=True):
        nets, cls = p.c_networks(), p.c_clusters()
        res, cand, st = p.alloc_outputs(details)
        work = np.zeros(1, dtype=np.uint64)
        rc = self.lib.bpemu_explore_batch(C.cast(nets, C.c_void_p), len(p.networks), C.cast(cls, C.c_void_p),
                                          len(p.clusters), p.queries.ctypes.data, p.queries.size, res.ctypes.data,
                                          None if cand is None else cand.ctypes.data,
                                          None if st is None else st.ctypes.data, work.ctypes.data)
        assert rc == 0, rc
        self.last_work = int(work[0])
        return res, cand, st
