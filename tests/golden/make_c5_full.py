"""Golden per-query results of the FULL C5 sweep from the reference itself.

Runs the reference's own explore() (oracle/_ref, compiled from
/root/reference) on all 65,536 queries with one worker per core and stores
the per-query result records (status, best kind/M/micro, makespan, peak
memory, max bandwidth demand) in c5_full_ref.npz.  ~1 h on 8 cores.
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
from pyoracle import RefOracle  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402

p = W.config_c5()
t = time.time()
res = RefOracle().explore_timed(p, threads=os.cpu_count())
dt = time.time() - t
np.savez_compressed(os.path.join(HERE, "c5_full_ref.npz"), res=res.view(np.uint8), seconds=np.array([dt]),
                    threads=np.array([os.cpu_count()]))
print(f"done in {dt:.0f} s; status hist {np.bincount(res['status'], minlength=7).tolist()}")
