"""Where the end-to-end C5 step goes (tool, not a test): table upload, batch
preparation on the host (layout, scheduling orders, pinned staging + one H2D),
the device run, and the result fetch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

p = W.config_c5()
ex = Explorer(0)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ex.load(p, force=True)
    t1 = time.perf_counter()
    b = ex.prepare(p, details=False)
    t2 = time.perf_counter()
    ex.run(b)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res, _, _ = ex.fetch(b, p)
    t4 = time.perf_counter()
    ex.free(b)
    t5 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.1f} ms  prepare {1e3*(t2-t1):.1f} ms  run {1e3*(t3-t2):.1f} ms  "
          f"fetch {1e3*(t4-t3):.1f} ms  free {1e3*(t5-t4):.1f} ms  total {1e3*(t5-t0):.1f} ms")
for rep in range(4):   # the public call, as bench.py's e2e leg makes it (its batch arena is reused)
    t = time.perf_counter()
    ex.load(p, force=True)
    r = ex.explore(p, details=False)
    print(f"explore() e2e {1e3*(time.perf_counter()-t):.1f} ms")
