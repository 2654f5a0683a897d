"""Tool (not collected by pytest): per-kernel and per-phase times of one
subset of the C5 sweep run alone (default: the N = 64 queries, the split's
first part), CUDA events around every launch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 64
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 64
full = W.config_c5()
n = full.queries["n_stages"]
p = W.subset(full, np.nonzero((n >= lo) & (n <= hi))[0])
ex = Explorer(0)
ex.split(False)
b = ex.prepare(p)
for _ in range(3):
    ex.run(b)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    ex.run(b)
e.record()
torch.cuda.synchronize()
print(f"N in [{lo}, {hi}]: {p.queries.size} queries, {a.elapsed_time(e) / 3:.2f} ms per run")
ex.profiling(True)
for _ in range(3):
    ex.run(b)
ex.fetch(b, p)
st = ex.kernel_stats()
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
    if v["ms"] / 3 > 0.05:
        print(f"  {k:24s} {v['ms'] / 3:8.3f} ms  work {v['work']:.4g}")
