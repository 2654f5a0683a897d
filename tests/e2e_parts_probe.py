"""Tool (not collected by pytest): the e2e step as bench.py times it, split
into the table upload (load), the explore() call and its pieces."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

p = W.config_c5()
ex = Explorer(0)
out = p.alloc_outputs(False, pinned=True)
sp = torch.cuda.Stream()
for _ in range(3):
    ex.load(p, force=True)
    ex.explore(p, details=False, stream=sp.cuda_stream, out=out)
torch.cuda.synchronize()
rows = []
for _ in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nets, cls = p.c_networks(), p.c_clusters()
    t1 = time.perf_counter()
    ex.lib.bp_set_networks(ex.ctx, nets, len(p.networks))
    t2 = time.perf_counter()
    ex.lib.bp_set_clusters(ex.ctx, cls, len(p.clusters))
    t3 = time.perf_counter()
    ex._keep, ex._loaded = (nets, cls), p
    ex.explore(p, details=False, stream=sp.cuda_stream, out=out)
    t4 = time.perf_counter()
    rows.append([1e3 * (b - a) for a, b in ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t0, t4))])
rows.sort(key=lambda r: r[-1])
r = rows[len(rows) // 2]
print(f"median step {r[4]:.2f} ms: c_tables {r[0]:.2f}, set_networks {r[1]:.2f}, set_clusters {r[2]:.2f}, explore {r[3]:.2f}")
