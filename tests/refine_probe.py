"""Tool (not collected by pytest): refine latency of the C5 sweep's longest
refine query (18895: N = 64, L = 128, 3255 boundary steps) run alone, next
to the full sweep's refine time.  Run under gpurun, optionally under ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.problem import Problem  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

full = W.config_c5()
q = full.queries
qid = int(sys.argv[1]) if len(sys.argv) > 1 else 18895
idx = np.array([qid])
p = Problem(networks=full.networks, clusters=full.clusters, name="probe")
p.set_queries(q["network"][idx], q["cluster"][idx], q["n_stages"][idx], q["mini_batch"][idx])
ex = Explorer(0)
ex.explore(p, details=False)
ex.profiling(True)
b = ex.prepare(p)
for _ in range(3):
    ex.run(b)
    ex.fetch(b, p)
st = ex.kernel_stats()
for k in ("refine", "refine_critical_path"):
    v = st.get(k, {})
    print(f"single query {qid}: {k:22s} {v.get('ms', 0) / max(1, v.get('launches', 1)):8.3f} ms  work={v.get('work', 0):.0f}")
