"""Tool (not collected by pytest): the refine phase on the C5 sweep's N = 64
queries only (every long walk, nothing else), beside the full sweep's."""
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
for label, sel in (("N=64 only", q["n_stages"] == 64), ("N<64 only", q["n_stages"] < 64)):
    idx = np.nonzero(sel)[0]
    p = Problem(networks=full.networks, clusters=full.clusters, name=label)
    p.set_queries(q["network"][idx], q["cluster"][idx], q["n_stages"][idx], q["mini_batch"][idx])
    ex = Explorer(0)
    ex.explore(p, details=False)
    ex.profiling(True)
    b = ex.prepare(p)
    for _ in range(3):
        ex.run(b)
        ex.fetch(b, p)
    st = ex.kernel_stats()
    r = st.get("refine", {})
    c = st.get("refine_critical_path", {})
    print(f"{label}: {idx.size} queries, refine {r.get('ms', 0) / max(1, r.get('launches', 1)):.2f} ms, "
          f"critical walk {c.get('work', 0):.0f} steps, steps {r.get('work', 0):.0f}")
    ex.close()
