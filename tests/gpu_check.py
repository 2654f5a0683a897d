"""Ad-hoc GPU parity + timing check (run under gpurun; not collected by pytest)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
from pyoracle import PortOracle, RefOracle, ref_available  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.problem import Problem  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

ref = RefOracle() if ref_available() else PortOracle()
port = PortOracle()
ex = Explorer(0)


def cmp(p, o, label):
    t = time.time()
    g = ex.explore(p, details=True)
    tg = time.time() - t
    t = time.time()
    w = o.explore(p, details=True)
    tw = time.time() - t
    bad = [int(sum(g[k][i].tobytes() != w[k][i].tobytes() for i in range(g[k].size))) for k in range(3)]
    print(f"{label:28s} badq={bad[0]} badc={bad[1]} bads={bad[2]} gpu={tg*1e3:.1f}ms {o.kind}={tw*1e3:.1f}ms "
          f"qstat={np.bincount(w[0]['status'], minlength=7).tolist()}", flush=True)
    if bad[1]:
        for i in [i for i in range(g[1].size) if g[1][i].tobytes() != w[1][i].tobytes()][:3]:
            print("   gpu", g[1][i])
            print("   ref", w[1][i])
    return sum(bad)


mode = sys.argv[1] if len(sys.argv) > 1 else "all"
tot = 0
if mode in ("all", "parity"):
    for name, p in [("C1", W.config_c1()), ("C2", W.config_c2()), ("C3", W.config_c3())]:
        tot += cmp(p, ref, name)
    for tier in ("onchip", "offchip", "homogeneous"):
        tot += cmp(W.config_c4(tier), port, "C4 " + tier)
    for s in range(4):
        tot += cmp(W.random_problem(s, n_queries=200), ref, f"rand{s}")
    for s in range(4):
        tot += cmp(W.random_problem(100 + s, n_queries=100, max_L=40, max_N=16, cap_range=(1000, 60000),
                                    bw_range=(1, 500), act_max=3000), ref, f"rand-heavy{s}")
full = W.config_c5()
if mode in ("all", "parity"):
    idx = np.arange(0, full.queries.size, 1031)
    p = Problem(networks=full.networks, clusters=full.clusters, name="C5 sample")
    q = full.queries[idx]
    p.set_queries(q["network"], q["cluster"], q["n_stages"], q["mini_batch"])
    tot += cmp(p, ref, "C5 1/1031 sample")
    print("TOTAL MISMATCHES", tot, flush=True)
if mode in ("all", "time"):
    ex.load(full)
    for it in range(3):
        t = time.time()
        res, _, _ = ex.explore(full, details=False)
        dt = time.time() - t
        print(f"C5 full sweep e2e: {dt*1e3:.1f} ms  ({full.total_candidates/dt:.3e} cand/s)", flush=True)
    ex.profiling(True)
    b = ex.prepare(full)
    for it in range(3):
        ex.run(b)
        r, _, _ = ex.fetch(b, full)
    for k, v in sorted(ex.kernel_stats().items(), key=lambda kv: -kv[1]["ms"]):
        print(f"  {k:18s} {v['ms']/max(1,v['launches']):9.3f} ms/launch  launches={v['launches']} work={v['work']:.3e}")
    print("status hist", np.bincount(r["status"], minlength=7).tolist(), "launches", ex.launches())
