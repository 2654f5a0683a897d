"""Generate the golden fixtures from the reference itself (dev container only).

Every fixture is computed by oracle/_ref (the UNMODIFIED reference headers
under /root/reference, compiled by oracle/Makefile) through its own public
explore()/balance_partition/estimate/simulate calls.  Scenarios:

  * the reference's own unit-test scenarios restated as explore() queries
    (proj/tests/test_explorer.cpp:60-172, test_partitioner.cpp:254-287,
    test_cost_models.cpp, test_simulator.cpp) -- inputs stored explicitly;
  * BASELINE configs C1-C4 and seeded random batches -- inputs regenerated
    from paper_2012_12544_b200.workloads (deterministic);
  * a 1/1024 query-stride sample of the C5 sweep.

Output: reference_fixtures.npz (raw result records) + reference_fixtures.json
(scenario index, readable key fields).  Run: python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
from pyoracle import RefOracle  # noqa: E402

import scenarios  # noqa: E402

if __name__ == "__main__":
    ref = RefOracle()
    arrays = {}
    index = []
    for name, build in scenarios.SCENARIOS:
        p = build()
        res, cand, st = ref.explore(p, details=True, threads=os.cpu_count())
        arrays[name + "/res"] = res.view(np.uint8)
        arrays[name + "/cand"] = cand.view(np.uint8)
        keep_stages = st.size <= 20000
        if keep_stages:
            arrays[name + "/stages"] = st.view(np.uint8)
        index.append({
            "name": name, "queries": int(p.queries.size), "candidates": int(cand.size),
            "stages_stored": keep_stages,
            "query_status": np.bincount(res["status"], minlength=7).tolist(),
            "candidate_status": np.bincount(cand["status"], minlength=11).tolist(),
            "best": [{"status": int(r["status"]), "kind": int(r["best_kind"]), "M": int(r["best_M"]),
                      "makespan": f"{int(r['best_makespan']['num'])}/{int(r['best_makespan']['den'])}"}
                     for r in res[:8]],
        })
        print(name, index[-1]["query_status"], flush=True)
    np.savez_compressed(os.path.join(HERE, "reference_fixtures.npz"), **arrays)
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (oracle/_ref = the reference itself)",
                   "scenarios": index}, f, indent=1)
