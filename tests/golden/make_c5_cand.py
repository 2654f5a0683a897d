"""Golden PER-CANDIDATE results of the FULL C5 sweep from the reference itself.

TEST INFRASTRUCTURE.  Runs oracle/_ref (the unmodified reference headers
compiled from /root/reference) in parity mode on all 65,536 C5 queries:
bapipe::explore() per query (explorer.hpp:80-155) for the ranking, then the
per-(kind, M) replay of explorer.hpp:96-132 through the public
balance_partition / estimate / simulate calls (oracle/ref_driver.cpp).  Every
one of the 2^20 candidates is reduced to a 64-bit digest of its bp_candidate
record plus its n_stages bp_stage records (tests/golden/digest.py), and the
full bp_query_result of every query is stored beside them:

    c5_cand_ref.npz: digest[2^20] u64, status[2^20] u8, rank[2^20] i8,
                     res[65536] (bp_query_result bytes), seconds, threads

About 2 h on 8 cores.  Resumable: finished query chunks are cached in
/tmp/c5_cand_chunks.
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)
import numpy as np  # noqa: E402
from digest import candidate_digests  # noqa: E402
from pyoracle import RefOracle  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.problem import CAND_DTYPE, RESULT_DTYPE, STAGE_DTYPE  # noqa: E402

CHUNK = 2048
CACHE = "/tmp/c5_cand_chunks"


def main(threads):
    os.makedirs(CACHE, exist_ok=True)
    p = W.config_c5()
    ref = RefOracle()
    nq = p.queries.size
    digest = np.zeros(p.total_candidates, dtype=np.uint64)
    status = np.zeros(p.total_candidates, dtype=np.uint8)
    rank = np.zeros(p.total_candidates, dtype=np.int8)
    res_all = np.zeros(nq, dtype=RESULT_DTYPE)
    t0 = time.time()
    spent = 0.0
    for q0 in range(0, nq, CHUNK):
        path = os.path.join(CACHE, f"{q0:06d}.npz")
        if os.path.exists(path):
            z = np.load(path)
            res, d, s, r, dt = z["res"].view(RESULT_DTYPE), z["digest"], z["status"], z["rank"], float(z["dt"])
        else:
            sub = W.subset(p, np.arange(q0, min(nq, q0 + CHUNK)))
            res = np.zeros(sub.queries.size, dtype=RESULT_DTYPE)
            cand = np.zeros(sub.total_candidates, dtype=CAND_DTYPE)
            st = np.zeros(sub.total_stages, dtype=STAGE_DTYPE)
            t = time.time()
            res, cand, st = ref.explore(sub, details=True, threads=threads)
            dt = time.time() - t
            d = candidate_digests(sub, cand, st)
            s = cand["status"].astype(np.uint8)
            r = np.clip(cand["rank"], -1, 127).astype(np.int8)
            np.savez(path, res=res.view(np.uint8), digest=d, status=s, rank=r, dt=np.array(dt))
        c0 = int(p.queries["cand_offset"][q0])
        digest[c0:c0 + d.size] = d
        status[c0:c0 + d.size] = s
        rank[c0:c0 + d.size] = r
        res_all[q0:q0 + res.size] = res
        spent += dt
        print(f"queries {q0 + res.size}/{nq}  ({time.time() - t0:.0f} s)", flush=True)
    np.savez_compressed(os.path.join(HERE, "c5_cand_ref.npz"), digest=digest, status=status, rank=rank,
                        res=res_all.view(np.uint8), seconds=np.array([spent]), threads=np.array([threads]))
    print(f"done: reference parity mode {spent:.0f} s on {threads} threads; "
          f"status hist {np.bincount(status, minlength=11).tolist()}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else os.cpu_count())
