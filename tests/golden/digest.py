"""TEST INFRASTRUCTURE: 64-bit digest of each candidate's full output.

digest[i] = blake2b-64 of bp_candidate record i followed by the n_stages
bp_stage records of that candidate (query stage_offset + slot * n_stages).
Equal digests mean byte-identical candidate and per-stage output.
"""
import hashlib

import numpy as np


def candidate_digests(p, cand, st):
    q = p.queries
    nst = np.where(q["n_stages"] > 0, q["n_stages"],
                   np.array([c.N for c in p.clusters], dtype=np.int64)[q["cluster"]]).astype(np.int64)
    ncand = p.n_candidates.astype(np.int64)
    # per-candidate stage start and length, in candidate order
    qi = np.repeat(np.arange(q.size), ncand)
    slot = np.arange(p.total_candidates, dtype=np.int64) - np.repeat(q["cand_offset"], ncand)
    s0 = q["stage_offset"][qi] + slot * nst[qi]
    s1 = s0 + nst[qi]
    cb = cand.view(np.uint8).reshape(cand.size, -1)
    sb = st.view(np.uint8).reshape(-1)
    w = st.dtype.itemsize
    out = np.empty(cand.size, dtype=np.uint64)
    for i in range(cand.size):
        h = hashlib.blake2b(cb[i].tobytes(), digest_size=8)
        h.update(sb[s0[i] * w:s1[i] * w].tobytes())
        out[i] = int.from_bytes(h.digest(), "little")
    return out
