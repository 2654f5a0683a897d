"""Multi-GPU sweep plumbing: query sharding and the best-record exchange.

The candidate space is sharded across ranks by whole queries (all candidates
of a query stay on one GPU, so the per-query DP / refine / ranking stay
local).  Each rank reduces its queries' bests to one bp_best_record on the
device (k_best), the records are exchanged with a single allgather, and every
rank takes the same deterministic argmin (bp_best_less: makespan, peak
memory, max bandwidth demand, M, kind -- explorer.hpp:144-151 -- then query
id).  There is no other collective on the data path.
"""
from __future__ import annotations

import numpy as np

from .problem import BEST_DTYPE
from .runtime import best_less


def best_record_from_results(res: np.ndarray, query_ids: np.ndarray) -> np.ndarray:
    """Host mirror of k_best (csrc/kernels.cu) over per-query results."""
    out = np.zeros(1, dtype=BEST_DTYPE)
    rec = out[0]
    rec["valid"] = 0
    rec["query_id"] = np.iinfo(np.int64).max
    for i in range(res.size):
        r = res[i]
        x = np.zeros(1, dtype=BEST_DTYPE)[0]
        x["valid"] = 1 if r["status"] == 0 else 0
        x["query_id"] = int(query_ids[i])
        if x["valid"]:
            x["makespan"] = r["best_makespan"]
            x["peak_memory"] = r["best_peak_memory"]
            x["max_bw"] = r["best_max_bw"]
            x["M"] = r["best_M"]
            x["kind"] = r["best_kind"]
        if best_less(x, rec):
            rec = x
    out[0] = rec
    return out


def argmin_records(records) -> np.ndarray:
    best = records[0]
    for r in records[1:]:
        if best_less(r, best):
            best = r
    return best


def allgather_best(local: np.ndarray, group=None) -> np.ndarray:
    """Exchange one best record per rank (torch.distributed all_gather) and
    return the global argmin.  Works with the nccl (device tensors) and gloo
    (host tensors) backends."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(local.view(np.uint8).copy()).to(dev)
    world = dist.get_world_size(group)
    bufs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    recs = [b.cpu().numpy().view(BEST_DTYPE)[0] for b in bufs]
    return argmin_records(recs)
