"""The strong-scaling path through the product kernels: world_size 2 over gloo.

Each rank evaluates its class-aligned shard of one C5 sweep (workloads.
shard_classes: whole dedup classes per rank, bench.py's split) with the CUDA
product, reduces its queries to one bp_best_record on the device
(bp_batch_best), maps the record's shard-local query index to the global
query id, exchanges records with one all_gather and takes the deterministic
argmin (bp_best_less).  Both ranks share the one GPU of the test box: their
kernels are independent (the only exchange is the host-side all_gather of
80-byte records), so this exercises the multi-rank code path, not NVLink.
Every rank must agree with the argmin of the unsharded sweep, and the shard
results must equal the unsharded per-query results.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu
MODELS = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2012_12544_b200 import workloads as W
    from paper_2012_12544_b200.problem import BEST_DTYPE
    from paper_2012_12544_b200.runtime import Explorer
    from paper_2012_12544_b200.sweep import argmin_records
    full = W.config_c5(models=MODELS)
    p = W.subset(full, W.shard_classes(full, world)[rank])
    ex = Explorer(0)
    b = ex.prepare(p)
    ex.run(b)
    res, _, _ = ex.fetch(b, p)
    rec = torch.zeros(BEST_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ex.best(b, rec.data_ptr())
    torch.cuda.synchronize()
    r = rec.cpu().numpy().view(BEST_DTYPE).copy()
    if r[0]["valid"]:
        r[0]["query_id"] = int(p.query_ids[int(r[0]["query_id"])])
    mine = torch.from_numpy(r.view(np.uint8).copy())
    allr = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine)
    best = argmin_records([a.numpy().view(BEST_DTYPE)[0] for a in allr])
    out[rank] = (bytes(np.array([best]).tobytes()), p.query_ids.tolist(), bytes(res.tobytes()))
    ex.free(b)
    ex.close()
    dist.destroy_process_group()


def test_two_ranks_class_shards_match_unsharded():
    from paper_2012_12544_b200 import workloads as W
    from paper_2012_12544_b200.problem import RESULT_DTYPE
    from paper_2012_12544_b200.runtime import Explorer
    from paper_2012_12544_b200.sweep import best_record_from_results
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    full = W.config_c5(models=MODELS)
    ex = Explorer(0)
    res, _, _ = ex.explore(full, details=False)
    ex.close()
    want = best_record_from_results(res, full.query_ids)
    assert out[0][0] == out[1][0] == want.tobytes()
    got = np.zeros_like(res)
    for r in range(world):
        ids = np.array(out[r][1])
        got[ids] = np.frombuffer(out[r][2], dtype=RESULT_DTYPE)
    assert got.tobytes() == res.tobytes()


def test_two_contexts_concurrent_batches():
    """Two contexts on one device, each with a batch of a different stage
    count range (different dynamic shared memory sizes), run concurrently on
    two streams: each equals the same queries run alone (the kernels' shared
    memory attributes are per device and set once, bp_create)."""
    import torch

    from paper_2012_12544_b200 import workloads as W
    from paper_2012_12544_b200.runtime import Explorer
    full = W.config_c5(models=16)
    n = full.queries["n_stages"]
    subs = [W.subset(full, np.nonzero(n >= 32)[0]), W.subset(full, np.nonzero(n < 32)[0])]
    alone = []
    for s in subs:
        ex = Explorer(0)
        alone.append(ex.explore(s, details=True))
        ex.close()
    exs = [Explorer(0), Explorer(0)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    bs = [e.prepare(s, details=True, stream=st.cuda_stream) for e, s, st in zip(exs, subs, streams)]
    for e, b, st in zip(exs, bs, streams):
        e.run(b, stream=st.cuda_stream)
    torch.cuda.synchronize()
    for e, b, s, st, want in zip(exs, bs, subs, streams, alone):
        got = e.fetch(b, s, details=True, stream=st.cuda_stream)
        for g, w in zip(got, want):
            assert g.tobytes() == w.tobytes()
        e.free(b)
        e.close()
