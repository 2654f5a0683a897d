"""The N>1 path on the CPU: world_size 2 over gloo.

Each rank takes its cost-balanced shard of a C5 subset, evaluates it (the
CPU replay of the product's phase code stands in for the GPU kernels, which
need a B200), reduces to one best record, exchanges records with one
allgather and takes the deterministic argmin.  The result must equal the
argmin over the unsharded batch, and the shards must partition the queries.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out, how="lpt"):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests", "emu"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pyemu

    from paper_2012_12544_b200 import workloads as W
    from paper_2012_12544_b200.sweep import allgather_best, best_record_from_results
    if how == "class":
        # bench.py's strong-scaling split: whole dedup classes per rank
        full = W.config_c5(models=2)
        p = W.subset(full, W.shard_classes(full, world)[rank])
    else:
        p = W.config_c5(models=2, shard=rank, n_shards=world)
    res, _, _ = pyemu.Emu().explore(p, details=False)
    local = best_record_from_results(res, p.query_ids)
    best = allgather_best(local)
    out[rank] = (bytes(best.tobytes()), p.query_ids.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("how", ["lpt", "class"])
def test_sharded_sweep_allgather_argmin_matches_unsharded(emu, how):
    from paper_2012_12544_b200 import workloads as W
    from paper_2012_12544_b200.sweep import best_record_from_results
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out, how), nprocs=world, join=True)
    full = W.config_c5(models=2)
    res, _, _ = emu.explore(full, details=False)
    want = best_record_from_results(res, full.query_ids)
    ids = sorted(out[0][1] + out[1][1])
    assert ids == list(range(full.queries.size))            # the shards partition the queries
    assert out[0][0] == out[1][0] == want.tobytes()           # every rank agrees with the unsharded argmin


def test_cost_balanced_shards():
    from paper_2012_12544_b200 import workloads as W
    full = W.config_c5(models=16)
    L = np.array([full.networks[i].L for i in full.queries["network"]])
    shards = W.shard_queries(L, full.queries["n_stages"], 8)
    cost = W.query_cost(L, full.queries["n_stages"])
    loads = [cost[s].sum() for s in shards]
    assert sum(len(s) for s in shards) == full.queries.size
    assert max(loads) / min(loads) < 1.05


def test_class_shards_keep_dedup_classes_whole():
    from paper_2012_12544_b200 import workloads as W
    full = W.config_c5(models=16)
    cls = W.query_classes(full)
    shards = W.shard_classes(full, 8)
    owner = np.empty(full.queries.size, dtype=np.int64)
    for r, s in enumerate(shards):
        owner[s] = r
    assert sorted(np.concatenate(shards).tolist()) == list(range(full.queries.size))
    for c in np.unique(cls):
        assert np.unique(owner[cls == c]).size == 1          # a class never spans two ranks
    cost = W.class_cost(full, cls)
    loads = [sum(cost[c] for c in np.unique(cls[s])) for s in shards]
    assert max(loads) / min(loads) < 1.1
