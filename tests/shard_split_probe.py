"""Tool (not collected by pytest): the slowest 8-way strong-scaling shard of
C5 as k concurrent batches (one context each): the N = 64 queries cut into
1, 2 or 4 groups of whole dedup classes, beside the rest."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

full = W.config_c5()
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shard = W.subset(full, W.shard_classes(full, world)[int(sys.argv[2]) if len(sys.argv) > 2 else 3])


def run(groups):
    subs = [W.subset(shard, g) for g in groups]
    exs = [Explorer(0) for _ in subs]
    for e in exs:
        e.split(False)
    sts = [torch.cuda.Stream() for _ in subs]
    bs = [e.prepare(s, stream=st.cuda_stream) for e, s, st in zip(exs, subs, sts)]
    main = torch.cuda.current_stream()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(main)
        for e, bb, st in zip(exs, bs, sts):
            st.wait_event(a)
            e.run(bb, stream=st.cuda_stream)
        for st in sts:
            main.wait_stream(st)
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    for e, bb in zip(exs, bs):
        e.free(bb)
        e.close()
    return sorted(ts[2:])[2]


n = shard.queries["n_stages"]
cls = W.query_classes(shard)
big = np.nonzero(n == n.max())[0]
rest = np.nonzero(n < n.max())[0]
ucls = np.unique(cls[big])
print(f"{world}-way shard: {shard.queries.size} queries, {ucls.size} classes with N = {n.max()}")
print(f"  one batch: {run([np.arange(shard.queries.size)]):.2f} ms")
for k in (1, 2, 4):
    parts = [big[np.isin(cls[big], ucls[i::k])] for i in range(k)]
    print(f"  N = {n.max()} in {k} group(s) + the rest: {run(parts + [rest]):.2f} ms")

# per-kernel profile of the two split parts of this shard, each alone
if "--profile" in sys.argv:
    for name, g in (("N = max", big), ("rest", rest)):
        sub = W.subset(shard, g)
        ex = Explorer(0)
        ex.split(False)
        b = ex.prepare(sub)
        ex.run(b)
        ex.profiling(True)
        for _ in range(3):
            ex.run(b)
        ex.fetch(b, sub)
        st = ex.kernel_stats()
        print(f"  part {name}: {sub.queries.size} queries")
        for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
            if v["ms"] / 3 > 0.15:
                print(f"    {k:24s} {v['ms'] / 3:8.3f} ms")
        ex.free(b)
        ex.close()
