"""Tool (not collected by pytest): the strong-scaling prediction on one GPU.
For world sizes 2, 4 and 8, each rank's class-aligned shard of the C5 sweep
(workloads.shard_classes, bench.py's split) is run alone and timed; the
step at N GPUs is the slowest shard (plus a ~20 us all_gather of 80-byte
records)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

full = W.config_c5()
ex = Explorer(0)


def timed(p, reps=5):
    b = ex.prepare(p)
    for _ in range(2):
        ex.run(b)
    ts = []
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        ex.run(b)
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    ex.free(b)
    return sorted(ts)[reps // 2]


t1 = timed(full)
print(f"1 GPU: {t1:.2f} ms")
for world in (2, 4, 8):
    ms = [timed(W.subset(full, s)) for s in W.shard_classes(full, world)]
    mx = max(ms)
    print(f"{world} GPUs: shard ms {[round(x, 2) for x in ms]}; step = max {mx:.2f} ms; "
          f"speed-up {t1 / mx:.2f}x, efficiency {t1 / mx / world:.2f}, imbalance max/mean {mx / (sum(ms) / world):.2f}")

# the slowest 8-way shard's phases (one batch, CUDA events around every launch)
shards = W.shard_classes(full, 8)
worst = max(range(8), key=lambda r: timed(W.subset(full, shards[r]), 3))
p = W.subset(full, shards[worst])
ex.split(False)
b = ex.prepare(p)
ex.run(b)
ex.profiling(True)
for _ in range(3):
    ex.run(b)
ex.fetch(b, p)
st = ex.kernel_stats()
ex.profiling(False)
print(f"8-way shard {worst}: {p.queries.size} queries, one batch {timed(p):.2f} ms")
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
    if v["ms"] / 3 > 0.1:
        print(f"  {k:24s} {v['ms'] / 3:8.3f} ms")
