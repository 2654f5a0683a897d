"""Tool (not collected by pytest): does running the C5 sweep as two batches
on two streams (the long-refine N = 64 classes beside the rest) overlap the
serial refine walks with the other batch's work?  Times each batch alone and
both concurrently (two contexts on one GPU), CUDA events around both."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

full = W.config_c5()
n = full.queries["n_stages"]
cut = int(sys.argv[1]) if len(sys.argv) > 1 else 64
groups = [np.nonzero(n >= cut)[0], np.nonzero(n < cut)[0]]
subs = [W.subset(full, g) for g in groups]
exs = [Explorer(0), Explorer(0)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
batches = [e.prepare(s, stream=st.cuda_stream) for e, s, st in zip(exs, subs, streams)]
main = torch.cuda.current_stream()


def timed(which, reps=5):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(main)
        for k in which:
            streams[k].wait_event(a)
            exs[k].run(batches[k], stream=streams[k].cuda_stream)
        for k in which:
            main.wait_stream(streams[k])
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts[2:])[reps // 2]


ta, tb, tab = timed([0]), timed([1]), timed([0, 1])
print(f"N >= {cut}: {groups[0].size} queries alone {ta:.2f} ms; the rest {groups[1].size} queries alone {tb:.2f} ms; "
      f"both concurrently {tab:.2f} ms (sum {ta + tb:.2f})")
full_b = exs[0].prepare(full, stream=streams[0].cuda_stream)
batches[0] = full_b
print(f"one batch: {timed([0]):.2f} ms")
