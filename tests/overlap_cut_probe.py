"""Tool (not collected by pytest): C5 as two concurrent batches cut by stage
count (n >= cut | n < cut; one context each, BP_OPT_SPLIT off inside), for
several cuts: each part alone and both concurrently (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

full = W.config_c5()
n = full.queries["n_stages"]


def run(groups, which):
    subs = [W.subset(full, g) for g in groups]
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
        for k in which:
            sts[k].wait_event(a)
            exs[k].run(bs[k], stream=sts[k].cuda_stream)
        for k in which:
            main.wait_stream(sts[k])
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    for e, bb in zip(exs, bs):
        e.free(bb)
        e.close()
    return sorted(ts[2:])[2]


cuts = [int(x) for x in sys.argv[1:]] or [16, 24, 32, 64]
for cut in cuts:
    g = [np.nonzero(n >= cut)[0], np.nonzero(n < cut)[0]]
    ta, tb, tab = run(g, [0]), run(g, [1]), run(g, [0, 1])
    print(f"cut {cut}: n>={cut} alone {ta:.2f} ms, n<{cut} alone {tb:.2f} ms, concurrent {tab:.2f} ms")
