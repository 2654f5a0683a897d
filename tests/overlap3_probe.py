"""Tool (not collected by pytest): C5 as 2, 3 or 4 concurrent batches split by stage count (one context each)."""
import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.runtime import Explorer
full = W.config_c5(); n = full.queries["n_stages"]
def run(groups):
    subs = [W.subset(full, g) for g in groups]
    exs = [Explorer(0) for _ in subs]
    for e in exs: e.split(False)
    sts = [torch.cuda.Stream() for _ in subs]
    bs = [e.prepare(s, stream=st.cuda_stream) for e, s, st in zip(exs, subs, sts)]
    main = torch.cuda.current_stream()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(main)
        for e, bb, st in zip(exs, bs, sts):
            st.wait_event(a); e.run(bb, stream=st.cuda_stream)
        for st in sts: main.wait_stream(st)
        b.record(main); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    for e, bb in zip(exs, bs): e.free(bb); e.close()
    return sorted(ts[2:])[2]
print("2-way 64|rest", run([np.nonzero(n == 64)[0], np.nonzero(n < 64)[0]]))
print("3-way 64|24-32|rest", run([np.nonzero(n == 64)[0], np.nonzero((n >= 24) & (n < 64))[0], np.nonzero(n < 24)[0]]))
print("3-way 64|32|rest", run([np.nonzero(n == 64)[0], np.nonzero(n == 32)[0], np.nonzero(n < 32)[0]]))
print("4-way 64|32|24|rest", run([np.nonzero(n == 64)[0], np.nonzero(n == 32)[0], np.nonzero(n == 24)[0], np.nonzero(n < 24)[0]]))
