"""Tool (not collected by pytest): e2e and device time of the C5 sweep with BP_OPT_SPLIT on and off."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.runtime import Explorer
p = W.config_c5(); p.pin()
ex = Explorer(0)
for split in (True, False, True, False, True, False):
    ex.split(split)
    for _ in range(3):
        ex.load(p, force=True); ex.explore(p, details=False)
    ts = []
    for _ in range(15):
        torch.cuda.synchronize(); t = time.perf_counter()
        ex.load(p, force=True); ex.explore(p, details=False)
        ts.append(1e3 * (time.perf_counter() - t))
    b = ex.prepare(p); ex.run(b); torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev = []
    for _ in range(5):
        a.record(); ex.run(b); e.record(); torch.cuda.synchronize(); dev.append(a.elapsed_time(e))
    ex.free(b)
    print(f"split={split}: e2e median {sorted(ts)[7]:.2f} ms (min {min(ts):.2f}), device median {sorted(dev)[2]:.2f} ms")

# where the end-to-end time goes: host wall time of explore() alone (tables
# already loaded) against the device time between events recorded on the
# call's stream just before and after it
ex.split(True)
s = torch.cuda.Stream()
for _ in range(3):
    ex.explore(p, details=False, stream=s.cuda_stream)
for _ in range(5):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    a.record(s)
    ex.explore(p, details=False, stream=s.cuda_stream)
    e.record(s)
    torch.cuda.synchronize()
    print(f"explore() without table upload: host {1e3 * (time.perf_counter() - t):.2f} ms, device span {a.elapsed_time(e):.2f} ms")
