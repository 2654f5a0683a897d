"""Tool (not collected by pytest): the e2e step against its pieces (wall ms, medians)."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.runtime import Explorer
p = W.config_c5(); ex = Explorer(0); out = p.alloc_outputs(False, pinned=True)
sp = torch.cuda.Stream()
def med(f, n=8):
    ts = []
    for _ in range(3): f()
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); ts.append(1e3 * (time.perf_counter() - t))
    ts.sort(); return ts[len(ts) // 2]
def v1():
    ex.load(p, force=True); ex.explore(p, details=False, stream=sp.cuda_stream, out=out)
def v2():
    ex.explore(p, details=False, stream=sp.cuda_stream, out=out)
r1, r2 = med(v1), med(v2)
parts = {}
for k in (2, 6, 8):
    ex.split(k)
    parts[k] = (med(v1), med(v3b) if False else None)
    ex.split(True)
b = ex.prepare(p, stream=sp.cuda_stream)
def v3():
    ex.run(b, stream=sp.cuda_stream); torch.cuda.synchronize()
def v4():
    bb = ex.prepare(p, stream=sp.cuda_stream); ex.run(bb, stream=sp.cuda_stream); ex.fetch(bb, p, stream=sp.cuda_stream); ex.free(bb)
print("load+explore %.2f  explore only %.2f  run only (resident) %.2f  prepare+run+fetch %.2f" % (r1, r2, med(v3), med(v4)))
print("load+explore with 2 parts %.2f, 6 parts %.2f, 8 parts %.2f" % (parts[2][0], parts[6][0], parts[8][0]))
