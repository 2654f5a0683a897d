"""Run the C5 sweep once (best-only) -- target for ncu captures."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2012_12544_b200 import workloads as W
from paper_2012_12544_b200.runtime import Explorer
p = W.config_c5()
ex = Explorer(0)
res, _, _ = ex.explore(p, details=False)
print("ok", res.size)
