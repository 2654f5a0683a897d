"""Tool (not collected by pytest): the launch timeline of one C5 sweep as the
headline runs it (BP_OPT_SPLIT on: the parts on their own streams).  Every
launch is bracketed by CUDA events (profiling on) and BP_TIMELINE makes the
library write each span's start / end relative to the first.  Prints the spans
in start order and, per part stream, the busy intervals -- which phases of
one part overlap which of the other, and what ends the step."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.join(tempfile.mkdtemp(), "timeline.txt")
os.environ["BP_TIMELINE"] = path
trace = os.path.join(os.path.dirname(path), "refine_trace.txt")
os.environ["BP_REFINE_TRACE"] = trace

import torch  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.runtime import Explorer  # noqa: E402

split = "--no-split" not in sys.argv
e2e = "--e2e" in sys.argv     # through explore(): tables and queries uploaded, results copied back
p = W.config_c5()
ex = Explorer(0)
ex.split(split)
ex.profiling(True)
if e2e:
    out = p.alloc_outputs(False, pinned=True)
    for _ in range(2):
        ex.load(p, force=True)
        ex.explore(p, details=False, out=out)
    open(path, "w").close()
    open(trace, "w").close()
    ex.load(p, force=True)
    ex.explore(p, details=False, out=out)
else:
    b = ex.prepare(p)
    for _ in range(2):
        ex.run(b)
    torch.cuda.synchronize()
    ex.fetch(b, p)              # the warm-up runs' spans and walks: discarded
    open(path, "w").close()
    open(trace, "w").close()
    ex.run(b)
    torch.cuda.synchronize()
    ex.fetch(b, p)
ex.profiling(False)
rows = []
for line in open(path):
    if line.startswith("--"):
        continue
    name, a, z = line.split()
    rows.append((float(a), float(z), name))
rows.sort()
end = max(z for _, z, _ in rows)
print(f"split={'on' if split else 'off'}: {len(rows)} spans, last ends at {end:.2f} ms")
for a, z, name in rows:
    if z - a < 0.05 and not name.startswith("phase"):
        continue
    bar = int(a / end * 60)
    width = max(1, int((z - a) / end * 60))
    print(f"{a:8.3f} {z:8.3f} {z - a:7.3f}  {name:<22} |{' ' * bar}{'#' * width}")

# the refine walks of the measured run: when the longest ones started and ended
walks = []
for line in open(trace):
    if line.startswith("--"):
        continue
    q, steps, t0, t1, sm = map(int, line.split())
    walks.append((t1 - t0, q, steps, t0, t1, sm))
if walks:
    base = min(w[3] for w in walks)
    starts = sorted(w[3] for w in walks if w[5] >= 262144)
    prunes = [w for w in walks if 131072 <= w[5] < 262144]
    walks = [w for w in walks if w[5] < 131072]
    for k, t in enumerate(starts):   # per refine launch sequence (one per part)
        mine = [w for w in walks if w[3] >= t and (k + 1 == len(starts) or w[3] < starts[k + 1])]
        if mine:
            print(f"refine sequence {k}: first walk starts {(min(w[3] for w in mine) - t) / 1e6:.3f} ms after "
                  f"k_refine_keys, last walk ends {(max(w[4] for w in mine) - t) / 1e6:.3f} ms after it")
    if prunes:
        pb = min(w[3] for w in prunes)
        print(f"{len(prunes)} pruned candidates with >= 4 fine-tune trials; the longest (ms from the first one's start):")
        for d, q, work, t0, t1, sm in sorted(prunes, reverse=True)[:8]:
            print(f"  candidate {q:8d} trials x stages {work:6d} start {(t0 - pb) / 1e6:6.3f} end {(t1 - pb) / 1e6:6.3f} "
                  f"dur {d / 1e6:6.3f} ms")
    gen = [w for w in walks if w[5] >= 65536]
    print(f"{len(walks) - len(gen)} slim refine walks, {len(gen)} in the general kernel "
          f"(its last ends at {max((w[4] for w in gen), default=base) / 1e6 - base / 1e6:.3f} ms, "
          f"longest {max((w[0] for w in gen), default=0) / 1e6:.3f} ms, steps max {max((w[2] for w in gen), default=0)}); "
          "the longest walks (ms from the first walk's start):")
    for d, q, steps, t0, t1, sm in sorted(walks, reverse=True)[:12]:
        share = sum(1 for w in walks if w[5] == sm and w[3] < t1 and w[4] > t0) - 1
        kern = "general" if sm >= 65536 else "slim"
        print(f"  {kern} query {q:6d} steps {steps:5d} start {(t0 - base) / 1e6:6.3f} end {(t1 - base) / 1e6:6.3f} "
              f"dur {d / 1e6:6.3f} ms ({d / max(steps, 1):7.0f} ns/step) SM {sm:3d}, overlapping walks on the SM: {share}")
