#!/usr/bin/env python3
"""Benchmark: BaPipe explore() candidates evaluated per second on B200.

Workload (BASELINE.json configs[4]): the sweep of 128
synthetic models x 64 cluster mixes x 8 stage counts x 8 micro-batch counts x
2 schedule kinds = 2^20 candidates (65,536 explore() queries).  A step is one
pass of the explore() path over that batch.  Scaling is weak: rank r sweeps
its own 2^20 candidates (models 128r..128r+127), so the whole job processes
N * 2^20 candidates per step; the per-rank best records are exchanged with
one NCCL allgather and reduced with the deterministic argmin.

  value   candidates/s with inputs resident in HBM (bp_batch_run), device
          time from CUDA events on the launching stream, max over ranks
  e2e     the same metric through the public C ABI with host buffers: every
          step uploads the network/cluster tables and the queries from pinned
          host memory (bp_set_networks / bp_set_clusters / bp_explore_batch)
          and reads the per-query results back
  --impl reference   the reference's own CPU explore() (oracle/_ref, built
          from /root/reference) on the host cores, bounded samples of C5

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.problem import BEST_DTYPE, Problem  # noqa: E402

METRIC = "partition candidates evaluated/sec (C5 sweep)"
UNIT = "candidates/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--models", type=int, default=128, help="models per rank (128 = full 2^20 sweep)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-stride", type=int, default=1021)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def cpu_baseline(problem, stride, threads):
    """The reference's own explore() (oracle/_ref) on a bounded C5 sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import PortOracle, RefOracle, ref_available
    oracle = RefOracle() if ref_available() else PortOracle()
    idx = np.arange(0, problem.queries.size, stride)
    sub = Problem(networks=problem.networks, clusters=problem.clusters)
    q = problem.queries[idx]
    sub.set_queries(q["network"], q["cluster"], q["n_stages"], q["mini_batch"])
    t = time.perf_counter()
    if oracle.kind == "reference":
        res = oracle.explore_timed(sub, threads=threads)
    else:
        res, _, _ = oracle.explore(sub, details=False)
        threads = 1
    dt = time.perf_counter() - t
    return {"value": sub.total_candidates / dt, "unit": UNIT, "cores": threads, "kind": oracle.kind,
            "sample": f"C5 1/{stride} query stride ({sub.queries.size} queries, {sub.total_candidates} "
                      f"candidates), explore() per query on {threads} host threads, {dt:.1f} s",
            "status_hist": np.bincount(res["status"], minlength=7).tolist()}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    p = W.config_c5(models=args.models)
    threads = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import PortOracle, RefOracle, ref_available
    oracle = RefOracle() if ref_available() else PortOracle()
    stride = 4093   # prime: ~16 queries (256 candidates) per step, rotating offsets
    times, cands = [], []
    for step in range(args.warmup + args.steps):
        idx = np.arange(step % stride, p.queries.size, stride)
        sub = Problem(networks=p.networks, clusters=p.clusters)
        q = p.queries[idx]
        sub.set_queries(q["network"], q["cluster"], q["n_stages"], q["mini_batch"])
        t = time.perf_counter()
        if oracle.kind == "reference":
            oracle.explore_timed(sub, threads=threads)
        else:
            oracle.explore(sub, details=False)
        dt = time.perf_counter() - t
        if step >= args.warmup:
            times.append(dt)
            cands.append(sub.total_candidates)
    value = sum(cands) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64/exact-rational",
            "data": "synthetic (C5 generator, mt19937_64 seeds of SURVEY.md 8d)",
            "config": {"workload": "C5 sweep sample: 1/4093 query stride per step (~16 queries, ~256 candidates), "
                                   "rotating offsets", "models": args.models},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if oracle.kind == "reference" else 1,
                             "kind": oracle.kind, "sample": "1/4093 query stride of C5 per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    from paper_2012_12544_b200.runtime import Explorer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream

    p = W.config_c5(models=args.models, model_base=rank * args.models)
    p.pin()
    ex = Explorer(local)
    ex.load(p)
    batch = ex.prepare(p, details=False, stream=sp)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    # ---- device-resident steps (value)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            ex.run(batch, stream=sp)
    torch.cuda.synchronize()
    ex.profiling(True)
    l0 = ex.launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()                       # L2 flush between steps (not timed)
                evs[i][0].record(stream)
                ex.run(batch, stream=sp)
                evs[i][1].record(stream)
        barrier()
    launches = ex.launches() - l0
    res, _, _ = ex.fetch(batch, p, details=False, stream=sp)
    stats = ex.kernel_stats()
    ex.profiling(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    cands_per_step = p.total_candidates * world
    value = cands_per_step * args.steps / (total_ms / 1e3)

    # ---- global best: per-rank record -> one allgather -> deterministic argmin
    rec = torch.zeros(BEST_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ex.best(batch, rec.data_ptr(), query_base=rank * p.queries.size, stream=sp)
    torch.cuda.synchronize()
    if world > 1:
        allrec = [torch.zeros_like(rec) for _ in range(world)]
        torch.distributed.all_gather(allrec, rec)
        recs = [r.cpu().numpy().view(BEST_DTYPE)[0] for r in allrec]
    else:
        recs = [rec.cpu().numpy().view(BEST_DTYPE)[0]]
    from paper_2012_12544_b200.runtime import best_less
    best = recs[0]
    for r in recs[1:]:
        if best_less(r, best):
            best = r

    # ---- end-to-end steps through the C ABI with host buffers (e2e)
    h0, d0 = ex.transfers()
    for _ in range(max(1, args.warmup)):
        ex.load(p, force=True)
        ex.explore(p, details=False, stream=sp)
    torch.cuda.synchronize()
    h1, d1 = ex.transfers()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ex.load(p, force=True)                 # H2D network + cluster tables (pinned host memory)
        r2, _, _ = ex.explore(p, details=False, stream=sp)   # H2D queries, kernels, D2H results
        e2e_ms.append(1e3 * (time.perf_counter() - t))
    barrier()
    h2, d2 = ex.transfers()
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = cands_per_step * args.steps / (e2e_total / 1e3)
    assert r2.tobytes() == res.tobytes(), "e2e results differ from the device-resident run"

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel
    peaks, peak_kind = measured_peaks()
    clocks = clk.summary()
    dom = max(stats.items(), key=lambda kv: kv[1]["ms"])
    f_clk = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    issue_peak = 148 * 128 * f_clk / 1e9          # lane-ops per ns == Gop/s
    dp = stats.get("minmax_dp", {"ms": 0.0, "work": 0.0})
    roof = {"kernel": dom[0], "bound": "issue", "unit": "Gop/s",
            "peak": issue_peak, "peak_source": f"148 SMs x 128 lanes x {f_clk/1e6:.0f} MHz (SM clock sampled "
                                                 f"during the timed region); {peak_kind} peaks file",
            "traffic": None}
    if dom[0] == "minmax_dp" and dp["ms"] > 0:
        ops = dp["work"] * 3.0          # sub, max, min per DP transition (SURVEY.md 8d c_dp)
        roof.update({"achieved": ops / (dp["ms"] * 1e6), "frac": ops / (dp["ms"] * 1e6) / issue_peak,
                     "work": f"{dp['work']/args.steps:.4g} DP transitions/launch x 3 ops"})
    else:
        roof.update({"achieved": None, "frac": None,
                     "work": f"dominant kernel {dom[0]} is latency-bound exact-rational code; see DESIGN.md"})
    kern = {k: {"ms_per_step": v["ms"] / args.steps, "launches": v["launches"]} for k, v in stats.items()}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64/exact-rational",
            "data": "synthetic (C5 generator, mt19937_64 seeds of SURVEY.md 8d; random-init layer tables)",
            "config": {"workload": "C5 sweep: 128 models x 64 cluster mixes x 8 stage counts x 8 M x 2 kinds "
                                   "= 2^20 candidates per GPU",
                       "queries_per_gpu": int(p.queries.size), "candidates_per_gpu": int(p.total_candidates),
                       "parallelism": f"weak x{world} (query shards per GPU, NCCL allgather of best records)",
                       "l2": "256 MiB buffer written between timed steps (L2 flush)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_total / args.steps,
                    "h2d_bytes_per_step": (h2 - h1) // args.steps, "d2h_bytes_per_step": (d2 - d1) // args.steps},
            "gpu_launches": launches,
            "clocks": clocks,
            "roofline": roof,
            "kernels": kern,
            "best": {"makespan": f"{int(best['makespan']['num'])}/{int(best['makespan']['den'])}",
                     "M": int(best["M"]), "kind": int(best["kind"]), "query_id": int(best["query_id"])},
            "query_status_hist": np.bincount(res["status"], minlength=7).tolist()}
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(p, args.cpu_sample_stride, os.cpu_count() or 1)
        except Exception as e:   # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
