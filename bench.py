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
    ap.add_argument("--cpu-sample-stride", type=int, default=127)
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


SMS, LANES = 148, 128          # B200: SMs x (4 SMSP x 32 lanes) issue slots per clock
OPS_PER_TRANSITION = 3         # DP: sub, max, min (SURVEY.md 8d c_dp, int32/int64-in-one-op path)
OPS_PER_EVENT = 3              # simulator: max, add, store-forward (SURVEY.md 8d c_sim)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")


OPS_PER_REFINE_STEP = 3        # refine boundary step: compare t_a/t_b, t_hi - t_lo, / (c_from + c_to)
OPS_PER_PRUNE_STAGE = 4        # estimate per stage: F+B, features + 2w, capacity test, link demand

WORK_UNITS = {"minmax_dp": ("DP transitions", OPS_PER_TRANSITION),
              "minmax_dp_coarse": ("DP transitions", OPS_PER_TRANSITION),
              "refine": ("refine boundary steps", OPS_PER_REFINE_STEP),
              "prune": ("candidate-stages estimated", OPS_PER_PRUNE_STAGE)}


def work_unit(name):
    if name in WORK_UNITS:
        return WORK_UNITS[name]
    if name.startswith("sim_"):
        return ("simulated events", OPS_PER_EVENT)
    return None


def kernel_work_ops(name, work):
    """Algorithmic lane-ops of one launch of `name` from its work counter
    (Rooflines), or None for kernels without a work count."""
    u = work_unit(name)
    return None if u is None else work * u[1]


def rooflines(stats, steps, clocks, problem, step_ms):
    """Per-kernel issue rooflines and the sweep-level bound of SURVEY.md 8d.

    Every kernel on this path is integer / exact-rational control flow (no
    dense contraction, no streaming): the bound is the SM issue rate,
    148 SMs x 128 lanes x f_clk, at the measured max SM clock.  `achieved` is
    the kernel's ALGORITHMIC lane-ops per launch (work counter x ops/unit)
    over its average launch time (CUDA events on its stream)."""
    peaks, peak_kind = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    issue_peak = SMS * LANES * f_max / 1e9              # Gop/s
    try:
        with open(TRAFFIC_FILE) as f:
            traffic = json.load(f)
    except Exception:
        traffic = {}
    # counters without launches (critical paths, moves, trials) are reported
    # beside the kernels, not as kernels
    counters = {k: stats[k]["work"] for k in list(stats) if stats[k]["launches"] == 0 and k != "refine_critical_path"}
    for k in counters:
        stats.pop(k)
    # phase spans (several launches over both streams) are reported apart
    phases = {k: stats.pop(k)["ms"] / steps for k in list(stats) if k.startswith("phase_")}
    # the prune phase is four launches (keys + list, representatives, members'
    # shared estimates, members' own prunes); its work counter covers all of
    # them, so its rate is quoted on the phase
    parts = [k for k in ("prune_list", "prune", "prune_members", "prune_members_full") if k in stats]
    if "prune" in stats and len(parts) > 1:
        stats["prune"] = {"ms": sum(stats.pop(k)["ms"] for k in parts if k != "prune") + stats["prune"]["ms"],
                          "launches": stats["prune"]["launches"], "work": stats["prune"]["work"]}
    kern = {}
    for k, v in stats.items():
        ms = v["ms"] / max(1, v["launches"])
        e = {"ms_per_step": v["ms"] / steps, "launches": v["launches"], "work_per_launch": v["work"]}
        ops = kernel_work_ops(k, v["work"])
        if ops is not None and ms > 0:
            e["achieved_gops"] = ops / (ms * 1e6)
            e["frac"] = e["achieved_gops"] / issue_peak
        kern[k] = e
    crit = stats.pop("refine_critical_path", None)
    kern.pop("refine_critical_path", None)
    kern["counters"] = counters
    kern["phases_ms_per_step"] = phases
    dom = max(stats, key=lambda k: stats[k]["ms"])
    d = kern[dom]
    u = work_unit(dom)
    roof = {"kernel": dom, "bound": "issue", "unit": "Gop/s", "peak": issue_peak,
            "achieved": d.get("achieved_gops"), "frac": d.get("frac"),
            "traffic": traffic.get(dom),
            "work": (f"{d['work_per_launch']:.4g} {u[0]}/launch x {u[1]} ops" if u and d.get("achieved_gops")
                     is not None else f"{dom}: no work count"),
            "peak_source": f"{SMS} SMs x {LANES} lanes x {f_max / 1e6:.0f} MHz (sm_max_mhz, {peak_kind} "
                           f"MEASURED_PEAKS.json); HBM {peaks.get('hbm_gbs')} GB/s"}
    if dom == "refine" and crit and crit["work"] > 0:
        # refine is a serial recurrence per query: its time is the longest
        # query's walk, so the meaningful bound is per-step latency on that path
        ms_launch = d["ms_per_step"]
        roof["critical_path"] = {"boundary_steps": crit["work"], "us_per_step": 1e3 * ms_launch / crit["work"],
                                 "cycles_per_step": ms_launch * 1e-3 * f_max / crit["work"],
                                 "note": "one query's intra_layer_refine walk is serial (each boundary step "
                                         "reads the stage times the previous step wrote)"}
    # sweep bound: t_roof = sum B_cost / BW + (X_dp * c_dp + X_sim * c_sim) / issue
    q = problem.queries
    U = np.array([problem.networks[i].L for i in q["network"]], dtype=np.float64)
    N = q["n_stages"].astype(np.float64)
    T = np.array([len(set(problem.clusters[c].types[:n].tolist())) for c, n in zip(q["cluster"], q["n_stages"])],
                 dtype=np.float64)
    b_cost = float(np.sum(8 * U * (2 * T + 2)))
    x_dp_ref = float(np.sum(np.where(U >= N, N * (U - N + 1) * (U - N + 2), 0)))
    x_sim = float(sum(v["work"] for k, v in stats.items() if k.startswith("sim_")))
    x_dp = float(sum(v["work"] for k, v in stats.items() if k.startswith("minmax_dp")))
    hbm = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    t_ref = b_cost / hbm + (x_dp_ref * OPS_PER_TRANSITION + x_sim * OPS_PER_EVENT) / (issue_peak * 1e9)
    t_own = b_cost / hbm + (x_dp * OPS_PER_TRANSITION + x_sim * OPS_PER_EVENT) / (issue_peak * 1e9)
    sweep = {"t_roof_ms_reference_dp": 1e3 * t_ref, "t_roof_ms_banded_dp": 1e3 * t_own, "t_measured_ms": step_ms,
             "frac": 1e3 * t_ref / step_ms,
             "x_dp_reference": x_dp_ref, "x_dp_performed": x_dp, "x_sim_events": x_sim, "b_cost_bytes": b_cost,
             "formula": "t_roof = B_cost/HBM + (X_dp*3 + X_sim*3)/(148*128*f_max); frac = t_roof(reference X_dp) / "
                        "t_measured (SURVEY.md 8d)"}
    return roof, kern, sweep


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
    stride = 257    # prime: 255-256 queries (~4,096 candidates) per step, rotating offsets
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
            "config": {"workload": "C5 sweep sample: 1/257 query stride per step (~256 queries, ~4,096 candidates), "
                                   "rotating offsets", "models": args.models},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if oracle.kind == "reference" else 1,
                             "kind": oracle.kind, "sample": "1/257 query stride of C5 per step, offset = step index"},
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

    # ---- the same steps with the batch dedup off (BP_OPT_DEDUP = 0: every
    # query and candidate solved on its own; identical results)
    ex.dedup(False)
    with torch.cuda.stream(stream):
        ex.run(batch, stream=sp)
    nd_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()
            nd_evs[i][0].record(stream)
            ex.run(batch, stream=sp)
            nd_evs[i][1].record(stream)
    barrier()
    ex.dedup(True)
    nd_ms = sum(a.elapsed_time(b) for a, b in nd_evs)
    if world > 1:
        t = torch.tensor([nd_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        nd_ms = float(t.item())
    value_nodedup = cands_per_step * args.steps / (nd_ms / 1e3)

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
    clocks = clk.summary()
    roof, kern, sweep = rooflines(stats, args.steps, clocks, p, total_ms / args.steps)

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
            "no_dedup": {"value": value_nodedup, "unit": UNIT, "ms_per_step": nd_ms / args.steps,
                         "note": "same steps with BP_OPT_DEDUP=0: identical subproblems of the batch not shared"},
            "gpu_launches": launches,
            "clocks": clocks,
            "roofline": roof,
            "sweep_roofline": sweep,
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
