#!/usr/bin/env python3
"""Benchmark: BaPipe explore() candidates evaluated per second on B200.

Workload (BASELINE.json configs[4]): the sweep of 128
synthetic models x 64 cluster mixes x 8 stage counts x 8 micro-batch counts x
2 schedule kinds = 2^20 candidates (65,536 explore() queries).  A step is one
pass of the explore() path over that batch.  Scaling is strong by default
(north_star: one 10^6-candidate sweep sharded over the GPUs): rank r runs the
queries of its shard of the ONE sweep -- whole batch-dedup classes assigned
by estimated cost (workloads.shard_classes) -- and the per-rank best records
are exchanged with one NCCL allgather and reduced with the deterministic
argmin.  --scaling weak gives every rank its own 2^20-candidate sweep.

  value   candidates/s with inputs resident in HBM (bp_batch_run), device
          time from CUDA events on the launching stream, max over ranks
  e2e     the same metric through the public C ABI with host buffers: every
          step uploads the network/cluster tables and the queries from pinned
          host memory (bp_set_networks / bp_set_clusters / bp_explore_batch)
          and reads the per-query results back into a pinned buffer the caller
          allocated once
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
from paper_2012_12544_b200.problem import BEST_DTYPE  # noqa: E402

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
    ap.add_argument("--no-per-call", action="store_true")
    ap.add_argument("--cpu-sample-stride", type=int, default=127)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
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
        if ops is not None and ms > 0 and not k.startswith("sim_"):
            e["achieved_gops"] = ops / (ms * 1e6)
            e["frac"] = e["achieved_gops"] / issue_peak
        elif k.startswith("sim_"):
            # the simulator classes run concurrently on two streams: a
            # kernel's event-timed span includes the other stream's work, so
            # rates are quoted on the phase (phases_ms_per_step), not here
            e["note"] = "overlapped on two streams; see phases_ms_per_step"
        kern[k] = e
    crit = stats.pop("refine_critical_path", None)
    kern.pop("refine_critical_path", None)
    kern["counters"] = counters
    kern["phases_ms_per_step"] = phases
    # the simulator classes overlap on two streams: as a group they are one
    # "kernel" (the phase span, all simulated events)
    sims = [k for k in stats if k.startswith("sim_") and k not in ("sim_prep", "sim_share")]
    if sims and "phase_sims" in phases:
        ev = sum(stats[k]["work"] for k in sims)
        kern["simulate"] = {"ms_per_step": phases["phase_sims"], "launches": steps, "work_per_launch": ev,
                            "achieved_gops": ev * OPS_PER_EVENT / (phases["phase_sims"] * 1e6),
                            "note": "all simulator kernels of the step (both streams): phase span, all events"}
        kern["simulate"]["frac"] = kern["simulate"]["achieved_gops"] / issue_peak
    cands = {k: kern[k]["ms_per_step"] for k in kern if isinstance(kern[k], dict) and "ms_per_step" in kern[k]
             and not k.startswith("sim_")}
    dom = max(cands, key=cands.get)
    d = kern[dom]
    u = ("simulated events", OPS_PER_EVENT) if dom == "simulate" else work_unit(dom)
    roof = {"kernel": dom, "bound": "issue", "unit": "Gop/s", "peak": issue_peak,
            "achieved": d.get("achieved_gops"), "frac": d.get("frac"),
            "traffic": traffic.get(dom),
            "work": (f"{d['work_per_launch']:.4g} {u[0]}/launch x {u[1]} ops" if u and d.get("achieved_gops")
                     is not None else f"{dom}: no work count"),
            "peak_source": f"{SMS} SMs x {LANES} lanes x {f_max / 1e6:.0f} MHz (sm_max_mhz, {peak_kind} "
                           f"MEASURED_PEAKS.json); HBM {peaks.get('hbm_gbs')} GB/s"}
    refine_lat = None
    if crit and crit["work"] > 0 and "refine" in kern:
        # refine is a serial recurrence per query: its time is the longest
        # query's walk, so the meaningful bound is per-step latency on that path
        ms_launch = kern["refine"]["ms_per_step"]
        refine_lat = {"longest_walk_steps": crit["work"], "refine_ms_per_step": ms_launch,
                      "us_per_step_in_sweep": 1e3 * ms_launch / crit["work"],
                      "cycles_per_step_in_sweep": ms_launch * 1e-3 * f_max / crit["work"],
                      "note": "one query's intra_layer_refine walk is serial (each boundary step reads the stage "
                              "times the previous step wrote): the refine launch cannot end before its longest "
                              "walk, so its bound is that walk's latency alone on an idle GPU (walk_alone)"}
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
    # a cheaper DP must charge the work it performs, so the
    # fraction is t_roof(performed X_dp, simulated events) / t_measured.  The
    # reference's X_dp at the same pace is a work-equivalence figure only.
    sweep = {"t_roof_ms": 1e3 * t_own, "t_measured_ms": step_ms, "frac": 1e3 * t_own / step_ms,
             "x_dp_performed": x_dp, "x_sim_events": x_sim, "b_cost_bytes": b_cost,
             "formula": "t_roof = B_cost/HBM + (X_dp*3 + X_sim*3)/(148*128*f_max) over the work performed; "
                        "frac = t_roof / t_measured (SURVEY.md 8d)",
             "work_equivalence": {"x_dp_reference": x_dp_ref, "t_roof_ms_reference_dp": 1e3 * t_ref,
                                  "ratio": 1e3 * t_ref / step_ms,
                                  "note": "the reference's own DP transitions (3L^2-class loops) at roofline pace "
                                          "against our measured step: how much reference work one step replaces, "
                                          "not a roofline fraction"}}
    return roof, kern, sweep, refine_lat


def cpu_baseline(problem, stride, threads):
    """The reference's own explore() (oracle/_ref) on a bounded C5 sample:
    the -O3 -march=native timing build, and the bounds-checking parity build
    beside it."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import PortOracle, RefOracle, ref_available
    idx = np.arange(0, problem.queries.size, stride)
    sub = W.subset(problem, idx)

    def timed(oracle):
        t = time.perf_counter()
        if oracle.kind == "reference":
            res = oracle.explore_timed(sub, threads=threads)
            n = threads
        else:
            res, _, _ = oracle.explore(sub, details=False)
            n = 1
        return time.perf_counter() - t, res, n

    if not ref_available():
        oracle = PortOracle()
        dt, res, n = timed(oracle)
        return {"value": sub.total_candidates / dt, "unit": UNIT, "cores": n, "kind": "port",
                "sample": f"C5 1/{stride} query stride ({sub.total_candidates} candidates), {dt:.1f} s"}
    fast = RefOracle(fast=True)
    dt, res, n = timed(fast)
    out = {"value": sub.total_candidates / dt, "unit": UNIT, "cores": n, "kind": "reference", "build": fast.build,
           "sample": f"C5 1/{stride} query stride ({sub.queries.size} queries, {sub.total_candidates} "
                     f"candidates), explore() per query on {n} host threads, {dt:.1f} s",
           "status_hist": np.bincount(res["status"], minlength=7).tolist()}
    checked = RefOracle()
    if checked.build != fast.build:
        dt2, _, _ = timed(checked)
        out["checking_build"] = {"value": sub.total_candidates / dt2, "build": checked.build, "seconds": dt2}
    return out


def per_call(reps_small=20, reps_c4=3):
    """explore() on single queries, one call at a time (BASELINE.md's CPU
    plan: C1-C3 >= 20 repetitions, C4 in its variants): the drop-in's
    explore() (include/bapipe_b200/explorer.hpp, host structs in, result out,
    every candidate on the GPU) against the reference's own explore() on one
    host core (-O3 -march=native) and, as aggregate calls/s, on every core."""
    import tempfile
    prod = os.path.join(ROOT, "paper_2012_12544_b200", "bin", "percall")
    ref = os.path.join(ROOT, "oracle", "_ref", "percall_ref")
    if not os.path.exists(prod):
        return {"error": "paper_2012_12544_b200/bin/percall not built"}
    out = {"cases": [], "note": "wall ms per explore() call; product: first call of a context excluded (2 warm-up "
                                "calls per case)"}
    with tempfile.TemporaryDirectory() as d:
        groups = {"small": [], "c4": []}
        for name, p, types in W.single_query_configs():
            q = p.queries[0]
            nf, cf = os.path.join(d, f"{len(out['cases'])}_net.json"), os.path.join(d, f"{len(out['cases'])}_cl.json")
            with open(nf, "w") as f:
                json.dump(W.network_json(p.networks[0], types), f)
            with open(cf, "w") as f:
                json.dump(W.cluster_json(p.clusters[0], types), f)
            groups["c4" if name.startswith("C4") else "small"].append((name, str(int(q["mini_batch"])), nf, cf))
            out["cases"].append(name)

        def run(exe, reps, cases, threads=0):
            cmd = [exe] + (["--threads", str(threads)] if threads else []) + [str(reps)]
            for _, mb, nf, cf in cases:
                cmd += [mb, nf, cf]
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
            return [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]

        res = {}
        for who, exe, threads in (("b200", prod, 0), ("reference", ref, os.cpu_count() or 1)):
            if not os.path.exists(exe):
                res[who] = None
                continue
            rows = run(exe, reps_small, groups["small"], threads) + run(exe, reps_c4, groups["c4"], 0)
            res[who] = {name: {k: v for k, v in r.items() if k != "ms" and k != "case"}
                        for name, r in zip([c[0] for c in groups["small"] + groups["c4"]], rows)}
        out.update(res)
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    p = W.config_c5(models=args.models)
    threads = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import PortOracle, RefOracle, ref_available
    oracle = RefOracle(fast=True) if ref_available() else PortOracle()
    stride = 257    # prime: 255-256 queries (~4,096 candidates) per step, rotating offsets
    times, cands = [], []
    for step in range(args.warmup + args.steps):
        idx = np.arange(step % stride, p.queries.size, stride)
        sub = W.subset(p, idx)
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
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int64/exact-rational",
            "data": "synthetic (C5 generator, mt19937_64 seeds of SURVEY.md 8d)",
            "config": {"workload": "C5 sweep sample: 1/257 query stride per step (~256 queries, ~4,096 candidates), "
                                   "rotating offsets", "models": args.models},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if oracle.kind == "reference" else 1,
                             "kind": oracle.kind, "build": getattr(oracle, "build", "port"),
                             "sample": "1/257 query stride of C5 per step, offset = step index"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


LONGEST_WALK_QUERY = 18895     # C5's longest refine walk (N = 64, L = 128, 3,255 boundary steps)


def walk_alone(ex, full, sp):
    """The refine launch of a batch holding only C5's longest-walk query:
    its walk's latency on an otherwise idle GPU (the refine phase's floor)."""
    one = W.subset(full, [LONGEST_WALK_QUERY])
    b = ex.prepare(one, details=False, stream=sp)
    ex.run(b, stream=sp)
    ex.profiling(True)
    for _ in range(3):
        ex.run(b, stream=sp)
    ex.fetch(b, one, stream=sp)
    st = ex.kernel_stats()
    ex.profiling(False)
    ex.free(b)
    r = st.get("refine", {})
    return {"query": LONGEST_WALK_QUERY, "steps": st.get("refine_critical_path", {}).get("work", 0),
            "ms": r.get("ms", 0) / max(1, r.get("launches", 1))}


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

    if args.scaling == "strong":
        # ONE sweep, sharded: whole dedup classes per rank, balanced by cost
        full = W.config_c5(models=args.models)
        p = W.subset(full, W.shard_classes(full, world)[rank]) if world > 1 else full
        cands_per_step = full.total_candidates
    else:
        full = W.config_c5(models=args.models, model_base=rank * args.models)
        p = full
        cands_per_step = p.total_candidates * world
    qids = getattr(p, "query_ids", np.arange(p.queries.size, dtype=np.int64))
    p.pin()
    ex = Explorer(local)
    ex.load(p)
    batch = ex.prepare(p, details=False, stream=sp)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x, [x]
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        torch.distributed.all_gather(allt, t)
        v = [float(a.item()) for a in allt]
        return max(v), v

    # ---- device-resident steps (value)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            ex.run(batch, stream=sp)
    torch.cuda.synchronize()
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
    step_ms = [a.elapsed_time(b) for a, b in evs]

    # ---- per-kernel breakdown (CUDA events around every launch), on the same
    # steps run as ONE batch (BP_OPT_SPLIT off): with the split, the parts run
    # concurrently and their kernel spans would overlap
    ex.split(False)
    kb = ex.prepare(p, details=False, stream=sp)
    with torch.cuda.stream(stream):
        ex.run(kb, stream=sp)
    torch.cuda.synchronize()
    ex.profiling(True)
    kb_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()
            kb_evs[i][0].record(stream)
            ex.run(kb, stream=sp)
            kb_evs[i][1].record(stream)
    torch.cuda.synchronize()
    res_kb, _, _ = ex.fetch(kb, p, details=False, stream=sp)
    stats = ex.kernel_stats()
    ex.profiling(False)
    ex.free(kb)
    ex.split(True)
    assert res_kb.tobytes() == res.tobytes(), "one-batch and split runs differ"
    kb_ms = sum(a.elapsed_time(b) for a, b in kb_evs) / args.steps
    total_ms, rank_ms = max_over_ranks(sum(step_ms))
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
    nd_ms, _ = max_over_ranks(sum(a.elapsed_time(b) for a, b in nd_evs))
    value_nodedup = cands_per_step * args.steps / (nd_ms / 1e3)

    # ---- the same steps with BP_OPT_PRUNE_LB: scaled-integer
    # candidates dominated by their query's best are not simulated; every
    # per-query result is identical (checked)
    ex.prune_lb(True)
    with torch.cuda.stream(stream):
        ex.run(batch, stream=sp)
    lb_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()
            lb_evs[i][0].record(stream)
            ex.run(batch, stream=sp)
            lb_evs[i][1].record(stream)
    barrier()
    res_lb, _, _ = ex.fetch(batch, p, details=False, stream=sp)
    ex.prune_lb(False)
    assert res_lb.tobytes() == res.tobytes(), "BP_OPT_PRUNE_LB changed a per-query result"
    lb_ms, _ = max_over_ranks(sum(a.elapsed_time(b) for a, b in lb_evs))
    value_lb = cands_per_step * args.steps / (lb_ms / 1e3)

    # ---- global best: per-rank record -> one allgather -> deterministic argmin
    rec = torch.zeros(BEST_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ex.best(batch, rec.data_ptr(), query_base=0, stream=sp)
    torch.cuda.synchronize()
    r0 = rec.cpu().numpy().view(BEST_DTYPE).copy()
    if r0[0]["valid"]:
        r0[0]["query_id"] = int(qids[int(r0[0]["query_id"])])   # shard-local -> global query id
    rec.copy_(torch.from_numpy(r0.view(np.uint8)).to(rec.device))
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
    # the caller's result buffer: pinned host memory, allocated once and
    # reused by every call (the D2H of each step lands in it)
    out = p.alloc_outputs(False, pinned=True)
    for _ in range(max(1, args.warmup)):
        ex.load(p, force=True)
        ex.explore(p, details=False, stream=sp, out=out)
    torch.cuda.synchronize()
    h1, d1 = ex.transfers()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ex.load(p, force=True)                 # H2D network + cluster tables (pinned host memory)
        r2, _, _ = ex.explore(p, details=False, stream=sp, out=out)   # H2D queries, kernels, D2H results
        e2e_ms.append(1e3 * (time.perf_counter() - t))
    barrier()
    h2, d2 = ex.transfers()
    e2e_total, _ = max_over_ranks(sum(e2e_ms))
    e2e_value = cands_per_step * args.steps / (e2e_total / 1e3)
    assert r2.tobytes() == res.tobytes(), "e2e results differ from the device-resident run"

    # ---- the same, returning every candidate record too (the drop-in's whole
    # ExplorationResult: ranked lists need them), into pinned buffers
    outc = p.alloc_outputs("candidates", pinned=True)
    ex.load(p, force=True)
    ex.explore(p, details="candidates", stream=sp, out=outc)
    torch.cuda.synchronize()
    hc0, dc0 = ex.transfers()
    cand_ms = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ex.load(p, force=True)
        r3, _, _ = ex.explore(p, details="candidates", stream=sp, out=outc)
        cand_ms.append(1e3 * (time.perf_counter() - t))
    hc1, dc1 = ex.transfers()
    assert r3.tobytes() == res.tobytes(), "e2e (candidate records) results differ"
    cand_total, _ = max_over_ranks(sum(cand_ms))
    e2e_cand = {"value": cands_per_step * 3 / (cand_total / 1e3), "unit": UNIT, "ms_per_step": cand_total / 3,
                "h2d_bytes_per_step": (hc1 - hc0) // 3, "d2h_bytes_per_step": (dc1 - dc0) // 3,
                "note": "e2e with every bp_candidate record returned as well (details=candidates), 3 steps"}

    alone = walk_alone(ex, full, sp) if (rank == 0 and args.models == 128 and args.scaling == "strong") else None
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel
    clocks = clk.summary()
    roof, kern, sweep, refine_lat = rooflines(stats, args.steps, clocks, p, total_ms / args.steps)
    if refine_lat is not None and alone is not None and alone["ms"] > 0:
        refine_lat["walk_alone"] = alone
        refine_lat["latency_bound_frac"] = alone["ms"] / refine_lat["refine_ms_per_step"]
    mean_ms = sum(rank_ms) / len(rank_ms)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64/exact-rational",
            "data": "synthetic (C5 generator, mt19937_64 seeds of SURVEY.md 8d; random-init layer tables)",
            "config": {"workload": "C5 sweep: 128 models x 64 cluster mixes x 8 stage counts x 8 M x 2 kinds "
                                   "= 2^20 candidates" + (" in total, sharded over the GPUs" if args.scaling == "strong"
                                                          else " per GPU"),
                       "queries": int(full.queries.size) if args.scaling == "strong" else int(p.queries.size) * world,
                       "candidates_per_step": int(cands_per_step),
                       "parallelism": (f"strong x{world} (whole dedup classes per GPU, cost-balanced; NCCL allgather "
                                       f"of one best record per rank)" if args.scaling == "strong" else
                                       f"weak x{world} (a 2^20-candidate sweep per GPU; NCCL allgather of best "
                                       f"records)"),
                       "l2": "256 MiB buffer written between timed steps (L2 flush)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_total / args.steps,
                    "h2d_bytes_per_step": (h2 - h1) // args.steps, "d2h_bytes_per_step": (d2 - d1) // args.steps},
            "e2e_candidates": e2e_cand,
            "no_dedup": {"value": value_nodedup, "unit": UNIT, "ms_per_step": nd_ms / args.steps,
                         "note": "same steps with BP_OPT_DEDUP=0: identical subproblems of the batch not shared"},
            "lb_pruned": {"value": value_lb, "unit": UNIT, "ms_per_step": lb_ms / args.steps,
                          "note": "same steps with BP_OPT_PRUNE_LB=1 (SPEC.md:320 estimate-based pruning): scaled-"
                                  "integer candidates whose makespan lower bound exceeds their query's best are not "
                                  "simulated; per-query results byte-identical (asserted). Not the headline: every "
                                  "candidate of the headline value is simulated"},
            "ranks": {"ms_per_step": [x / args.steps for x in rank_ms],
                      "imbalance_max_over_mean": max(rank_ms) / mean_ms if mean_ms > 0 else None,
                      "queries_rank0": int(p.queries.size)},
            "gpu_launches": launches,
            "clocks": clocks,
            "roofline": roof,
            "sweep_roofline": sweep,
            "refine_latency": refine_lat,
            "kernels": kern,
            "kernels_note": (f"per-kernel CUDA-event spans of the same steps run as one batch (BP_OPT_SPLIT off: "
                             f"{kb_ms:.2f} ms per step); the headline runs the batch as concurrent parts by stage count"),
            "best": {"makespan": f"{int(best['makespan']['num'])}/{int(best['makespan']['den'])}",
                     "M": int(best["M"]), "kind": int(best["kind"]), "query_id": int(best["query_id"])},
            "query_status_hist": np.bincount(res["status"], minlength=7).tolist()}
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(full, args.cpu_sample_stride, os.cpu_count() or 1)
        except Exception as e:   # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if not args.no_per_call:
        ex.close()
        try:
            line["per_call"] = per_call()
        except Exception as e:
            line["per_call"] = {"error": str(e)}
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
