#!/usr/bin/env python3
"""Summarise this round's ncu output into profiles/ (tracked).

  python profiles/ncu_summarize.py TAG gpurun_out/<dir>/launches.csv gpurun_out/<dir>/full.ncu-rep

writes
  profiles/<TAG>_launches.md   per-kernel launch list of one bench.py run
                               (--metrics gpu__time_duration.sum
                               --clock-control none): count, total, share
                               of the product kernels' time.  Per-launch
                               times are cold-cache and serialised: compare
                               SHARES with bench.py's CUDA-event breakdown,
                               not absolutes.
  profiles/<TAG>_ncu_full.md   key metrics of the `--set full` capture
                               (issue activity, warps active, SIMT efficiency,
                               DRAM bytes, top stall reasons) per kernel
  profiles/traffic.json        DRAM bytes (read + write) per launch of each
                               captured kernel, keyed by bench.py's kernel
                               names; bench.py reports it as roofline.traffic
"""
import csv
import re
import json
import os
import subprocess
import sys
from collections import OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))

# CUDA kernel -> bench.py / bp_kernel_stats name.  k_partition runs twice per
# step: the whole-layer DP first, then the coarse DPs.
def bench_name(kernel, seen):
    k = kernel.split("(")[0].replace("void ", "")
    k = re.sub(r"^.*::", "", k.split("<")[0]) + (k[k.index("<"):] if "<" in k else "")
    if k.startswith("k_partition"):
        n = seen.get("k_partition", 0)
        seen["k_partition"] = n + 1
        return "minmax_dp" if n % 2 == 0 else "minmax_dp_coarse"
    if k.startswith("k_sim_fast"):
        g = k.split("<")[1].rstrip(">").replace(" ", "").split(",")
        return f"sim_fast_g{g[0]}" + (f"s{g[1]}" if g[1] != "1" else "")
    k = k.replace("<unnamed>::", "")
    if k.startswith("k_sim_flow"):
        return "sim_flow" + k.split("<")[1].rstrip(">").strip()
    return {"k_refine": "refine", "k_refine_smem": "refine", "k_refine_list": "refine", "k_refine_keys": "refine", "k_refine_fast": "refine",
            "k_scatter_results": "fetch", "k_scatter_records": "fetch",
            "k_lb_bound": "lb_prune", "k_lb_round1": "lb_prune", "k_lb_incumbent": "lb_prune",
            "k_lb_decide": "lb_prune", "k_lb_finish": "lb_prune", "k_best_merge": "best", "k_prune": "prune",
            "k_prune_key": "prune", "k_prune_members": "prune", "k_sim_exact": "sim_exact",
            "k_xsort_count": "sim_exact", "k_xsort_scan": "sim_exact", "k_xsort_scatter": "sim_exact",
            "k_setup": "setup", "k_bottleneck": "bottleneck", "k_coarse_queue": "bottleneck", "k_rank": "rank",
            "k_sim_prep": "sim_prep", "k_sim_classify": "sim_prep", "k_best": "best",
            "k_cost_prefix": "cost_prefix", "k_dedup_insert": "dedup", "k_dedup_resolve": "dedup",
            "k_dedup_copy_dp": "dedup_copy", "k_dedup_copy_refine": "dedup_copy", "k_coarse_copy": "dedup_copy",
            "k_sim_share": "sim_share"}.get(k, k)


def launches(path, tag):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r["Metric Unit"]]
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * scale))
    agg = OrderedDict()
    seen = {}
    for k, ms in rows:
        if "bpk::" not in k:
            name = "(torch) " + k.split("(")[0][:60]
        else:
            name = bench_name(k, seen)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    ours = sum(v[1] for k, v in agg.items() if not k.startswith("(torch)"))
    out = [f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
           f"Source: `{os.path.basename(path)}` ({len(rows)} launches). Times are ncu's serialised, "
           "cold-cache per-launch durations; the share column is what must agree with bench.py's breakdown.", "",
           "| kernel | launches | total ms | mean ms | share of product time |", "|---|---:|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = "" if k.startswith("(torch)") else f"{100 * ms / ours:.1f}%"
        out.append(f"| {k} | {n} | {ms:.3f} | {ms / n:.3f} | {share} |")
    return "\n".join(out) + "\n"


WANT = [("gpu__time_duration.sum", "time"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/instr"),
        ("smsp__inst_executed.sum", "warp instrs"),
        ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"),
        ("launch__block_size", "block"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write")]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


def full(path, tag):
    csvtxt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(csvtxt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = [f"# {tag}: `ncu --set full --clock-control none --import-source on` (one capture per kernel)", "",
           f"Source: `{os.path.basename(path)}`.", ""]
    traffic = {}
    seen = {}
    for r in rows[2:]:
        raw = r[hdr.index("Kernel Name")]
        name = bench_name(raw, seen)
        short = re.sub(r"^.*::", "", raw.split("(")[0].replace("void ", "").split("<")[0])
        out.append(f"## {name}" + (f" (`{short}`)" if short.lstrip("k_") != name else ""))
        out.append("")
        for key, label in WANT:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"* {label}: {r[i]} {units[i]}".rstrip())
        rd = wr = None
        if "dram__bytes_read.sum" in hdr:
            i, j = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            rd, wr = to_bytes(r[i], units[i]), to_bytes(r[j], units[j])
            traffic[name] = traffic.get(name, 0.0) + rd + wr   # a phase's launches add up
        stalls = [(hdr[i], r[i]) for i in range(len(hdr))
                  if hdr[i].startswith("smsp__average_warps_issue_stalled_")
                  and hdr[i].endswith("_per_issue_active.ratio") and r[i] not in ("", "nan", "-nan")]
        stalls.sort(key=lambda kv: -float(kv[1]))
        out.append("* top stalls (warps per issue-active cycle): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
            f"={float(v):.2f}" for k, v in stalls[:6]))
        out.append("")
    return "\n".join(out), traffic


def main():
    tag, launch_csv, rep = sys.argv[1:4]
    with open(os.path.join(HERE, f"{tag}_launches.md"), "w") as f:
        f.write(launches(launch_csv, tag))
    text, traffic = full(rep, tag)
    with open(os.path.join(HERE, f"{tag}_ncu_full.md"), "w") as f:
        f.write(text)
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump({"source": f"{tag}_ncu_full.md", **traffic}, f, indent=1)
    print(open(os.path.join(HERE, f"{tag}_launches.md")).read())
    print(text)


if __name__ == "__main__":
    main()
