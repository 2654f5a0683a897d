"""Golden outputs of the `bapipe` CLI (validate / plan / explore / simulate)
from the reference.

Writes the input files under tests/golden/cli/ (networks and clusters of the
reference's explorer unit tests, C1 and C3 of SURVEY.md 8d, a heterogeneous
random chain, and malformed / schema-violating inputs), then runs
paper_2012_12544_b200/cli/bapipe.cpp built with -DUSE_REFERENCE against the
reference headers (oracle/Makefile target `cli`) on every case, with argv[0] =
"bapipe" and cwd = tests/golden/cli, and stores stdout, stderr, the exit code
and any -o / --gantt file in tests/golden/cli/expected.json.  Plan files for
`simulate` are hand-written (valid whole-layer and fractional plans, and
invalid ones) or made by the reference's own `plan -o` (plan_c1/c3/rand).
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CLI_DIR = os.path.join(HERE, "cli")
sys.path.insert(0, ROOT)

from paper_2012_12544_b200 import workloads as W  # noqa: E402

KINDS = ["1f1b-as", "fbp-as", "1f1b-sno", "1f1b-so"]


def net_json(net, types, name):
    layers = []
    for j in range(net.L):
        fp = {types[t]: int(net.fp[t, j]) for t in range(net.T) if net.fp[t, j] > 0}
        bp = {types[t]: int(net.bp[t, j]) for t in range(net.T) if net.bp[t, j] > 0}
        layers.append({"name": f"l{j}", "fp_us": fp, "bp_us": bp, "weight_bytes": int(net.w[j]),
                       "out_activation_bytes": int(net.a[j])})
    return {"name": name, "layers": layers}


def cluster_json(cl, types, n=None):
    n = cl.N if n is None else n
    accels = []
    for i in range(n):
        a = {"id": f"acc{i}", "type": types[int(cl.types[i])], "mem_capacity_bytes": int(cl.cap[i])}
        mm = {KINDS[k]: int(cl.min_micro[i, k]) for k in range(4) if cl.min_micro[i, k] != 1}
        if mm:
            a["min_micro_batch"] = mm
        accels.append(a)
    return {"execution_mode": "async" if cl.mode == 1 else "sync", "accelerators": accels,
            "link_bandwidth_bytes_per_us": [int(b) for b in cl.bw[:n - 1]]}


def tri_net():
    return {"name": "tri", "layers": [{"name": f"layer{i}", "fp_us": {"gpu": 10}, "bp_us": {"gpu": 20},
                                       "weight_bytes": 100, "out_activation_bytes": 50} for i in range(3)]}


def tri_cluster(mode, caps, floor=None):
    accels = []
    for i, c in enumerate(caps):
        a = {"id": f"g{i}", "type": "gpu", "mem_capacity_bytes": c}
        if floor:
            a["min_micro_batch"] = floor
        accels.append(a)
    return {"execution_mode": mode, "accelerators": accels, "link_bandwidth_bytes_per_us": [50, 50]}


def write_inputs():
    os.makedirs(CLI_DIR, exist_ok=True)
    files = {
        "tri_net.json": tri_net(),
        "tri_tight.json": tri_cluster("sync", [400, 1000000, 1000000]),
        "tri_roomy.json": tri_cluster("sync", [1000000, 1000000, 1000000]),
        "tri_floor.json": tri_cluster("async", [600, 600, 600], {"1f1b-as": 4}),
        "tri_tiny.json": tri_cluster("sync", [1, 1, 1]),
    }
    p1 = W.config_c1()
    files["c1_vgg16.json"] = net_json(p1.networks[0], ["v100"], "vgg16")
    files["c1_cluster.json"] = cluster_json(p1.clusters[0], ["v100"])
    p3 = W.config_c3()
    files["c3_gnmt.json"] = net_json(p3.networks[0], ["v100", "p100"], "gnmt16")
    files["c3_cluster.json"] = cluster_json(p3.clusters[0], ["v100", "p100"])
    pr = W.random_problem(5, n_queries=1, max_L=30, max_N=8, cap_range=(2000, 200000), bw_range=(1, 500),
                          act_max=3000)
    q = pr.queries[0]
    tys = ["fpga", "gpu", "tpu"]
    files["rand_net.json"] = net_json(pr.networks[int(q["network"])], tys, "rand5")
    rc = pr.clusters[int(q["cluster"])]
    files["rand_cluster.json"] = cluster_json(rc, tys, int(q["n_stages"]) or rc.N)
    # schema violations and malformed input
    bad = tri_net()
    bad["layers"][1]["color"] = "red"
    files["bad_unknown_key.json"] = bad
    bad = tri_net()
    bad["layers"][2]["fp_us"] = {"gpu": "10"}
    files["bad_type.json"] = bad
    bad = tri_net()
    del bad["layers"][0]["weight_bytes"]
    files["bad_missing.json"] = bad
    bad = tri_cluster("sometimes", [1000, 1000, 1000])
    files["bad_mode.json"] = bad
    bad = tri_cluster("sync", [1000, 1000, 1000], {"gpipe": 2})
    files["bad_kind.json"] = bad
    for name, obj in files.items():
        with open(os.path.join(CLI_DIR, name), "w") as f:
            json.dump(obj, f, indent=1)
    # plans for `simulate`
    def stage(acc, lo, hi, lead="1", trail="1"):
        return {"accelerator": acc, "layers": [lo, hi], "leading_fraction": lead, "trailing_fraction": trail}
    plans = {
        "plan_tri_whole.json": [stage("g0", 1, 1), stage("g1", 2, 2), stage("g2", 3, 3)],
        "plan_tri_frac.json": [stage("g0", 1, 2, "1", "1/2"), stage("g1", 2, 3, "1/2", "1/3"),
                               stage("g2", 3, 3, "2/3", "1")],
        "plan_tri_twostage.json": [stage("g0", 1, 2), stage("g1", 3, 3)],
        "plan_bad_range.json": [stage("g0", 1, 1), stage("g1", 2, 2), stage("g2", 3, 4)],
        "plan_bad_cover.json": [stage("g0", 1, 2, "1", "1/2"), stage("g1", 2, 3, "1/3", "1"),
                                stage("g2", 3, 3, "1/2", "1")],
        "plan_bad_frac.json": [stage("g0", 1, 1), stage("g1", 2, 2, "1", "3/2"), stage("g2", 3, 3)],
        "plan_bad_contig.json": [stage("g0", 1, 1), stage("g1", 3, 3), stage("g2", 3, 3)],
    }
    for name, st in plans.items():
        with open(os.path.join(CLI_DIR, name), "w") as f:
            json.dump({"stages": st}, f, indent=1)
    with open(os.path.join(CLI_DIR, "bad_syntax.json"), "w") as f:
        f.write('{"name": "x", "layers": [}\n')
    with open(os.path.join(CLI_DIR, "bad_array.json"), "w") as f:
        f.write("[1, 2, 3]\n")


CASES = [
    ["validate", "tri_net.json", "tri_roomy.json"],
    ["validate", "tri_net.json", "tri_roomy.json", "--format", "json"],
    ["explore", "tri_net.json", "tri_tight.json", "--minibatch", "4", "--micro-set", "4"],
    ["explore", "tri_net.json", "tri_roomy.json", "--minibatch", "4", "--micro-set", "4", "--format", "json"],
    ["explore", "tri_net.json", "tri_roomy.json", "--minibatch", "1", "--format", "json"],
    ["explore", "tri_net.json", "tri_floor.json", "--minibatch", "8", "--format", "json", "-o", "best_plan.json"],
    ["explore", "tri_net.json", "tri_floor.json", "--minibatch", "8", "-o", "best_plan.json"],
    ["explore", "tri_net.json", "tri_tiny.json", "--minibatch", "2"],
    ["explore", "tri_net.json", "tri_roomy.json", "--minibatch", "128", "--micro-set", "8", "3"],
    ["explore", "tri_net.json", "tri_roomy.json", "--minibatch", "16", "--dp-baseline", "123.5", "--format", "json"],
    ["explore", "c1_vgg16.json", "c1_cluster.json", "--minibatch", "32", "--format", "json"],
    ["explore", "c1_vgg16.json", "c1_cluster.json", "--minibatch", "32"],
    ["explore", "c3_gnmt.json", "c3_cluster.json", "--minibatch", "64", "--format", "json"],
    ["explore", "rand_net.json", "rand_cluster.json", "--minibatch", "16", "--format", "json"],
    ["explore", "bad_unknown_key.json", "tri_roomy.json", "--minibatch", "4"],
    ["explore", "bad_unknown_key.json", "tri_roomy.json", "--minibatch", "4", "--lenient", "--format", "json"],
    ["validate", "bad_type.json", "tri_roomy.json"],
    ["validate", "bad_missing.json", "tri_roomy.json"],
    ["validate", "tri_net.json", "bad_mode.json"],
    ["validate", "tri_net.json", "bad_kind.json"],
    ["validate", "bad_syntax.json", "tri_roomy.json"],
    ["validate", "bad_array.json", "tri_roomy.json"],
    ["validate", "missing_file.json", "tri_roomy.json"],
    ["validate", "tri_net.json", "c3_cluster.json"],
    # plan (tools/bapipe.cpp:152-190): balance_partition + estimate, no min-micro filter
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-sno", "--micro", "4"],
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-so", "--micro", "4", "--format", "json",
     "-o", "best_plan.json"],
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-sno", "--minibatch", "8"],
    ["plan", "tri_net.json", "tri_floor.json", "--schedule", "1f1b-as", "--micro", "8", "--minibatch", "8",
     "--format", "json"],
    ["plan", "tri_net.json", "tri_floor.json", "--schedule", "fbp-as", "--micro", "2", "--minibatch", "8"],
    ["plan", "tri_net.json", "tri_tight.json", "--schedule", "1f1b-so", "--micro", "2", "--minibatch", "8"],
    ["plan", "tri_net.json", "tri_tiny.json", "--schedule", "1f1b-sno", "--micro", "2"],
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-as", "--micro", "4"],
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "gpipe", "--micro", "4"],
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-sno"],
    ["plan", "tri_net.json", "tri_roomy.json", "--schedule", "1f1b-sno", "--micro", "3", "--minibatch", "8"],
    ["plan", "c1_vgg16.json", "c1_cluster.json", "--schedule", "1f1b-sno", "--micro", "8", "--minibatch", "32",
     "--format", "json"],
    ["plan", "c3_gnmt.json", "c3_cluster.json", "--schedule", "1f1b-so", "--micro", "16", "--minibatch", "64"],
    # simulate (tools/bapipe.cpp:234-256): full timeline, --trace / --gantt
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_whole.json", "--schedule", "1f1b-sno", "--micro", "4"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_whole.json", "--schedule", "1f1b-so", "--micro", "4",
     "--format", "json", "--trace"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_whole.json", "--schedule", "1f1b-sno", "--micro", "3",
     "--gantt", "gantt.csv"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_frac.json", "--schedule", "1f1b-so", "--micro", "3",
     "--minibatch", "6", "--format", "json", "--trace", "--gantt", "gantt.svg"],
    ["simulate", "tri_net.json", "tri_floor.json", "plan_tri_whole.json", "--schedule", "1f1b-as", "--micro", "4",
     "--trace"],
    ["simulate", "tri_net.json", "tri_floor.json", "plan_tri_frac.json", "--schedule", "fbp-as", "--micro", "5",
     "--format", "json", "--trace"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_twostage.json", "--schedule", "1f1b-sno", "--micro", "2"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_bad_range.json", "--schedule", "1f1b-sno", "--micro", "2"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_bad_cover.json", "--schedule", "1f1b-sno", "--micro", "2"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_bad_frac.json", "--schedule", "1f1b-sno", "--micro", "2"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_bad_contig.json", "--schedule", "1f1b-sno", "--micro", "2"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_whole.json", "--schedule", "fbp-as", "--micro", "2"],
    ["simulate", "tri_net.json", "tri_roomy.json", "plan_tri_whole.json", "--schedule", "1f1b-sno", "--micro", "3",
     "--minibatch", "4"],
    ["simulate", "c1_vgg16.json", "c1_cluster.json", "plan_c1.json", "--schedule", "1f1b-sno", "--micro", "8",
     "--minibatch", "32", "--format", "json", "--trace"],
    ["simulate", "c3_gnmt.json", "c3_cluster.json", "plan_c3.json", "--schedule", "1f1b-so", "--micro", "16",
     "--minibatch", "64", "--gantt", "gantt.svg"],
    ["simulate", "rand_net.json", "rand_cluster.json", "plan_rand.json", "--schedule", "RAND_KIND", "--micro", "16",
     "--minibatch", "16", "--format", "json", "--trace"],
    ["plan", "rand_net.json", "rand_cluster.json", "--schedule", "RAND_KIND", "--micro", "4", "--minibatch", "16"],
]

# plans made by the reference's own `plan -o` (written before the cases run)
PLAN_SOURCES = [
    ("plan_c1.json", ["plan", "c1_vgg16.json", "c1_cluster.json", "--schedule", "1f1b-sno", "--micro", "8",
                      "--minibatch", "32"]),
    ("plan_c3.json", ["plan", "c3_gnmt.json", "c3_cluster.json", "--schedule", "1f1b-so", "--micro", "16",
                      "--minibatch", "64"]),
    ("plan_rand.json", ["plan", "rand_net.json", "rand_cluster.json", "--schedule", "RAND_KIND", "--micro", "16",
                        "--minibatch", "16"]),
]

OUT_FILES = ("best_plan.json", "gantt.csv", "gantt.svg")


def rand_kind():
    with open(os.path.join(CLI_DIR, "rand_cluster.json")) as f:
        return "1f1b-so" if json.load(f)["execution_mode"] == "sync" else "fbp-as"


def resolve(args):
    return [rand_kind() if a == "RAND_KIND" else a for a in args]


def run_case(exe, args):
    for name in OUT_FILES:
        if os.path.exists(os.path.join(CLI_DIR, name)):
            os.remove(os.path.join(CLI_DIR, name))
    p = subprocess.run(["bapipe"] + args, executable=exe, cwd=CLI_DIR, capture_output=True, text=True, timeout=600)
    rec = {"args": args, "rc": p.returncode, "stdout": p.stdout, "stderr": p.stderr}
    for name in OUT_FILES:
        path = os.path.join(CLI_DIR, name)
        if os.path.exists(path):
            rec["out_file" if name == "best_plan.json" else name] = open(path).read()
            os.remove(path)
    return rec


def main():
    write_inputs()
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "cli"], check=True)
    exe = os.path.join(ROOT, "oracle", "_ref", "bapipe_ref")
    for name, args in PLAN_SOURCES:
        p = subprocess.run(["bapipe"] + resolve(args) + ["-o", name], executable=exe, cwd=CLI_DIR,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, (name, p.stderr)
    expected = [run_case(exe, resolve(c)) for c in CASES]
    with open(os.path.join(CLI_DIR, "expected.json"), "w") as f:
        json.dump(expected, f, indent=1)
    for r in expected:
        print(r["rc"], " ".join(r["args"]), r["stderr"].strip()[:100])


if __name__ == "__main__":
    main()
