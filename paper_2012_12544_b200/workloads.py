"""Synthetic workloads: the BASELINE.json configs and the
reference tests' seeded generators, as `Problem`s.

  C1  VGG-16 (16 layers) on 4 homogeneous v100, sync, mini-batch 32
  C2  ResNet-50 (18 units) on 8 accelerators with 1 GiB caps, sync, mini-batch 64
  C3  GNMT-16 (21 layers) on a [v100,v100,p100,p100]x2 chain, per-link bandwidths
  C4  synthetic 1000 layers, 64 alternating vcu118/vcu129 FPGAs, async, two
      memory tiers (on-chip / off-chip) plus a homogeneous variant
  C5  the 2^20-candidate sweep: 128 models x 64 cluster mixes x 8 stage counts
      x 8 micro-batch counts x 2 kinds (65,536 queries)

Layer times follow SURVEY.md 8d: fp_us = max(1, ceil(FLOPs / rate)),
bp_us = 2 fp_us, weight_bytes = 4 params, out_activation_bytes = 4 outputs.
All random draws use std::mt19937_64 (re-implemented below, vectorised).
"""
from __future__ import annotations

import math

import numpy as np

from .abi import MODE_ASYNC, MODE_SYNC
from .problem import Cluster, Network, Problem

# --------------------------------------------------------------------------- mt19937_64
_NN, _MM = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)


class MT19937_64:
    """std::mt19937_64 (same output sequence), twist vectorised with numpy."""

    def __init__(self, seed: int):
        mt = np.zeros(_NN, dtype=np.uint64)
        mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        with np.errstate(over="ignore"):
            for i in range(1, _NN):
                prev = int(mt[i - 1])
                mt[i] = np.uint64((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = mt
        self.buf = np.empty(0, dtype=np.uint64)
        self.pos = 0

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)

        def step(i0, i1, nxt, far):
            y = (mt[i0:i1] & _UM) | (nxt & _LM)
            mag = np.where((y & one) != 0, _MATRIX_A, np.uint64(0))
            mt[i0:i1] = far ^ (y >> one) ^ mag

        step(0, _NN - _MM, mt[1:_NN - _MM + 1].copy(), mt[_MM:_NN].copy())
        step(_NN - _MM, _NN - 1, mt[_NN - _MM + 1:_NN].copy(), mt[0:_MM - 1].copy())
        y = (mt[_NN - 1] & _UM) | (mt[0] & _LM)
        mt[_NN - 1] = mt[_MM - 1] ^ (y >> one) ^ (_MATRIX_A if int(y) & 1 else np.uint64(0))
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        return x

    def draw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        got = 0
        while got < n:
            if self.pos >= self.buf.size:
                self.buf = self._twist()
                self.pos = 0
            k = min(n - got, self.buf.size - self.pos)
            out[got:got + k] = self.buf[self.pos:self.pos + k]
            self.pos += k
            got += k
        return out

    def __call__(self) -> int:
        return int(self.draw(1)[0])


def _mod(r, m):
    return (r % np.uint64(m)).astype(np.int64)


# --------------------------------------------------------------------------- model tables
def _times(flops, rates):
    """fp_us per type = max(1, ceil(FLOPs / rate)), rate in FLOP/us."""
    fp = np.array([[max(1, math.ceil(f / r)) for f in flops] for r in rates], dtype=np.int64)
    return fp, 2 * fp


def vgg16_layers():
    """(FLOPs, params, outputs) per unit: 13 convs (pools folded) + 3 FC, 224^2."""
    cfg = [(224, 3, 64, False), (224, 64, 64, True), (112, 64, 128, False), (112, 128, 128, True),
           (56, 128, 256, False), (56, 256, 256, False), (56, 256, 256, True),
           (28, 256, 512, False), (28, 512, 512, False), (28, 512, 512, True),
           (14, 512, 512, False), (14, 512, 512, False), (14, 512, 512, True)]
    rows = []
    for hw, cin, cout, pool in cfg:
        macs = hw * hw * cin * cout * 9
        out_hw = hw // 2 if pool else hw
        rows.append((2 * macs, cin * cout * 9 + cout, out_hw * out_hw * cout))
    for fin, fout in [(7 * 7 * 512, 4096), (4096, 4096), (4096, 1000)]:
        rows.append((2 * fin * fout, fin * fout + fout, fout))
    return rows


def resnet50_units():
    """stem, 16 bottlenecks (torchvision v1.5 strides), fc."""
    rows = [(2 * 112 * 112 * 3 * 64 * 49, 3 * 64 * 49, 56 * 56 * 64)]
    cin = 64
    for hw_in, mid, blocks, stride in [(56, 64, 3, 1), (56, 128, 4, 2), (28, 256, 6, 2), (14, 512, 3, 2)]:
        out = 4 * mid
        hw = hw_in // stride
        for b in range(blocks):
            s_hw_in = hw_in if b == 0 else hw
            macs = s_hw_in * s_hw_in * cin * mid + hw * hw * mid * mid * 9 + hw * hw * mid * out
            params = cin * mid + mid * mid * 9 + mid * out
            if b == 0:
                macs += hw * hw * cin * out
                params += cin * out
            rows.append((2 * macs, params, hw * hw * out))
            cin = out
        hw_in = hw
    rows.append((2 * 2048 * 1000, 2048 * 1000 + 1000, 1000))
    return rows


def gnmt16_layers(T=50, h=1024, V=32000):
    lstm = (T * 16 * h * h, 4 * (2 * h * h + h), T * h)
    rows = [(0, V * h, T * h)]                                  # encoder embedding
    rows += [lstm] * 8
    rows += [(0, V * h, T * h)]                                 # decoder embedding
    rows += [(2 * T * T * h * 2 + 2 * T * 2 * h * h, 2 * h * h, T * h)]   # attention
    rows += [lstm] * 8
    rows += [(2 * T * h * V, h * V, T * V)]                     # logits
    rows += [(5 * T * V, 0, T)]                                 # loss
    return rows


def table_network(rows, rates, name):
    flops = [r[0] for r in rows]
    fp, bp = _times(flops, rates)
    w = np.array([4 * r[1] for r in rows], dtype=np.int64)
    a = np.array([4 * r[2] for r in rows], dtype=np.int64)
    return Network(fp, bp, w, a, name=name)


V100, P100 = 14e6, 9e6      # FLOP per microsecond (14 / 9 TFLOP/s)
GIB = 1 << 30


def config_c1() -> Problem:
    p = Problem(name="C1 VGG-16 / 4 homogeneous GPUs, sync, mini-batch 32")
    p.add_network(table_network(vgg16_layers(), [V100], "vgg16"))
    p.add_cluster(Cluster(MODE_SYNC, [0] * 4, [16 * GIB] * 4, [12000] * 3))
    p.set_queries([0], 0, 0, 32)
    return p


def config_c2() -> Problem:
    p = Problem(name="C2 ResNet-50 / 8 accelerators, 1 GiB caps, sync, mini-batch 64")
    p.add_network(table_network(resnet50_units(), [V100], "resnet50"))
    p.add_cluster(Cluster(MODE_SYNC, [0] * 8, [GIB] * 8, [12000] * 7))
    p.set_queries([0], 0, 0, 64)
    return p


def config_c3() -> Problem:
    p = Problem(name="C3 GNMT-16 / heterogeneous 8-chain, per-link bandwidths, sync, mini-batch 64")
    p.add_network(table_network(gnmt16_layers(), [V100, P100], "gnmt16"))
    types = [0, 0, 1, 1] * 2
    caps = [16 * GIB if t == 0 else 12 * GIB for t in types]
    bw = [3000 if k % 4 == 2 else 12000 for k in range(7)]
    p.add_cluster(Cluster(MODE_SYNC, types, caps, bw))
    p.set_queries([0], 0, 0, 64)
    return p


def synth_layers(L, seed, n_types=2):
    """Layer-major draws fp_a, bp_a, fp_b, bp_b, w, a."""
    per = 2 * n_types + 2
    r = MT19937_64(seed).draw(L * per).reshape(L, per)
    fp = np.stack([1 + _mod(r[:, 2 * t], 100) for t in range(n_types)])
    bp = np.stack([1 + _mod(r[:, 2 * t + 1], 200) for t in range(n_types)])
    w = _mod(r[:, 2 * n_types], 1_000_000)
    a = _mod(r[:, 2 * n_types + 1], 100_000)
    return Network(fp, bp, w, a, name=f"synth{L}_{seed}")


ONCHIP_CAP = (43_237_500, 56_862_500)     # vcu118 / vcu129 on-chip bytes


def config_c4(tier="onchip") -> Problem:
    p = Problem(name=f"C4 synthetic 1000 layers / 64 FPGAs, async, {tier}")
    p.add_network(synth_layers(1000, 12544))
    types = [k % 2 for k in range(64)]
    if tier == "onchip":
        caps = [ONCHIP_CAP[t] for t in types]
    elif tier == "offchip":
        caps = [8 * GIB] * 64
    elif tier == "homogeneous":
        types = [1] * 64
        caps = [8 * GIB] * 64
    else:
        raise ValueError(tier)
    p.add_cluster(Cluster(MODE_ASYNC, types, caps, [12500] * 63))
    p.set_queries([0], 0, 0, 128)
    return p


C5_LAYERS = (64, 96, 128, 192, 256, 384, 512, 1000)
C5_STAGES = (2, 4, 8, 12, 16, 24, 32, 64)
C5_CAPS = (64 << 20, 256 << 20, 2 << 30, 16 << 30)


def c5_cluster(c: int) -> Cluster:
    mode = MODE_ASYNC if c & 1 else MODE_SYNC
    pat = (c >> 1) & 3
    cap = C5_CAPS[(c >> 3) & 3]
    slow = (c >> 5) & 1
    types = [0 if (pat == 0 or (pat == 2 and k % 2 == 0) or (pat == 3 and k < 32)) else 1
             for k in range(64)]
    bw = [1250 if (slow and k % 4 == 3) else 12500 for k in range(63)]
    return Cluster(mode, types, [cap] * 64, bw)


def config_c5(models=128, shard=0, n_shards=1, model_base=0) -> Problem:
    """The sweep.  Query q = (i*64 + c)*8 + n over models i, clusters c, stage
    counts n.  `shard/n_shards` selects a cost-balanced
    subset of queries (multi-GPU); `model_base` offsets model seeds (weak
    scaling: each rank sweeps its own 2^20 candidates)."""
    p = Problem(name=f"C5 sweep ({models} models x 64 clusters x 8 stage counts)")
    for i in range(models):
        gi = model_base + i
        p.add_network(synth_layers(C5_LAYERS[(gi // 16) % 8], 0x2012125440 + gi))
    for c in range(64):
        p.add_cluster(c5_cluster(c))
    q = np.arange(models * 512)
    net, cl, ns = q // 512, (q // 8) % 64, np.array(C5_STAGES)[q % 8]
    if n_shards > 1:
        sel = shard_queries([p.networks[i].L for i in net], ns, n_shards)[shard]
        net, cl, ns = net[sel], cl[sel], ns[sel]
        p.query_ids = (model_base * 512 + q[sel]).astype(np.int64)
    else:
        p.query_ids = (model_base * 512 + q).astype(np.int64)
    p.set_queries(net, cl, ns, 128)
    return p


KINDS = ("1f1b-as", "fbp-as", "1f1b-sno", "1f1b-so")


def network_json(net: Network, type_names, name="net") -> dict:
    """NetworkProfile in the reference's JSON schema (profiles.hpp:194-217,
    274-290); type_names maps type ids to accelerator type strings."""
    layers = []
    for j in range(net.L):
        fp = {type_names[t]: int(net.fp[t, j]) for t in range(net.T) if net.fp[t, j] > 0}
        bp = {type_names[t]: int(net.bp[t, j]) for t in range(net.T) if net.bp[t, j] > 0}
        layers.append({"name": f"l{j}", "fp_us": fp, "bp_us": bp, "weight_bytes": int(net.w[j]),
                       "out_activation_bytes": int(net.a[j])})
    return {"name": name, "layers": layers}


def cluster_json(cl: Cluster, type_names, n=None) -> dict:
    """ClusterSpec in the reference's JSON schema (profiles.hpp:219-261,
    292-303), the first n accelerators."""
    n = cl.N if n is None else n
    accels = []
    for i in range(n):
        a = {"id": f"acc{i}", "type": type_names[int(cl.types[i])], "mem_capacity_bytes": int(cl.cap[i])}
        mm = {KINDS[k]: int(cl.min_micro[i, k]) for k in range(4) if cl.min_micro[i, k] != 1}
        if mm:
            a["min_micro_batch"] = mm
        accels.append(a)
    return {"execution_mode": "async" if cl.mode == MODE_ASYNC else "sync", "accelerators": accels,
            "link_bandwidth_bytes_per_us": [int(b) for b in cl.bw[:n - 1]]}


def single_query_configs():
    """(name, Problem, type names) of the one-query configs C1-C4 (SURVEY.md
    8d) -- the reference's own per-call use of explore()."""
    return [("C1", config_c1(), ["v100"]), ("C2", config_c2(), ["v100"]), ("C3", config_c3(), ["v100", "p100"]),
            ("C4 onchip", config_c4("onchip"), ["vcu118", "vcu129"]),
            ("C4 offchip", config_c4("offchip"), ["vcu118", "vcu129"]),
            ("C4 homogeneous", config_c4("homogeneous"), ["vcu118", "vcu129"])]


def subset(p: Problem, idx) -> Problem:
    """The queries `idx` of `p` as their own batch: same network and cluster
    tables, queries in the given order, dense offsets re-laid out.  Global
    query ids carry over (`query_ids`)."""
    idx = np.asarray(idx, dtype=np.int64)
    s = Problem(networks=p.networks, clusters=p.clusters, name=f"{p.name} [{idx.size} queries]")
    q = np.ascontiguousarray(p.queries[idx])
    s.m_lists = p.m_lists          # explicit M lists stay alive (pointers are copied)
    s.queries = q
    s.layout()
    ids = getattr(p, "query_ids", None)
    s.query_ids = (np.arange(p.queries.size, dtype=np.int64) if ids is None else ids)[idx]
    return s


def query_classes(p: Problem):
    """Batch-dedup class of every query: (network, stage count, accelerator
    type chain of the used prefix) -- the key under which the engine shares
    the whole-layer DP and refine (kernels.cu k_dedup_*).  Returns the class
    index per query (classes numbered in first-appearance order)."""
    q = p.queries
    keys = {}
    out = np.empty(q.size, dtype=np.int64)
    for i in range(q.size):
        cl = p.clusters[int(q["cluster"][i])]
        n = int(q["n_stages"][i]) or cl.N
        k = (int(q["network"][i]), n, cl.types[:n].tobytes())
        out[i] = keys.setdefault(k, len(keys))
    return out


def class_cost(p: Problem, cls):
    """Estimated cost of each dedup class: one DP fill (~U^2 transitions after
    the banded DP's early exits) and one refine walk (~N x U boundary-step
    units) per class, plus the class's simulated events (2NM, +2(N-1)M sync,
    per query and M).  Relative units; used only to balance shards."""
    q = p.queries
    ncls = int(cls.max()) + 1 if cls.size else 0
    cost = np.zeros(ncls)
    seen = np.zeros(ncls, dtype=bool)
    Ms = np.array([1, 2, 4, 8, 16, 32, 64, 128], dtype=np.float64)
    for i in range(q.size):
        c = int(cls[i])
        L = float(p.networks[int(q["network"][i])].L)
        n = float(int(q["n_stages"][i]) or p.clusters[int(q["cluster"][i])].N)
        sync = p.clusters[int(q["cluster"][i])].mode == MODE_SYNC
        if not seen[c]:
            seen[c] = True
            cost[c] += L * L + 40.0 * n * L
        ev = 2 * n * Ms + (2 * (n - 1) * Ms if sync else 0)
        cost[c] += 2.0 * float(ev.sum())
    return cost


def shard_classes(p: Problem, n_shards: int):
    """Strong-scaling shards of one sweep: whole dedup classes (so no rank
    re-solves another's DP / refine), assigned heaviest-first to the least
    loaded rank (LPT) by class_cost.  Returns the sorted query indices of each
    shard."""
    cls = query_classes(p)
    cost = class_cost(p, cls)
    owner = np.empty(cost.size, dtype=np.int64)
    load = np.zeros(n_shards)
    for c in np.argsort(-cost, kind="stable"):
        r = int(np.argmin(load))
        owner[c] = r
        load[r] += cost[c]
    qo = owner[cls]
    return [np.nonzero(qo == r)[0] for r in range(n_shards)]


def query_cost(L, N):
    """Estimated relative work of one query (DP rows x windows + simulation)."""
    L = np.asarray(L, dtype=np.float64)
    N = np.asarray(N, dtype=np.float64)
    return 3.0 * L * L + 2.0 * N * 128.0 * 16 + 40.0 * N * L


def shard_queries(L, N, n_shards):
    """Greedy LPT split of queries over ranks by estimated cost."""
    cost = query_cost(L, N)
    order = np.argsort(-cost, kind="stable")
    load = np.zeros(n_shards)
    owner = np.empty(cost.size, dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += cost[i]
    return [np.sort(np.nonzero(owner == r)[0]) for r in range(n_shards)]


# --------------------------------------------------------------------------- test generators
def uniform_network(L, fp, bp, w, a, n_types=1):
    """synth_uniform_network (profiles.hpp:316-337)."""
    return Network(np.full((n_types, L), fp), np.full((n_types, L), bp), np.full(L, w), np.full(L, a))


def random_problem(seed, n_queries=64, max_L=14, max_N=5, n_types=2, mini_batches=(1, 2, 4, 6, 8, 12, 16),
                   cap_range=(50, 200_000), act_max=1000, w_max=1000, t_max=60, bw_range=(1, 2000),
                   min_micro_p=0.1):
    """Seeded random small queries stressing every branch (comm-bound cuts,
    refine, fine-tune, rejections).  Sizes stay small so the O(N U^2)
    restatement oracle finishes in well under a second per query."""
    rng = np.random.default_rng(seed)
    p = Problem(name=f"random seed={seed}")
    for qi in range(n_queries):
        N = int(rng.integers(1, max_N + 1))
        L = int(rng.integers(max(1, N - 1), max_L + 1))
        fp = rng.integers(1, t_max + 1, size=(n_types, L))
        bp = rng.integers(1, t_max + 1, size=(n_types, L))
        w = rng.integers(0, w_max + 1, size=L)
        a = rng.integers(0, act_max + 1, size=L)
        if rng.random() < 0.3:
            a = np.where(rng.random(L) < 0.5, rng.integers(0, 20, size=L), a)
        p.add_network(Network(fp, bp, w, a))
        types = rng.integers(0, n_types, size=N) if rng.random() < 0.5 else np.zeros(N, dtype=np.int64)
        cap = rng.integers(cap_range[0], cap_range[1] + 1, size=N)
        if rng.random() < 0.3:
            cap = np.full(N, int(rng.integers(cap_range[0], cap_range[1] + 1)))
        bw = rng.integers(bw_range[0], bw_range[1] + 1, size=max(0, N - 1))
        mm = np.ones((N, 4), dtype=np.int64)
        if rng.random() < min_micro_p:
            mm[rng.integers(0, N), rng.integers(0, 4)] = int(rng.integers(1, 5))
        p.add_cluster(Cluster(int(rng.integers(0, 2)), types, cap, bw, mm))
    mb = rng.choice(np.array(mini_batches), size=n_queries)
    p.set_queries(np.arange(n_queries), np.arange(n_queries), 0, mb)
    return p
