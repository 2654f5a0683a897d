"""Named explore() scenarios shared by the golden generator and the tests.

The first group restates the reference's own unit-test scenarios as
explore() queries (file:line of /root/reference/proj/tests cited per entry);
the rest are the BASELINE configs and seeded random batches.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2012_12544_b200 import workloads as W  # noqa: E402
from paper_2012_12544_b200.abi import MODE_ASYNC, MODE_SYNC  # noqa: E402
from paper_2012_12544_b200.problem import Cluster, Network, Problem  # noqa: E402

GB = 1_000_000_000


def single(net, cl, mini, m_list=None, name=""):
    p = Problem(name=name)
    p.add_network(net)
    p.add_cluster(cl)
    p.set_queries([0], 0, 0, mini, None if m_list is None else [m_list])
    return p


def uni(L, fp, bp, w, a):
    return W.uniform_network(L, fp, bp, w, a)


def tri_cluster(mode, caps, min_micro=None):            # test_explorer.cpp:14-21
    return Cluster(mode, [0, 0, 0], caps, [50, 50], min_micro)


def homo(n, cap=GB, bw=None):                            # test_partitioner.cpp:13-22
    return Cluster(MODE_SYNC, [0] * n, [cap] * n, bw if bw is not None else [1_000_000] * (n - 1))


def _heavy(a1):                                          # test_partitioner.cpp:274-285
    n = uni(6, 10, 20, 0, 100000)
    n.a[1] = a1
    return n


def _shift_net():                                        # test_partitioner.cpp:232-237
    n = uni(4, 5, 10, 1000, 10)
    n.fp[0, 3], n.bp[0, 3] = 15, 30
    return n


def _hetero_tail():                                      # test_cost_models.cpp:119-135
    n = uni(3, 10, 20, 0, 50)
    n.fp[0, 2] = 17
    return n


def _async_floor():                                      # test_explorer.cpp:108-132
    mm = np.ones((3, 4), dtype=np.int64)
    mm[:, 0] = 4
    return tri_cluster(MODE_ASYNC, [600, 600, 600], mm)


def c5_sample(stride=1021):   # prime stride: covers every (model, cluster, N) class
    full = W.config_c5()
    idx = np.arange(0, full.queries.size, stride)
    p = Problem(networks=full.networks, clusters=full.clusters, name=f"C5 1/{stride}")
    q = full.queries[idx]
    p.set_queries(q["network"], q["cluster"], q["n_stages"], q["mini_batch"])
    return p


def heavy_random(seed):
    return W.random_problem(seed, n_queries=60, max_L=40, max_N=16, cap_range=(1000, 60000), bw_range=(1, 500),
                            act_max=3000)


SCENARIOS = [
    # test_explorer.cpp
    ("explorer_memory_tight_sno", lambda: single(uni(3, 10, 20, 100, 50), tri_cluster(MODE_SYNC, [400, 10**6, 10**6]), 4, [4])),
    ("explorer_abundant_so", lambda: single(uni(3, 10, 20, 100, 50), tri_cluster(MODE_SYNC, [10**6] * 3), 4, [4])),
    ("explorer_m1_tie_sno", lambda: single(uni(3, 10, 20, 100, 50), tri_cluster(MODE_SYNC, [10**6] * 3), 1)),
    ("explorer_async_fbp", lambda: single(uni(3, 10, 20, 100, 50), _async_floor(), 8)),
    ("explorer_capacity_tight", lambda: single(uni(3, 10, 20, 100, 50), tri_cluster(MODE_SYNC, [400, 10**6, 10**6]), 4)),
    ("explorer_capacity_roomy", lambda: single(uni(3, 10, 20, 100, 50), tri_cluster(MODE_SYNC, [GB] * 3), 4)),
    ("explorer_ranking", lambda: single(uni(6, 10, 20, 100, 40), tri_cluster(MODE_SYNC, [10**6] * 3), 8)),
    ("explorer_all_rejected", lambda: single(uni(3, 10, 20, 100, 50), tri_cluster(MODE_SYNC, [1, 1, 1]), 2)),
    # test_partitioner.cpp
    ("partition_balanced_flow", lambda: single(uni(6, 10, 20, 100, 40), homo(3), 6, [6])),
    ("partition_single_device", lambda: single(uni(6, 10, 20, 100, 40), homo(1), 6, [6])),
    ("partition_comm_coarse", lambda: single(_heavy(10), homo(2, GB, [10]), 4, [4])),
    ("partition_comm_infeasible", lambda: single(_heavy(100000), homo(2, GB, [10]), 4, [4])),
    ("finetune_shift", lambda: single(_shift_net(), Cluster(MODE_SYNC, [0, 0], [4100, 100000], [1_000_000]), 2, [2])),
    ("finetune_impossible", lambda: single(uni(4, 10, 20, 1_000_000, 10), homo(2, 1000), 2, [2])),
    ("refine_31_2", lambda: single(W.Network([[5, 5, 5]], [[5, 5, 6]], [0, 0, 0], [10, 10, 10]), homo(2), 1, [1])),
    # test_cost_models.cpp / test_simulator.cpp
    ("estimate_balanced", lambda: single(uni(4, 10, 20, 100, 50), Cluster(MODE_SYNC, [0] * 4, [100000] * 4, [25] * 3), 8, [8])),
    ("estimate_heuristic", lambda: single(_hetero_tail(), Cluster(MODE_ASYNC, [0] * 3, [100000] * 3, [50, 50]), 8, [8, 2])),
    ("simulator_plan_level", lambda: single(uni(4, 10, 20, 100, 50), Cluster(MODE_SYNC, [0, 0], [10**6] * 2, [25]), 4, [4])),
    # BASELINE configs
    ("C1_vgg16", W.config_c1),
    ("C2_resnet50", W.config_c2),
    ("C3_gnmt16", W.config_c3),
    ("C4_onchip", lambda: W.config_c4("onchip")),
    ("C4_offchip", lambda: W.config_c4("offchip")),
    ("C4_homogeneous", lambda: W.config_c4("homogeneous")),
    # seeded random batches
    ("random_0", lambda: W.random_problem(0, n_queries=100)),
    ("random_1", lambda: W.random_problem(1, n_queries=100)),
    ("random_2", lambda: W.random_problem(2, n_queries=100)),
    ("random_3", lambda: W.random_problem(3, n_queries=100)),
    ("random_heavy_100", lambda: heavy_random(100)),
    ("random_heavy_101", lambda: heavy_random(101)),
    ("random_heavy_102", lambda: heavy_random(102)),
    ("random_heavy_103", lambda: heavy_random(103)),
    ("C5_stride1021", c5_sample),
]

SMALL = [n for n, _ in SCENARIOS if not n.startswith(("C4", "C5"))]


def build(name):
    return dict(SCENARIOS)[name]()
