"""Inputs of the fr_layout parity cases (shared by the golden generator and
the tests): the reference tests' own graphs (pkg/tests/test_graphio.py:
169-185, test_acceptance.py:97-103) and a few more shapes."""

from __future__ import annotations

import numpy as np

from paper_2411_09809_b200.configs import random_graph


def _k5():
    return np.array([(a, b) for a in range(5) for b in range(a + 1, 5)], dtype=np.int64)


def _sparse_ids():
    # non-contiguous ids, a self-loop and a duplicate (dropped by normalize_edges)
    e = random_graph(150, 400, seed=11) * 7 + 3
    return np.concatenate([e, [[3, 3], [e[0, 1], e[0, 0]]]])


def _two_components():
    a = random_graph(60, 150, seed=12)
    b = random_graph(40, 90, seed=13) + 1000
    return np.concatenate([a, b])


CASES = {
    "ref_test_30_60": (random_graph(30, 60, seed=7), {"iterations": 40, "seed": 8, "extent": 10.0}),
    "ref_test_k5": (_k5(), {"iterations": 60, "seed": 3, "extent": 10.0}),
    "rg_200_600": (random_graph(200, 600, seed=1), {"iterations": 50, "seed": 1, "extent": 100.0}),
    "rg_1000_5000": (random_graph(1000, 5000, seed=3), {"iterations": 10, "seed": 4, "extent": 100.0}),
    "sparse_ids": (_sparse_ids(), {"iterations": 25, "seed": 5, "extent": 50.0}),
    "two_components": (_two_components(), {"iterations": 30, "seed": 6, "extent": 100.0}),
    "single_edge": (np.array([[4, 9]], dtype=np.int64), {"iterations": 5, "seed": 0, "extent": 1.0}),
    "acceptance_4000_80000": (random_graph(4000, 80000, seed=500),
                              {"iterations": 2, "seed": 600, "extent": 100.0}),
}
