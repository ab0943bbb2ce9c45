"""Inputs of the strip-sweep parity cases (shared by the golden generator and
the tests): the reference tests' graphs (pkg/tests/test_enhanced.py) and
random / tie-heavy layouts, each with (fraction, orientation) settings."""

from __future__ import annotations

import numpy as np

from paper_2411_09809_b200.configs import random_graph


def _random_layout(edges, extent, seed):
    ids = np.unique(edges)
    xy = np.random.default_rng(seed).uniform(0.0, extent, size=(len(ids), 2))
    return ids, xy, edges


def _lattice(seed=5, side=12, m=400):
    rng = np.random.default_rng(seed)
    gx, gy = np.meshgrid(np.arange(side, dtype=np.float64), np.arange(side, dtype=np.float64))
    xy = np.stack([gx.ravel(), gy.ravel()], 1)
    u = rng.integers(0, side * side, 3 * m)
    v = rng.integers(0, side * side, 3 * m)
    keep = u != v
    return np.arange(side * side), xy, np.stack([u[keep], v[keep]], 1)[:m]


def _off_boundary():
    return (np.arange(4), np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 0.7], [1.0, 0.2]]),
            np.array([[0, 1], [2, 3]]))


def _on_boundary():
    return (np.arange(4), np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 1.0], [1.0, 0.0]]),
            np.array([[0, 1], [2, 3]]))


GRAPHS = {
    "off_boundary": _off_boundary(),
    "on_boundary": _on_boundary(),
    "rg_40_100": _random_layout(random_graph(40, 100, seed=13), 10.0, 14),
    "rg_80_300": _random_layout(random_graph(80, 300, seed=17), 30.0, 18),
    "rg_1000_5000": _random_layout(random_graph(1000, 5000, seed=2), 100.0, 3),
    "lattice_ties": _lattice(),
}

SETTINGS = {
    "off_boundary": [(0.25, "vertical")],
    "on_boundary": [(0.5, "vertical"), (0.5, "both")],
    "rg_40_100": [(0.2, "vertical"), (0.2, "horizontal"), (0.2, "both")],
    "rg_80_300": [(0.1, "vertical"), (0.03, "horizontal"), (0.45, "both")],
    "rg_1000_5000": [(0.05, "vertical"), (0.1, "horizontal"), (0.01, "both")],
    "lattice_ties": [(0.25, "vertical"), (0.1, "horizontal"), (0.34, "both")],
}
