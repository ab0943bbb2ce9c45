"""Strip-sweep approximations against the reference's
own outputs (tests/golden/strip_golden.json, tests/golden/make_golden_strips.py):
counts exact, deviation sums at 1e-9."""

from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import strip_cases
from conftest import strict_close

HERE = os.path.dirname(os.path.abspath(__file__))
IDEAL = math.radians(70.0)


@pytest.fixture(scope="module")
def strip_golden():
    with open(os.path.join(HERE, "golden", "strip_golden.json")) as fh:
        return json.load(fh)


def _graph(name):
    from paper_2411_09809_b200.model import LayoutGraph

    ids, xy, pairs = strip_cases.GRAPHS[name]
    return LayoutGraph(ids, xy, pairs)


def test_strip_bounds_match_reference_recipe():
    from paper_2411_09809_b200.enhanced import strip_bounds

    xy = np.array([[0.1, 5.0], [0.9, -2.0], [0.35, 1.0]])
    b = strip_bounds(xy, 0.3, "vertical")
    assert len(b) == 5 and b[0] == 0.1 and b[-1] == 0.9
    width = (0.9 - 0.1) / 4
    assert b[1] == 0.1 + 1 * width and b[2] == 0.1 + 2 * width
    h = strip_bounds(xy, 0.5, "horizontal")
    assert h[0] == -2.0 and h[-1] == 5.0


def test_strip_parameter_errors_mirror_reference():
    from paper_2411_09809_b200 import InputError, ParameterError, edge_crossing_enhanced
    from paper_2411_09809_b200.enhanced import strip_bounds

    g = _graph("rg_40_100")
    with pytest.raises(ParameterError):
        edge_crossing_enhanced(g, 1.0)
    with pytest.raises(ParameterError):
        edge_crossing_enhanced(g, 0.2, orientation="diagonal")
    with pytest.raises(InputError):
        strip_bounds(np.array([[1.0, 0.0], [1.0, 2.0]]), 0.5, "vertical")
    # fewer than two edges: 0 before any fraction check (enhanced.py:239-240)
    lonely = _graph("off_boundary")
    from paper_2411_09809_b200.model import LayoutGraph

    one = LayoutGraph(np.arange(2), np.array([[0.0, 0.0], [1.0, 1.0]]), np.array([[0, 1]]))
    assert edge_crossing_enhanced(one, 5.0) == 0
    assert lonely.num_edges == 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(strip_cases.GRAPHS))
def test_gpu_strip_sweeps_match_reference(gpu, strip_golden, name):
    from paper_2411_09809_b200 import crossing_angle_stats, edge_crossing_enhanced

    g = _graph(name)
    for row in strip_golden["cases"][name]:
        frac, orient = row["fraction"], row["orientation"]
        assert edge_crossing_enhanced(g, frac, orient) == row["ec"], (name, frac, orient)
        c, d = crossing_angle_stats(g, frac, IDEAL, orient)
        assert c == row["count"], (name, frac, orient)
        assert strict_close(d, row["dev"]), (name, frac, orient, d, row["dev"])


@pytest.mark.gpu
def test_gpu_strip_properties(gpu):
    """Reference invariants (test_enhanced.py): a lower bound of the exact
    count; "both" is the larger orientation; angle score of a single visible
    crossing equals the exact one."""
    from paper_2411_09809_b200 import (edge_crossing, edge_crossing_angle,
                                       edge_crossing_angle_enhanced, edge_crossing_enhanced,
                                       node_occlusion, node_occlusion_grid)
    from paper_2411_09809_b200.model import LayoutGraph

    rng = np.random.default_rng(700)
    from paper_2411_09809_b200.configs import random_graph

    for seed in range(6):
        n = int(rng.integers(6, 80))
        m = min(4 * n, n * (n - 1) // 2)
        e = random_graph(n, m, seed=seed)
        ids = np.unique(e)
        xy = np.random.default_rng(seed + 9).uniform(0, 20.0, (len(ids), 2))
        g = LayoutGraph(ids, xy, e)
        frac = float(rng.uniform(0.02, 0.5))
        exact = edge_crossing(g)
        v = edge_crossing_enhanced(g, frac, "vertical")
        h = edge_crossing_enhanced(g, frac, "horizontal")
        assert v <= exact and h <= exact
        assert edge_crossing_enhanced(g, frac, "both") == max(v, h)
        assert node_occlusion_grid(g, 0.7) == node_occlusion(g, 0.7)
    g = _graph("off_boundary")
    assert edge_crossing_angle_enhanced(g, 0.25, IDEAL) == pytest.approx(
        edge_crossing_angle(g, IDEAL))
    assert edge_crossing_angle_enhanced(_graph("on_boundary"), 0.5, IDEAL) == 1.0


@pytest.mark.parametrize("name", sorted(strip_cases.GRAPHS))
def test_oracle_strip_restatement_matches_reference(strip_golden, name):
    from oracle.glare_oracle import strip_crossings

    g = _graph(name)
    ideal = strip_golden["ideal"]
    for row in strip_golden["cases"][name]:
        frac, orient = row["fraction"], row["orientation"]
        if orient == "both":
            v = strip_crossings(g.xy, g.edges, frac, "vertical", ideal)
            h = strip_crossings(g.xy, g.edges, frac, "horizontal", ideal)
            got = v if v[0] >= h[0] else h
        else:
            got = strip_crossings(g.xy, g.edges, frac, orient, ideal)
        assert got[0] == row["count"]
        assert strict_close(got[1], row["dev"])


@pytest.mark.gpu
def test_gpu_strips_random_against_oracle(gpu):
    """Random layouts (continuous and integer-lattice coordinates), random
    fractions, both single orientations: GPU == oracle restatement."""
    from oracle.glare_oracle import strip_crossings
    from paper_2411_09809_b200 import crossing_angle_stats
    from paper_2411_09809_b200.configs import random_graph
    from paper_2411_09809_b200.model import LayoutGraph

    rng = np.random.default_rng(11)
    for trial in range(24):
        n = int(rng.integers(8, 400))
        m = min(int(rng.integers(n, 6 * n)), n * (n - 1) // 2)
        e = random_graph(n, m, seed=trial)
        ids = np.unique(e)
        if trial % 3 == 0:
            xy = rng.integers(0, 9, (len(ids), 2)).astype(np.float64)
            keep = np.any(xy[np.searchsorted(ids, e[:, 0])] != xy[np.searchsorted(ids, e[:, 1])], 1)
            e = e[keep]
            if len(e) < 2:
                continue
            ids2 = np.unique(e)
            xy = xy[np.searchsorted(ids, ids2)]
            ids = ids2
        else:
            xy = rng.uniform(-5, 5, (len(ids), 2))
        g = LayoutGraph(ids, xy, e)
        frac = float(rng.uniform(0.01, 0.6))
        for orient in ("vertical", "horizontal"):
            c, d = crossing_angle_stats(g, frac, IDEAL, orient)
            wc, wd = strip_crossings(g.xy, g.edges, frac, orient, IDEAL)
            assert c == wc, (trial, orient)
            assert strict_close(d, wd), (trial, orient, d, wd)
