"""Pins the CPU oracle (oracle/) to the reference implementation.

The golden JSON files were produced by running the reference's own serial
oracle (glare.metrics.exact, /root/reference/pkg/src/glare/metrics/exact.py)
on the inputs of tests/cases.py and paper_2411_09809_b200/configs.py
(tests/golden/make_golden.py).  Counts must match exactly, reals within the
reference's 1e-9 (and 1e-9 relative).  The oracle is the checker for the GPU
tests, so it is pinned here first.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import cases
from conftest import graph_from, rel_close, strict_close
from oracle import glare_oracle as O
from oracle import sweep as S
from paper_2411_09809_b200 import configs
from paper_2411_09809_b200.configs import fingerprint

IDEAL = configs.IDEAL_70


def _check(g, want, use_c=False):
    assert fingerprint(g) == want["fingerprint"]
    r = want["radius"]
    if isinstance(want["nc"], int):
        got = S.node_occlusion(g.xy, r) if use_c else O.node_occlusion(g.xy, r)
        assert got == want["nc"]
    c, d = (S.crossing_scan if use_c else O.crossing_scan)(g.xy, g.edges, IDEAL)
    assert c == want["ec"]
    assert strict_close(d, want["dev"])
    if isinstance(want["ma"], float):
        assert strict_close(O.minimum_angle(g.xy, g.edges), want["ma"])
    if isinstance(want["ml"], float):
        assert strict_close(O.edge_length_variation(g.xy, g.edges), want["ml"])
    if isinstance(want["eca"], float):
        assert strict_close(O.edge_crossing_angle(g.xy, g.edges, IDEAL), want["eca"])


@pytest.mark.parametrize("name", sorted(cases.KNOWN))
def test_known_answers(golden_small, name):
    _check(graph_from(cases.KNOWN[name]), golden_small["known"][name])


def test_reference_test_values(golden_small):
    """Hand-computed values asserted by the reference's own tests
    (tests/test_metrics_exact.py:29-155, tests/test_engine.py:22-30)."""
    k = golden_small["known"]
    assert k["x_graph"]["ec"] == 1
    assert k["parallel"]["ec"] == 0
    assert k["triangle_centre"]["ec"] == 0
    assert k["three_mutual"]["ec"] == 3
    assert k["occ_one_pair"]["nc"] == 1
    assert k["occ_boundary"]["nc"] == 0 and k["occ_boundary"]["nc_r1.0000001"] == 1
    assert k["occ_three"]["nc"] == 3
    assert k["x_graph"]["eca"] == pytest.approx(5.0 / 7.0)
    assert k["ideal_crossing"]["eca"] == pytest.approx(1.0)
    assert k["parallel"]["eca"] == 1.0
    assert k["right_angle"]["ma"] == pytest.approx(1.0 - 0.5 / 3.0)
    assert k["star6"]["ma"] == pytest.approx(1.0)
    assert k["right_angle_isolated"]["ma"] == pytest.approx(k["right_angle"]["ma"])
    assert k["lengths_1_3"]["ml"] == pytest.approx(0.5)
    g = graph_from(cases.occ_boundary)
    assert O.node_occlusion(g.xy, 1.0000001) == 1
    assert float(O.crossing_angles(0.1, 3.0)) == 0.2415926535897932


@pytest.mark.parametrize("name", sorted(cases.ADVERSARIAL_SMALL) + sorted(cases.ADVERSARIAL_ARRAYS))
def test_adversarial(golden_small, name):
    builder = cases.ADVERSARIAL_SMALL.get(name) or cases.ADVERSARIAL_ARRAYS[name]
    _check(graph_from(builder), golden_small["adversarial"][name])


def test_adversarial_c_oracle(golden_small):
    """The C restatement (x-sorted sweep, pthreads) agrees too."""
    for name, builder in {**cases.ADVERSARIAL_SMALL, **cases.ADVERSARIAL_ARRAYS}.items():
        _check(graph_from(builder), golden_small["adversarial"][name], use_c=True)


def test_criterion1_random_graphs(golden_small):
    rng = np.random.default_rng(42)
    for i, want in enumerate(golden_small["criterion1"]):
        ids, xy, edges = cases.criterion1_case(i, rng)
        from paper_2411_09809_b200.model import LayoutGraph

        g = LayoutGraph(ids, xy, edges)
        _check(g, want, use_c=(i % 2 == 1))


def test_paper_oracle_semantics():
    """bbox prefilter, index-based adjacency,
    np.mod edge cases."""
    assert O.edge_crossing(*_arrays(cases.collinear_disjoint)) == 0
    assert O.edge_crossing(*_arrays(cases.coincident_ids)) == 1
    assert O.edge_crossing(*_arrays(cases.shared_vertex)) == 0
    assert O.axis_angles(0.0, 0.0, -1.0, 0.0) == 0.0
    assert math.copysign(1.0, float(np.mod(-0.0, np.pi))) == 1.0
    assert float(np.mod(-1e-17, np.pi)) == np.pi


def _arrays(builder):
    g = graph_from(builder)
    return g.xy, g.edges


def test_unit_range_partials_compose():
    """Partials over any partition of the tile-pair unit space sum to the
    whole scan (the sharding contract of glr_crossing_pairs /
    glr_occlusion_count), including diagonal tiles and ragged last tiles."""
    g = graph_from(cases.lattice_stress)
    tile = 512
    T = -(-g.num_edges // tile)
    U = T * (T + 1) // 2
    full = O.crossing_scan(g.xy, g.edges, IDEAL)
    cuts = [0, 1, 5, U // 2, U - 1, U]
    parts = [O.crossing_scan_units(g.xy, g.edges, IDEAL, tile, a, b) for a, b in zip(cuts, cuts[1:])]
    assert sum(p[0] for p in parts) == full[0]
    assert rel_close(sum(p[1] for p in parts), full[1])
    # banded unit order (the crossing kernels' order) is a permutation of the
    # triangle: every tile pair once, for any band width
    for band in (1, 2, 3, 5, T):
        seen = [O._band_coords(u, T, band) for u in range(U)]
        assert sorted(seen) == [(a, b) for a in range(T) for b in range(a, T)]
    small = 96
    Ts = -(-g.num_edges // small)
    Us = Ts * (Ts + 1) // 2
    cuts = [0, 7, Us // 3, Us - 5, Us]
    parts = [O.crossing_scan_units(g.xy, g.edges, IDEAL, small, a, b, band=4)
             for a, b in zip(cuts, cuts[1:])]
    assert sum(p[0] for p in parts) == full[0]
    tile_v = 1024
    Tv = -(-g.num_vertices // tile_v)
    Uv = Tv * (Tv + 1) // 2
    occ = sum(O.node_occlusion_units(g.xy, 1.0, tile_v, u, u + 1) for u in range(Uv))
    assert occ == O.node_occlusion(g.xy, 1.0)


def test_grid_occlusion_matches_dense():
    for name in ("lattice_stress", "occlusion_ties", "near_collinear"):
        g = graph_from(cases.ADVERSARIAL_ARRAYS[name])
        r = cases.ADVERSARIAL_RADIUS[name]
        assert O.node_occlusion_grid(g.xy, r) == O.node_occlusion(g.xy, r)
