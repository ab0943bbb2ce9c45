"""GPU parity: the drop-in functions, through the C ABI on a B200, against the
reference's golden values and the pinned oracle.

Counts bit-exact; reals within 1e-9 relative (strict_close) -- the north-star
tolerance -- which also implies the reference's own rel_close.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import cases
from conftest import graph_from, strict_close

pytestmark = pytest.mark.gpu

IDEAL = 7.0 * math.pi / 18.0


def _metrics(g, r):
    import paper_2411_09809_b200 as G

    out = {}
    for key, fn in (("nc", lambda: G.node_occlusion(g, r)), ("ma", lambda: G.minimum_angle(g)),
                    ("ml", lambda: G.edge_length_variation(g)),
                    ("eca", lambda: G.edge_crossing_angle(g, IDEAL))):
        try:
            out[key] = fn()
        except Exception as exc:
            out[key] = {"error": type(exc).__name__}
    out["ec"] = G.edge_crossing(g)
    out["scan"] = G._crossing_scan(g, IDEAL)
    return out


def _check(got, want):
    assert got["ec"] == want["ec"]
    assert got["scan"][0] == want["ec"]
    assert strict_close(got["scan"][1], want["dev"])
    assert got["nc"] == want["nc"]
    for key in ("ma", "ml", "eca"):
        if isinstance(want[key], dict):
            assert got[key] == want[key], key
        else:
            assert isinstance(got[key], float), key
            assert strict_close(got[key], want[key]), (key, got[key], want[key])
    assert isinstance(got["ec"], int) and isinstance(got["nc"], int)


@pytest.mark.parametrize("name", sorted(cases.KNOWN))
def test_known_answers(gpu, golden_small, name):
    want = golden_small["known"][name]
    _check(_metrics(graph_from(cases.KNOWN[name]), want["radius"]), want)


def test_reference_known_values(gpu):
    import paper_2411_09809_b200 as G

    x = graph_from(cases.x_graph)
    assert G.edge_crossing(x) == 1
    assert G.edge_crossing_angle(x) == pytest.approx(5.0 / 7.0)
    assert G.node_occlusion(graph_from(cases.occ_boundary), 1.0) == 0
    assert G.node_occlusion(graph_from(cases.occ_boundary), 1.0000001) == 1
    assert G.node_occlusion(graph_from(cases.occ_three), 1.0) == 3
    assert G.edge_crossing(graph_from(cases.three_mutual)) == 3
    assert G.minimum_angle(graph_from(cases.right_angle)) == pytest.approx(1.0 - 0.5 / 3.0)
    assert G.edge_length_variation(graph_from(cases.lengths_1_3)) == pytest.approx(0.5)


@pytest.mark.parametrize("name", sorted(cases.ADVERSARIAL_SMALL) + sorted(cases.ADVERSARIAL_ARRAYS))
def test_adversarial(gpu, golden_small, name):
    builder = cases.ADVERSARIAL_SMALL.get(name) or cases.ADVERSARIAL_ARRAYS[name]
    want = golden_small["adversarial"][name]
    _check(_metrics(graph_from(builder), want["radius"]), want)


def test_fast_and_general_sign_paths_selected(gpu):
    from paper_2411_09809_b200 import metrics as M

    for name, fast in (("lattice_stress", True), ("big_fast", True), ("small_fast", True),
                       ("huge_coords", False), ("tiny_coords", False),
                       ("small_general", False)):
        g = graph_from(cases.ADVERSARIAL_ARRAYS[name])
        assert M.CrossingRecords(M.DeviceGraph.from_graph(g)).fast_path() is fast, name


def test_criterion1_random_graphs(gpu, golden_small):
    from paper_2411_09809_b200.model import LayoutGraph

    rng = np.random.default_rng(42)
    for i, want in enumerate(golden_small["criterion1"]):
        ids, xy, edges = cases.criterion1_case(i, rng)
        _check(_metrics(LayoutGraph(ids, xy, edges), want["radius"]), want)


def test_parameter_errors_match_reference(gpu):
    import paper_2411_09809_b200 as G

    x = graph_from(cases.x_graph)
    with pytest.raises(G.ParameterError):
        G.node_occlusion(x, 0.0)
    with pytest.raises(G.ParameterError):
        G.node_occlusion(x, -2.0)
    with pytest.raises(G.ParameterError):
        G.edge_crossing_angle(x, ideal_angle=0.0)
    with pytest.raises(G.ParameterError):
        G.edge_crossing_angle(x, ideal_angle=math.pi)
    with pytest.raises(OverflowError):  # (2r)**2 overflows in Python, as in exact.py:63
        G.node_occlusion(x, 1e200)


def test_degenerate_returns(gpu):
    import paper_2411_09809_b200 as G

    lonely = G.LayoutGraph.from_positions({0: (0.0, 0.0), 1: (1.0, 1.0)}, [])
    assert G.minimum_angle(lonely) == 1.0
    assert G.edge_crossing(lonely) == 0
    assert G.edge_crossing_angle(lonely) == 1.0
    assert G._crossing_scan(lonely, IDEAL) == (0, 0.0)
    one = G.LayoutGraph.from_positions({0: (0.0, 0.0), 1: (1.0, 1.0)}, [(0, 1)])
    assert G.edge_length_variation(one) == 0.0
    single = G.LayoutGraph.from_positions({0: (0.0, 0.0)}, [])
    assert G.node_occlusion(single, 1.0) == 0


def test_similarity_invariance(gpu):
    """Acceptance criterion 11 (test_acceptance.py:356-395) on the GPU path."""
    import paper_2411_09809_b200 as G
    from paper_2411_09809_b200.configs import random_graph

    rng = np.random.default_rng(17)
    for i in range(10):
        n = int(rng.integers(10, 81))
        m = int(rng.integers(n, min(4 * n, n * (n - 1) // 2) + 1))
        ids, xy, edges = cases.random_layout_arrays(random_graph(n, m, seed=i), 10.0, 3000 + i)
        g = G.LayoutGraph(ids, xy, edges)
        base = (G.edge_crossing(g), G.minimum_angle(g), G.edge_length_variation(g),
                G.edge_crossing_angle(g))
        for ang, sc, sh in ((1.234, 2.37, (-3.1, 8.9)), (0.3, 1.0, (0.0, 0.0))):
            c, s = math.cos(ang), math.sin(ang)
            rot = np.array([[c, -s], [s, c]])
            g2 = g.with_xy((g.xy @ rot.T) * sc + np.asarray(sh))
            got = (G.edge_crossing(g2), G.minimum_angle(g2), G.edge_length_variation(g2),
                   G.edge_crossing_angle(g2))
            assert got[0] == base[0]
            assert all(abs(a - b) <= 1e-9 * max(1, abs(a), abs(b)) for a, b in zip(base[1:], got[1:]))


def test_unit_range_partials_sum_to_whole(gpu):
    """Sharding contract on one device: disjoint unit ranges add up exactly,
    and match the oracle's unit-range partials."""
    import torch

    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import metrics as M
    from paper_2411_09809_b200 import sharding

    g = graph_from(cases.lattice_stress)
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg)
    full = rec.partial(IDEAL, 0, rec.units).tolist()
    tile = M._lib.lib().glr_crossing_tile()
    for world in (2, 3, 4, 8):
        parts = [rec.partial(IDEAL, *sharding.shard_range(rec.units, r, world)).tolist()
                 for r in range(world)]
        assert sum(p[0] for p in parts) == full[0]
        assert strict_close(sum(p[1] for p in parts), full[1])
        for r, p in enumerate(parts):
            b, e = sharding.shard_range(rec.units, r, world)
            oc, od = O.crossing_scan_units(g.xy, g.edges, IDEAL, tile, b, e,
                                           band=M._lib.lib().glr_crossing_band())
            assert p[0] == oc
            assert strict_close(p[1], od, floor=1e-9)
    n = g.num_vertices
    U = M.occlusion_units(n)
    thr = M.occlusion_threshold(1.0)
    whole = M.occlusion_partial(dg, thr, 0, U).item()
    assert sum(M.occlusion_partial(dg, thr, *sharding.shard_range(U, r, 4)).item()
               for r in range(4)) == whole
    out = sharding.sharded_evaluate(dg, 1.0, IDEAL, 0, 1)
    torch.cuda.synchronize()
    assert out.tolist()[0] == full[0] and out.tolist()[2] == whole


def test_reference_layoutgraph_duck_typing(gpu):
    """A graph object exposing only xy/edges/num_vertices/num_edges (the
    reference LayoutGraph's attributes) is accepted."""
    import paper_2411_09809_b200 as G

    g = graph_from(cases.three_mutual)

    class Duck:
        xy = g.xy
        edges = g.edges
        num_vertices = g.num_vertices
        num_edges = g.num_edges

    assert G.edge_crossing(Duck()) == 3


def test_device_graph_input(gpu):
    import torch

    import paper_2411_09809_b200 as G

    g = graph_from(cases.lattice_stress)
    dg = G.DeviceGraph(torch.from_numpy(g.xy).cuda(), torch.from_numpy(g.edges).cuda())
    assert G.edge_crossing(dg) == 4194903
    assert G.node_occlusion(dg, 1.0) == 9588


def test_balanced_shards_sum_to_whole(gpu):
    """Cost-balanced unit ranges (CrossingRecords.shard) tile the unit space
    and their partials add up exactly, dense and culled."""
    from paper_2411_09809_b200 import metrics as M

    g = graph_from(cases.lattice_stress)
    dg = M.DeviceGraph.from_graph(g)
    for strategy in ("dense", "culled"):
        rec = M.CrossingRecords(dg, strategy)
        full = rec.partial(IDEAL, 0, rec.units).tolist()
        for world in (2, 5, 8):
            ranges = [rec.shard(r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == rec.units
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            parts = [rec.partial(IDEAL, b, e).tolist() for b, e in ranges]
            assert sum(p[0] for p in parts) == full[0] == 4194903
            assert strict_close(sum(p[1] for p in parts), full[1])


@pytest.mark.parametrize("m", [2, 3, 255, 256, 257, 511, 512, 513, 1023, 1025])
def test_tile_boundaries_dense_and_culled(gpu, m):
    """Edge counts around the 256-edge tile (padding, diagonal tiles, ragged
    last tile) on a degenerate-heavy integer lattice, against the oracle."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import metrics as M
    from paper_2411_09809_b200.model import LayoutGraph

    rng = np.random.default_rng(m)
    n = max(4, m // 2)
    xy = rng.integers(0, 12, (n, 2)).astype(np.float64)
    pairs = rng.integers(0, n, (3 * m, 2))
    pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
    g = LayoutGraph(np.arange(n), xy, pairs)
    e = g.edges[:m]
    g = LayoutGraph(np.arange(n), xy, e)
    want_c, want_d = O.crossing_scan(g.xy, g.edges, IDEAL)
    want_nc = O.node_occlusion(g.xy, 0.7)
    for strategy in ("dense", "culled"):
        c, d = M._crossing_scan(g, IDEAL, strategy=strategy)
        assert c == want_c, strategy
        assert strict_close(d, want_d), strategy
        assert M.node_occlusion(g, 0.7, strategy=strategy) == want_nc, strategy


def test_vertex_tile_boundaries(gpu):
    """Vertex counts around the 1024-vertex occlusion tile."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import metrics as M
    from paper_2411_09809_b200.model import LayoutGraph

    for n in (2, 1023, 1024, 1025, 2049):
        xy = np.random.default_rng(n).integers(0, 40, (n, 2)).astype(np.float64)
        g = LayoutGraph(np.arange(n), xy, [])
        want = O.node_occlusion(g.xy, 1.0)
        for strategy in ("dense", "culled"):
            assert M.node_occlusion(g, 1.0, strategy=strategy) == want, (n, strategy)


def test_random_degenerate_graphs(gpu):
    """Many small graphs on tiny integer grids (collinear, overlapping,
    coincident and touching segments everywhere) against the oracle."""
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G

    rng = np.random.default_rng(123)
    for trial in range(40):
        n = int(rng.integers(3, 60))
        side = int(rng.integers(2, 8))
        xy = rng.integers(0, side, (n, 2)).astype(np.float64)
        if trial % 3 == 0:
            xy = xy * 0.1 - 0.3  # non-integer, negative, still degenerate
        pairs = rng.integers(0, n, (int(rng.integers(1, 150)), 2))
        pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
        if len(pairs) == 0:
            continue
        g = G.LayoutGraph(np.arange(n), xy, pairs)
        c, d = G._crossing_scan(g, IDEAL)
        oc, od = O.crossing_scan(g.xy, g.edges, IDEAL)
        assert c == oc and strict_close(d, od), trial
        r = float(rng.uniform(0.05, 1.0))
        assert G.node_occlusion(g, r) == O.node_occlusion(g.xy, r), trial
        assert strict_close(G.minimum_angle(g), O.minimum_angle(g.xy, g.edges)), trial
        if g.num_edges > 1:
            assert strict_close(G.edge_length_variation(g),
                                O.edge_length_variation(g.xy, g.edges)), trial


def test_interleaved_shards_sum_to_whole(gpu):
    """Interleaved chunk ownership (the multi-GPU default): ranks' partials
    sum exactly to the whole, dense and culled, and match the oracle."""
    from paper_2411_09809_b200 import metrics as M

    g = graph_from(cases.lattice_stress)
    dg = M.DeviceGraph.from_graph(g)
    for strategy in ("dense", "culled"):
        rec = M.CrossingRecords(dg, strategy)
        for world in (1, 2, 3, 8):
            parts = [rec.partial_interleaved(IDEAL, r, world).tolist() for r in range(world)]
            assert sum(p[0] for p in parts) == 4194903, (strategy, world)
            assert strict_close(sum(p[1] for p in parts), 1475177.8703388437)
