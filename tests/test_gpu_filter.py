"""GPU: the certified packed-FP32 crossing filter (pair-kernel mode 2, the
default inside the fast window) against the general exact-comparison kernel
(mode 0), the FP64 float-view sign kernel (mode 1) and the C oracle, on
inputs built to defeat a filter: near-collinear triples, exact collinear
lattice points, coordinates far from the origin, mixed scales, very short
edges, hubs (shared vertices) and coincident vertices with distinct ids.

Counts must agree exactly; dev_sum differs between modes only in the order
the per-thread sums absorb the terms (mode 2 adds a block's uncertain pairs
after its certain ones, mode 1 subtracts its adjacency correction at the
end), so it is compared at 1e-12.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import strict_close

pytestmark = pytest.mark.gpu

IDEAL = 7.0 * math.pi / 18.0


def _graph(xy, pairs):
    from paper_2411_09809_b200.model import LayoutGraph

    xy = np.asarray(xy, dtype=np.float64)
    return LayoutGraph(np.arange(len(xy)), xy, np.asarray(pairs, dtype=np.int64))


def _random_pairs(rng, n, m):
    u = rng.integers(0, n, 3 * m)
    v = rng.integers(0, n, 3 * m)
    keep = u != v
    p = np.stack([u[keep], v[keep]], 1)[:m]
    return p


def near_collinear(seed=1, lines=60, per_line=20):
    """Points on random lines, perturbed by ~1e-9 of the extent: many cross
    products within the filter's uncertainty band."""
    rng = np.random.default_rng(seed)
    pts = []
    for _ in range(lines):
        p0 = rng.uniform(0, 1, 2)
        d = rng.normal(size=2)
        d /= np.linalg.norm(d)
        t = rng.uniform(-0.5, 0.5, per_line)
        q = p0 + t[:, None] * d + rng.normal(scale=1e-9, size=(per_line, 2))
        pts.append(q)
    xy = np.concatenate(pts)
    n = len(xy)
    pairs = [(i, i + 1) for i in range(0, n - 1)] + [tuple(p) for p in _random_pairs(rng, n, n)]
    return xy, pairs


def exact_lattice(seed=2, side=6, m=1500):
    """Integer lattice with many exactly collinear vertex/edge triples."""
    rng = np.random.default_rng(seed)
    gx, gy = np.meshgrid(np.arange(side), np.arange(side))
    xy = np.stack([gx.ravel(), gy.ravel()], 1).astype(np.float64)
    return xy, _random_pairs(rng, len(xy), m)


def far_offset(seed=3, n=600, m=2000, offset=2.0 ** 40):
    """Coordinates 2^40 + small integers/halves: the FP32 filter must work on
    translated coordinates."""
    rng = np.random.default_rng(seed)
    xy = offset + rng.integers(0, 200, (n, 2)).astype(np.float64) * 0.5
    xy = np.unique(xy, axis=0)
    return xy, _random_pairs(rng, len(xy), m)


def mixed_scales(seed=4, n=800, m=2500):
    """A dense cluster of extent 1e-7 plus long edges spanning [0, 1]."""
    rng = np.random.default_rng(seed)
    cluster = 0.5 + rng.uniform(0, 1e-7, (n, 2))
    far = rng.uniform(0, 1, (50, 2))
    xy = np.concatenate([cluster, far])
    pairs = _random_pairs(rng, n, m - 100)
    pairs = np.concatenate([pairs, _random_pairs(rng, len(xy), 100)])
    return xy, pairs


def short_edges(seed=5, n=3000):
    """Edges of length ~1e-6 in a unit square (C3-like, extreme)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0, 1, (n, 2))
    b = a + rng.normal(scale=1e-6, size=(n, 2))
    c = a + rng.normal(scale=1e-6, size=(n, 2))
    xy = np.concatenate([a, b, c])
    pairs = [(i, n + i) for i in range(n)] + [(n + i, 2 * n + i) for i in range(n)]
    return xy, pairs


def hubs(seed=6, n=2000, m=4000):
    """A few hubs holding most edges, some spokes exactly collinear."""
    rng = np.random.default_rng(seed)
    xy = rng.integers(0, 64, (n, 2)).astype(np.float64)
    xy = np.unique(xy, axis=0)
    n = len(xy)
    hub = rng.integers(0, 5, m)
    other = rng.integers(5, n, m)
    return xy, np.stack([hub, other], 1)


def coincident(seed=7, n=400, m=1500):
    """Distinct vertex ids sharing coordinates."""
    rng = np.random.default_rng(seed)
    half = n // 2
    base = rng.uniform(0, 1, (half, 2))
    xy = np.concatenate([base, base])
    p = _random_pairs(rng, len(xy), 2 * m)
    p = p[(p[:, 0] % half) != (p[:, 1] % half)][:m]  # no zero-length edges
    return xy, p


def lattice_c5_like(seed=8, n=3000, m=6000):
    rng = np.random.default_rng(seed)
    xy = rng.integers(0, 2 ** 16, (n, 2)).astype(np.float64)
    return xy, _random_pairs(rng, n, m)


def tight_clusters(seed=9, clusters=24, per=300):
    """Clusters that fill whole tiles with tight per-unit thresholds (small
    box D, long edges L ~ 2D): packed near-parallel long edges, near-collinear
    chains with T-junctions, pencils of lines at 1e-7 rad through one point,
    and crossing fans -- the unit threshold, not the global bound, decides
    every pair inside them (tests/test_filter_bound.py checks the same
    families with exact rationals)."""
    rng = np.random.default_rng(seed)
    segs = []
    for c in range(clusters):
        off = rng.uniform(0.05, 0.9, 2)
        D = float(10.0 ** rng.uniform(-6, -2))
        kind = c % 4
        for _ in range(per):
            if kind == 0:
                y = rng.uniform(0, D)
                segs.append((off + [0, y], off + [D, y + rng.normal(scale=D * 1e-6)]))
            elif kind == 1:
                d = np.array([0.6, 0.8])
                s0, s1 = np.sort(rng.uniform(0, D, 2))
                nrm = np.array([-0.8, 0.6]) * rng.normal(scale=D * 1e-9)
                segs.append((off + s0 * d + nrm, off + s1 * d))
            elif kind == 2:
                ang = rng.normal(scale=1e-7)
                v = np.array([math.cos(ang), math.sin(ang)]) * D / 2
                q = off + rng.normal(scale=D * 1e-9, size=2)
                segs.append((q - v, q + v))
            else:
                if rng.random() < 0.5:
                    y = rng.uniform(0, D)
                    segs.append((off + [0, y], off + [D, y + rng.uniform(-D, D) * 1e-3]))
                else:
                    x = rng.uniform(0, D)
                    segs.append((off + [x, -D * 0.1], off + [x + rng.uniform(-D, D), D * 1.1]))
    pts = np.array([p for sgm in segs for p in sgm], dtype=np.float64)
    xy, inv = np.unique(pts, axis=0, return_inverse=True)
    pairs = inv.reshape(-1, 2)
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    return xy, pairs


CASES = {f.__name__: f for f in (near_collinear, exact_lattice, far_offset, mixed_scales,
                                  short_edges, hubs, coincident, lattice_c5_like,
                                  tight_clusters)}


def _run(dg, mode, ideal):
    from paper_2411_09809_b200 import metrics as M

    rec = M.CrossingRecords(dg)
    got_mode = rec.set_mode(mode).mode()
    out = rec.partial(ideal, 0, rec.units).tolist()
    return got_mode, int(out[0]), out[1]


@pytest.mark.parametrize("name", sorted(CASES))
def test_filter_modes_agree_with_oracle(gpu, name):
    from oracle import sweep as S
    from paper_2411_09809_b200 import metrics as M

    g = _graph(*CASES[name]())
    dg = M.DeviceGraph.from_graph(g)
    assert M.CrossingRecords(dg).mode() == M.CrossingRecords.MODE_FILTER
    m2, c2, d2 = _run(dg, 2, IDEAL)
    m1, c1, d1 = _run(dg, 1, IDEAL)
    m0, c0, d0 = _run(dg, 0, IDEAL)
    assert (m0, m1, m2) == (0, 1, 2)
    assert c2 == c0 == c1
    # modes differ only in the order uncertain pairs are accumulated
    assert abs(d2 - d0) <= 1e-12 * max(abs(d0), 1e-300)
    assert abs(d1 - d0) <= 1e-12 * max(abs(d0), 1e-300)
    cw, dw = S.crossing_scan(g.xy, g.edges, IDEAL)
    assert c2 == cw
    assert strict_close(d2, dw)
    # count-only instantiation
    _, c2n, _ = _run(dg, 2, None)
    assert c2n == cw


def lattice_local(seed=10, side=120):
    """Jittered unit lattice with nearest-neighbour edges (C4-like): after
    the Morton sort the culled units are spatially local, so the per-unit
    certification threshold drops far below 1."""
    rng = np.random.default_rng(seed)
    gx, gy = np.meshgrid(np.arange(side, dtype=np.float64), np.arange(side, dtype=np.float64))
    xy = np.stack([gx.ravel(), gy.ravel()], 1) + rng.uniform(-1e-3, 1e-3, (side * side, 2))
    idx = np.arange(side * side).reshape(side, side)
    pairs = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                            np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1),
                            np.stack([idx[:-1, :-1].ravel(), idx[1:, 1:].ravel()], 1),
                            np.stack([idx[:-1, 1:].ravel(), idx[1:, :-1].ravel()], 1)])
    return xy, pairs


@pytest.mark.parametrize("name", sorted(CASES) + ["lattice_local"])
def test_filter_culled_units_agree_with_oracle(gpu, name):
    """Culled (Morton-ordered, spatially local) units use tightened per-unit
    thresholds: mode 2 must still equal mode 0 and the oracle."""
    from oracle import sweep as S
    from paper_2411_09809_b200 import metrics as M

    builder = CASES.get(name) or lattice_local
    g = _graph(*builder())
    dg = M.DeviceGraph.from_graph(g)
    res = {}
    for mode in (2, 0):
        rec = M.CrossingRecords(dg, "culled")
        rec.set_mode(mode)
        res[mode] = rec.partial(IDEAL, 0, rec.units).tolist()
    cw, dw = S.crossing_scan(g.xy, g.edges, IDEAL)
    assert int(res[2][0]) == int(res[0][0]) == cw
    assert strict_close(res[2][1], dw) and strict_close(res[0][1], dw)


@pytest.mark.parametrize("name", ["near_collinear", "hubs", "exact_lattice"])
def test_filter_unit_partials_and_shards(gpu, name):
    from paper_2411_09809_b200 import metrics as M

    g = _graph(*CASES[name]())
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg)
    whole = rec.partial(IDEAL, 0, rec.units).tolist()
    U = rec.units
    cuts = [0, U // 3, U // 2, U]
    parts = [rec.partial(IDEAL, a, b).tolist() for a, b in zip(cuts, cuts[1:])]
    assert sum(int(p[0]) for p in parts) == int(whole[0])
    assert strict_close(sum(p[1] for p in parts), whole[1])
    shares = [rec.partial_interleaved(IDEAL, r, 3).tolist() for r in range(3)]
    assert sum(int(p[0]) for p in shares) == int(whole[0])
    assert strict_close(sum(p[1] for p in shares), whole[1])


def test_set_mode_outside_fast_window_degrades(gpu):
    from paper_2411_09809_b200 import metrics as M

    rng = np.random.default_rng(9)
    xy = rng.uniform(0, 1, (300, 2)) * 2.0 ** 600  # outside [2^-160, 2^500]
    g = _graph(xy, _random_pairs(rng, 300, 600))
    rec = M.CrossingRecords(M.DeviceGraph.from_graph(g))
    assert rec.mode() == 0
    assert rec.set_mode(2).mode() == 0
    with pytest.raises(Exception):
        rec.set_mode(3)


def uniform_long(seed=11, n=6000, m=24000):
    """Long random edges in the unit square (C5-like mix, ~100 tiles): after
    a theta sort almost every off-diagonal unit is one shift class."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, (n, 2)), _random_pairs(rng, n, m)


@pytest.mark.parametrize("name", ["uniform_long", "lattice_c5_like", "near_collinear", "hubs",
                                  "exact_lattice"])
def test_theta_order_shift_classes(gpu, name):
    """Dense records over theta-ordered edges (glr_theta_sort_edges) evaluate
    the deviation as |theta_j - (theta_i + s)| in classified units
    (crossing.cu unit_shift).  Ascending order exercises the s = ideal and
    s = pi - ideal classes, a host-side descending order the s = -ideal and
    s = ideal - pi classes; several ideal angles move the class borders.
    Counts must equal the oracle's exactly, dev_sum within 1e-9."""
    import torch

    from oracle import sweep as S
    from paper_2411_09809_b200 import metrics as M

    g = _graph(*(CASES.get(name) or uniform_long)())
    th = np.mod(np.arctan2(g.xy[g.edges[:, 1], 1] - g.xy[g.edges[:, 0], 1],
                           g.xy[g.edges[:, 1], 0] - g.xy[g.edges[:, 0], 0]), np.pi)
    desc = g.edges[np.argsort(-th, kind="stable")]
    dg = M.DeviceGraph.from_graph(g)
    dd = M.DeviceGraph(dg.xy, torch.as_tensor(desc, device=dg.xy.device))
    for ideal in (0.1, 1.0, IDEAL, 1.3, math.pi / 2):
        cw, dw = S.crossing_scan(g.xy, g.edges, ideal)
        asc = M.CrossingRecords(dg, "dense", "theta")
        c, d = asc.partial(ideal, 0, asc.units).tolist()
        assert int(c) == cw and strict_close(d, dw), (name, ideal, "ascending")
        rd = M.CrossingRecords(dd, "dense", "input")
        c, d = rd.partial(ideal, 0, rd.units).tolist()
        assert int(c) == cw and strict_close(d, dw), (name, ideal, "descending")
        # interleaved shards of the theta-ordered records sum to the whole
        parts = [asc.partial_interleaved(ideal, r, 3).tolist() for r in range(3)]
        assert sum(int(p[0]) for p in parts) == cw
        assert strict_close(sum(p[1] for p in parts), dw)
    assert M._crossing_scan(g, IDEAL)[0] == S.crossing_scan(g.xy, g.edges, IDEAL)[0]


def star_graphs(seed=12):
    """Hubs only: one star (every pair shares the centre: E_c = 0, E_ca = 1)
    and two interleaved stars whose spokes cross each other."""
    rng = np.random.default_rng(seed)
    n = 3000
    xy = rng.uniform(0, 1, (n, 2))
    one = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1)
    two = np.concatenate([np.stack([np.zeros(1499, np.int64), np.arange(2, 1501)], 1),
                          np.stack([np.ones(1499, np.int64), np.arange(1501, 3000)], 1)])
    return (xy, one), (xy, two)


@pytest.mark.parametrize("which", [0, 1])
def test_star_tiles_skip_exactly(gpu, which):
    """Units of two star tiles of one vertex are skipped (crossing.cu
    TileBox.star): dense input order, direction order with hub groups
    (2,999 spokes > the hub degree) and the culled plan all equal the
    oracle."""
    from oracle import sweep as S
    from paper_2411_09809_b200 import metrics as M

    g = _graph(*star_graphs()[which])
    dg = M.DeviceGraph.from_graph(g)
    cw, dw = S.crossing_scan(g.xy, g.edges, IDEAL)
    if which == 0:
        assert cw == 0
    for strategy, order in (("dense", "input"), ("dense", "theta"), ("culled", "input")):
        rec = M.CrossingRecords(dg, strategy, order)
        c, d = rec.partial(IDEAL, 0, rec.units).tolist()
        assert int(c) == cw and strict_close(d, dw), (strategy, order)
        c0, _ = rec.partial(None, 0, rec.units).tolist()
        assert int(c0) == cw
    assert M.edge_crossing_angle(g, IDEAL) == pytest.approx(
        1.0 if cw == 0 else 1.0 - (dw / IDEAL) / cw, rel=1e-9)


@pytest.mark.parametrize("strategy,order", [("dense", "theta"), ("dense", "input"),
                                            ("culled", "input")])
def test_repeatable_bit_for_bit(gpu, strategy, order):
    """Slices go to warps dynamically and uncertain pairs are queued per warp,
    yet count and dev_sum are identical bit for bit across runs (integer
    counts, per-slice 2^-50 fixed-point angle sums, queue order fixed by the
    slice)."""
    from paper_2411_09809_b200 import metrics as M

    g = _graph(*uniform_long(seed=13, n=5000, m=30000))
    dg = M.DeviceGraph.from_graph(g)
    runs = []
    for _ in range(3):
        rec = M.CrossingRecords(dg, strategy, order)
        runs.append(tuple(rec.partial(IDEAL, 0, rec.units).tolist()))
    assert runs[0] == runs[1] == runs[2], runs


@pytest.mark.parametrize("hub", [1, 2, 64, 10**9])
def test_theta_order_hub_degree_is_only_an_order(gpu, hub, monkeypatch):
    """glr_theta_sort_edges' hub groups (every edge grouped by its
    higher-degree endpoint at hub degree 1, none at 10^9) change the edge
    order only: counts exact and dev_sum within 1e-9 of the oracle."""
    from oracle import sweep as S
    from paper_2411_09809_b200 import metrics as M

    monkeypatch.setattr(M, "HUB_DEGREE", hub)
    g = _graph(*hubs())
    dg = M.DeviceGraph.from_graph(g)
    cw, dw = S.crossing_scan(g.xy, g.edges, IDEAL)
    rec = M.CrossingRecords(dg, "dense", "theta")
    c, d = rec.partial(IDEAL, 0, rec.units).tolist()
    assert int(c) == cw and strict_close(d, dw)
