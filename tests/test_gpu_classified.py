"""Classified candidate lists (glr_crossing_candidates_classified): units
certified "none" are dropped and units certified "full" are counted without a
per-pair predicate (crossing.cu tile_class_kernel / cross_full_kernel).  The
certificates are checked unit by unit against the oracle, and the plans'
totals against the oracle and the dense pass (exact.py:145-222)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import strict_close

pytestmark = pytest.mark.gpu
IDEAL = 7.0 * math.pi / 18.0


def _graph(xy, pairs):
    from paper_2411_09809_b200.model import LayoutGraph, normalize_edges

    pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
    e, _, _ = normalize_edges(pairs)
    return LayoutGraph.from_normalized(xy, e)


def long_uniform(seed=0, n=3000, m=12000):
    rng = np.random.default_rng(seed)
    return _graph(rng.random((n, 2)), rng.integers(0, n, (m, 2)))


def long_lattice(seed=1, n=3000, m=12000, side=1024):
    """Integer lattice: exact collinear, touching and coincident-endpoint cases."""
    rng = np.random.default_rng(seed)
    return _graph(rng.integers(0, side, (n, 2)).astype(np.float64), rng.integers(0, n, (m, 2)))


def crossing_bundles(seed=2, k=600, touch=True):
    """Two bundles of long edges between small clusters that cross everywhere
    (full units), plus edges whose endpoints lie exactly on a bundle's lines
    (orientation exactly 0: touching counts, so such units must not be
    certified) and a parallel bundle (no crossings: certified none)."""
    rng = np.random.default_rng(seed)
    c = lambda x, y, s=16: np.stack([x + rng.integers(0, s, k), y + rng.integers(0, s, k)], 1)
    pts = [c(0, 0), c(4000, 4000), c(0, 4000), c(4000, 0), c(0, 200), c(4000, 4200)]
    if touch:
        # on the line y = x of bundle 0's main diagonal
        t = rng.integers(1000, 3000, k)
        pts += [np.stack([t, t], 1).astype(np.int64), c(2000, 6000)]
    xy = np.concatenate(pts).astype(np.float64)
    off = np.arange(len(pts)) * k
    idx = np.arange(k)
    pairs = [np.stack([off[0] + idx, off[1] + idx], 1), np.stack([off[2] + idx, off[3] + idx], 1),
             np.stack([off[4] + idx, off[5] + idx], 1)]
    if touch:
        pairs.append(np.stack([off[6] + idx, off[7] + idx], 1))
    # also the exact main diagonal (0, 0)-(4000, 4000)
    xy = np.concatenate([xy, [[0.0, 0.0], [4000.0, 4000.0]]])
    pairs.append(np.array([[len(xy) - 2, len(xy) - 1]]))
    return _graph(xy, np.concatenate(pairs))


def chung_lu_small(seed=3):
    from paper_2411_09809_b200 import configs

    rng = np.random.default_rng(seed)
    xy = rng.integers(0, 2 ** 16, (20000, 2)).astype(np.float64)
    e = configs.chung_lu(20000, 60000, 2.3, rng, xy)
    return _graph(xy, e)


GRAPHS = {"long_uniform": long_uniform, "long_lattice": long_lattice,
          "bundles": crossing_bundles, "chung_lu": chung_lu_small}


def _sorted_edges(dg):
    import torch

    from paper_2411_09809_b200 import _lib

    es = torch.empty_like(dg.edges)
    st = torch.cuda.current_stream().cuda_stream
    rc = _lib.lib().glr_spatial_sort_edges(dg.xy.data_ptr(), dg.num_vertices,
                                           dg.edges.data_ptr(), dg.num_edges, es.data_ptr(), st)
    assert rc == 0
    return es.cpu().numpy()


@pytest.fixture(scope="module", params=sorted(GRAPHS))
def plan(request):
    from paper_2411_09809_b200 import metrics as M

    g = GRAPHS[request.param]()
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg, "culled")
    return request.param, g, dg, rec, _sorted_edges(dg)


def test_classified_totals(plan):
    """Classified culled plan == oracle == dense pass (count exact, dev 1e-9)."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import metrics as M

    name, g, dg, rec, _ = plan
    if g.num_edges > 20000:
        from oracle import sweep  # the C restatement, pinned like the numpy one

        want_c, want_d = sweep.crossing_scan(g.xy, g.edges, IDEAL)
    else:
        want_c, want_d = O.crossing_scan(g.xy, g.edges, IDEAL)
    c, d = rec.partial(IDEAL, 0, rec.units).tolist()
    assert int(c) == want_c and strict_close(d, want_d), (name, c, want_c, d, want_d)
    c0 = rec.partial(None, 0, rec.units)[0].item()
    assert int(c0) == want_c
    dense = M.CrossingRecords(dg, "dense", "theta")
    dc, dd = dense.partial(IDEAL, 0, dense.units).tolist()
    assert int(dc) == want_c and strict_close(dd, want_d)
    if name in ("bundles", "chung_lu"):
        assert rec.n_full > 0, name
    if name == "bundles":
        assert want_c > 0


def test_full_units_cross_everywhere(plan):
    """Every certified full unit: the oracle counts na * nb crossings and the
    same deviation sum."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    tile = _lib.lib().glr_crossing_tile()
    m = len(edges)
    lst = rec.list.cpu().numpy()
    full = lst[rec.n_mixed:]
    rng = np.random.default_rng(5)
    pick = rng.choice(len(full), min(60, len(full)), replace=False) if len(full) else []
    for k in pick:
        ti, tj = (int(v) for v in full[k])
        assert ti < tj
        na = min(tile, m - ti * tile)
        nb = min(tile, m - tj * tile)
        oc, od = O.crossing_scan_tiles(g.xy, edges, IDEAL, tile, [(ti, tj)])
        assert oc == na * nb, (name, ti, tj, oc, na * nb)
        u = rec.n_mixed + int(k)
        gc, gd = rec.partial(IDEAL, u, u + 1).tolist()
        assert int(gc) == oc and strict_close(gd, od, floor=0.0), (name, ti, tj, gd, od)


def test_dropped_units_have_no_crossings(plan):
    """Tile pairs absent from the list (bbox-disjoint or certified none): the
    oracle finds no crossing in them."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    tile = _lib.lib().glr_crossing_tile()
    T = -(-len(edges) // tile)
    kept = {(int(a), int(b)) for a, b in rec.list.cpu().numpy()}
    dropped = [(i, j) for i in range(T) for j in range(i, T) if (i, j) not in kept]
    rng = np.random.default_rng(6)
    pick = rng.choice(len(dropped), min(150, len(dropped)), replace=False) if dropped else []
    for k in pick:
        oc, _ = O.crossing_scan_tiles(g.xy, edges, None, tile, [dropped[k]])
        assert oc == 0, (name, dropped[k])


def test_mixed_units_match_oracle(plan):
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    tile = _lib.lib().glr_crossing_tile()
    lst = rec.list.cpu().numpy()
    rng = np.random.default_rng(7)
    pick = rng.choice(rec.n_mixed, min(40, rec.n_mixed), replace=False)
    for u in pick.tolist():
        oc, od = O.crossing_scan_tiles(g.xy, edges, IDEAL, tile, [tuple(lst[u])])
        gc, gd = rec.partial(IDEAL, u, u + 1).tolist()
        assert int(gc) == oc and strict_close(gd, od), (name, u)


def test_classified_interleaved_ranks_sum(plan):
    """Interleaved ownership over the classified list: ranks' partials sum to
    the whole (both parts are dealt in chunks)."""
    name, g, dg, rec, edges = plan
    c, d = rec.partial(IDEAL, 0, rec.units).tolist()
    for world in (2, 3, 8):
        cs, ds = 0, 0.0
        for r in range(world):
            pc, pd = rec.partial_interleaved(IDEAL, r, world).tolist()
            cs += int(pc)
            ds += pd
        assert cs == int(c) and strict_close(ds, d), (name, world)


def test_classified_abi_ranges(gpu, plan):
    """Arbitrary unit ranges straddling the mixed/full boundary sum exactly;
    out-of-range requests fail with GLR_EARG."""
    import torch

    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    L = _lib.lib()
    U = rec.units
    c, d = rec.partial(IDEAL, 0, U).tolist()
    cuts = sorted({0, U, rec.n_mixed, max(rec.n_mixed - 3, 0), min(rec.n_mixed + 5, U), U // 3})
    cs, ds = 0, 0.0
    for a, b in zip(cuts[:-1], cuts[1:]):
        pc, pd = rec.partial(IDEAL, a, b).tolist()
        cs += int(pc)
        ds += pd
    assert cs == int(c) and strict_close(ds, d)
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    rc = L.glr_crossing_pairs_classified(rec.buf.data_ptr(), rec.n, rec.m, 1, IDEAL,
                                         rec.list.data_ptr(), rec.sub.data_ptr(), rec.n_mixed,
                                         rec.n_full, 0, U + 1, 0, 1, out.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.GLR_EARG


def test_sub_masks_sound(plan):
    """Sub-unit masks: every (warp slice x j-quarter) block marked empty has no
    crossing by the reference predicate, and the plan gives the same result
    with the masks ignored."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    tile = _lib.lib().glr_crossing_tile()
    slice_, quarter = 128, tile // 4
    m = len(edges)
    lst = rec.list.cpu().numpy()[:rec.n_mixed]
    sub = rec.sub.cpu().numpy()[:rec.n_mixed].astype(np.int64) & 0xFFFF
    marked = np.nonzero(sub)[0]
    if name in ("chung_lu",):
        assert len(marked) > 0
    xy = g.xy
    rng = np.random.default_rng(8)
    for u in rng.choice(marked, min(40, len(marked)), replace=False) if len(marked) else []:
        ti, tj = (int(v) for v in lst[u])
        assert ti != tj
        for bit in range(8):
            if not (sub[u] >> bit) & 1:
                continue
            s, q = divmod(bit, 4)
            I = np.arange(ti * tile + s * slice_, min(m, ti * tile + (s + 1) * slice_))
            J = np.arange(tj * tile + q * quarter, min(m, tj * tile + (q + 1) * quarter))
            if len(I) == 0 or len(J) == 0:
                continue
            ii, jj = np.meshgrid(I, J, indexing="ij")
            ii, jj = ii.ravel(), jj.ravel()
            a, b, c, d = xy[edges[ii, 0]], xy[edges[ii, 1]], xy[edges[jj, 0]], xy[edges[jj, 1]]
            hit = O.straddle_mask(a[:, 0], a[:, 1], b[:, 0], b[:, 1], c[:, 0], c[:, 1], d[:, 0],
                                  d[:, 1])
            box = ((np.maximum(c[:, 0], d[:, 0]) >= np.minimum(a[:, 0], b[:, 0]))
                   & (np.maximum(a[:, 0], b[:, 0]) >= np.minimum(c[:, 0], d[:, 0]))
                   & (np.maximum(c[:, 1], d[:, 1]) >= np.minimum(a[:, 1], b[:, 1]))
                   & (np.maximum(a[:, 1], b[:, 1]) >= np.minimum(c[:, 1], d[:, 1])))
            assert not np.any(hit & box), (name, u, bit)
    with_masks = rec.partial(IDEAL, 0, rec.units).tolist()
    rec.use_sub_masks = False
    try:
        without = rec.partial(IDEAL, 0, rec.units).tolist()
    finally:
        rec.use_sub_masks = True
    assert with_masks[0] == without[0] and strict_close(with_masks[1], without[1])


def test_sub_full_blocks_cross_everywhere(plan):
    """Sub-unit masks, upper bits: every (warp slice x j-quarter) block marked
    full has all its pairs crossing by the reference predicate (bboxes
    overlapping, no shared vertex), and a plan restricted to such units gives
    the oracle's count and deviation sum for them."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    L = _lib.lib()
    tile, Q = L.glr_crossing_tile(), L.glr_crossing_sub_quarters()
    slice_, quarter = 128, tile // Q
    nb = (tile // slice_) * Q
    m = len(edges)
    lst = rec.list.cpu().numpy()[:rec.n_mixed]
    sub = rec.sub.cpu().numpy()[:rec.n_mixed].astype(np.int64)
    fullbits = (sub >> nb) & ((1 << nb) - 1)
    assert not np.any(fullbits & sub & ((1 << nb) - 1)), "a block is both empty and full"
    marked = np.nonzero(fullbits)[0]
    if name in ("chung_lu", "bundles"):
        assert len(marked) > 0, name
    xy = g.xy
    rng = np.random.default_rng(9)
    for u in rng.choice(marked, min(30, len(marked)), replace=False) if len(marked) else []:
        ti, tj = (int(v) for v in lst[u])
        assert ti != tj
        for bit in range(nb):
            if not (fullbits[u] >> bit) & 1:
                continue
            s, q = divmod(bit, Q)
            I = np.arange(ti * tile + s * slice_, min(m, ti * tile + (s + 1) * slice_))
            J = np.arange(tj * tile + q * quarter, min(m, tj * tile + (q + 1) * quarter))
            assert len(I) and len(J)
            ii, jj = np.meshgrid(I, J, indexing="ij")
            ii, jj = ii.ravel(), jj.ravel()
            a, b, c, d = xy[edges[ii, 0]], xy[edges[ii, 1]], xy[edges[jj, 0]], xy[edges[jj, 1]]
            hit = O.straddle_mask(a[:, 0], a[:, 1], b[:, 0], b[:, 1], c[:, 0], c[:, 1], d[:, 0],
                                  d[:, 1])
            box = ((np.maximum(c[:, 0], d[:, 0]) >= np.minimum(a[:, 0], b[:, 0]))
                   & (np.maximum(a[:, 0], b[:, 0]) >= np.minimum(c[:, 0], d[:, 0]))
                   & (np.maximum(c[:, 1], d[:, 1]) >= np.minimum(a[:, 1], b[:, 1]))
                   & (np.maximum(a[:, 1], b[:, 1]) >= np.minimum(c[:, 1], d[:, 1])))
            share = ((edges[ii, 0] == edges[jj, 0]) | (edges[ii, 0] == edges[jj, 1])
                     | (edges[ii, 1] == edges[jj, 0]) | (edges[ii, 1] == edges[jj, 1]))
            assert np.all(hit & box & ~share), (name, u, bit)
        # the unit through the kernels (filter on the rest + sub-full blocks)
        oc, od = O.crossing_scan_tiles(g.xy, edges, IDEAL, tile, [(ti, tj)])
        gc, gd = rec.partial(IDEAL, int(u), int(u) + 1).tolist()
        assert int(gc) == oc and strict_close(gd, od), (name, u, gc, oc)
        assert int(rec.partial(None, int(u), int(u) + 1)[0].item()) == oc


def test_row_dealt_plans_partition_the_list(plan):
    """glr_crossing_candidates_rows: the ranks' lists partition the full
    classified list by tile row, each rank's partial equals the oracle's
    share of those rows, and the partials sum to the whole."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib, metrics as M

    name, g, dg, rec, edges = plan
    tile = _lib.lib().glr_crossing_tile()
    whole = rec.partial(IDEAL, 0, rec.units).tolist()
    full_list = {(int(a), int(b)) for a, b in rec.list.cpu().numpy()}
    for world in (2, 3, 8):
        seen = set()
        cs, ds = 0, 0.0
        for r in range(world):
            part = M.CrossingRecords(dg, "culled", rows=(r, world))
            assert part.rows == (r, world)
            lst = {(int(a), int(b)) for a, b in part.list.cpu().numpy()} if part.units else set()
            assert all(a % world == r for a, _ in lst)
            assert not (seen & lst)
            seen |= lst
            pc, pd = part.partial_interleaved(IDEAL, r, world).tolist()
            if g.num_edges <= 20000 and world == 3:
                oc, od = O.crossing_scan_rows(g.xy, edges, IDEAL, tile, r, world)
                assert int(pc) == oc and strict_close(pd, od), (name, world, r)
            cs += int(pc)
            ds += pd
            with pytest.raises(Exception):
                part.partial_interleaved(IDEAL, (r + 1) % world, world)
        assert seen == full_list, (name, world)
        assert cs == int(whole[0]) and strict_close(ds, whole[1]), (name, world)


def test_rows_bad_arguments(gpu, plan):
    """glr_crossing_candidates_rows rejects rank >= world and world < 1."""
    import ctypes

    import torch

    from paper_2411_09809_b200 import _lib

    name, g, dg, rec, edges = plan
    L = _lib.lib()
    counts = (ctypes.c_uint64 * 2)()
    st = torch.cuda.current_stream().cuda_stream
    for rank, world in ((2, 2), (-1, 2), (0, 0)):
        rc = L.glr_crossing_candidates_rows(rec.buf.data_ptr(), rec.n, rec.m, None, None, 0,
                                            counts, rank, world, st)
        assert rc == _lib.GLR_EARG, (rank, world)


@pytest.mark.parametrize("ideal", [2.0 ** -120, 1e-9, math.pi / 2])
def test_classified_extreme_ideal_angles(plan, ideal):
    """Ideal angles at the ends of (0, pi/2]: below 2^-100 the filter kernel
    stands down (the FP64 sign kernel scans the mixed units, masks ignored,
    full blocks not counted apart); at pi/2 three kinks of the deviation
    coincide.  Totals must still equal the oracle's."""
    from oracle import glare_oracle as O

    name, g, dg, rec, _ = plan
    if g.num_edges > 20000:
        from oracle import sweep

        want_c, want_d = sweep.crossing_scan(g.xy, g.edges, ideal)
    else:
        want_c, want_d = O.crossing_scan(g.xy, g.edges, ideal)
    c, d = rec.partial(ideal, 0, rec.units).tolist()
    assert int(c) == want_c and strict_close(d, want_d), (name, ideal, c, want_c, d, want_d)
    parts = [rec.partial_interleaved(ideal, r, 2).tolist() for r in range(2)]
    assert sum(int(p[0]) for p in parts) == want_c
    assert strict_close(sum(p[1] for p in parts), want_d)
