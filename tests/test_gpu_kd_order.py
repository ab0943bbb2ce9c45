"""k-d edge order of the culled plan for long edges (spatial.cu kd_sort,
behind glr_spatial_sort_edges).  The order may only permute rows -- the
reference visits every unordered pair once whatever the order
(exact.py:145-222) -- so the checks are: the output is a row permutation,
deterministic; tiles, slices and quarters are k-d cells (tighter than the
Morton order's); the plans built on it give the oracle's results."""

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


def uniform(seed, n, m):
    rng = np.random.default_rng(seed)
    return _graph(rng.random((n, 2)), rng.integers(0, n, (m, 2)))


def hubs(seed=4, n=30000, m=90000):
    """A few vertices above the culled order's hub degree (16,384)."""
    rng = np.random.default_rng(seed)
    xy = rng.integers(0, 2 ** 16, (n, 2)).astype(np.float64)
    a = rng.integers(0, n, m)
    b = rng.integers(0, n, m)
    a[:20000] = 7
    a[20000:38000] = 11
    return _graph(xy, np.stack([a, b], 1))


def flat_axis(seed=5, n=4000, m=9000):
    """All P.x equal to all Q.x within two columns: two coordinates carry no
    extent, and many coordinates tie."""
    rng = np.random.default_rng(seed)
    xy = np.stack([np.repeat([0.0, 1000.0], n // 2), rng.integers(0, 500, n).astype(np.float64)], 1)
    a = rng.integers(0, n // 2, m)
    b = rng.integers(n // 2, n, m)
    return _graph(xy, np.stack([a, b], 1))


GRAPHS = {
    "uniform_ragged": lambda: uniform(0, 5000, 20011),   # m not a multiple of 64
    "uniform_small": lambda: uniform(1, 200, 150),       # less than one tile
    "one_leaf": lambda: uniform(2, 40, 50),              # less than one quarter
    "hubs": hubs,
    "flat_axis": flat_axis,
}


def _sort(dg, kd):
    import torch

    from paper_2411_09809_b200 import _lib

    L = _lib.lib()
    was = L.glr_spatial_set_kd(2 if kd else 0)
    try:
        es = torch.empty_like(dg.edges)
        rc = L.glr_spatial_sort_edges(dg.xy.data_ptr(), dg.num_vertices, dg.edges.data_ptr(),
                                      dg.num_edges, es.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream)
        assert rc == 0, _lib.last_error()
        return es.cpu().numpy()
    finally:
        L.glr_spatial_set_kd(was)


def _pq(xy, e):
    a, b = xy[e[:, 0]], xy[e[:, 1]]
    pa = (a[:, 0] < b[:, 0]) | ((a[:, 0] == b[:, 0]) & (a[:, 1] <= b[:, 1]))
    return np.concatenate([np.where(pa[:, None], a, b), np.where(pa[:, None], b, a)], 1)


def _block_extent(c, block):
    """Sum over aligned blocks of the four coordinate extents."""
    tot = 0.0
    for s in range(0, len(c), block):
        blk = c[s:s + block]
        tot += float((blk.max(0) - blk.min(0)).sum())
    return tot


@pytest.fixture(scope="module", params=sorted(GRAPHS))
def case(request):
    from paper_2411_09809_b200 import metrics as M

    g = GRAPHS[request.param]()
    dg = M.DeviceGraph.from_graph(g)
    return request.param, g, dg


def test_kd_order_is_a_row_permutation(case):
    name, g, dg = case
    es = _sort(dg, True)
    assert es.shape == g.edges.shape
    key = lambda e: np.sort(e[:, 0] * (g.num_vertices + 1) + e[:, 1])  # noqa: E731
    assert np.array_equal(key(es), key(g.edges)), name
    assert np.array_equal(es, _sort(dg, True)), "not deterministic"


def test_kd_cells_are_tighter_than_morton(case):
    """Tiles (256), slices (128) and quarters (64) of the k-d order have
    smaller boxes in total than the Morton order's."""
    name, g, dg = case
    if g.num_edges < 1024:
        pytest.skip("a handful of blocks")
    kd, mo = _pq(g.xy, _sort(dg, True)), _pq(g.xy, _sort(dg, False))
    for block in (256, 128, 64):
        assert _block_extent(kd, block) < _block_extent(mo, block), (name, block)


def test_kd_blocks_keep_one_orientation(case):
    """Below the (hub group, orientation) runs every aligned 64-block holds one
    diagonal orientation, except the blocks a run boundary falls into."""
    name, g, dg = case
    es = _sort(dg, True)
    c = _pq(g.xy, es)
    up = (c[:, 2] - c[:, 0]) * (c[:, 3] - c[:, 1]) >= 0
    mixed = sum(1 for s in range(0, len(up), 64) if up[s:s + 64].min() != up[s:s + 64].max())
    runs = 1 + int(np.count_nonzero(np.diff(up.astype(np.int8))))
    assert mixed <= runs and runs <= 2 * (1 + 8), (name, mixed, runs)


def test_plans_on_kd_order_match_oracle(case):
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib, metrics as M

    name, g, dg = case
    if g.num_edges > 30000:
        from oracle import sweep

        want_c, want_d = sweep.crossing_scan(g.xy, g.edges, IDEAL)
    else:
        want_c, want_d = O.crossing_scan(g.xy, g.edges, IDEAL)
    L = _lib.lib()
    for kd in (2, 0):
        was = L.glr_spatial_set_kd(kd)
        try:
            rec = M.CrossingRecords(dg, "culled")
            c, d = rec.partial_interleaved(IDEAL, 0, 1).tolist()
            c0 = rec.partial_interleaved(None, 0, 1)[0].item()
        finally:
            L.glr_spatial_set_kd(was)
        assert int(c) == want_c == int(c0) and strict_close(d, want_d), (name, kd, c, want_c)


def test_kd_beats_morton_on_classification():
    """Long random edges at tile scale: fewer mixed units with the k-d order."""
    from paper_2411_09809_b200 import _lib, metrics as M

    g = uniform(9, 40000, 120000)
    dg = M.DeviceGraph.from_graph(g)
    L = _lib.lib()
    mixed = {}
    for kd in (2, 0):
        was = L.glr_spatial_set_kd(kd)
        try:
            rec = M.CrossingRecords(dg, "culled")
            mixed[kd] = rec.n_mixed
            res = rec.partial_interleaved(IDEAL, 0, 1).tolist()
        finally:
            L.glr_spatial_set_kd(was)
        mixed[("res", kd)] = res
    assert mixed[2] < mixed[0], mixed
    assert mixed[("res", 2)][0] == mixed[("res", 0)][0]
    assert strict_close(mixed[("res", 2)][1], mixed[("res", 0)][1])


def test_kd_default_threshold():
    """Default setting: the tree is built from 131,072 edges on (the Morton
    order below), and the knob reports its previous value."""
    from paper_2411_09809_b200 import _lib, metrics as M

    L = _lib.lib()
    assert L.glr_spatial_set_kd(-1) == 1
    small = M.DeviceGraph.from_graph(uniform(11, 3000, 20000))
    big = M.DeviceGraph.from_graph(uniform(12, 60000, 140000))
    import torch

    def default_sort(dg):
        es = torch.empty_like(dg.edges)
        assert L.glr_spatial_sort_edges(dg.xy.data_ptr(), dg.num_vertices, dg.edges.data_ptr(),
                                        dg.num_edges, es.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream) == 0
        return es.cpu().numpy()

    assert np.array_equal(default_sort(small), _sort(small, False))
    assert np.array_equal(default_sort(big), _sort(big, True))
    assert not np.array_equal(default_sort(big), _sort(big, False))
