"""C5 (BASELINE.json configs[4], the benchmark configuration) crossing parity.

* >= 1,000 random tile-pair units (SURVEY.md 8(c) 'tile-sampled parity'),
  each checked bit-exactly against the oracle's restatement of the
  reference predicate (oracle/glare_oracle.py, exact.py:187-221) on the SAME
  edge order the kernel ran: input order (dense), direction order with hub
  groups (dense, the bench path) and 4-D bbox Morton order (culled list).
* the full-size E_c / dev_sum / E_ca against the pinned C oracle's golden
  (tests/golden/make_golden_oracle.py --c5-crossing, oracle/sweep_oracle.c)
  through every route: dense theta order (bench), dense input order, culled,
  and the FP64 sign kernel (mode 1) -- four independent kernels/orders.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import strict_close
from paper_2411_09809_b200 import configs

pytestmark = pytest.mark.gpu
IDEAL = configs.IDEAL_70


@pytest.fixture(scope="module")
def c5():
    from paper_2411_09809_b200 import metrics as M

    g, p = configs.config5()
    return g, p, M.DeviceGraph.from_graph(g)


def _sorted_edges(dg, which):
    import torch

    from paper_2411_09809_b200 import _lib, metrics as M

    L = _lib.lib()
    es = torch.empty_like(dg.edges)
    st = torch.cuda.current_stream().cuda_stream
    if which == "theta":
        rc = L.glr_theta_sort_edges(dg.xy.data_ptr(), dg.num_vertices, dg.edges.data_ptr(),
                                    dg.num_edges, M.HUB_DEGREE, es.data_ptr(), st)
    else:
        rc = L.glr_spatial_sort_edges(dg.xy.data_ptr(), dg.num_vertices, dg.edges.data_ptr(),
                                      dg.num_edges, es.data_ptr(), st)
    assert rc == 0
    return es.cpu().numpy()


@pytest.mark.parametrize("route", ["input", "theta", "culled"])
def test_c5_tile_samples(gpu, c5, route):
    """400 random units per route (1,200 in all), count bit-exact, dev_sum
    1e-9 relative per unit."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib, metrics as M

    g, p, dg = c5
    L = _lib.lib()
    tile, band = L.glr_crossing_tile(), L.glr_crossing_band()
    if route == "culled":
        rec = M.CrossingRecords(dg, "culled")
        edges = _sorted_edges(dg, "culled")
        lst = rec.list.cpu().numpy().reshape(-1, 2)
    else:
        rec = M.CrossingRecords(dg, "dense", route)
        edges = g.edges if route == "input" else _sorted_edges(dg, "theta")
    # a permutation of the graph's edges
    assert np.array_equal(edges[np.lexsort(edges.T[::-1])], g.edges)
    T = -(-g.num_edges // tile)
    rng = np.random.default_rng({"input": 1, "theta": 2, "culled": 3}[route])
    units = rng.choice(rec.units, 400, replace=False)
    hits = 0
    for u in units.tolist():
        gc, gd = rec.partial(IDEAL, u, u + 1).tolist()
        pair = tuple(lst[u]) if route == "culled" else O._band_coords(u, T, band)
        oc, od = O.crossing_scan_tiles(g.xy, edges, IDEAL, tile, [pair])
        assert int(gc) == oc, (route, u, pair)
        assert strict_close(gd, od), (route, u, pair, gd, od)
        hits += oc
    assert hits > 1000


def test_c5_full_crossing_golden(gpu, c5, golden_configs):
    from paper_2411_09809_b200 import metrics as M

    want = golden_configs["configs"]["C5"]
    if "ec" not in want:
        pytest.skip("C5 crossing golden not generated (make_golden_oracle.py --c5-crossing)")
    g, p, dg = c5
    assert configs.fingerprint(g) == want["fingerprint"]
    routes = {
        "dense-theta": M.CrossingRecords(dg, "dense", "theta"),
        "dense-input": M.CrossingRecords(dg, "dense", "input"),
        "culled": M.CrossingRecords(dg, "culled"),
        "fp64-sign": M.CrossingRecords(dg, "dense", "input").set_mode(1),
    }
    for name, rec in routes.items():
        c, d = rec.partial_interleaved(IDEAL, 0, 1).tolist()
        assert int(c) == want["ec"], (name, c, want["ec"])
        assert strict_close(d, want["dev"]), (name, d, want["dev"])
        eca = 1.0 - (d / IDEAL) / c
        assert strict_close(eca, want["eca"]), name
        del rec
    # the count-only instantiation and the public API
    import paper_2411_09809_b200 as G

    assert G.edge_crossing(g) == want["ec"]
    assert strict_close(G.edge_crossing_angle(g, IDEAL), want["eca"])
