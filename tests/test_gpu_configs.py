"""Config-scale GPU parity (BASELINE.json configs), against golden values from
the reference (C1, C2, C3, C4 at 1/10 scale) and the C oracle."""

from __future__ import annotations

import pytest

from conftest import strict_close
from paper_2411_09809_b200 import configs

pytestmark = pytest.mark.gpu
IDEAL = configs.IDEAL_70


def _all(g, p):
    import paper_2411_09809_b200 as G

    c, d = G._crossing_scan(g, IDEAL)
    return {"nc": G.node_occlusion(g, p["radius"]), "ma": G.minimum_angle(g),
            "ml": G.edge_length_variation(g), "ec": c, "dev": d,
            "eca": G.edge_crossing_angle(g, IDEAL)}


@pytest.mark.parametrize("key,builder", [("C1", configs.config1), ("C2", configs.config2),
                                         ("C4_R316", lambda: configs.config4(R=316))])
def test_config_golden(gpu, golden_configs, key, builder):
    g, p = builder()
    want = golden_configs["configs"][key]
    assert configs.fingerprint(g) == want["fingerprint"]
    got = _all(g, p)
    assert got["nc"] == want["nc"]
    assert got["ec"] == want["ec"]
    for k in ("dev", "ma", "ml", "eca"):
        assert strict_close(got[k], want[k]), (k, got[k], want[k])


def test_config3_golden(gpu, golden_configs):
    import paper_2411_09809_b200 as G

    g, p = configs.config3()
    want = golden_configs["configs"]["C3"]
    assert configs.fingerprint(g) == want["fingerprint"]
    c, d = G._crossing_scan(g, IDEAL)
    assert c == want["ec"]
    assert strict_close(d, want["dev"])
    assert G.node_occlusion(g, p["radius"]) == want["nc"]


def test_config4_full(gpu, golden_configs):
    """C4 at full size (1M vertices, 2,996,001 edges) against the pinned
    oracle: E_c = 0 (shared-endpoint exclusion on a mesh), N_c, M_a, M_l."""
    import paper_2411_09809_b200 as G

    g, p = configs.config4()
    want = golden_configs["configs"]["C4"]
    assert configs.fingerprint(g) == want["fingerprint"]
    c, d = G._crossing_scan(g, IDEAL)
    assert (c, d) == (want["ec"], want["dev"]) == (0, 0.0)
    assert G.edge_crossing_angle(g, IDEAL) == 1.0
    assert G.node_occlusion(g, p["radius"]) == want["nc"]
    assert strict_close(G.minimum_angle(g), want["ma"])
    assert strict_close(G.edge_length_variation(g), want["ml"])


def test_config5_occlusion_and_tile_samples(gpu, golden_configs):
    """C5: N_c against the pinned oracle; E_c/E_ca on 24 random tile-pair
    units checked bit-exactly against the oracle's unit restatement
    (SURVEY.md 8(c) 'tile-sampled parity'), and 3 random 30k-edge subgraphs
    against the C oracle."""
    import numpy as np

    import paper_2411_09809_b200 as G
    from oracle import glare_oracle as O
    from oracle import sweep as S
    from paper_2411_09809_b200 import metrics as M

    g, p = configs.config5()
    want = golden_configs["configs"]["C5"]
    assert configs.fingerprint(g) == want["fingerprint"]
    assert G.node_occlusion(g, p["radius"]) == want["nc"]
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg, "dense")
    tile = M._lib.lib().glr_crossing_tile()
    rng = np.random.default_rng(2024)
    for u in rng.integers(0, rec.units, 24).tolist():
        gc, gd = rec.partial(IDEAL, u, u + 1).tolist()
        oc, od = O.crossing_scan_units(g.xy, g.edges, IDEAL, tile, u, u + 1,
                                       band=M._lib.lib().glr_crossing_band())
        assert gc == oc
        assert strict_close(gd, od, floor=1e-9)
    for seed in range(3):
        sub = np.sort(np.random.default_rng(seed).choice(g.num_edges, 30_000, replace=False))
        e = g.edges[sub]
        sg = G.LayoutGraph.from_normalized(g.xy, e)
        c, d = G._crossing_scan(sg, IDEAL)
        oc, od = S.crossing_scan(g.xy, e, IDEAL)
        assert c == oc and strict_close(d, od)


@pytest.mark.slow
def test_config5_dense_equals_culled(gpu):
    """Full C5 E_c/E_ca two independent ways: dense (input order, run reuse)
    and culled (Morton order, candidate list) -- identical counts."""
    from paper_2411_09809_b200 import metrics as M

    g, p = configs.config5()
    dg = M.DeviceGraph.from_graph(g)
    a = M.CrossingRecords(dg, "dense")
    b = M.CrossingRecords(dg, "culled")
    ca, da = a.partial(IDEAL, 0, a.units).tolist()
    cb, db = b.partial(IDEAL, 0, b.units).tolist()
    assert ca == cb
    assert strict_close(da, db)
