"""Culled variants (Morton order + candidate tile pairs) give exactly the
dense results."""

from __future__ import annotations

import math

import numpy as np
import pytest

import cases
from conftest import graph_from, strict_close
from paper_2411_09809_b200 import configs

pytestmark = pytest.mark.gpu
IDEAL = 7.0 * math.pi / 18.0


def _both(g, r):
    import paper_2411_09809_b200 as G
    from paper_2411_09809_b200 import metrics as M

    out = {}
    for s in ("dense", "culled"):
        out[s] = (M._crossing_scan(g, IDEAL, strategy=s), M.node_occlusion(g, r, strategy=s))
    return out


@pytest.mark.parametrize("name", sorted(cases.ADVERSARIAL_ARRAYS))
def test_adversarial_culled_equals_dense(gpu, golden_small, name):
    want = golden_small["adversarial"][name]
    g = graph_from(cases.ADVERSARIAL_ARRAYS[name])
    res = _both(g, want["radius"])
    for s in ("dense", "culled"):
        (c, d), nc = res[s]
        assert c == want["ec"], s
        assert strict_close(d, want["dev"]), s
        assert nc == want["nc"], s


def test_criterion1_culled(gpu, golden_small):
    from paper_2411_09809_b200 import metrics as M
    from paper_2411_09809_b200.model import LayoutGraph

    rng = np.random.default_rng(42)
    for i, want in enumerate(golden_small["criterion1"][:60]):
        ids, xy, edges = cases.criterion1_case(i, rng)
        g = LayoutGraph(ids, xy, edges)
        c, d = M._crossing_scan(g, IDEAL, strategy="culled")
        assert c == want["ec"] and strict_close(d, want["dev"])
        assert M.node_occlusion(g, want["radius"], strategy="culled") == want["nc"]


def test_c3_culled_matches_reference(gpu, golden_configs):
    from paper_2411_09809_b200 import metrics as M

    g, p = configs.config3()
    want = golden_configs["configs"]["C3"]
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg, "auto")
    assert rec.culled and rec.units < 0.01 * M.crossing_units(g.num_edges)
    c, d = rec.partial(IDEAL, 0, rec.units).tolist()
    assert c == want["ec"] and strict_close(d, want["dev"])
    plan = M.OcclusionPlan(dg, p["radius"], "auto")
    assert plan.culled
    assert plan.partial(0, plan.units).item() == want["nc"]


def test_c4_small_culled(gpu, golden_configs):
    import paper_2411_09809_b200 as G

    g, p = configs.config4(R=316)
    want = golden_configs["configs"]["C4_R316"]
    assert G.edge_crossing(g, strategy="culled") == want["ec"] == 0
    assert G.edge_crossing_angle(g, strategy="culled") == 1.0
    assert G.node_occlusion(g, p["radius"], strategy="culled") == want["nc"]


def test_culled_unit_ranges_sum(gpu):
    """Sharding a candidate list: disjoint list ranges sum exactly, including
    the adjacency correction assigned by tile-pair key."""
    from paper_2411_09809_b200 import metrics as M
    from paper_2411_09809_b200 import sharding

    g, _ = configs.config3()
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg, "culled")
    full = rec.partial(IDEAL, 0, rec.units).tolist()
    for world in (2, 3, 8):
        parts = [rec.partial(IDEAL, *sharding.shard_range(rec.units, r, world)).tolist()
                 for r in range(world)]
        assert sum(p[0] for p in parts) == full[0]
        assert strict_close(sum(p[1] for p in parts), full[1])
    plan = M.OcclusionPlan(dg, 2.5e-4, "culled")
    whole = plan.partial(0, plan.units).item()
    assert sum(plan.partial(*sharding.shard_range(plan.units, r, 4)).item()
               for r in range(4)) == whole


def test_strategy_validation(gpu):
    import paper_2411_09809_b200 as G

    with pytest.raises(G.ParameterError):
        G.edge_crossing(graph_from(cases.x_graph), strategy="fast")
