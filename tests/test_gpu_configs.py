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
