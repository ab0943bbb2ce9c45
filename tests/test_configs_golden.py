"""Config generators reproduce the inputs the golden values were taken on,
and the oracle reproduces the reference's config-scale values.

golden.json holds the reference's own outputs on C1, C2, C3 and C4 at 1/10
scale (tests/golden/make_golden.py --configs).  C3's golden was produced
with the reference's _crossing_scan (72 s) and its exact grid occlusion.
"""

from __future__ import annotations

import pytest

from conftest import strict_close
from oracle import glare_oracle as O
from oracle import sweep as S
from paper_2411_09809_b200 import configs
from paper_2411_09809_b200.configs import fingerprint, verify_contract

IDEAL = configs.IDEAL_70


def test_c1_matches_reference(golden_configs):
    g, p = configs.config1()
    want = golden_configs["configs"]["C1"]
    verify_contract(g)
    assert fingerprint(g) == want["fingerprint"]
    assert O.node_occlusion(g.xy, p["radius"]) == want["nc"] == 159
    c, d = S.crossing_scan(g.xy, g.edges, IDEAL)
    assert c == want["ec"] == 2965010
    assert strict_close(d, want["dev"])
    assert strict_close(O.minimum_angle(g.xy, g.edges), want["ma"])
    assert strict_close(O.edge_length_variation(g.xy, g.edges), want["ml"])


def test_c2_matches_reference(golden_configs):
    g, p = configs.config2()
    want = golden_configs["configs"]["C2"]
    verify_contract(g)
    assert fingerprint(g) == want["fingerprint"]
    c, d = S.crossing_scan(g.xy, g.edges, IDEAL)
    assert c == want["ec"]
    assert strict_close(d, want["dev"])
    assert S.node_occlusion(g.xy, p["radius"]) == want["nc"]
    assert strict_close(O.minimum_angle(g.xy, g.edges), want["ma"])
    assert strict_close(O.edge_length_variation(g.xy, g.edges), want["ml"])


def test_c4_small_matches_reference(golden_configs):
    g, p = configs.config4(R=316)
    want = golden_configs["configs"]["C4_R316"]
    verify_contract(g)
    assert g.num_edges == 315 * (3 * 316 - 1)
    assert fingerprint(g) == want["fingerprint"]
    assert want["ec"] == 0 and want["nc"] == 0
    assert S.crossing_scan(g.xy, g.edges, None)[0] == 0
    assert strict_close(O.minimum_angle(g.xy, g.edges), want["ma"])
    assert strict_close(O.edge_length_variation(g.xy, g.edges), want["ml"])


@pytest.mark.slow
def test_c3_matches_reference(golden_configs):
    g, p = configs.config3()
    want = golden_configs["configs"]["C3"]
    verify_contract(g)
    assert fingerprint(g) == want["fingerprint"]
    c, d = S.crossing_scan(g.xy, g.edges, IDEAL)
    assert c == want["ec"]
    assert strict_close(d, want["dev"])
    assert O.node_occlusion_grid(g.xy, p["radius"]) == want["nc"]


def test_c4_c5_shapes():
    """Full-size generators hit the BASELINE.json sizes (cheap checks)."""
    xy, e = configs.triangular_lattice(40)
    assert len(e) == 39 * (3 * 40 - 1)
    g, p = configs.config5(n=20_000, m=50_000)
    verify_contract(g)
    assert g.num_edges == 50_000
