"""GPU parity of M_a's hand-written per-vertex segmented sort
(csrc/length_angle.cu: warp class deg <= 32, block class <= 4096, hub class
above) against the pinned oracle (oracle/glare_oracle.py:91-116, the
restatement of exact.py:88-124).

The sort only permutes values, so every d_v equals the reference's up to the
atan2 ulp; M_a is held to 1e-9 relative.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import strict_close

pytestmark = pytest.mark.gpu


def _star(d: int, rng, side: int, ties: bool):
    """Hub 0 at the centre of a side x side integer lattice, d distinct
    leaves; with ties, leaves are drawn on a few rays so many incident angles
    coincide exactly (gap 0) or differ by one lattice step."""
    c = side // 2
    pts = set()
    out = []
    while len(out) < d:
        if ties and rng.random() < 0.7:
            dx, dy = [(1, 0), (0, 1), (1, 1), (-2, 1), (3, -1)][int(rng.integers(0, 5))]
            k = int(rng.integers(1, side // 4))
            p = (c + dx * k, c + dy * k)
        else:
            p = (int(rng.integers(0, side)), int(rng.integers(0, side)))
        if p != (c, c) and p not in pts:
            pts.add(p)
            out.append(p)
    xy = np.array([(c, c)] + out, dtype=np.float64)
    edges = np.stack([np.zeros(d, np.int64), np.arange(1, d + 1)], axis=1)
    return xy, edges


@pytest.mark.parametrize("d", [1, 2, 3, 7, 8, 9, 31, 32, 33, 64, 255, 1000, 4095, 4096, 4097,
                               8191, 8192, 8193, 12289, 54873])
@pytest.mark.parametrize("ties", [False, True])
def test_star_size_classes(gpu, d, ties):
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G

    rng = np.random.default_rng(d * 2 + int(ties))
    xy, edges = _star(d, rng, 1 << 12, ties)
    g = G.LayoutGraph(np.arange(len(xy)), xy, edges)
    got, want = G.minimum_angle(g), O.minimum_angle(g.xy, g.edges)
    assert strict_close(got, want), (d, ties, got, want)


def test_hub_alone_matches_reference_formula(gpu):
    """One hub whose d_v dominates: with every leaf of degree 1, M_a is a
    closed form of the hub's min gap, so a wrong hub sort moves it visibly."""
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G

    rng = np.random.default_rng(7)
    d = 20000
    theta = np.sort(rng.uniform(0, 2 * np.pi, d))
    xy = np.concatenate([[[0.0, 0.0]], np.stack([np.cos(theta), np.sin(theta)], 1) * 1e3])
    perm = rng.permutation(d)  # scatter order unrelated to angle order
    edges = np.stack([np.zeros(d, np.int64), perm + 1], axis=1)
    g = G.LayoutGraph(np.arange(d + 1), xy, edges)
    dev = O.vertex_angle_deviations(g.xy, g.edges)
    assert strict_close(G.minimum_angle(g), 1.0 - float(np.mean(dev)))


def test_many_hubs_chung_lu(gpu):
    """C5-shaped degrees (Chung-Lu, gamma 2.3) at 1/20 size: every class at
    once, hubs of several thousand, on the integer lattice (exact ties)."""
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G
    from paper_2411_09809_b200 import configs

    g, _ = configs.config5(seed=3, n=75_000, m=200_000)
    deg = np.bincount(g.edges.ravel(), minlength=g.num_vertices)
    assert deg.max() > 4096 and (deg > 32).sum() > 10
    assert strict_close(G.minimum_angle(g), O.minimum_angle(g.xy, g.edges))


def test_mixed_degrees_random(gpu):
    """Random graphs whose vertices land in all three classes, plus isolated
    vertices (ignored by the mean, exact.py:115-124)."""
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G

    rng = np.random.default_rng(11)
    for trial in range(6):
        n = int(rng.integers(5000, 20000))
        hubs = rng.integers(0, n, 8)
        a = np.concatenate([rng.integers(0, n, 30000), np.repeat(hubs, int(rng.integers(40, 6000)))])
        b = rng.integers(0, n, len(a))
        keep = a != b
        xy = rng.integers(0, 1 << 10, (n, 2)).astype(np.float64)
        keep &= np.any(xy[a] != xy[b], axis=1)
        g = G.LayoutGraph(np.arange(n), xy, np.stack([a[keep], b[keep]], 1))
        assert strict_close(G.minimum_angle(g), O.minimum_angle(g.xy, g.edges)), trial
