"""GPU: the crossing-angle deviation sum (exact.py:219-221) at 1e-9
RELATIVE with no absolute floor, including sums of a few tiny deviations.

The inputs are built so that every axis angle is exactly representable and
numpy's and CUDA's atan2 agree bit for bit (axis-parallel edges: 0 and
fl(pi/2); slopes of 2^-40: atan2 returns the ratio), so the only differences
left are the kernels' own accumulation -- which is exact (per-warp fixed
point in units of 2^-1074, crossing.cu xacc_add) and therefore must not
lose digits when the total is 1e-12.  Long runs of non-crossing edges put
many missed pairs (whose cleared deviations leave subnormal leftovers) into
the same slices as the hits.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HALF_PI = 1.5707963267948966


def _graph(xy, pairs):
    from paper_2411_09809_b200.model import LayoutGraph

    xy = np.asarray(xy, dtype=np.float64)
    return LayoutGraph(np.arange(len(xy)), xy, np.asarray(pairs, dtype=np.int64))


def grid_crossings(k: int, filler: int = 600, seed: int = 3):
    """k horizontal/vertical crossing pairs (angle fl(pi/2)) far apart, plus
    `filler` short horizontal edges that cross nothing."""
    rng = np.random.default_rng(seed)
    xy, pairs = [], []
    for c in range(k):
        x0 = 100.0 * c
        base = len(xy)
        xy += [(x0, 0.0), (x0 + 2.0, 0.0), (x0 + 1.0, -1.0), (x0 + 1.0, 1.0)]
        pairs += [(base, base + 1), (base + 2, base + 3)]
    for f in range(filler):
        x = float(rng.integers(0, 2**20)) * 8.0 + 5000.0
        y = 50.0 + 4.0 * f
        base = len(xy)
        xy += [(x, y), (x + 1.0, y)]
        pairs.append((base, base + 1))
    return xy, pairs


def shallow_crossings(k: int, filler: int = 600):
    """k pairs crossing at the angle 2^-40: a horizontal edge and an edge of
    slope 2^-40 through its midpoint (theta exactly 2^-40 in numpy and
    CUDA), plus filler."""
    xy, pairs = [], []
    L = 2.0**20
    for c in range(k):
        y0 = 10.0 * c
        base = len(xy)
        xy += [(0.0, y0), (2 * L, y0), (0.0, y0 - L * 2.0**-40), (2 * L, y0 + L * 2.0**-40)]
        pairs += [(base, base + 1), (base + 2, base + 3)]
    for f in range(filler):
        base = len(xy)
        y = 1e6 + 3.0 * f
        xy += [(0.0, y), (1.0, y)]
        pairs.append((base, base + 1))
    return xy, pairs


def _check(g, ideal, strategy):
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G

    c_ref, d_ref = O.crossing_scan(g.xy, g.edges, ideal)
    c, d = G._crossing_scan(g, ideal, strategy=strategy)
    assert c == c_ref
    assert d_ref > 0.0
    assert abs(d - d_ref) <= 1e-9 * d_ref, (d, d_ref)  # no absolute floor
    return c, d, d_ref


@pytest.mark.parametrize("k", [1, 2, 5, 10])
@pytest.mark.parametrize("strategy", ["dense", "culled"])
def test_tiny_deviation_sums_right_angles(gpu, k, strategy):
    xy, pairs = grid_crossings(k)
    g = _graph(xy, pairs)
    for delta in (1e-12, 3.7e-14, 2.0**-45):
        ideal = HALF_PI - delta  # deviation per crossing = HALF_PI - ideal, exact
        c, d, d_ref = _check(g, ideal, strategy)
        assert c == k
        assert d == d_ref  # every term exact: the exact accumulator reproduces it bit for bit


@pytest.mark.parametrize("k", [1, 3, 10])
def test_tiny_deviation_sums_shallow_angles(gpu, k):
    xy, pairs = shallow_crossings(k)
    g = _graph(xy, pairs)
    for ideal in (2.0**-39, 2.0**-40 + 2.0**-80, 3.0 * 2.0**-41):
        c, d, d_ref = _check(g, ideal, "dense")
        assert c == k


def test_zero_deviation_is_exactly_zero(gpu):
    """Crossings exactly at the ideal angle: the reference's dev_sum is 0.0,
    so the kernels' cleared-miss leftovers must not survive."""
    import paper_2411_09809_b200 as G

    xy, pairs = grid_crossings(4)
    g = _graph(xy, pairs)
    c, d = G._crossing_scan(g, HALF_PI, strategy="dense")
    assert (c, d) == (4, 0.0)
    assert G.edge_crossing_angle(g, HALF_PI) == 1.0


def test_large_and_small_terms_mixed(gpu):
    """Relative accuracy of a sum dominated by one large deviation with many
    tiny ones beside it (no absolute quantum)."""
    from oracle import glare_oracle as O
    import paper_2411_09809_b200 as G

    xy, pairs = grid_crossings(8)
    g = _graph(xy, pairs)
    ideal = 0.25
    c_ref, d_ref = O.crossing_scan(g.xy, g.edges, ideal)
    c, d = G._crossing_scan(g, ideal)
    assert c == c_ref == 8
    assert abs(d - d_ref) <= 1e-12 * d_ref


def full_grid(h: int = 600, v: int = 600):
    """h horizontal edges crossing v vertical ones everywhere (h * v crossings
    at the angle fl(pi/2), every theta exactly 0 or fl(pi/2)): in the culled
    plan most of them sit in certified-full units and blocks, whose
    deviations come from closed forms or piecewise-linear sums
    (cross_full_kernel / cross_subfull_kernel) unless the mean is small."""
    L = 2.0**12
    xy, pairs = [], []
    for i in range(h):
        base = len(xy)
        xy += [(0.0, 1.0 + i), (2.0 * L, 1.0 + i)]
        pairs.append((base, base + 1))
    for j in range(v):
        base = len(xy)
        xy += [(L / 2 + j, 0.0), (L / 2 + j, 2.0 * L)]
        pairs.append((base, base + 1))
    return xy, pairs


@pytest.mark.parametrize("delta", [1e-12, 2.0**-30, 1e-5, 2.0**-12 * 0.9, 2.0**-12 * 1.1, 1e-3, 0.3])
def test_full_units_small_and_large_deviations(gpu, delta):
    """dev_sum of certified-full units at 1e-9 relative (no floor) from tiny
    to ordinary deviations, on both sides of the per-pair fallback's
    threshold (mean deviation 2^-12)."""
    from paper_2411_09809_b200 import metrics as M

    xy, pairs = full_grid()
    g = _graph(xy, pairs)
    ideal = HALF_PI - delta
    c, d, d_ref = _check(g, ideal, "culled")
    assert c == 600 * 600
    rec = M.CrossingRecords(M.DeviceGraph.from_graph(g), "culled")
    assert rec.n_full > 0
    if delta < 2.0**-13:
        assert d == d_ref  # per-pair fallback: every term exact, exact accumulation
