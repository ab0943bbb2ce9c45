"""CPU check of the one-DADD angle deviation of classified units
(csrc/crossing.cu unit_shift, DESIGN.md 4 K2 "Edge order").

A unit whose theta difference dt = theta_j - theta_i keeps one side of 0 and
of +-pi/2 for all its pairs (tile theta bounds) evaluates the reference's
|ideal - min(d, pi - d)|, d = |theta_i - theta_j| (exact.py:217-220,
geometry.py:107-110), as |theta_j - (theta_i + s)| with s chosen per unit.
Here the classification is restated in Python and checked on random tiles
against the reference formula (float64, 1e-15 absolute: a few ulps of pi),
for several ideal angles including pi/2 and tiny ones.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

HALF_PI = 1.5707963267948966
PI = 3.141592653589793


def unit_shift(lo_i, hi_i, lo_j, hi_j, ideal):
    """crossing.cu unit_shift on (outward-rounded) tile theta bounds."""
    lo, hi = lo_j - hi_i, hi_j - lo_i
    if not lo <= hi:
        return None
    if lo >= 0.0 and hi <= HALF_PI:
        return 0, ideal
    if lo >= HALF_PI:
        return 1, PI - ideal
    if hi <= 0.0 and lo >= -HALF_PI:
        return 2, -ideal
    if hi <= -HALF_PI:
        return 3, ideal - PI
    return None


def reference_dev(ti, tj, ideal):
    d = np.abs(ti - tj)
    return np.abs(ideal - np.minimum(d, PI - d))


@pytest.mark.parametrize("ideal", [1e-6, 0.3, math.radians(70.0), 1.3, HALF_PI])
def test_shift_classes_match_reference(ideal):
    rng = np.random.default_rng(int(ideal * 1e6) % 2**32)
    hits = {}
    for _ in range(4000):
        wi, wj = rng.uniform(0, 0.3, 2) * rng.choice([1e-4, 1e-2, 1.0], 2)
        ci, cj = rng.uniform(0, PI, 2)
        ti = np.clip(ci + rng.uniform(0, wi, 64), 0, np.nextafter(PI, 0))
        tj = np.clip(cj + rng.uniform(0, wj, 64), 0, np.nextafter(PI, 0))
        cls = unit_shift(ti.min(), ti.max(), tj.min(), tj.max(), ideal)
        if cls is None:
            continue
        hits[cls[0]] = hits.get(cls[0], 0) + 1
        s = cls[1]
        got = np.abs(tj[None, :] - (ti[:, None] + s))
        want = reference_dev(ti[:, None], tj[None, :], ideal)
        assert np.max(np.abs(got - want)) <= 4e-16 * 4, (ideal, s)
    # all four classes occur
    assert len(hits) == 4, hits


def test_straddling_units_are_not_classified():
    # a unit whose theta difference crosses 0 or pi/2 keeps the general formula
    assert unit_shift(1.0, 1.2, 1.1, 1.3, 0.5) is None           # crosses 0
    assert unit_shift(0.1, 0.2, 1.6, 1.9, 0.5) is None           # crosses pi/2
    assert unit_shift(0.1, 0.2, 0.3, 0.4, 0.5) == (0, 0.5)
    assert unit_shift(2.9, 3.0, 0.1, 0.2, 0.5) == (3, 0.5 - PI)
    assert unit_shift(float("inf"), -float("inf"), 0.1, 0.2, 0.5) is None  # empty tile


SIGN_MARGIN = 2.0 ** -8


def range_kink(lo_i, hi_i, lo_j, hi_j, ideal):
    """crossing.cu range_kink on tile theta bounds: (beta, f(beta), minus) of
    the one kink the unit's dt range may hold, or None."""
    lo, hi = lo_j - hi_i, hi_j - lo_i
    if not lo <= hi:
        return None
    pmi, hmi, mg = PI - ideal, HALF_PI - ideal, SIGN_MARGIN
    table = ((-PI, -pmi, -HALF_PI - mg, 0, hmi), (-pmi + mg, -HALF_PI, -ideal - mg, 1, hmi),
             (-HALF_PI + mg, -ideal, -mg, 0, hmi), (-ideal + mg, 0.0, ideal - mg, 1, ideal),
             (mg, ideal, HALF_PI - mg, 0, hmi), (ideal + mg, HALF_PI, pmi - mg, 1, hmi),
             (HALF_PI + mg, pmi, PI, 0, hmi))
    for left, beta, right, minus, fbeta in table:
        if lo >= left and hi <= right:
            return beta, fbeta, minus
    return None


@pytest.mark.parametrize("ideal", [1e-6, 0.02, 0.3, math.radians(70.0), 1.3, HALF_PI - 1e-3, HALF_PI])
def test_one_kink_units_match_reference(ideal):
    """Every pair of a unit range_kink accepts: |theta_j - (theta_i + beta)|
    (or f(beta) minus it) equals the reference deviation to a few ulps of pi,
    the second kind's terms stay >= the margin, and all seven kinks occur."""
    rng = np.random.default_rng(int(ideal * 1e6) % 2**32 + 7)
    seen = set()
    for _ in range(6000):
        wi, wj = rng.uniform(0, 0.5, 2) * rng.choice([1e-4, 1e-2, 1.0], 2)
        ci, cj = rng.uniform(0, PI, 2)
        ti = np.clip(ci + rng.uniform(0, wi, 48), 0, np.nextafter(PI, 0))
        tj = np.clip(cj + rng.uniform(0, wj, 48), 0, np.nextafter(PI, 0))
        cls = range_kink(ti.min(), ti.max(), tj.min(), tj.max(), ideal)
        if cls is None:
            continue
        beta, fbeta, minus = cls
        seen.add(round(beta, 9))
        v = np.abs(tj[None, :] - (ti[:, None] + beta))
        got = fbeta - v if minus else v
        want = reference_dev(ti[:, None], tj[None, :], ideal)
        assert np.max(np.abs(got - want)) <= 4e-15, (ideal, beta, minus)
        if minus:
            assert got.min() >= SIGN_MARGIN * (1 - 1e-9)
    if 0.02 <= ideal <= 1.3:  # nearer 0 or pi/2 some kinks sit inside their neighbours' margins
        assert len(seen) == 7, seen
