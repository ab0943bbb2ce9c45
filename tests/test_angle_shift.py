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
