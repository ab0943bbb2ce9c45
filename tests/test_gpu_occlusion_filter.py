"""GPU: the certified FP32 occlusion filter (default) against the FP64 kernel
and the oracle, on inputs with exact ties, near-threshold pairs, offsets,
tiny and huge radii, coincident points and culled (spatially local) plans."""

from __future__ import annotations

import numpy as np
import pytest

import cases
from conftest import graph_from

pytestmark = pytest.mark.gpu


def _both(g, r, strategy):
    from paper_2411_09809_b200 import _lib, node_occlusion

    L = _lib.lib()
    prev = L.glr_occlusion_set_filter(1)
    try:
        f = node_occlusion(g, r, strategy=strategy)
        L.glr_occlusion_set_filter(0)
        e = node_occlusion(g, r, strategy=strategy)
    finally:
        L.glr_occlusion_set_filter(prev)
    return f, e


def _random(seed, n, kind):
    from paper_2411_09809_b200.model import LayoutGraph

    rng = np.random.default_rng(seed)
    if kind == "lattice":
        xy = rng.integers(0, 200, (n, 2)).astype(np.float64)
    elif kind == "offset":
        xy = 2.0 ** 40 + rng.integers(0, 300, (n, 2)).astype(np.float64) * 0.25
    elif kind == "ring":
        # pairs at distance 2r (r = 0.75 here) scaled by 1 +- k 2^-52 and by
        # 1 +- 2^-24 (the FP32 resolution), in random directions, around
        # random centres at an offset: every folded-test band case
        c = 1000.0 + rng.uniform(0, 50, (n // 2, 2))
        ang = rng.uniform(0, 2 * np.pi, n // 2)
        f = 1.0 + rng.choice([0, 1, -1, 2, -2, 2 ** 28, -(2 ** 28)], n // 2) * 2.0 ** -52
        d = 1.5 * f
        xy = np.concatenate([c, c + d[:, None] * np.stack([np.cos(ang), np.sin(ang)], 1)])
    elif kind == "cluster":
        xy = np.concatenate([rng.uniform(0, 1e-6, (n // 2, 2)), rng.uniform(0, 10, (n - n // 2, 2))])
    else:
        xy = rng.uniform(0, 100, (n, 2))
    return LayoutGraph(np.arange(n), xy, np.empty((0, 2), dtype=np.int64))


@pytest.mark.parametrize("kind,r", [("lattice", 1.0), ("lattice", 2.5), ("offset", 0.5), ("ring", 0.75),
                                    ("cluster", 1e-7), ("cluster", 0.3), ("uniform", 0.7),
                                    ("uniform", 1e-9), ("uniform", 1e9)])
@pytest.mark.parametrize("strategy", ["dense", "culled"])
def test_filter_equals_fp64_and_oracle(gpu, kind, r, strategy):
    from oracle import sweep as S

    g = _random(sum(map(ord, kind)) + int(abs(np.log2(r))), 3000, kind)
    f, e = _both(g, r, strategy)
    assert f == e == S.node_occlusion(g.xy, r)


def test_filter_on_adversarial_sets(gpu):
    for name in ("occlusion_ties", "lattice_stress", "signed_zero_mix", "huge_coords",
                 "tiny_coords"):
        builder = cases.ADVERSARIAL_ARRAYS.get(name)
        if builder is None:
            continue
        g = graph_from(builder)
        for r in (0.5, 1.0, 2.0):
            f, e = _both(g, r, "dense")
            assert f == e, (name, r)
