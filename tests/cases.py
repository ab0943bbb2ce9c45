"""Deterministic test inputs shared by the golden-fixture generator and the
tests: the reference's own known-answer graphs (pkg/tests/conftest.py and
pkg/tests/test_metrics_exact.py), adversarial degenerate sets (SURVEY.md 0.1
and 8(c)) and seeded random layouts (criterion-1 style, test_acceptance.py:
117-142).

Every builder returns ``(positions: dict id->(x, y), edge id pairs)`` or
arrays, so the same input can be wrapped by this package's LayoutGraph or by
the reference's.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2411_09809_b200.configs import random_graph

IDEAL = 7.0 * math.pi / 18.0


# -- known answers of the reference's own tests ------------------------------

def x_graph():
    return {0: (0.0, 0.0), 1: (1.0, 1.0), 2: (0.0, 1.0), 3: (1.0, 0.0)}, [(0, 1), (2, 3)]


def star_graph(k=6):
    pos = {0: (0.0, 0.0)}
    edges = []
    for i in range(k):
        a = 2.0 * math.pi * i / k
        pos[i + 1] = (math.cos(a), math.sin(a))
        edges.append((0, i + 1))
    return pos, edges


def parallel_graph():
    return {0: (0.0, 0.0), 1: (1.0, 0.0), 2: (0.0, 1.0), 3: (1.0, 1.0)}, [(0, 1), (2, 3)]


def triangle_centre():
    return ({0: (0.0, 0.0), 1: (4.0, 0.0), 2: (2.0, 3.0), 3: (2.0, 1.0)},
            [(0, 1), (1, 2), (0, 2), (0, 3), (1, 3), (2, 3)])


def three_mutual():
    return ({0: (0.0, 1.0), 1: (4.0, 1.2), 2: (1.0, 0.0), 3: (2.5, 3.0),
             4: (3.0, 0.0), 5: (1.5, 3.0)}, [(0, 1), (2, 3), (4, 5)])


def ideal_crossing():
    th = 7.0 * math.pi / 18.0
    return ({0: (-1.0, 0.0), 1: (1.0, 0.0), 2: (-math.cos(th), -math.sin(th)),
             3: (math.cos(th), math.sin(th))}, [(0, 1), (2, 3)])


def right_angle():
    return {0: (0.0, 0.0), 1: (1.0, 0.0), 2: (0.0, 1.0)}, [(0, 1), (0, 2)]


def right_angle_isolated():
    return {0: (0.0, 0.0), 1: (1.0, 0.0), 2: (0.0, 1.0), 9: (5.0, 5.0)}, [(0, 1), (0, 2)]


def lengths_1_3():
    return {0: (0.0, 0.0), 1: (1.0, 0.0), 2: (0.0, 5.0), 3: (3.0, 5.0)}, [(0, 1), (2, 3)]


def occ_one_pair():
    return {0: (0.0, 0.0), 1: (1.0, 0.0), 2: (10.0, 10.0)}, [(0, 1)]


def occ_boundary():
    return {0: (0.0, 0.0), 1: (2.0, 0.0)}, [(0, 1)]


def occ_three():
    return {0: (0.0, 0.0), 1: (0.1, 0.0), 2: (0.0, 0.1)}, []


KNOWN = {
    "x_graph": x_graph,
    "star6": star_graph,
    "parallel": parallel_graph,
    "triangle_centre": triangle_centre,
    "three_mutual": three_mutual,
    "ideal_crossing": ideal_crossing,
    "right_angle": right_angle,
    "right_angle_isolated": right_angle_isolated,
    "lengths_1_3": lengths_1_3,
    "occ_one_pair": occ_one_pair,
    "occ_boundary": occ_boundary,
    "occ_three": occ_three,
}


# -- adversarial degenerate sets -------------------------------

def collinear_disjoint():
    return {0: (0.0, 0.0), 1: (1.0, 0.0), 2: (2.0, 0.0), 3: (3.0, 0.0)}, [(0, 1), (2, 3)]


def collinear_overlap():
    return {0: (0.0, 0.0), 1: (2.0, 0.0), 2: (1.0, 0.0), 3: (3.0, 0.0)}, [(0, 1), (2, 3)]


def t_junction():
    return {0: (0.0, 0.0), 1: (2.0, 0.0), 2: (1.0, 0.0), 3: (1.0, 1.0)}, [(0, 1), (2, 3)]


def coincident_ids():
    return {0: (0.0, 0.0), 1: (1.0, 1.0), 2: (1.0, 1.0), 3: (2.0, 0.0)}, [(0, 1), (2, 3)]


def shared_vertex():
    return {0: (0.0, 0.0), 1: (1.0, 1.0), 2: (2.0, 0.0)}, [(0, 1), (1, 2)]


def corner_touch():
    return {0: (0.0, 0.0), 1: (1.0, 1.0), 2: (1.0, 2.0), 3: (2.0, 1.0)}, [(0, 1), (2, 3)]


def collinear_chain():
    # many collinear segments on one line, some sharing vertices, some overlapping
    pos = {i: (float(i), 2.0 * float(i)) for i in range(12)}
    edges = [(0, 3), (1, 2), (2, 5), (4, 6), (6, 9), (7, 8), (8, 11), (10, 11), (0, 11)]
    return pos, edges


ADVERSARIAL_SMALL = {
    "collinear_disjoint": collinear_disjoint,
    "collinear_overlap": collinear_overlap,
    "t_junction": t_junction,
    "coincident_ids": coincident_ids,
    "shared_vertex": shared_vertex,
    "corner_touch": corner_touch,
    "collinear_chain": collinear_chain,
}


def lattice_stress(seed=7, n=3000, m=6000, side=64):
    """Integer-lattice graph dense in exact collinear/coincident/tie cases
    (SURVEY.md appendix A)."""
    rng = np.random.default_rng(seed)
    xy = rng.integers(0, side, (n, 2)).astype(np.float64)
    pairs = rng.integers(0, n, (m, 2))
    pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
    return np.arange(n), xy, pairs


def near_collinear(seed=11, lines=300, per_line=6, scale=1.0):
    """Edges whose endpoints sit within ~1e-16 relative of other edges' lines:
    the set where FMA contraction flips orientation signs (SURVEY.md 0.1
    item 2)."""
    rng = np.random.default_rng(seed)
    pts = []
    edges = []
    for _ in range(lines):
        a = rng.uniform(-1, 1, 2) * scale
        b = rng.uniform(-1, 1, 2) * scale
        base = len(pts)
        pts.extend([a, b])
        edges.append((base, base + 1))
        for _k in range(per_line):
            t1, t2 = rng.uniform(-0.5, 1.5, 2)
            p = a + t1 * (b - a) + rng.normal(0, 1e-16 * scale, 2)
            q = a + t2 * (b - a) + rng.normal(0, 1e-16 * scale, 2)
            if np.all(p == q):
                continue
            i = len(pts)
            pts.extend([p, q])
            edges.append((i, i + 1))
        # a crossing edge through the line
        c = 0.5 * (a + b) + rng.normal(0, 0.3 * scale, 2)
        d = 0.5 * (a + b) - (c - 0.5 * (a + b))
        if not np.all(c == d):
            i = len(pts)
            pts.extend([c, d])
            edges.append((i, i + 1))
    xy = np.asarray(pts, dtype=np.float64)
    return np.arange(len(xy)), xy, np.asarray(edges, dtype=np.int64)


def occlusion_ties(side=40, spacing=2.0):
    """Square lattice at spacing 2 with r = 1: every neighbour pair sits at
    exactly 2r (not occluding) plus jittered extras that do occlude."""
    g = np.arange(side, dtype=np.float64) * spacing
    X, Y = np.meshgrid(g, g)
    xy = np.stack([X.ravel(), Y.ravel()], 1)
    rng = np.random.default_rng(3)
    extra = xy[rng.integers(0, len(xy), 200)] + rng.uniform(-1.5, 1.5, (200, 2))
    xy = np.concatenate([xy, extra])
    edges = np.stack([np.arange(0, len(xy) - 1, 7), np.arange(1, len(xy), 7)], 1)
    return np.arange(len(xy)), xy, edges


def scaled_lattice(scale, seed=13):
    """Lattice stress graph scaled by a power of two: huge (1e200) or tiny
    (1e-300) magnitudes exercise the general (non-fast) sign path."""
    ids, xy, pairs = lattice_stress(seed=seed, n=600, m=1200, side=24)
    return ids, xy * scale, pairs


def signed_zero_mix(seed=17):
    """Coordinates drawn from {-1, -0.0, +0.0, 1, 0.5} so -0.0/+0.0 ties hit the
    bbox ranks and the sign tests."""
    rng = np.random.default_rng(seed)
    vals = np.array([-1.0, -0.0, 0.0, 1.0, 0.5, -0.5])
    xy = vals[rng.integers(0, len(vals), (400, 2))]
    pairs = rng.integers(0, 400, (900, 2))
    pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
    return np.arange(400), xy, pairs


ADVERSARIAL_ARRAYS = {
    "lattice_stress": lattice_stress,
    "near_collinear": near_collinear,
    "occlusion_ties": occlusion_ties,
    "huge_coords": lambda: scaled_lattice(2.0 ** 660),
    "tiny_coords": lambda: scaled_lattice(2.0 ** -990),
    "big_fast": lambda: scaled_lattice(2.0 ** 400),
    "small_fast": lambda: scaled_lattice(2.0 ** -150),
    "small_general": lambda: scaled_lattice(2.0 ** -300),
    "signed_zero_mix": signed_zero_mix,
}

ADVERSARIAL_RADIUS = {
    "lattice_stress": 1.0,
    "near_collinear": 0.01,
    "occlusion_ties": 1.0,
    "huge_coords": 2.0 ** 500,
    "tiny_coords": 2.0 ** -990,
    "big_fast": 2.0 ** 400,
    "small_fast": 2.0 ** -150,
    "small_general": 2.0 ** -300,
    "signed_zero_mix": 0.25,
}


# -- seeded random layouts ----------------------------------------------------

def random_layout_arrays(edges, extent=100.0, seed=0):
    """Uniform positions in [0, extent]^2 for every endpoint id, drawn like
    the reference's random_layout (graphio.py:141-148)."""
    ids = np.unique(np.asarray(edges, dtype=np.int64))
    xy = np.random.default_rng(seed).uniform(0.0, extent, size=(len(ids), 2))
    return ids, xy, edges


def criterion1_case(i, rng):
    """One of the 200 acceptance-criterion-1 style graphs (|V| <= 300,
    |E| <= 1000, [0, 100]^2; test_acceptance.py:117-142 draws sizes the same
    way from one generator)."""
    n = int(rng.integers(4, 301))
    m = int(rng.integers(1, min(1000, n * (n - 1) // 2) + 1))
    edges = random_graph(n, m, seed=1000 + i)
    return random_layout_arrays(edges, extent=100.0, seed=2000 + i)
