"""CPU check of the tile-pair certificates of the classified candidate list
(csrc/crossing.cu tile_pq_kernel / orient_ranges / unit_class; K6).

The kernel's classification is restated here with the same IEEE double
operations (round-to-nearest subtractions and products, min / max, the
margin rounded up), and checked two ways:

* the error bound the certificate rests on, with exact rationals: for every
  corner line and point, and for the reference's own FP64 cross products
  (geometry.py:62-79), |fl(c) - c_exact| <= 2^-49 Ux Uy, Ux / Uy the extents
  of the union of the unit's four endpoint boxes;
* end to end: on tile pairs from several families (random, integer lattice,
  crossing bundles, near-degenerate points 1 ulp off a line, large offsets,
  tiny coordinates), every pair of a unit certified "full" passes the
  reference predicate and shares no vertex, and no pair of a unit certified
  "none" passes it.
"""

from __future__ import annotations

import math
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle.glare_oracle import straddle_mask

MARGIN = 2.0 ** -47


def up(x: Fr) -> float:
    """Round an exact rational up to a double."""
    f = float(x)
    return f if Fr(f) >= x else math.nextafter(f, math.inf)


def pq_box(ax, ay, bx, by):
    """tile_pq_kernel: boxes of the P (smaller x, ties smaller y) and Q endpoints."""
    pa = (ax < bx) | ((ax == bx) & (ay <= by))
    px, py = np.where(pa, ax, bx), np.where(pa, ay, by)
    qx, qy = np.where(pa, bx, ax), np.where(pa, by, ay)
    return (px.min(), px.max(), py.min(), py.max(), qx.min(), qx.max(), qy.min(), qy.max())


def orient_ranges(L, R):
    """crossing.cu orient_ranges: computed (lo, hi) of (Q - P) x (r - P) for r
    in R's P box and Q box."""
    lo, hi = [math.inf, math.inf], [-math.inf, -math.inf]
    rb = ((R[0], R[1], R[2], R[3]), (R[4], R[5], R[6], R[7]))
    for c in range(16):
        px = L[1] if c & 1 else L[0]
        py = L[3] if c & 2 else L[2]
        qx = L[5] if c & 4 else L[4]
        qy = L[7] if c & 8 else L[6]
        a, b = qx - px, qy - py
        for k in range(2):
            t1a, t1b = a * (rb[k][2] - py), a * (rb[k][3] - py)
            t2a, t2b = b * (rb[k][0] - px), b * (rb[k][1] - px)
            lo[k] = min(lo[k], min(t1a, t1b) - max(t2a, t2b))
            hi[k] = max(hi[k], max(t1a, t1b) - min(t2a, t2b))
    return lo, hi


def extents(A, B):
    x0 = min(A[0], A[4], B[0], B[4])
    x1 = max(A[1], A[5], B[1], B[5])
    y0 = min(A[2], A[6], B[2], B[6])
    y1 = max(A[3], A[7], B[3], B[7])
    return x0, x1, y0, y1


def unit_class(A, B):
    """crossing.cu unit_class: 0 none, 1 mixed, 2 full."""
    x0, x1, y0, y1 = extents(A, B)
    ux, uy = up(Fr(x1) - Fr(x0)), up(Fr(y1) - Fr(y0))
    thr = up(Fr(up(Fr(up(Fr(ux) * Fr(uy))) * Fr(MARGIN * (1.0 + 2.0 ** -20)))) + Fr(2) ** -1000)
    la, ha = orient_ranges(A, B)
    lb, hb = orient_ranges(B, A)
    pa0, na0, pa1, na1 = la[0] > thr, ha[0] < -thr, la[1] > thr, ha[1] < -thr
    pb0, nb0, pb1, nb1 = lb[0] > thr, hb[0] < -thr, lb[1] > thr, hb[1] < -thr
    if (pa0 and pa1) or (na0 and na1) or (pb0 and pb1) or (nb0 and nb1):
        return 0
    if ((pa0 and na1) or (na0 and pa1)) and ((pb0 and nb1) or (nb0 and pb1)):
        return 2
    return 1


def exact_orient(px, py, qx, qy, rx, ry):
    return (Fr(qx) - Fr(px)) * (Fr(ry) - Fr(py)) - (Fr(qy) - Fr(py)) * (Fr(rx) - Fr(px))


def ref_c(ax, ay, bx, by, cx, cy):
    """The reference's c1 (geometry.py:71) in IEEE doubles."""
    return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)


# ---- tile families ---------------------------------------------------------


def _bundle(rng, k, p0, p1, s):
    a = np.asarray(p0, float) + rng.random((k, 2)) * s
    b = np.asarray(p1, float) + rng.random((k, 2)) * s
    return a, b


def fam_random(rng, k):
    return (rng.random((k, 2)), rng.random((k, 2))), (rng.random((k, 2)), rng.random((k, 2)))


def fam_lattice(rng, k):
    """Two tiles of long lattice edges (2^16 grid) from small endpoint clusters."""
    c = lambda: rng.integers(0, 2 ** 16, 2)  # noqa: E731
    out = []
    for _ in range(2):
        p, q, s = c(), c(), int(rng.integers(1, 2048))
        out.append((p + rng.integers(0, s, (k, 2)), q + rng.integers(0, s, (k, 2))))
    return tuple((a.astype(float), b.astype(float)) for a, b in out)


def fam_cross(rng, k):
    """Bundles that cross everywhere, at random scales and offsets."""
    off = rng.choice([0.0, 1e6, 2.0 ** 40, -3.5e9])
    sc = rng.choice([1.0, 2.0 ** -150, 1e-3, 2.0 ** 100])
    s = rng.random() * 0.2
    A = _bundle(rng, k, (0, 0), (1, 1), s)
    B = _bundle(rng, k, (0, 1), (1, 0), s)
    return tuple((off + sc * a, off + sc * b) for a, b in (A, B))


def fam_touch(rng, k):
    """B's endpoints on (or 1 ulp beside) A's lines: orientations ~ 0."""
    A = _bundle(rng, k, (0, 0), (1, 1), 0.0)
    t = rng.random(k)
    c = np.stack([t, t], 1)
    step = rng.integers(-1, 2, k)  # 1 ulp below, on, 1 ulp above the line
    c[:, 1] = np.where(step == 0, c[:, 1], np.nextafter(c[:, 1], step * np.inf))
    d = np.stack([rng.random(k), 2 + rng.random(k)], 1)
    return A, (c, d)


def fam_parallel(rng, k):
    """Near-parallel bundles a tiny gap apart (certified none, or mixed)."""
    gap = rng.choice([1e-3, 1e-9, 2.0 ** -40])
    A = _bundle(rng, k, (0, 0), (1, 1), 0.0)
    a, b = A
    B = (a + [0.0, gap], b + [0.0, gap])
    return A, B


FAMILIES = {"random": fam_random, "lattice": fam_lattice, "cross": fam_cross,
            "touch": fam_touch, "parallel": fam_parallel}


def _tiles(fam, rng, k):
    (a1, b1), (a2, b2) = FAMILIES[fam](rng, k)
    keep1 = np.any(a1 != b1, axis=1)
    keep2 = np.any(a2 != b2, axis=1)
    return (a1[keep1], b1[keep1]), (a2[keep2], b2[keep2])


def _box(t):
    a, b = t
    return pq_box(a[:, 0], a[:, 1], b[:, 0], b[:, 1])


@pytest.mark.parametrize("fam", sorted(FAMILIES))
def test_certificates_are_sound(fam):
    rng = np.random.default_rng(sorted(FAMILIES).index(fam))
    seen = {0: 0, 1: 0, 2: 0}
    for _ in range(150):
        A, B = _tiles(fam, rng, int(rng.integers(1, 24)))
        if len(A[0]) == 0 or len(B[0]) == 0:
            continue
        cls = unit_class(_box(A), _box(B))
        seen[cls] += 1
        if cls == 1:
            continue
        (a, b), (c, d) = A, B
        I, J = np.meshgrid(np.arange(len(a)), np.arange(len(c)), indexing="ij")
        I, J = I.ravel(), J.ravel()
        hit = straddle_mask(a[I, 0], a[I, 1], b[I, 0], b[I, 1], c[J, 0], c[J, 1], d[J, 0], d[J, 1])
        box = ((np.maximum(c[J, 0], d[J, 0]) >= np.minimum(a[I, 0], b[I, 0]))
               & (np.maximum(a[I, 0], b[I, 0]) >= np.minimum(c[J, 0], d[J, 0]))
               & (np.maximum(c[J, 1], d[J, 1]) >= np.minimum(a[I, 1], b[I, 1]))
               & (np.maximum(a[I, 1], b[I, 1]) >= np.minimum(c[J, 1], d[J, 1])))
        if cls == 2:
            assert np.all(hit & box), fam
            # no shared point: every exact orientation is nonzero
            assert not np.any(np.all(a[I] == c[J], axis=1) | np.all(a[I] == d[J], axis=1)
                              | np.all(b[I] == c[J], axis=1) | np.all(b[I] == d[J], axis=1))
        else:
            assert not np.any(hit & box), fam
    if fam == "cross":
        assert seen[2] > 50
    if fam == "parallel":
        assert seen[0] > 20
    if fam == "touch":
        assert seen[2] == 0


@pytest.mark.parametrize("fam", sorted(FAMILIES))
def test_error_bound_exact(fam):
    """|fl(c) - c| <= 2^-49 Ux Uy for the corner evaluations (orient_ranges'
    differences form) and for the reference's c1 (base point a, either
    endpoint order), in exact rational arithmetic."""
    rng = np.random.default_rng(100 + sorted(FAMILIES).index(fam))
    worst = Fr(0)
    for _ in range(60):
        A, B = _tiles(fam, rng, int(rng.integers(1, 6)))
        if len(A[0]) == 0 or len(B[0]) == 0:
            continue
        BA, BB = _box(A), _box(B)
        x0, x1, y0, y1 = extents(BA, BB)
        bound = Fr(2) ** -49 * (Fr(x1) - Fr(x0)) * (Fr(y1) - Fr(y0))
        if bound == 0:
            continue
        # corner lines of A against corners of B's boxes (orient_ranges)
        for c in rng.integers(0, 16, 4):
            px = BA[1] if c & 1 else BA[0]
            py = BA[3] if c & 2 else BA[2]
            qx = BA[5] if c & 4 else BA[4]
            qy = BA[7] if c & 8 else BA[6]
            rx, ry = BB[int(rng.integers(0, 2))], BB[2 + int(rng.integers(0, 2))]
            got = (qx - px) * (ry - py) - (qy - py) * (rx - px)
            err = abs(Fr(got) - exact_orient(px, py, qx, qy, rx, ry))
            assert err <= bound, fam
            worst = max(worst, err / bound)
        # the reference's own c1 / c2 for actual pairs (a, b) x (c, d)
        (a, b), (c, d) = A, B
        for i in range(len(a)):
            for j in range(len(c)):
                for (sx, sy, ex, ey) in ((a[i], None, b[i], None), (b[i], None, a[i], None)):
                    for r in (c[j], d[j]):
                        got = ref_c(sx[0], sx[1], ex[0], ex[1], r[0], r[1])
                        err = abs(Fr(got) - exact_orient(sx[0], sx[1], ex[0], ex[1], r[0], r[1]))
                        assert err <= bound, fam
                        worst = max(worst, err / bound)
    assert worst <= 1
