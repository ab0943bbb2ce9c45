"""CPU check of the certified FP32 filter's error analysis (K2;
csrc/crossing.cu frec_kernel / filter_m).

The kernel's FP32 records and cross products are re-evaluated here with
exact rational arithmetic for the roundings (RN to FP32 of exact values, so
FFMA's single rounding is modelled exactly), and compared with the exact
cross product of the original FP64 coordinates:

    |c~ - sigma * c_exact| <= sigma * E / 2,   E = 2^-23 (1 + 3 L)
    |c~| <= sigma * C,                          C = L/2 (1 + 2^-20) + E

and every pair the filter would certify has the sign of the exact
orientation.  Inputs include near-collinear triples, shared endpoints,
large offsets and tiny edges.
"""

from __future__ import annotations

import math
from fractions import Fraction as Fr

import numpy as np


def rn32(x: Fr) -> Fr:
    """Round an exact rational to the nearest FP32 value (ties to even)."""
    if x == 0:
        return Fr(0)
    sign = -1 if x < 0 else 1
    a = abs(x)
    e = math.floor(math.log2(a.numerator) - math.log2(a.denominator))
    # fix the exponent estimate
    while Fr(2) ** e > a:
        e -= 1
    while Fr(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)
    ulp = Fr(2) ** (e - 23)
    q = a / ulp
    n = q.numerator // q.denominator
    r = q - n
    if r > Fr(1, 2) or (r == Fr(1, 2) and n % 2 == 1):
        n += 1
    return sign * n * ulp


def rn64(x: Fr) -> Fr:
    return Fr(float(x))  # Python float() of a Fraction rounds to nearest


def rd32_of_float(v: float) -> Fr:
    f = np.float32(v)
    if float(f) > v:
        f = np.nextafter(f, np.float32(-np.inf))
    return Fr(float(f))


def records(ax, ay, bx, by, x0, y0, s):
    """frec_kernel for one edge: scaled FP32 endpoints and scaled line."""
    def q(v, o):
        return rn32(rn64(Fr(v) - Fr(o)) * Fr(s))

    A = (q(ax, x0), q(ay, y0))
    B = (q(bx, x0), q(by, y0))
    abx, aby = rn32(B[0] - A[0]), rn32(B[1] - A[1])
    ka = rn64(abx * A[1] - aby * A[0])
    L = float(abs(abx) + abs(aby))
    if L == 0:
        return A, B, Fr(0), Fr(0), Fr(0), 0.0, 0.0, 0.0
    E = 2.0 ** -23 * (1.0 + 3.0 * L)
    C = 0.5 * L * (1.0 + 2.0 ** -20) + E
    tau = E * C * (1.0 + 2.0 ** -20)
    sig = rd32_of_float((1.0 / math.sqrt(tau)) * (1.0 - 2.0 ** -40))
    return (A, B, rn32(sig * abx), rn32(-sig * aby), rn32(-sig * ka), float(sig), E, C)


def cross_tilde(rec, P):
    """Two FFMAs: c~ = RN(sabx*Py + RN(nsaby*Px + nska))."""
    _, _, sabx, nsaby, nska, _, _, _ = rec
    inner = rn32(nsaby * P[0] + nska)
    return rn32(sabx * P[1] + inner)


def exact_cross(a, b, p):
    ax, ay = Fr(a[0]), Fr(a[1])
    bx, by = Fr(b[0]), Fr(b[1])
    px, py = Fr(p[0]), Fr(p[1])
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax)


def _cases(rng):
    out = []
    for _ in range(300):  # generic
        out.append(rng.uniform(0, 1, (3, 2)))
    for _ in range(300):  # near-collinear: p on the line ab up to 1e-9
        a, b = rng.uniform(0, 1, (2, 2))
        t = rng.uniform(-1, 2)
        p = a + t * (b - a) + rng.normal(scale=1e-9, size=2)
        out.append(np.array([a, b, p]))
    for _ in range(100):  # exactly collinear lattice points
        a, d = rng.integers(0, 50, 2), rng.integers(-5, 6, 2)
        out.append(np.array([a, a + d, a + 3 * d], dtype=np.float64))
    for _ in range(100):  # shared endpoint
        a, b, c = rng.uniform(0, 1, (3, 2))
        out.append(np.array([a, b, [b, a][rng.integers(0, 2)]]))
    for _ in range(200):  # far offset + tiny edges
        base = 2.0 ** 30
        a = base + rng.uniform(0, 1, 2)
        b = a + rng.normal(scale=1e-6, size=2)
        p = base + rng.uniform(0, 1, 2)
        out.append(np.array([a, b, p]))
    return out


def test_cross_product_error_bound_and_certified_signs():
    rng = np.random.default_rng(2024)
    cases = _cases(rng)
    # one global translation/scale over all points, as frec_kernel does
    pts = np.concatenate(cases)
    x0, y0 = pts[:, 0].min(), pts[:, 1].min()
    W = max(pts[:, 0].max() - x0, pts[:, 1].max() - y0)
    s = 2.0 ** -(math.frexp(W)[1] - 1 + 2)
    for a, b, p in cases:
        rec = records(a[0], a[1], b[0], b[1], x0, y0, s)
        A, B, _, _, _, sig, E, C = rec
        if sig == 0.0:
            continue
        P = (rn32(rn64(Fr(p[0]) - Fr(x0)) * Fr(s)), rn32(rn64(Fr(p[1]) - Fr(y0)) * Fr(s)))
        ct = cross_tilde(rec, P)
        ce = exact_cross(a, b, p) * Fr(s) * Fr(s)
        err = abs(ct - Fr(sig) * ce)
        assert err <= Fr(sig) * Fr(E) / 2, (a, b, p, float(err), sig * E / 2)
        assert abs(ct) <= Fr(sig) * Fr(C)
        # certified (|c~| > sigma E) => exact sign equal, nonzero
        if abs(ct) > Fr(sig) * Fr(E):
            assert ce != 0 and (ce > 0) == (ct > 0)


def test_product_certification_threshold():
    """|RN(c~1 c~2)| > 1 implies |c~1| > sigma E and |c~2| > sigma E."""
    rng = np.random.default_rng(7)
    for _ in range(400):
        a, b, c, d = rng.uniform(0, 1, (4, 2))
        if rng.random() < 0.5:  # push c near the line ab
            c = a + rng.uniform(-1, 2) * (b - a) + rng.normal(scale=1e-7, size=2)
        rec = records(a[0], a[1], b[0], b[1], 0.0, 0.0, 0.5)
        _, _, _, _, _, sig, E, C = rec
        P1 = (rn32(Fr(c[0]) / 2), rn32(Fr(c[1]) / 2))
        P2 = (rn32(Fr(d[0]) / 2), rn32(Fr(d[1]) / 2))
        c1, c2 = cross_tilde(rec, P1), cross_tilde(rec, P2)
        prod = rn32(c1 * c2)
        if abs(prod) > 1:
            assert abs(c1) > Fr(sig) * Fr(E) and abs(c2) > Fr(sig) * Fr(E)
