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
    # f[kFSabx] = RN32(RN64(abx sig)) etc.: abx*sig and aby*sig are exact in
    # FP64 (24-bit factors); ka*sig is not, so the line constant is rounded
    # twice (RN64, then RN32) exactly as frec_kernel does
    return (A, B, rn32(sig * abx), -rn32(sig * aby), -rn32(rn64(ka * Fr(sig))), float(sig), E, C)


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


# ---------------------------------------------------------------------------
# Per-unit thresholds, the FOLD rule and the occlusion band, machine-checked.
#
# The kernel's decisions are replayed with exact rational arithmetic (every
# FP32/FP64 rounding modelled) and checked against the REFERENCE predicate
# evaluated in IEEE double exactly as geometry.py:62-79 / exact.py:187-221
# and exact.py:55-74 write it: a pair the filter certifies must get the
# reference's verdict.

def ru64(x: Fr) -> float:
    f = float(x)
    return f if Fr(f) >= x else float(np.nextafter(f, np.inf))


def ru32(x: float) -> float:
    f = np.float32(x)
    if float(f) < x:
        f = np.nextafter(f, np.float32(np.inf))
    return float(f)


def frame(points: np.ndarray):
    """frec_kernel's frame: x0/y0 = smallest endpoint coordinate, W = the
    larger extent rounded up, s = 2^-(ilogb(W) + 2)."""
    x0, y0 = float(points[:, 0].min()), float(points[:, 1].min())
    W = max(ru64(Fr(float(points[:, 0].max())) - Fr(x0)),
            ru64(Fr(float(points[:, 1].max())) - Fr(y0)))
    s = 2.0 ** -(math.frexp(W)[1] - 1 + 2)
    return x0, y0, s


def tile_box(recs):
    """tile_fbox_kernel: box of the scaled FP32 endpoints and the largest
    L = RU(|RN(bx - ax)| + |RN(by - ay)|) (FP32)."""
    xs = [float(v) for r in recs for v in (r[0][0], r[1][0])]
    ys = [float(v) for r in recs for v in (r[0][1], r[1][1])]
    lm = 0.0
    for A, B, *_ in recs:
        lx = abs(float(rn32(B[0] - A[0])))
        ly = abs(float(rn32(B[1] - A[1])))
        lm = max(lm, ru32(lx + ly) if Fr(ru32(lx + ly)) >= Fr(lx) + Fr(ly) else lx + ly)
    return min(xs), max(xs), min(ys), max(ys), lm


def unit_threshold(a, b) -> float:
    """crossing.cu unit_threshold (FP64 arithmetic, RU to FP32, capped at 1)."""
    D = max(max(a[1], b[1]) - min(a[0], b[0]), max(a[3], b[3]) - min(a[2], b[2]))
    Lm = max(a[4], b[4])
    t = (1.5 * D + 3.0 * Lm) * (3.5 * D + 3.0 * Lm) * (1.0 + 2.0 ** -18)
    return 1.0 if t >= 1.0 else ru32(t)


def ref_crosses(e1, e2) -> bool:
    """The reference's pair predicate in IEEE double (Python floats): closed
    bbox overlap, no shared vertex id, proper_intersection_mask."""
    (i1, j1, ax, ay, bx, by), (i2, j2, cx, cy, dx, dy) = e1, e2
    if max(ax, bx) < min(cx, dx) or max(cx, dx) < min(ax, bx):
        return False
    if max(ay, by) < min(cy, dy) or max(cy, dy) < min(ay, by):
        return False
    if len({i1, j1, i2, j2}) < 4:
        return False
    abx, aby = bx - ax, by - ay
    c1 = abx * (cy - ay) - aby * (cx - ax)
    c2 = abx * (dy - ay) - aby * (dx - ax)
    cdx, cdy = dx - cx, dy - cy
    c3 = cdx * (ay - cy) - cdy * (ax - cx)
    c4 = cdx * (by - cy) - cdy * (bx - cx)
    s_cd = (c1 <= 0.0 and c2 >= 0.0) or (c1 >= 0.0 and c2 <= 0.0)
    s_ab = (c3 <= 0.0 and c4 >= 0.0) or (c3 >= 0.0 and c4 <= 0.0)
    return s_cd and s_ab


def fold_class(p12: Fr, p34: Fr, t: float) -> str:
    """FOLD (filter_m<.., true> + filter_block's vote): M = signed-int max of
    the bit patterns of RN(c1 c2 + t), RN(c3 c4 + t); hit = M's sign bit,
    uncertain = M's bits <= bits(2t) (unsigned), else miss."""
    def bits(x: Fr) -> int:
        # sign bit of an RN result = exact value < 0 (a negative value that
        # underflows rounds to -0); +0 for an exact zero sum
        f = np.float32(float(rn32(x)))
        b = int(np.array(f, dtype=np.float32).view(np.uint32))
        if x < 0:
            b |= 0x80000000
        return b
    tt = Fr(t)
    b12, b34 = bits(p12 + tt), bits(p34 + tt)
    s12 = b12 - (1 << 32) if b12 >> 31 else b12
    s34 = b34 - (1 << 32) if b34 >> 31 else b34
    M = max(s12, s34) & 0xFFFFFFFF
    if M >> 31:
        return "hit"
    vbits = int(np.array(np.float32(2.0 * t), dtype=np.float32).view(np.uint32))
    return "uncertain" if M <= vbits else "miss"


def mul_class(p12: Fr, p34: Fr, t: float) -> str:
    """Non-FOLD: M = max(RN(c1 c2), RN(c3 c4)); hit M < -t, uncertain
    |M| <= t, else miss."""
    M = max(rn32(p12), rn32(p34))
    if M < -Fr(t):
        return "hit"
    return "uncertain" if abs(M) <= Fr(t) else "miss"


def _unit_sets(rng):
    """(tile A, tile B) edge sets aimed at tight per-unit thresholds: long
    parallel edges packed inside one small box, near-collinear chains with
    T-junctions, tiny crossing angles, lattice collinearity -- all placed far
    from the frame's origin so D is small against the frame."""
    sets = []
    for trial in range(24):
        kind = trial % 8
        off = rng.uniform(0.2, 0.45, 2)
        D = float(10.0 ** (rng.uniform(-4, -1) if kind in (5, 7) else rng.uniform(-7, -2)))
        edges = []
        if kind == 0:  # long parallel edges filling a D-box (L ~ 2D)
            for _ in range(24):
                y = rng.uniform(0, D)
                edges.append((off + [0, y], off + [D, y + rng.normal(scale=D * 1e-6)]))
        elif kind == 1:  # near-collinear chain with T-junction endpoints
            d = rng.normal(size=2)
            d /= np.linalg.norm(d)
            for _ in range(24):
                s, e = np.sort(rng.uniform(0, D, 2))
                nrm = np.array([-d[1], d[0]]) * rng.normal(scale=D * 1e-9)
                edges.append((off + s * d + nrm, off + e * d))
        elif kind == 2:  # tiny crossing angles through one point
            for _ in range(24):
                ang = rng.normal(scale=1e-7)
                v = np.array([math.cos(ang), math.sin(ang)]) * D / 2
                c = off + rng.normal(scale=D * 1e-9, size=2)
                edges.append((c - v, c + v))
        elif kind == 3:  # exact collinear lattice points, overlapping
            base = np.floor(off * 2 ** 20) / 2 ** 20
            q = 2.0 ** -30
            for _ in range(24):
                a = rng.integers(0, 64, 2)
                st = rng.integers(-3, 4, 2)
                if not st.any():
                    st[0] = 1
                k = int(rng.integers(1, 8))
                edges.append((base + a * q, base + (a + k * st) * q))
        elif kind == 4:  # shared endpoints (hub) inside the box
            c = off.copy()
            for _ in range(24):
                edges.append((c, c + rng.uniform(-D, D, 2)))
        elif kind == 5:  # generic random in a small box
            for _ in range(24):
                edges.append((off + rng.uniform(0, D, 2), off + rng.uniform(0, D, 2)))
        elif kind == 7:  # a fan of edges all crossing one band, plus the band
            for _ in range(12):
                y = rng.uniform(0, D)
                edges.append((off + [0, y], off + [D, y + rng.uniform(-D, D) * 1e-3]))
            for _ in range(12):
                x = rng.uniform(0, D)
                edges.append((off + [x, -D * 0.1], off + [x + rng.uniform(-D, D), D * 1.1]))
        else:  # very short edges near long ones
            for _ in range(12):
                y = rng.uniform(0, D)
                edges.append((off + [0, y], off + [D, y]))
            for _ in range(12):
                p = off + rng.uniform(0, D, 2)
                edges.append((p, p + rng.normal(scale=D * 1e-5, size=2)))
        edges = [(np.asarray(a, float), np.asarray(b, float)) for a, b in edges
                 if np.any(np.asarray(a) != np.asarray(b))]
        perm = rng.permutation(len(edges))
        edges = [edges[k] for k in perm]
        half = len(edges) // 2
        sets.append((edges[:half], edges[half:]))
    return sets


def _unit_check(tiles_a, tiles_b, anchors):
    pts = np.concatenate([np.array([p for e in tiles_a + tiles_b for p in e]), anchors])
    x0, y0, s = frame(pts)
    # vertex ids: equal coordinates share an id (hubs and chains share
    # endpoints by index, as in a normalized LayoutGraph)
    ids = {}

    def vid(p):
        return ids.setdefault((float(p[0]), float(p[1])), len(ids))

    def rec_of(e):
        a, b = e
        return records(a[0], a[1], b[0], b[1], x0, y0, s)

    def quant(p):
        return (rn32(rn64(Fr(float(p[0])) - Fr(x0)) * Fr(s)),
                rn32(rn64(Fr(float(p[1])) - Fr(y0)) * Fr(s)))

    ra = [rec_of(e) for e in tiles_a]
    rb = [rec_of(e) for e in tiles_b]
    t = unit_threshold(tile_box(ra), tile_box(rb))
    stats = {"t": t, "hit": 0, "miss": 0, "uncertain": 0}
    for ea, rA in zip(tiles_a, ra):
        for eb, rB in zip(tiles_b, rb):
            ref = ref_crosses((vid(ea[0]), vid(ea[1]), *ea[0], *ea[1]),
                              (vid(eb[0]), vid(eb[1]), *eb[0], *eb[1]))
            Cq, Dq = quant(eb[0]), quant(eb[1])
            c1, c2 = cross_tilde(rA, Cq), cross_tilde(rA, Dq)
            c3, c4 = cross_tilde(rB, rA[0]), cross_tilde(rB, rA[1])
            p12, p34 = c1 * c2, c3 * c4
            for cls in (fold_class(p12, p34, t), mul_class(p12, p34, t)):
                stats[cls] += 1
                if cls == "hit":
                    assert ref, (ea, eb, t)
                elif cls == "miss":
                    assert not ref, (ea, eb, t)
    return stats


def test_unit_threshold_certifies_adversarial_units():
    """unit_threshold (crossing.cu) with the FOLD and FMUL classifications:
    every certified hit / miss of every pair of every unit agrees with the
    reference predicate; the thresholds are well below the global 1."""
    rng = np.random.default_rng(31)
    anchors = np.array([[0.0, 0.0], [1.0, 1.0]])  # frame: the unit square
    ts, tot = [], {"hit": 0, "miss": 0, "uncertain": 0}
    for A, B in _unit_sets(rng):
        for ta, tb in ((A, B), (A, A)):  # off-diagonal and diagonal units
            st = _unit_check(ta, tb, anchors)
            ts.append(st["t"])
            for k in tot:
                tot[k] += st[k]
    assert min(ts) < 1e-6 and sum(t < 1.0 for t in ts) >= len(ts) - 2
    # the check is not vacuous: many decisions are certified both ways
    assert tot["hit"] > 100 and tot["miss"] > 1000, tot


def test_fold_rule_on_extreme_products():
    """FOLD's sign-bit hit and unsigned 2t vote against the exact products,
    on boundary values: products at exactly -t, t, -t +- ulp, zeros (+0/-0),
    subnormal products, and t from 2^-40 to 1."""
    rng = np.random.default_rng(5)
    ts = [1.0, 0.5, ru32(3e-3), ru32(1e-7), 2.0 ** -40, ru32(0.7)]
    for t in ts:
        T = Fr(t)
        specials = [T, -T, T * (1 + Fr(1, 2 ** 30)), -T * (1 + Fr(1, 2 ** 30)),
                    T * (1 - Fr(1, 2 ** 30)), -T * (1 - Fr(1, 2 ** 30)), Fr(0),
                    Fr(1, 2 ** 160), -Fr(1, 2 ** 160), 3 * T, -3 * T, Fr(2) * T, -2 * T]
        for _ in range(400):
            p12 = specials[int(rng.integers(len(specials)))] if rng.random() < 0.6 else \
                Fr(float(rng.normal() * t * 4))
            p34 = specials[int(rng.integers(len(specials)))] if rng.random() < 0.6 else \
                Fr(float(rng.normal() * t * 4))
            cls = fold_class(p12, p34, t)
            if cls == "hit":
                assert p12 < -T and p34 < -T, (t, p12, p34)
            elif cls == "miss":
                assert p12 > T or p34 > T, (t, p12, p34)
            # soundness both ways: a strictly certain exact case is never
            # lost to "uncertain" beyond the one rounding of the FFMA
            if p12 < -2 * T and p34 < -2 * T:
                assert cls == "hit"
            if p12 > 2 * T or p34 > 2 * T:
                assert cls == "miss"
            # the masked diagonal value 4 is always a miss (t <= 1)
        assert fold_class(Fr(4) - T, Fr(4) - T, t) == "miss"


# -- occlusion band (occlusion.cu occ_header_kernel / occ_filter_block) -----

def _occ_E(S: float) -> float:
    return 3.0 * 2.0 ** -25 * math.sqrt(2.01 * S) + 2.0 ** -21 * S + 2.0 ** -48


def _occ_header(xy: np.ndarray, thr: float):
    x0, y0 = float(xy[:, 0].min()), float(xy[:, 1].min())
    W = max(ru64(Fr(float(xy[:, 0].max())) - Fr(x0)), ru64(Fr(float(xy[:, 1].max())) - Fr(y0)))
    sc = 2.0 ** -(math.frexp(W)[1] - 1 + 2)
    T = thr * sc * sc
    tlo = float(rd32_of_float(T - _occ_E(T)))
    thi = ru32(T + _occ_E(4.0 * T))
    return x0, y0, sc, T, tlo, thi


def test_occlusion_band_certifies():
    """S~ = RN(dY dY + RN(dX dX)) of the packed filter: S~ < T_lo must be an
    occluding pair of the reference (FP64 dx*dx + dy*dy < (2r)^2, strict),
    S~ > T_hi a non-occluding one; and the folded form the kernel runs,
    d = RN(dY dY + RN(dX dX - T_lo)): d < 0 occluding, d > RU(T_hi - T_lo)
    not.  Exact ties and near-ties included."""
    rng = np.random.default_rng(17)
    checked = {"hit": 0, "miss": 0, "uncertain": 0}
    for trial in range(12):
        r = float(10.0 ** rng.uniform(-6, 1))
        thr = (2.0 * r) ** 2
        span = float(10.0 ** rng.uniform(0, 3)) * r
        off = float(rng.choice([0.0, 1.0, 2.0 ** 20, -(2.0 ** 12)]))
        pts = []
        for _ in range(60):
            p = off + rng.uniform(0, span, 2)
            ang = rng.uniform(0, 2 * math.pi)
            d = 2 * r * (1 + rng.choice([0.0, 1e-9, -1e-9, 1e-6, -1e-6, 1e-16, -1e-16]))
            q = p + d * np.array([math.cos(ang), math.sin(ang)])
            pts += [p, q]
        if trial % 3 == 0:  # lattice: exact ties dist^2 == thr
            k = 2.0 ** int(rng.integers(-10, 4))
            base = np.floor(rng.uniform(0, 64, (60, 2)))
            pts = list(np.concatenate([base, base + [[2, 0]]]) * k + off)
            thr = (2.0 * k) ** 2
        xy = np.array(pts, dtype=np.float64)
        x0, y0, sc, T, tlo, thi = _occ_header(xy, thr)
        q = [(rn32(rn64(Fr(float(x)) - Fr(x0)) * Fr(sc)), rn32(rn64(Fr(float(y)) - Fr(y0)) * Fr(sc)))
             for x, y in xy]
        for i in range(len(xy)):
            for j in range(i + 1, len(xy)):
                dX, dY = rn32(q[j][0] - q[i][0]), rn32(q[j][1] - q[i][1])
                S = rn32(dY * dY + rn32(dX * dX))  # FFMA(dy, dy, FMUL(dx, dx))
                dx, dy = float(xy[i, 0]) - float(xy[j, 0]), float(xy[i, 1]) - float(xy[j, 1])
                ref = dx * dx + dy * dy < thr
                # d = RN(S - tlo): sign bit <=> S < tlo
                if S < Fr(tlo):
                    assert ref, (trial, i, j)
                    checked["hit"] += 1
                elif S > Fr(thi):
                    assert not ref, (trial, i, j)
                    checked["miss"] += 1
                else:
                    checked["uncertain"] += 1
                # the folded evaluation the kernel runs (occlusion.cu occ_d):
                # d = RN(dY dY + RN(dX dX - tlo)); hit <=> the pre-rounding
                # value is negative (d's sign bit); miss <=> d > RU(thi - tlo)
                e = rn32(dX * dX - Fr(tlo))
                w = dY * dY + e
                dfold = rn32(w)
                if w < 0:
                    assert ref, ("fold", trial, i, j)
                    checked["fold_hit"] = checked.get("fold_hit", 0) + 1
                elif dfold > Fr(ru32(thi - tlo)):
                    assert not ref, ("fold", trial, i, j)
                # the error bound the band is built from
                St = Fr(dx * dx + dy * dy) * Fr(sc) * Fr(sc)
                if St < Fr(8 * T):
                    assert abs(S - St) <= Fr(_occ_E(float(St))), (trial, i, j)
    assert checked["hit"] > 50 and checked["miss"] > 1000 and checked["uncertain"] > 0, checked
    assert checked["fold_hit"] >= checked["hit"] // 2, checked
