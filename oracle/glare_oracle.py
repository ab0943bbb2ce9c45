"""CPU oracle for the exact readability-metric hot path -- TEST INFRASTRUCTURE.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2411_09809_b200``) never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

It restates, in numpy, the reference's serial oracle (the ``"oracle"`` mode of
``glare``; /root/reference/pkg/src/glare/engine.py:74-94) for the five exact
metrics, using the same IEEE ufunc sequence so counts are bit-identical and
reals agree to the last few ulps:

* ``node_occlusion``        -- reference src/metrics/exact.py:55-74
* ``minimum_angle``         -- reference src/metrics/exact.py:88-124, geometry.py:82-85
* ``edge_length_variation`` -- reference src/metrics/exact.py:127-142
* ``crossing_scan``         -- reference src/metrics/exact.py:145-222, geometry.py:62-79, 94-110
* ``edge_crossing`` / ``edge_crossing_angle`` -- src/metrics/exact.py:225-238

``crossing_scan`` is restated in the *dense tiled* form (no x-sort): for every
unordered pair (i < j) in original edge order it evaluates closed-bbox overlap
AND index-disjointness AND the four-cross-product straddle test.  The
reference's x-sort only prunes pairs whose bboxes cannot overlap, so the count
is identical; the deviation sum differs only in
summation order.

Parity pinning: tests/test_oracle_golden.py checks this module against the
reference's own known-answer tests and against golden values produced by the
reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi
_PAIR_BUDGET = 2_000_000


def occlusion_threshold(r: float) -> float:
    """(2r)^2 exactly as the reference computes it (src/metrics/exact.py:63)."""
    return (2.0 * r) ** 2


def node_occlusion(xy: np.ndarray, r: float) -> int:
    """Unordered vertex pairs with fl(fl(dx*dx)+fl(dy*dy)) < (2r)^2.

    Follows src/metrics/exact.py:55-74 (strict inequality, no FMA, every
    vertex including isolated ones).
    """
    n = len(xy)
    if n < 2:
        return 0
    x = np.ascontiguousarray(xy[:, 0])
    y = np.ascontiguousarray(xy[:, 1])
    thr = occlusion_threshold(r)
    total = 0
    block = max(1, _PAIR_BUDGET // n)
    for s in range(0, n - 1, block):
        e = min(n - 1, s + block)
        # rows s..e-1 against columns strictly to their right
        cols = slice(s + 1, n)
        dx = x[s:e, None] - x[None, cols]
        dy = y[s:e, None] - y[None, cols]
        close = dx * dx + dy * dy < thr
        upper = np.arange(s + 1, n)[None, :] > np.arange(s, e)[:, None]
        total += int(np.count_nonzero(close & upper))
    return total


def incident_angles(vx, vy, ux, uy):
    """Angle of u - v in [0, 2pi) -- src/geometry.py:82-85."""
    ang = np.arctan2(np.asarray(uy) - vy, np.asarray(ux) - vx)
    return np.where(ang < 0.0, ang + TWO_PI, ang)


def axis_angles(ax, ay, bx, by):
    """Undirected line angle mod pi -- src/geometry.py:94-97."""
    ang = np.arctan2(np.asarray(by) - ay, np.asarray(bx) - ax)
    return np.mod(ang, np.pi)


def crossing_angles(t1, t2):
    """Acute angle between two axis angles -- src/geometry.py:107-110."""
    d = np.abs(np.asarray(t1) - t2)
    return np.minimum(d, np.pi - d)


def vertex_angle_deviations(xy: np.ndarray, edges: np.ndarray) -> np.ndarray:
    """d_v per vertex of degree >= 1 -- src/metrics/exact.py:88-116."""
    v = np.concatenate([edges[:, 0], edges[:, 1]])
    u = np.concatenate([edges[:, 1], edges[:, 0]])
    ang = incident_angles(xy[v, 0], xy[v, 1], xy[u, 0], xy[u, 1])
    order = np.lexsort((ang, v))
    sv = v[order]
    sa = ang[order]
    starts = np.flatnonzero(np.concatenate(([True], sv[1:] != sv[:-1])))
    degs = np.diff(np.append(starts, len(sv)))
    wrap = TWO_PI - sa[starts + degs - 1] + sa[starts]
    diffs = np.diff(sa)
    diffs = np.where(sv[1:] == sv[:-1], diffs, np.inf)
    diffs = np.append(diffs, np.inf)
    inner = np.minimum.reduceat(diffs, starts)
    gap = np.minimum(inner, wrap)
    phi = TWO_PI / degs
    return (phi - gap) / phi


def minimum_angle(xy: np.ndarray, edges: np.ndarray) -> float:
    """1 - mean(d_v) over vertices of degree >= 1; 1.0 without edges
    (src/metrics/exact.py:119-124)."""
    if len(edges) == 0:
        return 1.0
    return 1.0 - float(np.mean(vertex_angle_deviations(xy, edges)))


def edge_lengths(xy: np.ndarray, edges: np.ndarray) -> np.ndarray:
    """sqrt(dx*dx + dy*dy) with d = b - a (src/metrics/exact.py:127-131)."""
    d = xy[edges[:, 1]] - xy[edges[:, 0]]
    return np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1])


def edge_length_variation(xy: np.ndarray, edges: np.ndarray) -> float:
    """Two-pass spread of edge lengths (src/metrics/exact.py:134-142)."""
    m = len(edges)
    if m <= 1:
        return 0.0
    lengths = edge_lengths(xy, edges)
    mean = float(np.mean(lengths))
    la = math.sqrt(float(np.sum((lengths - mean) ** 2)) / (m * mean * mean))
    return la / math.sqrt(m - 1)


def straddle_mask(ax, ay, bx, by, cx, cy, dx, dy):
    """The four cross products and straddle tests of src/geometry.py:62-79,
    same operand order, each product compared against zero separately."""
    abx = bx - ax
    aby = by - ay
    c1 = abx * (cy - ay) - aby * (cx - ax)
    c2 = abx * (dy - ay) - aby * (dx - ax)
    cdx = dx - cx
    cdy = dy - cy
    c3 = cdx * (ay - cy) - cdy * (ax - cx)
    c4 = cdx * (by - cy) - cdy * (bx - cx)
    s_cd = ((c1 <= 0.0) & (c2 >= 0.0)) | ((c1 >= 0.0) & (c2 <= 0.0))
    s_ab = ((c3 <= 0.0) & (c4 >= 0.0)) | ((c3 >= 0.0) & (c4 <= 0.0))
    return s_cd & s_ab


def crossing_scan(xy: np.ndarray, edges: np.ndarray, ideal=None):
    """(count, dev_sum) over unordered non-adjacent edge pairs.

    The predicate of src/metrics/exact.py:182-221 evaluated densely over the
    upper triangle in original edge order: closed bbox overlap in x and y,
    no shared vertex index, proper_intersection_mask.  dev_sum accumulates
    |ideal - crossing_angle| over hits (0.0 when ideal is None).
    """
    m = len(edges)
    if m < 2:
        return 0, 0.0
    e0 = edges[:, 0]
    e1 = edges[:, 1]
    ax, ay = xy[e0, 0], xy[e0, 1]
    bx, by = xy[e1, 0], xy[e1, 1]
    xmin = np.minimum(ax, bx)
    xmax = np.maximum(ax, bx)
    ymin = np.minimum(ay, by)
    ymax = np.maximum(ay, by)
    theta = axis_angles(ax, ay, bx, by) if ideal is not None else None
    total = 0
    dev = 0.0
    block = max(1, _PAIR_BUDGET // m)
    for s in range(0, m - 1, block):
        e = min(m - 1, s + block)
        i = np.arange(s, e)[:, None]
        j = np.arange(s + 1, m)[None, :]
        js = slice(s + 1, m)
        ok = j > i
        ok &= (xmax[None, js] >= xmin[s:e, None]) & (xmax[s:e, None] >= xmin[None, js])
        ok &= (ymax[None, js] >= ymin[s:e, None]) & (ymax[s:e, None] >= ymin[None, js])
        ok &= (e0[s:e, None] != e0[None, js]) & (e0[s:e, None] != e1[None, js])
        ok &= (e1[s:e, None] != e0[None, js]) & (e1[s:e, None] != e1[None, js])
        ii, jj = np.nonzero(ok)
        if len(ii) == 0:
            continue
        ii = ii + s
        jj = jj + s + 1
        hit = straddle_mask(ax[ii], ay[ii], bx[ii], by[ii], ax[jj], ay[jj], bx[jj], by[jj])
        total += int(np.count_nonzero(hit))
        if ideal is not None and np.any(hit):
            a = crossing_angles(theta[ii[hit]], theta[jj[hit]])
            dev += float(np.sum(np.abs(ideal - a)))
    return total, dev


def edge_crossing(xy, edges) -> int:
    """src/metrics/exact.py:225-227."""
    return crossing_scan(xy, edges)[0]


def edge_crossing_angle(xy, edges, ideal: float) -> float:
    """src/metrics/exact.py:230-238 (1.0 when there are no crossings)."""
    total, dev = crossing_scan(xy, edges, ideal)
    if total == 0:
        return 1.0
    return 1.0 - (dev / ideal) / total


def node_occlusion_grid(xy: np.ndarray, r: float) -> int:
    """Exact occlusion via cell bucketing, for sizes the dense oracle cannot
    reach.  Same predicate as node_occlusion; candidate pairs come from a
    2r-wide grid (the reference's exact grid variant, src/metrics/enhanced.py:
    56-127, is pinned to equal the dense oracle by its tests; this restates
    its idea with a 3x3 neighbourhood scan instead of multi-cell insertion).
    """
    n = len(xy)
    if n < 2:
        return 0
    thr = occlusion_threshold(r)
    w = 2.0 * r
    x = xy[:, 0]
    y = xy[:, 1]
    cx = np.floor((x - x.min()) / w).astype(np.int64)
    cy = np.floor((y - y.min()) / w).astype(np.int64)
    # floor rounding can misplace a point by one cell; scanning a 5x5
    # neighbourhood (offsets -2..2) makes the candidate set a safe superset
    ncy = int(cy.max()) + 5
    key = (cx + 2) * ncy + (cy + 2)
    order = np.argsort(key, kind="stable")
    skey = key[order]
    uniq, starts, counts = np.unique(skey, return_index=True, return_counts=True)
    total = 0
    for ox in range(-2, 3):
        for oy in range(-2, 3):
            off = ox * ncy + oy
            if (ox, oy) < (0, 0):
                continue
            # pair each point with points in the offset cell
            tgt = skey + off
            lo = np.searchsorted(skey, tgt, side="left")
            hi = np.searchsorted(skey, tgt, side="right")
            cnt = hi - lo
            src = np.repeat(np.arange(n), cnt)
            if len(src) == 0:
                continue
            base = np.repeat(lo, cnt)
            local = np.arange(len(src)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            dst = base + local
            if off == 0:
                keep = dst > src
                src = src[keep]
                dst = dst[keep]
            p = order[src]
            q = order[dst]
            ddx = x[p] - x[q]
            ddy = y[p] - y[q]
            total += int(np.count_nonzero(ddx * ddx + ddy * ddy < thr))
    return total


# -- unit-range partials (checks the kernels' tile-pair sharding contract) ----

def _tri_coords(u: int, T: int):
    """(ti, tj) of unit u in the row-major upper-triangular tile-pair order
    used by the kernels (paper_2411_09809_b200/csrc/common.cuh)."""
    ti = 0
    while u >= T - ti:
        u -= T - ti
        ti += 1
    return ti, ti + u


def _band_coords(u: int, T: int, W: int):
    """(ti, tj) of unit u in the banded order of the crossing pass: bands of W
    consecutive j-tiles; inside band [b0, e): rows ti < b0 (each over the
    band's w tiles), then the band's own triangle."""
    b0 = 0
    while True:
        e = min(T, b0 + W)
        w = e - b0
        count = b0 * w + w * (w + 1) // 2
        if u < count:
            break
        u -= count
        b0 = e
    if u < b0 * w:
        return u // w, b0 + u % w
    a, c = _tri_coords(u - b0 * w, w)
    return b0 + a, b0 + c


def crossing_scan_units(xy, edges, ideal, tile: int, ubeg: int, uend: int, band=None):
    """(count, dev_sum) restricted to pairs whose tile pair (i//tile, j//tile)
    has a unit index in [ubeg, uend) -- in the banded unit order with band
    width `band` tiles (None: one band, i.e. row-major).  Summing over a
    partition of [0, T(T+1)/2) gives crossing_scan()."""
    m = len(edges)
    T = max(1, -(-m // tile))
    W = T if band is None else int(band)
    e0, e1 = edges[:, 0], edges[:, 1]
    ax, ay, bx, by = xy[e0, 0], xy[e0, 1], xy[e1, 0], xy[e1, 1]
    xmin, xmax = np.minimum(ax, bx), np.maximum(ax, bx)
    ymin, ymax = np.minimum(ay, by), np.maximum(ay, by)
    theta = axis_angles(ax, ay, bx, by) if ideal is not None else None
    total, dev = 0, 0.0
    for u in range(ubeg, uend):
        ti, tj = _band_coords(u, T, W)
        I = np.arange(ti * tile, min(m, (ti + 1) * tile))[:, None]
        J = np.arange(tj * tile, min(m, (tj + 1) * tile))[None, :]
        if I.size == 0 or J.size == 0:
            continue
        ok = J > I
        ok &= (xmax[J] >= xmin[I]) & (xmax[I] >= xmin[J]) & (ymax[J] >= ymin[I]) & (ymax[I] >= ymin[J])
        ok &= (e0[I] != e0[J]) & (e0[I] != e1[J]) & (e1[I] != e0[J]) & (e1[I] != e1[J])
        ii, jj = np.nonzero(ok)
        ii = I[ii, 0]
        jj = J[0, jj]
        hit = straddle_mask(ax[ii], ay[ii], bx[ii], by[ii], ax[jj], ay[jj], bx[jj], by[jj])
        total += int(np.count_nonzero(hit))
        if ideal is not None and np.any(hit):
            dev += float(np.sum(np.abs(ideal - crossing_angles(theta[ii[hit]], theta[jj[hit]]))))
    return total, dev


def crossing_scan_tiles(xy, edges, ideal, tile: int, tile_pairs):
    """(count, dev_sum) over explicit tile pairs (ti, tj), ti <= tj, of the
    edge sequence `edges` (pairs j > i only when ti == tj) -- the unit of the
    culled candidate lists and of any edge order the kernels use."""
    m = len(edges)
    e0, e1 = edges[:, 0], edges[:, 1]
    ax, ay, bx, by = xy[e0, 0], xy[e0, 1], xy[e1, 0], xy[e1, 1]
    xmin, xmax = np.minimum(ax, bx), np.maximum(ax, bx)
    ymin, ymax = np.minimum(ay, by), np.maximum(ay, by)
    theta = axis_angles(ax, ay, bx, by) if ideal is not None else None
    total, dev = 0, 0.0
    for ti, tj in tile_pairs:
        I = np.arange(ti * tile, min(m, (ti + 1) * tile))[:, None]
        J = np.arange(tj * tile, min(m, (tj + 1) * tile))[None, :]
        if I.size == 0 or J.size == 0:
            continue
        ok = J > I
        ok &= (xmax[J] >= xmin[I]) & (xmax[I] >= xmin[J]) & (ymax[J] >= ymin[I]) & (ymax[I] >= ymin[J])
        ok &= (e0[I] != e0[J]) & (e0[I] != e1[J]) & (e1[I] != e0[J]) & (e1[I] != e1[J])
        ii, jj = np.nonzero(ok)
        ii = I[ii, 0]
        jj = J[0, jj]
        hit = straddle_mask(ax[ii], ay[ii], bx[ii], by[ii], ax[jj], ay[jj], bx[jj], by[jj])
        total += int(np.count_nonzero(hit))
        if ideal is not None and np.any(hit):
            dev += float(np.sum(np.abs(ideal - crossing_angles(theta[ii[hit]], theta[jj[hit]]))))
    return total, dev


# Interleaved ownership of the crossing pass's units across ranks (restates
# csrc/crossing.cu chunk_for and the chunk loop of the pair kernels: rank r
# of `world` takes the chunks ch = r, r + world, r + 2 world, ...).  The
# build-time constants are the library's defaults: 148 SMs (B200) x 4 CTAs
# per SM as the reference CTA count, chunks of at most 256 units.
CHUNK_CTA_REF = 148 * 4
CHUNK_MAX = 256


def interleaved_chunk(span: int, world: int) -> int:
    if span == 0 or world < 1:
        return 1
    c = span // (min(span, CHUNK_CTA_REF) * 8 * world)
    return max(1, min(CHUNK_MAX, c))


def interleaved_owner(u: int, ubeg: int, chunk: int, world: int) -> int:
    return ((u - ubeg) // chunk) % world


def crossing_scan_interleaved(xy, edges, ideal, tile: int, rank: int, world: int, band=None):
    """(count, dev_sum) of the units rank `rank` owns under interleaved chunk
    ownership of the whole unit space [0, T(T+1)/2)."""
    m = len(edges)
    T = max(1, -(-m // tile))
    U = T * (T + 1) // 2
    chunk = interleaved_chunk(U, world)
    total, dev = 0, 0.0
    for ch in range(rank, -(-U // chunk), world):
        b, e = ch * chunk, min(U, (ch + 1) * chunk)
        c, d = crossing_scan_units(xy, edges, ideal, tile, b, e, band)
        total += c
        dev += d
    return total, dev


def crossing_scan_rows(xy, edges, ideal, tile: int, rank: int, world: int):
    """(count, dev_sum) of the tile pairs (ti <= tj) whose row ti = rank (mod
    world): row ownership of the culled plan (glr_crossing_candidates_rows --
    the ranks' lists partition the classified list by rows, and the dropped
    tile pairs hold no crossing, so the ranks' shares partition the dense
    triangle the same way)."""
    m = len(edges)
    T = max(1, -(-m // tile))
    pairs = [(ti, tj) for ti in range(rank, T, world) for tj in range(ti, T)]
    return crossing_scan_tiles(xy, edges, ideal, tile, pairs)


def node_occlusion_units(xy, r, tile: int, ubeg: int, uend: int) -> int:
    """Occluding pairs restricted to vertex tile-pair units [ubeg, uend)."""
    n = len(xy)
    T = max(1, -(-n // tile))
    thr = occlusion_threshold(r)
    x, y = xy[:, 0], xy[:, 1]
    total = 0
    for u in range(ubeg, uend):
        ti, tj = _tri_coords(u, T)
        I = np.arange(ti * tile, min(n, (ti + 1) * tile))[:, None]
        J = np.arange(tj * tile, min(n, (tj + 1) * tile))[None, :]
        if I.size == 0 or J.size == 0:
            continue
        dx = x[I] - x[J]
        dy = y[I] - y[J]
        total += int(np.count_nonzero((dx * dx + dy * dy < thr) & (J > I)))
    return total


# ---- force-directed layout --------------------------

def fr_layout_positions(n: int, ei: np.ndarray, ej: np.ndarray, iterations: int, seed: int,
                        extent: float) -> np.ndarray:
    """Final positions of the reference's fr_layout (graphio.py:151-197) for n
    vertices and normalized index edges (ei, ej).

    Restated row by row: each vertex's repulsion is the numpy sum over the
    full row of (p_i - p_j) * k^2 / max(|p_i - p_j|^2, 1e-12), which numpy
    reduces with its pairwise summation, so the row sums are bit-identical
    to the reference's blocked evaluation; the spring pulls are scattered
    with np.add.at in edge order (first -pull at ei, then +pull at ej).
    """
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, extent, size=(n, 2))
    k = extent / math.sqrt(n)
    ksq = k * k
    t = extent / 10.0
    rows = max(1, 1_000_000 // n)
    for _ in range(iterations):
        disp = np.zeros((n, 2))
        for s in range(0, n, rows):
            e = min(n, s + rows)
            dx = pos[s:e, 0][:, None] - pos[:, 0][None, :]
            dy = pos[s:e, 1][:, None] - pos[:, 1][None, :]
            d2 = np.maximum(dx * dx + dy * dy, 1e-12)
            coef = ksq / d2
            disp[s:e, 0] += (dx * coef).sum(axis=1)
            disp[s:e, 1] += (dy * coef).sum(axis=1)
        dxy = pos[ei] - pos[ej]
        dist = np.sqrt(dxy[:, 0] * dxy[:, 0] + dxy[:, 1] * dxy[:, 1])
        pull = dxy * (dist / k)[:, None]
        np.add.at(disp, ei, -pull)
        np.add.at(disp, ej, pull)
        length = np.maximum(np.sqrt(disp[:, 0] * disp[:, 0] + disp[:, 1] * disp[:, 1]), 1e-12)
        pos = pos + disp * (np.minimum(length, t) / length)[:, None]
        t *= 0.95
    lo = pos.min(axis=0)
    span = pos.max(axis=0) - lo
    span[span <= 0] = 1.0
    return (pos - lo) / span * extent


# ---- strip sweeps -----------------------------------

def strip_crossings(xy: np.ndarray, edges: np.ndarray, fraction: float, orientation: str,
                    ideal=None):
    """(strip crossings, deviation sum) of one orientation of the reference's
    strip sweep (metrics/enhanced.py:133-215 strips, sweep.py:60-108 count,
    sweep.py:110-402 deviation), restated by pair enumeration per strip:
    a pair is counted when its l- and r-orders strictly disagree (the sweep's
    tie rule) and contributes |ideal - a_c|.  O(S^2) per strip: small inputs.
    """
    if orientation == "horizontal":
        axis_c, ord_c = xy[:, 1], xy[:, 0]
    else:
        axis_c, ord_c = xy[:, 0], xy[:, 1]
    lo, hi = float(axis_c.min()), float(axis_c.max())
    nstrips = math.ceil(1.0 / fraction)
    width = (hi - lo) / nstrips
    bounds = lo + np.arange(nstrips + 1) * width
    bounds[-1] = hi
    x0, y0 = axis_c[edges[:, 0]], ord_c[edges[:, 0]]
    x1, y1 = axis_c[edges[:, 1]], ord_c[edges[:, 1]]
    swap = x1 < x0
    sx0, sy0 = np.where(swap, x1, x0), np.where(swap, y1, y0)
    sx1, sy1 = np.where(swap, x0, x1), np.where(swap, y0, y1)
    kf = np.searchsorted(bounds, sx0, side="left")
    kl = np.searchsorted(bounds, sx1, side="right") - 1
    total, dev = 0, 0.0
    for k in range(nstrips):
        sel = np.flatnonzero((kf <= k) & (k < kl))
        if len(sel) < 2:
            continue
        slope = (sy1[sel] - sy0[sel]) / (sx1[sel] - sx0[sel])
        lv = sy0[sel] + slope * (bounds[k] - sx0[sel])
        rv = sy0[sel] + slope * (bounds[k + 1] - sx0[sel])
        i, j = np.triu_indices(len(sel), 1)
        inv = ((lv[i] < lv[j]) & (rv[i] > rv[j])) | ((lv[i] > lv[j]) & (rv[i] < rv[j]))
        total += int(np.count_nonzero(inv))
        if ideal is not None and inv.any():
            th = axis_angles(sx0[sel], sy0[sel], sx1[sel], sy1[sel])
            dev += float(np.sum(np.abs(ideal - crossing_angles(th[i[inv]], th[j[inv]]))))
    return total, dev
