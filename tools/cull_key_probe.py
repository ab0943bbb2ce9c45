"""CPU estimate of culled crossing plans for different edge orders on a
config (default C5): candidate tile pairs (tile bboxes overlap) and the
share of them that the filter kernel can run in the signed angle form
(crossing.cu unit_shift), plus a cost estimate  units * (signed ? 1 : r).

    python tools/cull_key_probe.py [config] [r]
"""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2411_09809_b200 import configs  # noqa: E402

TILE = 256
HALF_PI = math.pi / 2
MARGIN = 2.0**-8


def spread(v, bits, dims):
    out = np.zeros_like(v, dtype=np.uint64)
    for i in range(bits):
        out |= ((v >> np.uint64(i)) & np.uint64(1)) << np.uint64(dims * i)
    return out


def q(v, lo, hi, bits):
    s = (2**bits - 1) / (hi - lo) if hi > lo else 0.0
    return np.clip(((v - lo) * s), 0, 2**bits - 1).astype(np.uint64)


def hub_groups(edges, n, hub):
    deg = np.bincount(edges.ravel(), minlength=n)
    du, dv = deg[edges[:, 0]], deg[edges[:, 1]]
    h = np.where(du >= dv, edges[:, 0], edges[:, 1])
    return np.where(np.maximum(du, dv) >= hub, h + 1, 0).astype(np.uint64)


def key_box4(xy, edges, theta, n, bits=8, hub=16384):
    a, b = xy[edges[:, 0]], xy[edges[:, 1]]
    x0, x1 = xy[:, 0].min(), xy[:, 0].max()
    y0, y1 = xy[:, 1].min(), xy[:, 1].max()
    mk = (spread(q(np.minimum(a[:, 0], b[:, 0]), x0, x1, bits), bits, 4)
          | spread(q(np.maximum(a[:, 0], b[:, 0]), x0, x1, bits), bits, 4) << np.uint64(1)
          | spread(q(np.minimum(a[:, 1], b[:, 1]), y0, y1, bits), bits, 4) << np.uint64(2)
          | spread(q(np.maximum(a[:, 1], b[:, 1]), y0, y1, bits), bits, 4) << np.uint64(3))
    up = ((b[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]) >= 0).astype(np.uint64)
    return [hub_groups(edges, n, hub), mk, up]


def key_box5(xy, edges, theta, n, bits=6, tbits=6, hub=16384):
    a, b = xy[edges[:, 0]], xy[edges[:, 1]]
    x0, x1 = xy[:, 0].min(), xy[:, 0].max()
    y0, y1 = xy[:, 1].min(), xy[:, 1].max()
    qs = [q(np.minimum(a[:, 0], b[:, 0]), x0, x1, bits), q(np.maximum(a[:, 0], b[:, 0]), x0, x1, bits),
          q(np.minimum(a[:, 1], b[:, 1]), y0, y1, bits), q(np.maximum(a[:, 1], b[:, 1]), y0, y1, bits),
          q(theta, 0.0, math.pi, tbits)]
    mk = np.zeros(len(edges), dtype=np.uint64)
    for d, v in enumerate(qs):
        mk |= spread(v, max(bits, tbits), 5) << np.uint64(d)
    return [hub_groups(edges, n, hub), mk]


def key_theta_top(xy, edges, theta, n, tbits=3, bits=8, hub=16384):
    g, mk, up = key_box4(xy, edges, theta, n, bits, hub)
    return [g, q(theta, 0.0, math.pi, tbits), mk, up]


def evaluate(name, keys, xy, edges, theta, r):
    order = np.lexsort(keys[::-1])
    e = edges[order]
    th = theta[order]
    a, b = xy[e[:, 0]], xy[e[:, 1]]
    m = len(e)
    T = -(-m // TILE)
    pad = T * TILE - m

    def tiles(v, fill):
        return np.concatenate([v, np.full(pad, fill)]).reshape(T, TILE)

    bx0 = tiles(np.minimum(a[:, 0], b[:, 0]), np.inf).min(1)
    bx1 = tiles(np.maximum(a[:, 0], b[:, 0]), -np.inf).max(1)
    by0 = tiles(np.minimum(a[:, 1], b[:, 1]), np.inf).min(1)
    by1 = tiles(np.maximum(a[:, 1], b[:, 1]), -np.inf).max(1)
    tlo = tiles(th, np.inf).min(1)
    thi = tiles(th, -np.inf).max(1)
    cand = signed = 0
    for i in range(T):
        j = np.arange(i, T)
        ok = (bx1[j] >= bx0[i]) & (bx1[i] >= bx0[j]) & (by1[j] >= by0[i]) & (by1[i] >= by0[j])
        cand += int(ok.sum())
        j = j[ok & (j != i)]
        lo = tlo[j] - thi[i]
        hi = thi[j] - tlo[i]
        s = np.full(len(j), np.nan)
        c1 = (lo >= 0) & (hi <= HALF_PI)
        c2 = lo >= HALF_PI
        c3 = (hi <= 0) & (lo >= -HALF_PI)
        c4 = hi <= -HALF_PI
        s[c1] = IDEAL
        s[c2] = math.pi - IDEAL
        s[c3] = -IDEAL
        s[c4] = IDEAL - math.pi
        sg = (hi <= s - MARGIN) | (lo >= s + MARGIN)
        signed += int(sg.sum())
    U = T * (T + 1) // 2
    cost = signed + r * (cand - signed)
    print(f"{name:28s} candidates {cand:>11,d} ({cand / U:.3f})  signed {signed / max(cand, 1):.3f}  "
          f"cost {cost / U:.3f}", flush=True)


if __name__ == "__main__":
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    r = float(sys.argv[2]) if len(sys.argv) > 2 else 1.47
    g, p = configs.make(k)
    IDEAL = p["ideal"]
    xy, edges = g.xy, g.edges
    a, b = xy[edges[:, 0]], xy[edges[:, 1]]
    theta = np.mod(np.arctan2(b[:, 1] - a[:, 1], b[:, 0] - a[:, 0]), np.pi)
    n = g.num_vertices
    for name, fn in [
        ("box4 (current)", lambda: key_box4(xy, edges, theta, n)),
        ("theta3 + box4", lambda: key_theta_top(xy, edges, theta, n, 3)),
        ("theta4 + box4", lambda: key_theta_top(xy, edges, theta, n, 4)),
        ("theta5 + box4", lambda: key_theta_top(xy, edges, theta, n, 5)),
        ("box5 6/6", lambda: key_box5(xy, edges, theta, n, 6, 6)),
        ("box5 7/7", lambda: key_box5(xy, edges, theta, n, 7, 7)),
    ]:
        evaluate(name, fn(), xy, edges, theta, r)
