"""Fraction of culled C5 units (4-D bbox Morton order) whose theta-difference
range allows the one-DADD signed angle form (crossing.cu unit_shift), at
tile level and at finer (i-part x j-part) granularity with theta-sorted
tiles:  python tools/culled_angle_stats.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs, _lib

g, p = configs.config5()
ideal = p["ideal"]
dg = M.DeviceGraph.from_graph(g)
L = _lib.lib()
es = torch.empty_like(dg.edges)
L.glr_spatial_sort_edges(dg.xy.data_ptr(), dg.num_vertices, dg.edges.data_ptr(), dg.num_edges,
                         es.data_ptr(), torch.cuda.current_stream().cuda_stream)
rec = M.CrossingRecords(dg, "culled")
lst = rec.list.cpu().numpy().reshape(-1, 2).astype(np.int64)
E = es.cpu().numpy()
xy = g.xy
ax, ay, bx, by = xy[E[:, 0], 0], xy[E[:, 0], 1], xy[E[:, 1], 0], xy[E[:, 1], 1]
th = np.mod(np.arctan2(by - ay, bx - ax), np.pi)
m = len(E)
T = 256
nt = -(-m // T)
thp = np.concatenate([th, np.full(nt * T - m, np.nan)]).reshape(nt, T)
rng = np.random.default_rng(0)
sel = lst[rng.choice(len(lst), min(len(lst), 2_000_000), replace=False)]
sel = sel[sel[:, 0] != sel[:, 1]]
HP, MARGIN = np.pi / 2, 2.0 ** -8


def classified(lo_i, hi_i, lo_j, hi_j):
    lo = lo_j - hi_i
    hi = hi_j - lo_i
    sh = np.full(lo.shape, np.nan)
    sh[(lo >= 0) & (hi <= HP)] = ideal
    sh[lo >= HP] = np.pi - ideal
    sh[(hi <= 0) & (lo >= -HP)] = -ideal
    sh[hi <= -HP] = ideal - np.pi
    return ~np.isnan(sh) & ((hi <= sh - MARGIN) | (lo >= sh + MARGIN))


print(f"candidate units {len(lst)}, sampled {len(sel)}")
for parts_i, parts_j, sort in ((1, 1, False), (1, 1, True), (2, 1, True), (2, 2, True),
                               (2, 4, True), (2, 16, True), (2, 64, True)):
    tp = np.sort(thp, axis=1) if sort else thp
    wi, wj = T // parts_i, T // parts_j
    lo_i = np.nanmin(tp.reshape(nt, parts_i, wi), 2)
    hi_i = np.nanmax(tp.reshape(nt, parts_i, wi), 2)
    lo_j = np.nanmin(tp.reshape(nt, parts_j, wj), 2)
    hi_j = np.nanmax(tp.reshape(nt, parts_j, wj), 2)
    tot = 0.0
    for a in range(parts_i):
        for b in range(parts_j):
            tot += classified(lo_i[sel[:, 0], a], hi_i[sel[:, 0], a],
                              lo_j[sel[:, 1], b], hi_j[sel[:, 1], b]).mean()
    print(f"i parts {parts_i} x j parts {parts_j} (theta-sorted tiles: {sort}): "
          f"classified {tot / (parts_i * parts_j):.3f}; median tile theta span "
          f"{np.nanmedian(np.nanmax(thp, 1) - np.nanmin(thp, 1)):.3f}")
