"""How many (i-slice x j-block) pair blocks of the culled C5 plan have
disjoint bounding boxes (could be skipped exactly), at several block shapes,
and the pair-level bbox-overlap fraction, on a sample of candidate units:
    python tools/cull_block_stats.py [samples]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs, _lib

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
L = _lib.lib()
es = torch.empty_like(dg.edges)
L.glr_spatial_sort_edges(dg.xy.data_ptr(), dg.num_vertices, dg.edges.data_ptr(), dg.num_edges,
                         es.data_ptr(), torch.cuda.current_stream().cuda_stream)
rec = M.CrossingRecords(dg, "culled")
lst = rec.list.cpu().numpy().reshape(-1, 2)
E = es.cpu().numpy()
xy = g.xy
ax, ay, bx, by = xy[E[:, 0], 0], xy[E[:, 0], 1], xy[E[:, 1], 0], xy[E[:, 1], 1]
box = np.stack([np.minimum(ax, bx), np.maximum(ax, bx), np.minimum(ay, by), np.maximum(ay, by)], 1)
m = len(E)
T = 256
rng = np.random.default_rng(0)
pick = lst[rng.choice(len(lst), size=min(S, len(lst)), replace=False)]
print(f"candidate units {len(lst)} of {(m // T + 1) * (m // T + 2) // 2}")


def blocks(b, size):
    n = len(b) // size
    b = b[: n * size].reshape(n, size, 4)
    return np.stack([b[:, :, 0].min(1), b[:, :, 1].max(1), b[:, :, 2].min(1), b[:, :, 3].max(1)], 1)


pair_ov = []
res = {}
for ti, tj in pick:
    bi = box[ti * T:(ti + 1) * T]
    bj = box[tj * T:(tj + 1) * T]
    if len(bi) < T or len(bj) < T:
        continue
    ov = ((bi[:, None, 1] >= bj[None, :, 0]) & (bj[None, :, 1] >= bi[:, None, 0]) &
          (bi[:, None, 3] >= bj[None, :, 2]) & (bj[None, :, 3] >= bi[:, None, 2]))
    pair_ov.append(ov.mean())
    for si, sj in ((128, 4), (128, 8), (128, 16), (64, 4), (32, 4), (32, 8)):
        A, B = blocks(bi, si), blocks(bj, sj)
        o = ((A[:, None, 1] >= B[None, :, 0]) & (B[None, :, 1] >= A[:, None, 0]) &
             (A[:, None, 3] >= B[None, :, 2]) & (B[None, :, 3] >= A[:, None, 2]))
        res.setdefault((si, sj), []).append(o.mean())
print(f"pair-level bbox overlap in candidate units: {np.mean(pair_ov):.3f}")
for k, v in res.items():
    print(f"i-slice {k[0]:4d} x j-block {k[1]:3d}: overlapping blocks {np.mean(v):.3f}")
