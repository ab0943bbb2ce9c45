"""Small driver for ncu captures: one fused crossing pass and one occlusion
pass on synthetic uniform segments (m edges, 2m vertices)."""
import argparse, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2411_09809_b200 as G
from paper_2411_09809_b200 import metrics as M, configs

ap = argparse.ArgumentParser()
ap.add_argument('--m', type=int, default=100_000)
ap.add_argument('--config', type=int, default=0)
ap.add_argument('--reps', type=int, default=2)
a = ap.parse_args()
if a.config:
    g, p = configs.make(a.config)
else:
    n = 2 * a.m
    xy = np.random.default_rng(3).uniform(0, 1, (n, 2))
    e = np.stack([np.arange(0, n, 2), np.arange(1, n, 2)], 1)
    g = G.LayoutGraph.from_normalized(xy, e)
dg = M.DeviceGraph.from_graph(g)
for _ in range(a.reps):
    rec = M.CrossingRecords(dg)
    out = rec.partial(configs.IDEAL_70, 0, rec.units)
    out2 = rec.partial(None, 0, rec.units)
    o = M.occlusion_partial(dg, M.occlusion_threshold(1e-4), 0, M.occlusion_units(g.num_vertices))
torch.cuda.synchronize()
print('count', out.tolist(), out2.tolist(), o.item())
