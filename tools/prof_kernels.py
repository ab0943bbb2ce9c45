"""Small driver for ncu captures: one fused crossing pass, one E_c pass and one
occlusion pass on a C5-shaped graph (Chung-Lu, 2^16 lattice) with m edges."""
import argparse, sys
sys.path.insert(0, '.')
import torch
from paper_2411_09809_b200 import metrics as M, configs

ap = argparse.ArgumentParser()
ap.add_argument('--m', type=int, default=100_000)
ap.add_argument('--reps', type=int, default=2)
a = ap.parse_args()
g, _ = configs.config5(n=a.m * 3 // 8, m=a.m)
dg = M.DeviceGraph.from_graph(g)
for _ in range(a.reps):
    rec = M.CrossingRecords(dg, order="theta")
    out = rec.partial(configs.IDEAL_70, 0, rec.units)
    out2 = rec.partial(None, 0, rec.units)
    o = M.occlusion_partial(dg, M.occlusion_threshold(8.0), 0, M.occlusion_units(g.num_vertices))
torch.cuda.synchronize()
print('count', out.tolist(), out2.tolist(), o.item())
