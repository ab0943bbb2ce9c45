"""Dense C5 node-occlusion pass time (occlusion_filter_kernel):
    python tools/occ_time.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
n = g.num_vertices
thr = M.occlusion_threshold(p["radius"])
U = M.occlusion_units(n)
M.occlusion_partial(dg, thr, 0, U); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    out = M.occlusion_partial(dg, thr, 0, U)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"C5 dense N_c {out.item():.0f} in {ms:.1f} ms = {n * (n - 1) / 2 / ms / 1e9:.3f} Tpairs/s")
