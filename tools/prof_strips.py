"""One strip count on C5 (ncu launch list): python tools/prof_strips.py FRACTION"""
import sys; sys.path.insert(0, ".")
import torch
from paper_2411_09809_b200 import configs, edge_crossing_enhanced
from paper_2411_09809_b200 import metrics as M
g, p = configs.make(5)
dg = M.DeviceGraph.from_graph(g)
frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.05
print(edge_crossing_enhanced(dg, frac))
torch.cuda.synchronize()
