"""One fused E_c+E_ca launch over all of C5 (for ncu captures of the full
launch: ncu -k regex:cross_filter_kernel -c 1 python tools/c5_once.py)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg, order="theta")
out = rec.partial_interleaved(p["ideal"], 0, 1)
torch.cuda.synchronize()
print("mode", rec.mode(), "count", out[0].item(), "dev", out[1].item())
