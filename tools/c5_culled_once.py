"""One fused E_c+E_ca launch of the culled C5 plan (for ncu captures):
    ncu -k regex:cross_filter_kernel -c 1 python tools/c5_culled_once.py [world]
world > 1 keeps rank 0's interleaved share of the candidate list."""
import sys, torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs
world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg, "culled")
out = rec.partial_interleaved(p["ideal"], 0, world)
torch.cuda.synchronize()
print("units", rec.units, "count", out[0].item(), "dev", out[1].item())
