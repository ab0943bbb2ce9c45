"""One E_c+E_ca launch (or count-only with `count`) over C5, for ncu captures:
    ncu -k regex:cross_filter_kernel -c 1 python tools/c5_once.py [world] [count]
With world > 1 the launch covers rank 0's interleaved share (1/world of the
units, the same unit mix as the whole pass) so a full ncu replay stays short."""
import sys, torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs
world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
count_only = "count" in sys.argv[2:]
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg, order="theta")
out = rec.partial_interleaved(None if count_only else p["ideal"], 0, world)
torch.cuda.synchronize()
print("mode", rec.mode(), "count", out[0].item(), "dev", out[1].item())
