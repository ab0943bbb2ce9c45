"""Dense fused C5 pass time vs the hub-group degree of the direction order
(metrics.HUB_DEGREE; 0 = library default):
    python tools/hub_sweep.py 0 2048 4096 8192"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
ideal = p["ideal"]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for hd in [int(a) for a in sys.argv[1:]]:
    M.HUB_DEGREE = hd
    rec = M.CrossingRecords(dg, "dense", "theta")
    rec.partial(ideal, 0, 200)
    torch.cuda.synchronize()
    e0.record()
    out = rec.partial_interleaved(ideal, 0, 1)
    e1.record()
    torch.cuda.synchronize()
    print(f"hub_degree {hd}: {e0.elapsed_time(e1):.1f} ms count {out[0].item():.0f} "
          f"dev {out[1].item()!r}", flush=True)
    del rec
