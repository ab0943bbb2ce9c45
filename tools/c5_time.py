"""Time the full C5 fused crossing pass (and 8-way interleaved shares)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg)
rec.partial(p["ideal"], 0, 1000); torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); out = rec.partial_interleaved(p["ideal"], 0, 1); t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1)
times = []
for r in range(8):
    t0.record(); rec.partial_interleaved(p["ideal"], r, 8); t1.record(); torch.cuda.synchronize()
    times.append(t0.elapsed_time(t1))
print(f"full {ms:.0f} ms {8e12 / ms / 1e9:.3f} Tpairs/s count {out[0].item():.0f} | 8-way max {max(times):.0f} "
      f"mean {sum(times) / 8:.0f}", flush=True)
