"""Culled crossing plans by config: candidate units and fused time
    python tools/cull_probe.py [configs...]"""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

for k in [int(a) for a in sys.argv[1:]] or [3, 5]:
    g, p = configs.make(k)
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg, "culled")
    out = rec.partial(p["ideal"], 0, rec.units); torch.cuda.synchronize()
    t0 = time.perf_counter()
    rec = M.CrossingRecords(dg, "culled")
    out = rec.partial(p["ideal"], 0, rec.units).tolist(); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"C{k}: units {rec.units} of {M.crossing_units(g.num_edges)} "
          f"({rec.units / M.crossing_units(g.num_edges):.4f}) time {dt * 1e3:.1f} ms {out}", flush=True)
