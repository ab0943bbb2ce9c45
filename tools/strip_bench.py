"""Strip-sweep timing on the BASELINE configs (count only and with angle).
python tools/strip_bench.py [config ...]"""
import json, math, sys, time
sys.path.insert(0, ".")
import torch
from paper_2411_09809_b200 import configs, crossing_angle_stats, edge_crossing_enhanced
from paper_2411_09809_b200 import metrics as M

IDEAL = math.radians(70.0)
for k in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    g, p = configs.make(k)
    dg = M.DeviceGraph.from_graph(g)
    for frac in (0.05, 0.1):
        row = {"config": k, "m": g.num_edges, "fraction": frac}
        for name, fn in (("count", lambda: edge_crossing_enhanced(dg, frac)),
                         ("stats", lambda: crossing_angle_stats(dg, frac, IDEAL))):
            fn(); torch.cuda.synchronize()
            t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
            row[name] = {"s": round(time.perf_counter() - t0, 4), "result": r}
        print(json.dumps(row), flush=True)
