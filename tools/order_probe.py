"""C5 pair-kernel time by edge order over one unit range (count-only and
fused):  python tools/order_probe.py [units]   -- for ncu A/B captures."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
U = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
for order in ("input", "theta"):
    rec = M.CrossingRecords(dg, order=order)
    for angle in (None, p["ideal"]):
        rec.partial(angle, 0, 1000)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(); out = rec.partial(angle, 0, U); t1.record(); torch.cuda.synchronize()
        print(f"{order:5s} {'fused' if angle else 'count'} {t0.elapsed_time(t1):8.2f} ms "
              f"{out.tolist()}", flush=True)
