"""Per-phase device time of one bench step on C5 (records build by order,
pair pass):  python tools/step_probe.py"""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
ev = lambda: torch.cuda.Event(enable_timing=True)
for order in ("theta", "input"):
    for it in range(3):
        a, b, c = ev(), ev(), ev()
        torch.cuda.synchronize(); h0 = time.perf_counter()
        a.record()
        rec = M.CrossingRecords(dg, order=order)
        b.record(); h1 = time.perf_counter()
        out = rec.partial_interleaved(p["ideal"], 0, 1)
        c.record(); torch.cuda.synchronize()
        print(f"{order} it{it}: records {a.elapsed_time(b):.2f} ms (host {1e3 * (h1 - h0):.2f} ms) "
              f"pass {b.elapsed_time(c):.1f} ms", flush=True)
        del rec
