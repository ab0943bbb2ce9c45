"""Time the full C5 fused crossing pass (and 8-way interleaved shares) per
pair-kernel mode and edge order:
    python tools/c5_time.py [mode ...]   (default: 2 1; GLR_ORDER=input|theta|both)."""
import os
import sys, torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
modes = [int(a) for a in sys.argv[1:]] or [2, 1]
orders = {"both": ["theta", "input"]}.get(os.environ.get("GLR_ORDER", "both"),
                                           [os.environ.get("GLR_ORDER")])
for mode, order in [(m_, o_) for m_ in modes for o_ in orders]:
    rec = M.CrossingRecords(dg, order=order).set_mode(mode)
    rec.partial(p["ideal"], 0, 1000); torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    res = []
    for angle in (p["ideal"], None):
        t0.record(); out = rec.partial_interleaved(angle, 0, 1); t1.record(); torch.cuda.synchronize()
        res.append((t0.elapsed_time(t1), out.tolist()))
    times = []
    for r in range(8):
        t0.record(); rec.partial_interleaved(p["ideal"], r, 8); t1.record(); torch.cuda.synchronize()
        times.append(t0.elapsed_time(t1))
    (ms, o), (ms_ec, o_ec) = res
    print(f"order {order} mode {rec.mode()} fused {ms:.0f} ms {8e12 / ms / 1e9:.3f} Tpairs/s count {o[0]:.0f} dev {o[1]!r} "
          f"| ec {ms_ec:.0f} ms {8e12 / ms_ec / 1e9:.3f} Tpairs/s count {o_ec[0]:.0f} "
          f"| 8-way max {max(times):.0f} mean {sum(times) / 8:.0f}", flush=True)
