"""Time the C5 crossing pass the way the public API runs it: dense
direction-ordered fused E_c+E_ca, the count-only pass, and the culled plan
(plan build included), each repeated; prints counts, dev sums and times.
    python tools/c5_fused.py [reps]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
ideal = p["ideal"]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn):
    torch.cuda.synchronize()
    ev[0].record()
    out = fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]), out.tolist()


rec = M.CrossingRecords(dg, "dense", "theta")
rec.partial(ideal, 0, 100)
for r in range(reps):
    ms, o = timed(lambda: rec.partial_interleaved(ideal, 0, 1))
    print(f"dense theta fused: {ms:.1f} ms {8e12 / ms / 1e9:.4f} Tpairs/s count {o[0]:.0f} dev {o[1]!r}",
          flush=True)
for r in range(reps):
    ms, o = timed(lambda: rec.partial_interleaved(None, 0, 1))
    print(f"dense theta count: {ms:.1f} ms {8e12 / ms / 1e9:.4f} Tpairs/s count {o[0]:.0f}", flush=True)
del rec
for r in range(reps):
    t0 = time.perf_counter()
    ms, o = timed(lambda: M.CrossingRecords(dg, "culled").partial_interleaved(ideal, 0, 1))
    print(f"culled fused (plan incl.): {ms:.1f} ms {8e12 / ms / 1e9:.4f} Tpairs/s count {o[0]:.0f} "
          f"dev {o[1]!r}", flush=True)
