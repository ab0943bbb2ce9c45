"""Projected strong scaling: time each of G interleaved shares of the C5
fused pass back to back on one GPU (dense direction order and culled plan),
plus the per-rank plan build.   python tools/shares_time.py [G ...]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
ev = lambda: torch.cuda.Event(enable_timing=True)
for strategy, order in (("dense", "theta"), ("culled", "input")):
    a, b = ev(), ev()
    M.CrossingRecords(dg, strategy, order); torch.cuda.synchronize()
    a.record(); rec = M.CrossingRecords(dg, strategy, order); b.record(); torch.cuda.synchronize()
    plan_ms = a.elapsed_time(b)
    a.record(); whole = rec.partial_interleaved(p["ideal"], 0, 1); b.record(); torch.cuda.synchronize()
    t1 = a.elapsed_time(b)
    for G in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
        ts = []
        tot = 0.0
        for r in range(G):
            a.record(); out = rec.partial_interleaved(p["ideal"], r, G); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b)); tot += out[0].item()
        assert tot == whole[0].item()
        eff = (plan_ms + t1) / (G * (plan_ms + max(ts)))
        print(f"{strategy:6s} G={G}: plan {plan_ms:.1f} ms, whole {t1:.0f} ms, shares max {max(ts):.1f} "
              f"mean {sum(ts) / G:.1f} ms -> projected strong-scaling efficiency {eff:.3f}", flush=True)

# culled plan with the tile ROWS dealt to the ranks (what sharded_evaluate runs
# for world > 1): each rank's plan build + pass, wall clock
import time


def rank_time(rows):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rec = M.CrossingRecords(dg, "culled", rows=rows)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r, w = rows if rows else (0, 1)
    out = rec.partial_interleaved(p["ideal"], r, w)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return 1e3 * (t1 - t0), 1e3 * (t2 - t1), out[0].item()


rank_time(None)
plan1, pass1, whole = rank_time(None)
for G in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
    res = [rank_time((r, G)) for r in range(G)]
    assert sum(x[2] for x in res) == whole
    worst = max(a + b for a, b, _ in res)
    print(f"culled rows G={G}: whole plan {plan1:.0f} + pass {pass1:.0f} ms; per rank plan "
          f"{max(a for a, _, _ in res):.0f} ms, pass max {max(b for _, b, _ in res):.0f} "
          f"mean {sum(b for _, b, _ in res) / G:.0f} ms -> projected strong-scaling efficiency "
          f"{(plan1 + pass1) / (G * worst):.3f}", flush=True)
