"""Per-step timing of the culled C5 plan after two dense passes (the context of
bench.py's crossing_culled item): plan build, pass, release.
    python tools/culled_steps.py"""
import sys, time, torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs, sharding
g, p = configs.config5(); dg = M.DeviceGraph.from_graph(g); ideal = p["ideal"]
out = torch.zeros(3, dtype=torch.float64, device="cuda")
# mimic bench: dense steps first
for _ in range(2):
    rec = M.CrossingRecords(dg, order="theta"); rec.partial_interleaved(ideal, 0, 1, out=out[0:2]); del rec
torch.cuda.synchronize()
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rec = M.CrossingRecords(dg, "culled")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    rec.partial_interleaved(ideal, 0, 1, out=out[0:2])
    torch.cuda.synchronize(); t2 = time.perf_counter()
    del rec
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"step {i}: plan {1e3*(t1-t0):.1f} pass {1e3*(t2-t1):.1f} del {1e3*(t3-t2):.1f} ms", flush=True)
