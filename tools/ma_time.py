"""M_a device time (hand-written per-vertex segmented sort, csrc/length_angle.cu)
on C4 (1M vertices, degree <= 6) and on the C5 graph (degree up to ~55k):
    python tools/ma_time.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs

for name, (g, _) in (("C4", configs.config4()), ("C5-shape", configs.config5())):
    dg = M.DeviceGraph.from_graph(g)
    out = M.minimum_angle_device(dg)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        out = M.minimum_angle_device(dg, out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"{name}: n={g.num_vertices} m={g.num_edges} M_a={out[2].item():.12f} "
          f"{ms:.3f} ms per call (2m={2 * g.num_edges} angles)")
