"""Debug: sequence of partial calls on one CrossingRecords (mode 2)."""
import sys, time; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from test_gpu_filter import CASES, _graph, IDEAL
from paper_2411_09809_b200 import metrics as M
g = _graph(*CASES[sys.argv[1] if len(sys.argv) > 1 else 'near_collinear']())
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg)
U = rec.units
calls = [("whole", lambda: rec.partial(IDEAL, 0, U))]
cuts = [0, U // 3, U // 2, U]
for a, b in zip(cuts, cuts[1:]):
    calls.append((f"part {a}-{b}", lambda a=a, b=b: rec.partial(IDEAL, a, b)))
for r in range(3):
    calls.append((f"share {r}/3", lambda r=r: rec.partial_interleaved(IDEAL, r, 3)))
for name, fn in calls:
    t = time.time(); p = fn().tolist(); torch.cuda.synchronize()
    print(name, p, f"{time.time() - t:.3f}s", flush=True)
