"""Debug: interleaved shares of the near-collinear stress graph, one call per
process run (python tools/dbg_filter.py MODE RANK WORLD)."""
import sys, time; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from test_gpu_filter import CASES, _graph, IDEAL
from paper_2411_09809_b200 import metrics as M
mode, rank, world = (int(a) for a in sys.argv[1:4])
g = _graph(*CASES[sys.argv[4] if len(sys.argv) > 4 else 'near_collinear']())
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg).set_mode(mode)
t = time.time(); p = rec.partial_interleaved(IDEAL, rank, world).tolist(); torch.cuda.synchronize()
print(mode, rank, world, p, f"{time.time() - t:.3f}s", flush=True)
