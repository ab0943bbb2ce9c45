import sys, os, ctypes
sys.path.insert(0, ".")
from paper_2411_09809_b200 import _lib
_h = ctypes.CDLL(os.environ.get("GLARE_B200_LIB", _lib.LIB_PATH))
for _k in [k for k in _lib.SIGNATURES if not hasattr(_h, k)]:
    _lib.SIGNATURES.pop(_k)
import torch
from paper_2411_09809_b200 import metrics as M, configs
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg, "culled")
out = rec.partial_interleaved(p["ideal"], 0, 64)
torch.cuda.synchronize()
print("units", rec.units, "count", out[0].item(), "dev", out[1].item())
