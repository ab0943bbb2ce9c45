"""Stage-wait statistics of the filter kernel (library built with
-DGLR_XWAITSTAT, selected by GLARE_B200_LIB): share of warp time spent
waiting for j-tiles."""
import ctypes, os, sys; sys.path.insert(0, '.')
import torch
from paper_2411_09809_b200 import metrics as M, configs, _lib
m = int(sys.argv[1]) if len(sys.argv) > 1 else 400000
g, _ = configs.config5(n=m * 3 // 8, m=m)
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg)
L = _lib.lib()
f = L.glr_debug_wait_stats
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 5)()
for ideal in (configs.IDEAL_70, None):
    rec.partial(ideal, 0, rec.units); torch.cuda.synchronize()
    f(buf, 1)
    rec.partial(ideal, 0, rec.units); torch.cuda.synchronize()
    f(buf, 1)
    w_first, w_later, n_first, n_later, comp = list(buf)
    tot = w_first + w_later + comp
    print(f"angle={ideal is not None}: wait first {w_first / tot:.3f} later {w_later / tot:.3f} "
          f"compute {comp / tot:.3f}; waits {n_first}/{n_later}, mean later wait "
          f"{w_later / max(n_later, 1):.0f} cyc, mean unit {comp / max(n_later, 1):.0f} cyc")
