"""Culled fused E_c+E_ca time on the spatially local configs (C3, C4) and
C5 per variant library:  python tools/variant_local.py name1 name2 ..."""
import os, subprocess, sys
CHILD = r'''
import sys, time; sys.path.insert(0, ".")
import ctypes, os, torch
from paper_2411_09809_b200 import _lib
_h = ctypes.CDLL(os.environ["GLARE_B200_LIB"])
for _k in [k for k in _lib.SIGNATURES if not hasattr(_h, k)]:
    _lib.SIGNATURES.pop(_k)
from paper_2411_09809_b200 import metrics as M, configs
out = []
for k in (3, 4, 5):
    g, p = configs.make(k); dg = M.DeviceGraph.from_graph(g); ideal = configs.IDEAL_70
    rec = M.CrossingRecords(dg, "culled"); rec.partial(ideal, 0, rec.units); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3 if k < 5 else 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(); o = rec.partial_interleaved(ideal, 0, 1); e[1].record(); torch.cuda.synchronize()
        best = min(best, e[0].elapsed_time(e[1]))
    out.append(f"C{k} {best:.2f} ms ({o[0].item():.0f})")
print(" | ".join(out))
'''
for name in sys.argv[1:]:
    env = dict(os.environ, GLARE_B200_LIB=os.path.join("tools", "variants", name, "libglare_b200.so"))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(name, (out.stdout.strip().splitlines() or [out.stderr[-400:]])[-1], flush=True)
