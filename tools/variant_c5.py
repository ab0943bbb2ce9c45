"""Full-C5 fused crossing pass (dense theta and culled) per variant library:
    python tools/variant_c5.py name1 name2 ...   (tools/variants/<name>/)"""
import os, subprocess, sys
CHILD = r'''
import sys, time; sys.path.insert(0, ".")
import ctypes, os, torch
from paper_2411_09809_b200 import _lib
_h = ctypes.CDLL(os.environ["GLARE_B200_LIB"])  # older builds lack newer symbols
for _k in [k for k in _lib.SIGNATURES if not hasattr(_h, k)]:
    _lib.SIGNATURES.pop(_k)
from paper_2411_09809_b200 import metrics as M, configs
g, p = configs.config5(); dg = M.DeviceGraph.from_graph(g); ideal = p["ideal"]
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def t(fn):
    torch.cuda.synchronize(); e[0].record(); o = fn(); e[1].record(); torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]), o.tolist()
rec = M.CrossingRecords(dg, "dense", "theta"); rec.partial(ideal, 0, 100)
d = t(lambda: rec.partial_interleaved(ideal, 0, 1)); del rec
M.CrossingRecords(dg, "culled").partial(ideal, 0, 100)
c = t(lambda: M.CrossingRecords(dg, "culled").partial_interleaved(ideal, 0, 1))
print(f"dense {d[0]:.1f} ms culled {c[0]:.1f} ms count {d[1][0]:.0f}/{c[1][0]:.0f} dev {d[1][1]!r}/{c[1][1]!r}")
'''
for name in sys.argv[1:]:
    env = dict(os.environ, GLARE_B200_LIB=os.path.join("tools", "variants", name, "libglare_b200.so"))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(name, (out.stdout.strip().splitlines() or [out.stderr[-400:]])[-1], flush=True)
