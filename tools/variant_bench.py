"""Time the crossing / occlusion kernels of each variant library.

    python tools/variant_bench.py name1 name2 ...   (libraries in tools/variants/<name>/)
Each variant runs in its own subprocess (GLARE_B200_LIB selects the .so)."""
import json, os, subprocess, sys

CHILD = r'''
import sys, json, os; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2411_09809_b200 import metrics as M, configs, LayoutGraph
m = int(sys.argv[1])
g, _ = configs.config5(n=m * 3 // 8, m=m)   # C5 shape (Chung-Lu on the 2^16 lattice), scaled
dg = M.DeviceGraph.from_graph(g)
rec = M.CrossingRecords(dg, order=os.environ.get("VB_ORDER", "theta"))
res = {}
for name, ideal in (("ec", None), ("eca", configs.IDEAL_70)):
    rec.partial(ideal, 0, rec.units); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(3): out = rec.partial(ideal, 0, rec.units)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    res[name] = {"ms": ms, "Tpairs_s": m * (m - 1) / 2 / ms / 1e9, "count": out[0].item()}
print(json.dumps(res))
'''

if __name__ == "__main__":
    m = int(os.environ.get("VB_M", "400000"))
    for name in sys.argv[1:]:
        lib = os.path.join("tools", "variants", name, "libglare_b200.so")
        env = dict(os.environ, GLARE_B200_LIB=lib)
        out = subprocess.run([sys.executable, "-c", CHILD, str(m)], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        print(name, line, flush=True)
