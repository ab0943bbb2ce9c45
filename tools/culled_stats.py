"""Filter fallback statistics of the culled C5 plan (debug variant built with
-DGLR_XFSTATS: tools/build_variants.sh stats:-DGLR_XFSTATS)
    GLARE_B200_LIB=tools/variants/stats/libglare_b200.so python tools/culled_stats.py"""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs, _lib

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
L = _lib.lib()
buf = (ctypes.c_ulonglong * 2)()
rec = M.CrossingRecords(dg, "culled")
for angle in (None, p["ideal"]):
    L.glr_debug_fstats(buf, 1)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(); out = rec.partial_interleaved(angle, 0, 1); t1.record(); torch.cuda.synchronize()
    L.glr_debug_fstats(buf, 1)
    print(f"culled {'fused' if angle else 'count'} {t0.elapsed_time(t1):8.1f} ms fallback blocks "
          f"{buf[0]:.3e} uncertain pairs {buf[1]:.3e} {out.tolist()}", flush=True)
