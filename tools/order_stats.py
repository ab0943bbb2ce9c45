"""Filter fallback statistics of the C5 fused pass by edge order and hub degree (debug
variant built with -DGLR_XFSTATS: tools/build_variants.sh stats:-DGLR_XFSTATS)
    GLARE_B200_LIB=tools/variants/stats/libglare_b200.so python tools/order_stats.py [hub_degree ...]"""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_2411_09809_b200 import metrics as M, configs, _lib

g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
L = _lib.lib()
buf = (ctypes.c_ulonglong * 2)()
stats = hasattr(L, "glr_debug_fstats")  # debug variant only
if not stats:
    L.glr_debug_fstats = lambda b, r: 0
runs = [("input", 0)] + [("theta", int(d)) for d in (sys.argv[1:] or ["1024"])]
for order, hub in runs:
    M.HUB_DEGREE = hub
    rec = M.CrossingRecords(dg, order=order)
    for angle in (None, p["ideal"]):
        L.glr_debug_fstats(buf, 1)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(); out = rec.partial(angle, 0, rec.units); t1.record(); torch.cuda.synchronize()
        L.glr_debug_fstats(buf, 1)
        print(f"{order:5s} hub {hub:>10d} {'fused' if angle else 'count'} {t0.elapsed_time(t1):8.1f} ms "
              f"fallback blocks {buf[0]:.3e} uncertain pairs {buf[1]:.3e} {out.tolist()}", flush=True)
