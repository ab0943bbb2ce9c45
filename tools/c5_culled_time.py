"""Time the culled C5 plan: build (box sort, prepare, classified candidates)
and the fused E_c + E_ca pass over it, checked against the C5 golden:
    python tools/c5_culled_time.py [reps] [alt]   (alt: odd reps ignore the sub-unit masks)"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2411_09809_b200 import configs, metrics as M  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
want = json.load(open("tests/golden/golden.json"))["configs"]["C5"]
g, p = configs.config5()
dg = M.DeviceGraph.from_graph(g)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for r in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    rec = M.CrossingRecords(dg, "culled")
    rec.use_sub_masks = r % 2 == 0 or len(sys.argv) < 3
    torch.cuda.synchronize()
    build = time.perf_counter() - t
    a, b = ev(), ev()
    a.record()
    c, d = rec.partial_interleaved(p["ideal"], 0, 1).tolist()
    b.record()
    torch.cuda.synchronize()
    fused = a.elapsed_time(b)
    a.record()
    c0 = rec.partial_interleaved(None, 0, 1)[0].item()
    b.record()
    torch.cuda.synchronize()
    ec = a.elapsed_time(b)
    ok = int(c) == want["ec"] and int(c0) == want["ec"] and abs(d - want["dev"]) <= 1e-9 * want["dev"]
    print(json.dumps({"rep": r, "build_ms": round(build * 1e3, 1), "fused_ms": round(fused, 1),
                      "ec_ms": round(ec, 1), "sub_masks": rec.use_sub_masks, "mixed": rec.n_mixed, "full": rec.n_full,
                      "dense_units": M.crossing_units(g.num_edges), "count": int(c),
                      "dev": d, "golden_ok": ok}), flush=True)
    del rec
