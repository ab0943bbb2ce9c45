"""Generate tests/golden/*.json from the REFERENCE implementation itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py [--configs]

The reference package (glare, pure Python + numpy) is imported from
/root/reference/pkg/src and its serial oracle functions
(metrics/exact.py:55-238) are evaluated on the inputs built by tests/cases.py
and paper_2411_09809_b200/configs.py.  Inputs are identified by a content
fingerprint so the GPU-side tests can check they regenerated the same graph.
The GPU box never runs this script (no /root/reference there); it only reads
the committed JSON.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from glare.metrics import exact as ref  # noqa: E402
from glare.metrics.enhanced import node_occlusion_grid as ref_grid  # noqa: E402
from glare.model import LayoutGraph as RefGraph  # noqa: E402

import cases  # noqa: E402
from paper_2411_09809_b200 import configs  # noqa: E402

IDEAL = configs.IDEAL_70


def fp(xy, edges):
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(xy, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(edges, dtype=np.int64).tobytes())
    return h.hexdigest()[:16]


def _try(fn, cast):
    """Value, or {"error": ExceptionName} when the reference raises."""
    try:
        return cast(fn())
    except Exception as exc:  # the drop-in must raise the same type
        return {"error": type(exc).__name__}


def all_metrics(g, r):
    out = {
        "n": int(g.num_vertices),
        "m": int(g.num_edges),
        "fingerprint": fp(g.xy, g.edges),
        "radius": r,
        "nc": _try(lambda: ref.node_occlusion(g, r), int),
        "ma": _try(lambda: ref.minimum_angle(g), float),
        "ml": _try(lambda: ref.edge_length_variation(g), float),
    }
    c, d = ref._crossing_scan(g, IDEAL)
    out["ec"] = int(c)
    out["dev"] = float(d)
    out["eca"] = _try(lambda: ref.edge_crossing_angle(g, IDEAL), float)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", action="store_true", help="also run C1-C4 (minutes)")
    args = ap.parse_args()
    doc = {"meta": {"source": "reference glare oracle, /root/reference/pkg/src",
                    "numpy": np.__version__, "ideal": IDEAL}}
    known = {}
    for name, fn in cases.KNOWN.items():
        pos, edges = fn()
        g = RefGraph.from_positions(pos, edges)
        r = 1.0 if name.startswith("occ") else 0.1
        known[name] = all_metrics(g, r)
    # radius variants pinned by the reference's tests (test_metrics_exact.py:30-43)
    pos, edges = cases.occ_boundary()
    g = RefGraph.from_positions(pos, edges)
    known["occ_boundary"]["nc_r1.0000001"] = int(ref.node_occlusion(g, 1.0000001))
    doc["known"] = known

    adv = {}
    for name, fn in cases.ADVERSARIAL_SMALL.items():
        pos, edges = fn()
        adv[name] = all_metrics(RefGraph.from_positions(pos, edges), 0.5)
    for name, fn in cases.ADVERSARIAL_ARRAYS.items():
        ids, xy, pairs = fn()
        g = RefGraph(ids, xy, pairs)
        adv[name] = all_metrics(g, cases.ADVERSARIAL_RADIUS[name])
    doc["adversarial"] = adv

    rng = np.random.default_rng(42)
    crit = []
    t = time.time()
    for i in range(200):
        ids, xy, edges = cases.criterion1_case(i, rng)
        g = RefGraph(ids, xy, edges)
        r = 0.5 + (i % 7)
        crit.append(all_metrics(g, r))
    doc["criterion1"] = crit
    print(f"criterion1: {time.time() - t:.1f}s", flush=True)

    if args.configs:
        cfg = {}
        for k in (1, 2):
            t = time.time()
            g, p = configs.make(k)
            rg = RefGraph(g.ids, g.xy, g.edges)
            cfg[f"C{k}"] = all_metrics(rg, p["radius"])
            cfg[f"C{k}"]["source"] = "reference oracle"
            print(f"C{k}: {time.time() - t:.1f}s", cfg[f"C{k}"], flush=True)
        # C4 at 1/10 scale (R=316): the survey's probe recipe
        t = time.time()
        g, p = configs.config4(R=316)
        rg = RefGraph(g.ids, g.xy, g.edges)
        cfg["C4_R316"] = all_metrics(rg, p["radius"])
        cfg["C4_R316"]["source"] = "reference oracle"
        print(f"C4_R316: {time.time() - t:.1f}s", cfg["C4_R316"], flush=True)
        # C3: full reference crossing scan and grid occlusion (exact)
        t = time.time()
        g, p = configs.config3()
        rg = RefGraph(g.ids, g.xy, g.edges)
        c, d = ref._crossing_scan(rg, IDEAL)
        cfg["C3"] = {"n": g.num_vertices, "m": g.num_edges, "fingerprint": fp(g.xy, g.edges),
                     "radius": p["radius"], "ec": int(c), "dev": float(d),
                     "eca": float(1.0 - (d / IDEAL) / c) if c else 1.0,
                     "nc": int(ref_grid(rg, p["radius"])),
                     "source": "reference oracle (_crossing_scan; node_occlusion_grid)"}
        print(f"C3: {time.time() - t:.1f}s", cfg["C3"], flush=True)
        doc["configs"] = cfg
    out = os.path.join(HERE, "golden.json" if args.configs else "golden_small.json")
    if args.configs:
        # keep the small sets in their own file; configs file holds only configs
        doc = {"meta": doc["meta"], "configs": doc["configs"]}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    print("wrote", out)


if __name__ == "__main__":
    main()
