"""Generate tests/golden/layout_golden.json from the REFERENCE's fr_layout.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_layout.py

Each case records the edge list recipe, the fr_layout arguments and the
SHA-256 of the reference's final positions (float64 bytes), plus the full
positions of the small cases.  The GPU box only reads the committed JSON.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from glare.graphio import fr_layout as ref_fr  # noqa: E402

import layout_cases  # noqa: E402


def main():
    out = {"generator": "reference glare.graphio.fr_layout (graphio.py:151-197)", "cases": {}}
    for name, (edges, kw) in layout_cases.CASES.items():
        t0 = time.perf_counter()
        g = ref_fr(edges, **kw)
        dt = time.perf_counter() - t0
        xy = np.ascontiguousarray(g.xy, dtype=np.float64)
        rec = {"kwargs": kw, "n": int(len(xy)), "m": int(g.num_edges),
               "sha256": hashlib.sha256(xy.tobytes()).hexdigest(),
               "first": [float(v) for v in xy[:2].ravel()], "seconds": round(dt, 3)}
        if len(xy) <= 64:
            rec["xy_hex"] = [v.hex() for v in xy.ravel().tolist()]
        out["cases"][name] = rec
        print(name, rec["n"], rec["m"], f"{dt:.2f}s", flush=True)
    with open(os.path.join(HERE, "layout_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
