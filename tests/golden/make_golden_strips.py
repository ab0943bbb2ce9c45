"""Generate tests/golden/strip_golden.json from the REFERENCE's strip sweeps
(metrics/enhanced.py edge_crossing_enhanced / crossing_angle_stats).

    python tests/golden/make_golden_strips.py
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from glare.metrics.enhanced import crossing_angle_stats, edge_crossing_enhanced  # noqa: E402
from glare.model import LayoutGraph as RefGraph  # noqa: E402

import strip_cases  # noqa: E402

IDEAL = math.radians(70.0)


def main():
    out = {"generator": "reference glare.metrics.enhanced", "ideal": IDEAL, "cases": {}}
    for name, (ids, xy, pairs) in strip_cases.GRAPHS.items():
        g = RefGraph(ids, xy, pairs)
        rows = []
        for frac, orient in strip_cases.SETTINGS[name]:
            t0 = time.perf_counter()
            ec = edge_crossing_enhanced(g, frac, orient)
            c, d = crossing_angle_stats(g, frac, IDEAL, orient)
            rows.append({"fraction": frac, "orientation": orient, "ec": int(ec), "count": int(c),
                         "dev": float(d), "seconds": round(time.perf_counter() - t0, 3)})
            print(name, rows[-1], flush=True)
        out["cases"][name] = rows
    with open(os.path.join(HERE, "strip_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
