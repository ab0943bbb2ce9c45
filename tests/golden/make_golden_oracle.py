"""Add full-size C4 and C5 goldens to tests/golden/golden.json from the PINNED
oracle (oracle/sweep_oracle.c and oracle/glare_oracle.py, themselves checked
against the reference's own outputs by tests/test_oracle_golden.py and
tests/test_configs_golden.py).  The reference is too slow at these sizes
(C4 crossing ~20-30 min, C5 days).

    python tests/golden/make_golden_oracle.py               # C4 all, C5 occlusion
    python tests/golden/make_golden_oracle.py --c5-crossing # C5 E_c/E_ca (hours)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import glare_oracle as O  # noqa: E402
from oracle import sweep as S  # noqa: E402
from paper_2411_09809_b200 import configs  # noqa: E402


def c5_crossing():
    """Full C5 E_c / dev_sum with the C oracle on all host cores (~2 h on 8
    cores); stored beside the C5 occlusion golden."""
    path = os.path.join(HERE, "golden.json")
    g, p = configs.config5()
    c, d = S.crossing_scan(g.xy, g.edges, p["ideal"])
    doc = json.load(open(path))
    assert doc["configs"]["C5"]["fingerprint"] == configs.fingerprint(g)
    doc["configs"]["C5"].update({"ec": c, "dev": d,
                                 "eca": 1.0 if c == 0 else 1 - (d / p["ideal"]) / c,
                                 "source_ec": "pinned oracle: oracle/sweep_oracle.c, all host threads"})
    json.dump(doc, open(path, "w"), indent=1, sort_keys=True)
    print(doc["configs"]["C5"])


def main():
    if "--c5-crossing" in sys.argv:
        return c5_crossing()
    path = os.path.join(HERE, "golden.json")
    doc = json.load(open(path))
    g, p = configs.config4()
    c, d = S.crossing_scan(g.xy, g.edges, p["ideal"])
    doc["configs"]["C4"] = {
        "n": g.num_vertices, "m": g.num_edges, "fingerprint": configs.fingerprint(g),
        "radius": p["radius"], "ec": c, "dev": d, "eca": 1.0 if c == 0 else 1 - (d / p["ideal"]) / c,
        "nc": S.node_occlusion(g.xy, p["radius"]),
        "ma": O.minimum_angle(g.xy, g.edges), "ml": O.edge_length_variation(g.xy, g.edges),
        "source": "pinned oracle: oracle/sweep_oracle.c (ec, nc), oracle/glare_oracle.py (ma, ml)"}
    g, p = configs.config5()
    nc = S.node_occlusion(g.xy, p["radius"])
    assert nc == O.node_occlusion_grid(g.xy, p["radius"])
    doc["configs"]["C5"] = {
        "n": g.num_vertices, "m": g.num_edges, "fingerprint": configs.fingerprint(g),
        "radius": p["radius"], "nc": nc,
        "source": "pinned oracle: x-sorted sweep (sweep_oracle.c) == grid occlusion (glare_oracle.py)"}
    json.dump(doc, open(path, "w"), indent=1, sort_keys=True)
    print(doc["configs"]["C4"], doc["configs"]["C5"])


if __name__ == "__main__":
    main()
