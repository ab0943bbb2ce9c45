"""Generate tests/golden/io_golden.json from the REFERENCE's loaders
(graphio.parse_edgelist / read_layout) on tests/io_cases.py's texts.

    python tests/golden/make_golden_io.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from glare.graphio import parse_edgelist, read_layout  # noqa: E402

import io_cases  # noqa: E402


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(fn, text, summarize):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "f.txt")
        if isinstance(text, bytes):
            with open(path, "wb") as fh:
                fh.write(text)
        else:
            with open(path, "w", encoding="utf-8", newline="") as fh:
                fh.write(text)
        try:
            return {"ok": summarize(fn(path))}
        except Exception as exc:  # noqa: BLE001 - the reference's error is the golden
            return {"error": [type(exc).__name__, str(exc).replace(path, "<path>")]}


def main():
    out = {"generator": "reference glare.graphio", "edgelists": {}, "layouts": {}}
    for name, text in io_cases.EDGELISTS.items():
        out["edgelists"][name] = run(parse_edgelist, text,
                                     lambda e: {"m": int(len(e)), "sha256": _sha(e.astype(np.int64))})
    for name, text in io_cases.LAYOUTS.items():
        def summ(pos):
            ids = np.fromiter(pos.keys(), dtype=np.int64, count=len(pos))
            xy = np.array(list(pos.values()), dtype=np.float64).reshape(-1, 2)
            return {"n": int(len(ids)), "ids_sha256": _sha(ids), "xy_sha256": _sha(xy)}
        out["layouts"][name] = run(read_layout, text, summ)
    for k in ("edgelists", "layouts"):
        for name, v in out[k].items():
            print(k, name, v)
    with open(os.path.join(HERE, "io_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
