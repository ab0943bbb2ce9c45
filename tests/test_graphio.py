"""Native edge-list / layout loaders against the
reference's own results and errors (tests/golden/io_golden.json, made by
tests/golden/make_golden_io.py).  CPU only: the loaders are host code."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import io_cases

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def io_golden():
    with open(os.path.join(HERE, "golden", "io_golden.json")) as fh:
        return json.load(fh)


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _write(tmp_path, text):
    path = tmp_path / "f.txt"
    if isinstance(text, bytes):
        with open(path, "wb") as fh:
            fh.write(text)
    else:
        with open(path, "w", encoding="utf-8", newline="") as fh:
            fh.write(text)
    return str(path)


def _run(fn, path, summarize):
    try:
        return {"ok": summarize(fn(path))}
    except Exception as exc:  # noqa: BLE001
        return {"error": [type(exc).__name__, str(exc).replace(path, "<path>")]}


@pytest.mark.parametrize("name", sorted(io_cases.EDGELISTS))
def test_parse_edgelist_matches_reference(io_golden, tmp_path, name):
    from paper_2411_09809_b200.graphio import parse_edgelist

    path = _write(tmp_path, io_cases.EDGELISTS[name])
    got = _run(parse_edgelist, path, lambda e: {"m": int(len(e)), "sha256": _sha(e.astype(np.int64))})
    assert got == io_golden["edgelists"][name]


@pytest.mark.parametrize("name", sorted(io_cases.LAYOUTS))
def test_read_layout_matches_reference(io_golden, tmp_path, name):
    from paper_2411_09809_b200.graphio import read_layout

    def summ(pos):
        ids = np.fromiter(pos.keys(), dtype=np.int64, count=len(pos))
        xy = np.array(list(pos.values()), dtype=np.float64).reshape(-1, 2)
        return {"n": int(len(ids)), "ids_sha256": _sha(ids), "xy_sha256": _sha(xy)}

    path = _write(tmp_path, io_cases.LAYOUTS[name])
    assert _run(read_layout, path, summ) == io_golden["layouts"][name]


def test_every_text_is_parsed_natively():
    """No Python parsing path is left: the native parsers answer every case
    with a result or a GLR_PARSE_* error (never the old fallback code)."""
    import ctypes

    from paper_2411_09809_b200 import _lib, graphio

    assert not hasattr(graphio, "_edge_pairs_py") and not hasattr(graphio, "_layout_py")
    L = _lib.host_lib()
    n = ctypes.c_int64(0)
    for texts, fn in ((io_cases.EDGELISTS, L.glr_parse_edgelist),
                      (io_cases.LAYOUTS, None)):
        for name, text in texts.items():
            raw = text if isinstance(text, bytes) else text.encode("utf-8")
            if fn is None:
                rc = L.glr_parse_layout(raw, len(raw), None, None, 0, ctypes.byref(n))
            else:
                rc = fn(raw, len(raw), None, 0, ctypes.byref(n))
            assert rc in (_lib.GLR_OK, _lib.GLR_EPARSE), (name, rc)


def test_load_graph(tmp_path):
    from paper_2411_09809_b200.graphio import load_graph

    e = _write(tmp_path, "0 1\n1 2\n")
    (tmp_path / "l.csv").write_text("id,x,y\n2,1,1\n0,0,0\n1,1,0\n")
    g = load_graph(e, str(tmp_path / "l.csv"))
    assert g.ids.tolist() == [0, 1, 2] and g.xy.tolist() == [[0, 0], [1, 0], [1, 1]]
    assert g.num_edges == 2
