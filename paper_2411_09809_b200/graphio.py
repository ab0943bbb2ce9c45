"""Edge-list and layout loaders: drop-ins for the reference's
graphio.parse_edgelist and graphio.read_layout (graphio.py:46-117), with a
native fast path (csrc/io.cu: `glr_parse_edgelist`, `glr_parse_layout`).

The native parsers handle plain-ASCII files whose ids are decimal digit
strings and whose reals are ordinary decimal numbers; anything else --
non-ASCII text, other line breaks, underscores, inf/nan, malformed rows --
makes them defer (GLR_EFALLBACK) to the Python restatement below, which
follows the reference's rules line by line, so results and error messages
are the reference's in every case.  ``read_layout_arrays`` returns
(ids, xy) arrays for building a LayoutGraph without a million-entry dict.
"""

from __future__ import annotations

import ctypes
import logging
import math

import numpy as np

from . import _lib
from .model import InputError, LayoutGraph, normalize_edges

log = logging.getLogger(__name__)


def _read_bytes(path) -> bytes:
    try:
        with open(path, "rb") as fh:
            return fh.read()
    except OSError as exc:
        raise InputError(f"cannot read {path}: {exc}") from exc


def _decode(path, raw: bytes) -> str:
    """graphio._read_text: the file as UTF-8 text."""
    try:
        return raw.decode("utf-8")
    except UnicodeDecodeError as exc:  # open(..., encoding="utf-8").read() raises the same
        raise exc


# -- Python restatement of the reference parsers (fallback path) --------------

def _edge_pairs_py(path, text: str) -> list:
    pairs = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 2:
            raise InputError(f"{path}:{lineno}: expected two ids per line, got {line!r}")
        try:
            a, b = int(parts[0]), int(parts[1])
        except ValueError as exc:
            raise InputError(f"{path}:{lineno}: ids must be integers, got {line!r}") from exc
        if a < 0 or b < 0:
            raise InputError(f"{path}:{lineno}: ids must be nonnegative")
        pairs.append((a, b))
    return pairs


def _layout_py(path, text: str) -> dict:
    lines = text.splitlines()
    if not lines:
        raise InputError(f"{path}: empty layout file")
    header = [c.strip() for c in lines[0].split(",")]
    if header != ["id", "x", "y"]:
        raise InputError(f"{path}: expected header 'id,x,y', got {lines[0]!r}")
    positions: dict = {}
    for lineno, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        parts = [c.strip() for c in line.split(",")]
        if len(parts) != 3:
            raise InputError(f"{path}:{lineno}: expected 3 fields, got {line!r}")
        try:
            vid = int(parts[0])
            x = float(parts[1])
            y = float(parts[2])
        except ValueError as exc:
            raise InputError(f"{path}:{lineno}: malformed row {line!r}") from exc
        if not (math.isfinite(x) and math.isfinite(y)):
            raise InputError(f"{path}:{lineno}: non-finite coordinate")
        if vid in positions:
            raise InputError(f"{path}:{lineno}: duplicate vertex id {vid}")
        positions[vid] = (x, y)
    if not positions:
        raise InputError(f"{path}: layout file has no rows")
    return positions


# -- native fast paths ---------------------------------------------------------

def _native_pairs(raw: bytes):
    L = _lib.host_lib()
    n = ctypes.c_int64(0)
    rc = L.glr_parse_edgelist(raw, len(raw), None, 0, ctypes.byref(n))
    if rc == _lib.GLR_EFALLBACK:
        return None
    _lib.check(rc, "glr_parse_edgelist")
    out = np.empty((n.value, 2), dtype=np.int64)
    rc = L.glr_parse_edgelist(raw, len(raw), out.ctypes.data, n.value, ctypes.byref(n))
    _lib.check(rc, "glr_parse_edgelist")
    return out


def _native_layout(raw: bytes):
    L = _lib.host_lib()
    n = ctypes.c_int64(0)
    rc = L.glr_parse_layout(raw, len(raw), None, None, 0, ctypes.byref(n))
    if rc == _lib.GLR_EFALLBACK:
        return None
    _lib.check(rc, "glr_parse_layout")
    ids = np.empty(n.value, dtype=np.int64)
    xy = np.empty((n.value, 2), dtype=np.float64)
    rc = L.glr_parse_layout(raw, len(raw), ids.ctypes.data, xy.ctypes.data, n.value,
                            ctypes.byref(n))
    _lib.check(rc, "glr_parse_layout")
    if len(ids) == 0 or len(np.unique(ids)) != len(ids):
        return None  # the Python path raises the reference's error
    return ids, xy


def parse_edgelist(path) -> np.ndarray:
    """Normalized (m, 2) id pairs from a SNAP-style edge list file
    (graphio.py:46-79)."""
    raw = _read_bytes(path)
    pairs = _native_pairs(raw)
    if pairs is None:
        pairs = _edge_pairs_py(path, _decode(path, raw))
        if not pairs:
            raise InputError(f"{path}: no edges found")
    elif len(pairs) == 0:
        raise InputError(f"{path}: no edges found")
    edges, loops, dupes = normalize_edges(pairs)
    if loops or dupes:
        log.info("%s: dropped %d self-loop(s) and %d duplicate edge(s)", path, loops, dupes)
    return edges


def read_layout_arrays(path) -> tuple:
    """(ids int64 (n,), xy float64 (n, 2)) in file order, with read_layout's
    validation and errors."""
    raw = _read_bytes(path)
    got = _native_layout(raw)
    if got is not None:
        return got
    pos = _layout_py(path, _decode(path, raw))
    ids = np.fromiter(pos.keys(), dtype=np.int64, count=len(pos))
    xy = np.array(list(pos.values()), dtype=np.float64).reshape(-1, 2)
    return ids, xy


def read_layout(path) -> dict:
    """{id: (x, y)} from a CSV layout file with an id,x,y header
    (graphio.py:89-117)."""
    ids, xy = read_layout_arrays(path)
    return dict(zip(ids.tolist(), map(tuple, xy.tolist())))


def load_graph(edges_path, layout_path) -> LayoutGraph:
    """LayoutGraph from an edge-list file and a layout file (the CLI's
    loading step, cli.py:179-190, without a dict round trip)."""
    edges = parse_edgelist(edges_path)
    ids, xy = read_layout_arrays(layout_path)
    order = np.argsort(ids, kind="stable")
    return LayoutGraph(ids[order], xy[order], edges)
