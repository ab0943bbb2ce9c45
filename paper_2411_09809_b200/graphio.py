"""Edge-list and layout loaders: drop-ins for the reference's
graphio.parse_edgelist and graphio.read_layout (graphio.py:46-117).

All parsing is native (csrc/io.cu: ``glr_parse_edgelist`` /
``glr_parse_layout``), over the reference's whole input grammar -- UTF-8,
str.splitlines() line boundaries, str.isspace() whitespace, and int() /
float() of a str.  A malformed input comes back as a ``GLR_PARSE_*`` kind
with a line number and the byte span of the offending line
(``glr_parse_status``); ``_raise`` below turns that into the exception the
reference raises, with its message (the quoted line is ``repr`` of the
decoded span, as the reference's f-strings do).
``read_layout_arrays`` returns (ids, xy) arrays for building a LayoutGraph
without a million-entry dict.

One deliberate difference: a layout id beyond the int64 range raises the
``OverflowError`` that any int64 id array raises (the reference's dict would
hold it and fail later, when a LayoutGraph is built from it).
"""

from __future__ import annotations

import ctypes
import logging

import numpy as np

from . import _lib
from .model import InputError, LayoutGraph, normalize_edges

log = logging.getLogger(__name__)

# message templates of the reference's loaders (graphio.py:59-79, 89-117),
# by GLR_PARSE_* kind ({q}: repr of the quoted line)
_MESSAGES = {
    2: "expected two ids per line, got {q}",
    3: "ids must be integers, got {q}",
    4: "ids must be nonnegative",
    5: "no edges found",
    7: "empty layout file",
    8: "expected header 'id,x,y', got {q}",
    9: "expected 3 fields, got {q}",
    10: "malformed row {q}",
    11: "non-finite coordinate",
    12: "duplicate vertex id {vid}",
    13: "layout file has no rows",
}
_KIND_UTF8, _KIND_OVERFLOW, _KIND_HEADER = 1, 6, 8


def _read_bytes(path) -> bytes:
    try:
        with open(path, "rb") as fh:
            return fh.read()
    except OSError as exc:
        raise InputError(f"cannot read {path}: {exc}") from exc


def _raise(path, raw: bytes) -> None:
    """Raise what the reference raises for the parse failure just reported."""
    info = (ctypes.c_int64 * 4)()
    _lib.host_lib().glr_parse_status(info)
    kind, lineno, a, b = info
    if kind == _KIND_UTF8:
        # the reference reads the file as UTF-8 text (graphio.py:_read_text);
        # the same read raises the same UnicodeDecodeError here
        with open(path, encoding="utf-8") as fh:
            fh.read()
        raise InputError(f"{path}: invalid UTF-8")  # unreachable: the decoder agrees
    if kind == _KIND_OVERFLOW:
        raise OverflowError("Python int too large to convert to C long")
    msg = _MESSAGES[kind].format(q=repr(raw[a:b].decode("utf-8")), vid=a)
    where = f"{path}:{lineno}" if lineno and kind != _KIND_HEADER else f"{path}"
    raise InputError(f"{where}: {msg}")


def _native_pairs(path, raw: bytes) -> np.ndarray:
    L = _lib.host_lib()
    n = ctypes.c_int64(0)
    rc = L.glr_parse_edgelist(raw, len(raw), None, 0, ctypes.byref(n))
    if rc == _lib.GLR_EPARSE:
        _raise(path, raw)
    _lib.check(rc, "glr_parse_edgelist")
    out = np.empty((n.value, 2), dtype=np.int64)
    rc = L.glr_parse_edgelist(raw, len(raw), out.ctypes.data, n.value, ctypes.byref(n))
    _lib.check(rc, "glr_parse_edgelist")
    return out


def _native_layout(path, raw: bytes):
    L = _lib.host_lib()
    n = ctypes.c_int64(0)
    rc = L.glr_parse_layout(raw, len(raw), None, None, 0, ctypes.byref(n))
    if rc == _lib.GLR_EPARSE:
        _raise(path, raw)
    _lib.check(rc, "glr_parse_layout")
    ids = np.empty(n.value, dtype=np.int64)
    xy = np.empty((n.value, 2), dtype=np.float64)
    rc = L.glr_parse_layout(raw, len(raw), ids.ctypes.data, xy.ctypes.data, n.value,
                            ctypes.byref(n))
    _lib.check(rc, "glr_parse_layout")
    return ids, xy


def parse_edgelist(path) -> np.ndarray:
    """Normalized (m, 2) id pairs from a SNAP-style edge list file
    (graphio.py:46-79)."""
    pairs = _native_pairs(path, _read_bytes(path))
    edges, loops, dupes = normalize_edges(pairs)
    if loops or dupes:
        log.info("%s: dropped %d self-loop(s) and %d duplicate edge(s)", path, loops, dupes)
    return edges


def read_layout_arrays(path) -> tuple:
    """(ids int64 (n,), xy float64 (n, 2)) in file order, with read_layout's
    validation and errors."""
    return _native_layout(path, _read_bytes(path))


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
