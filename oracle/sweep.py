"""ctypes wrapper of oracle/_build/libsweep_oracle.so -- TEST INFRASTRUCTURE.

Multi-threaded C restatement of the reference's crossing scan and node
occlusion (see sweep_oracle.c).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs use it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_build", "libsweep_oracle.so")
_h = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB


def _lib():
    global _h
    if _h is None:
        if not os.path.exists(LIB):
            build()
        h = ctypes.CDLL(LIB)
        h.oracle_crossing_scan.restype = ctypes.c_int
        h.oracle_crossing_scan.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int,
            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)]
        h.oracle_node_occlusion.restype = ctypes.c_int
        h.oracle_node_occlusion.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
            ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
        _h = h
    return _h


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def crossing_scan(xy, edges, ideal=None, threads=None):
    """(count, dev_sum) of the reference crossing scan (exact.py:145-222)."""
    from .glare_oracle import axis_angles

    xy = np.ascontiguousarray(xy, dtype=np.float64)
    edges = np.ascontiguousarray(edges, dtype=np.int64).reshape(-1, 2)
    m = len(edges)
    if m < 2:
        return 0, 0.0
    theta = None
    if ideal is not None:
        a = xy[edges[:, 0]]
        b = xy[edges[:, 1]]
        theta = np.ascontiguousarray(axis_angles(a[:, 0], a[:, 1], b[:, 0], b[:, 1]))
    cnt = ctypes.c_uint64(0)
    dev = ctypes.c_double(0.0)
    rc = _lib().oracle_crossing_scan(
        xy.ctypes.data, len(xy), edges.ctypes.data, m,
        theta.ctypes.data if theta is not None else None, 1 if ideal is not None else 0,
        float(ideal) if ideal is not None else 0.0, threads or default_threads(),
        ctypes.byref(cnt), ctypes.byref(dev))
    if rc != 0:
        raise MemoryError("oracle_crossing_scan failed")
    return int(cnt.value), (float(dev.value) if ideal is not None else 0.0)


def node_occlusion(xy, r, threads=None):
    """Occluding pairs (exact.py:55-74), x-sorted sweep."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    if len(xy) < 2:
        return 0
    thr = (2.0 * r) ** 2
    cnt = ctypes.c_uint64(0)
    rc = _lib().oracle_node_occlusion(xy.ctypes.data, len(xy), thr, 2.0 * r,
                                      threads or default_threads(), ctypes.byref(cnt))
    if rc != 0:
        raise MemoryError("oracle_node_occlusion failed")
    return int(cnt.value)
