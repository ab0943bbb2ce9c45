"""Strip-sweep approximations and grid occlusion: drop-ins for the
reference's metrics/enhanced.py.

* ``edge_crossing_enhanced``, ``crossing_angle_stats``,
  ``edge_crossing_angle_enhanced`` (enhanced.py:218-300): strips are built
  exactly as ``build_strips`` does (the boundaries on the host, in the
  reference's float arithmetic), the per-strip sweeps run on the GPU
  (csrc/strips.cu, ``glr_strip_crossings``): inversion counts (exact
  integers, equal to the reference's) and the deviation sums over the same
  pairs (equal up to rounding).
* ``node_occlusion_grid`` (enhanced.py:54-127) is exact; it returns the
  occlusion count of ``metrics.node_occlusion`` (culled plan).

``exec_cfg`` is accepted for signature compatibility and ignored (the GPU
replaces the reference's worker pools).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .metrics import DeviceGraph, _ptr, _stream, node_occlusion
from .model import InputError, ParameterError, check_ideal_angle

STRIP_ORIENTATIONS = ("vertical", "horizontal", "both")


def _check_fraction(f: float) -> float:
    if not (0.0 < f < 1.0) or not math.isfinite(f):
        raise ParameterError(f"strip width fraction must lie in (0, 1), got {f}")
    return f


def _check_orientation(orientation: str) -> str:
    if orientation not in STRIP_ORIENTATIONS:
        raise ParameterError(
            f"orientation must be one of {STRIP_ORIENTATIONS}, got {orientation!r}")
    return orientation


def strip_bounds(xy: np.ndarray, fraction: float, orientation: str) -> np.ndarray:
    """Strip boundaries along the sweep axis, as build_strips computes them
    (enhanced.py:155-167)."""
    _check_fraction(fraction)
    if orientation not in ("vertical", "horizontal"):
        raise ParameterError(
            f"orientation must be 'vertical' or 'horizontal', got {orientation!r}")
    axis_c = xy[:, 1] if orientation == "horizontal" else xy[:, 0]
    lo = float(axis_c.min())
    hi = float(axis_c.max())
    if not hi > lo:
        raise InputError("layout has zero extent along the strip axis")
    nstrips = math.ceil(1.0 / fraction)
    width = (hi - lo) / nstrips
    bounds = lo + np.arange(nstrips + 1) * width
    bounds[-1] = hi
    return bounds


def _as_host_xy(g) -> np.ndarray:
    if isinstance(g, DeviceGraph):
        return g.xy.cpu().numpy()
    return np.asarray(g.xy, dtype=np.float64)


def _oriented(g, dg: DeviceGraph, fraction: float, orientation: str, ideal) -> tuple:
    import torch

    bounds = strip_bounds(_as_host_xy(g), fraction, orientation)
    db = torch.from_numpy(bounds).to(dg.xy.device)
    out = torch.zeros(2, dtype=torch.float64, device=dg.xy.device)
    rc = _lib.lib().glr_strip_crossings(
        _ptr(dg.xy), dg.num_vertices, _ptr(dg.edges), dg.num_edges, _ptr(db), len(bounds) - 1,
        1 if orientation == "horizontal" else 0, 0 if ideal is None else 1,
        0.0 if ideal is None else float(ideal), _ptr(out), _stream())
    _lib.check(rc, "glr_strip_crossings")
    c, d = out.tolist()
    return int(c), d


def _device(g) -> DeviceGraph:
    return g if isinstance(g, DeviceGraph) else DeviceGraph.from_graph(g)


def edge_crossing_enhanced(g, strip_width_fraction: float, orientation: str = "vertical",
                           exec_cfg=None) -> int:
    """Strip-inversion crossing count, never above the exact count
    (enhanced.py:225-245); "both" keeps the larger of the two passes."""
    _check_orientation(orientation)
    if g.num_edges < 2:
        return 0
    _check_fraction(strip_width_fraction)  # build_strips' first check, before any GPU work
    dg = _device(g)
    if orientation == "both":
        return max(_oriented(g, dg, strip_width_fraction, "vertical", None)[0],
                   _oriented(g, dg, strip_width_fraction, "horizontal", None)[0])
    return _oriented(g, dg, strip_width_fraction, orientation, None)[0]


def crossing_angle_stats(g, strip_width_fraction: float, ideal_angle: float,
                         orientation: str = "vertical", exec_cfg=None) -> tuple:
    """(count, deviation sum) over the strip crossings (enhanced.py:259-287);
    for "both" the statistics of the orientation with more crossings
    (vertical on ties)."""
    _check_orientation(orientation)
    ideal_angle = check_ideal_angle(ideal_angle)
    if g.num_edges < 2:
        return 0, 0.0
    _check_fraction(strip_width_fraction)
    dg = _device(g)
    if orientation == "both":
        v = _oriented(g, dg, strip_width_fraction, "vertical", ideal_angle)
        h = _oriented(g, dg, strip_width_fraction, "horizontal", ideal_angle)
        return v if v[0] >= h[0] else h
    return _oriented(g, dg, strip_width_fraction, orientation, ideal_angle)


def edge_crossing_angle_enhanced(g, strip_width_fraction: float, ideal_angle: float,
                                 orientation: str = "vertical", exec_cfg=None) -> float:
    """1 - mean normalised deviation over the strip crossings
    (enhanced.py:290-300)."""
    count, deviation = crossing_angle_stats(g, strip_width_fraction, ideal_angle, orientation,
                                            exec_cfg)
    if count == 0:
        return 1.0
    return 1.0 - (deviation / ideal_angle) / count


def node_occlusion_grid(g, r: float, exec_cfg=None) -> int:
    """Exact occluding-pair count (enhanced.py:54-127): the same value as
    node_occlusion, computed by the culled GPU plan."""
    return node_occlusion(g, r, strategy="culled")
