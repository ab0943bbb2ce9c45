"""Layout generators: drop-ins for the reference's graphio.random_layout,
graphio.fr_layout and engine.generate_layout.

`fr_layout` runs the O(n^2) force-directed iteration on the GPU
(csrc/layout.cu, `glr_fr_layout`), bit-for-bit equal to the reference's numpy
implementation (graphio.py:151-197): same seeded start (numpy's
default_rng(seed).uniform, a host call), same IEEE operations, numpy's
pairwise summation order for the repulsion row sums and np.add.at's order for
the spring pulls.  Validation and error messages mirror the reference.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .model import InputError, LayoutGraph, ParameterError, normalize_edges


def _vertex_ids(edges) -> np.ndarray:
    """graphio.py:134-138."""
    arr = np.asarray(edges, dtype=np.int64)
    if arr.size == 0:
        raise InputError("cannot lay out a graph with no edges")
    return np.unique(arr)


def _check_extent(extent: float) -> None:
    if not (extent > 0 and math.isfinite(extent)):
        raise ParameterError(f"extent must be finite and > 0, got {extent}")


def random_layout(edges, extent: float = 100.0, seed: int = 0) -> LayoutGraph:
    """Independent uniform coordinates in [0, extent]^2 for every endpoint id
    (graphio.py:141-148; O(n) host work, no kernel)."""
    _check_extent(extent)
    ids = _vertex_ids(edges)
    rng = np.random.default_rng(seed)
    xy = rng.uniform(0.0, extent, size=(len(ids), 2))
    return LayoutGraph(ids, xy, edges)


def fr_layout(edges, iterations: int = 50, seed: int = 0, extent: float = 100.0,
              device=None) -> LayoutGraph:
    """Force-directed layout (graphio.py:151-197) on the GPU."""
    import torch

    if iterations < 1:
        raise ParameterError(f"iterations must be >= 1, got {iterations}")
    _check_extent(extent)
    ids = _vertex_ids(edges)
    n = len(ids)
    norm_edges, _, _ = normalize_edges(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    ei = np.searchsorted(ids, norm_edges[:, 0])
    ej = np.searchsorted(ids, norm_edges[:, 1])
    rng = np.random.default_rng(seed)
    pos0 = rng.uniform(0.0, extent, size=(n, 2))
    L = _lib.lib()
    dev = torch.device("cuda") if device is None else torch.device(device)
    pos = torch.from_numpy(np.ascontiguousarray(pos0)).to(dev)
    tei = torch.from_numpy(np.ascontiguousarray(ei, dtype=np.int64)).to(dev)
    tej = torch.from_numpy(np.ascontiguousarray(ej, dtype=np.int64)).to(dev)
    m = len(norm_edges)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.glr_fr_layout(pos.data_ptr(), n, tei.data_ptr() if m else None,
                         tej.data_ptr() if m else None, m, int(iterations), float(extent), stream)
    _lib.check(rc, "glr_fr_layout")
    return LayoutGraph(ids, pos.cpu().numpy(), norm_edges)


def generate_layout(edges, kind: str = "random", seed: int = 0, extent: float = 100.0,
                    iterations: int = 50) -> LayoutGraph:
    """Seeded layout for an edge set (engine.py generate_layout)."""
    if kind == "random":
        return random_layout(edges, extent=extent, seed=seed)
    if kind == "fr":
        return fr_layout(edges, iterations=iterations, seed=seed, extent=extent)
    raise ParameterError(f"layout kind must be 'random' or 'fr', got {kind!r}")
