"""Seeded synthetic inputs for the five BASELINE.json configurations.

There is no public dataset for this path: BASELINE.json's configs are
generator recipes; these functions realise them with fixed
seeds so the GPU box, the tests and the golden fixtures see identical graphs.

* C1  uniform G(1000, 5000) via the reference's random_graph algorithm
      (graphio.py:200-231, restated) + uniform [0,1]^2 positions
* C2  Barabasi-Albert n=20,000, 2 edges per node (networkx) + 20-Gaussian
      mixture positions (sigma 0.05)
* C3  random geometric graph, 100,000 uniform points, radius for ~500k edges
* C4  1000x1000 jittered triangular lattice (~3M edges)
* C5  Chung-Lu power law (gamma 2.3), 4,000,000 edges over 1,500,000
      vertices on the integer 2^16 x 2^16 lattice

Each returns ``(LayoutGraph, params)`` with params = {"radius", "ideal",
"metrics"}.  Graph builders emit canonical edge lists directly and wrap them
with ``LayoutGraph.from_normalized`` (the contract's checks that matter --
zero-length edges, duplicates, loops -- are enforced by construction and
re-checked by ``verify_contract``).
"""

from __future__ import annotations

import math

import numpy as np

from .model import LayoutGraph, normalize_edges

IDEAL_70 = math.radians(70.0)  # bit-identical to 7*pi/18


def random_graph(n: int, m: int, seed: int = 0) -> np.ndarray:
    """Uniform simple graph with exactly m edges on vertices 0..n-1, drawing
    the same random stream as the reference's generator (graphio.py:200-231)
    so seeded graphs coincide with the reference's."""
    max_m = n * (n - 1) // 2
    if m == 0:
        return np.empty((0, 2), dtype=np.int64)
    rng = np.random.default_rng(seed)
    if 3 * m > max_m and max_m <= 20_000_000:
        iu, ju = np.triu_indices(n, k=1)
        take = rng.choice(max_m, size=m, replace=False)
        return np.column_stack((iu[take], ju[take])).astype(np.int64)
    seen: set = set()
    out: list = []
    while len(out) < m:
        want = (m - len(out)) * 2 + 16
        a = rng.integers(0, n, size=want).tolist()
        b = rng.integers(0, n, size=want).tolist()
        for p, q in zip(a, b):
            if p == q:
                continue
            key = (p, q) if p < q else (q, p)
            if key in seen:
                continue
            seen.add(key)
            out.append(key)
            if len(out) == m:
                break
    return np.asarray(out, dtype=np.int64)


def _canonical(edges: np.ndarray, n: int) -> np.ndarray:
    """Sorted unique small-first rows via int64 keys (n^2 < 2^63)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    keep = lo != hi
    key = np.unique(lo[keep] * np.int64(n) + hi[keep])
    return np.stack([key // n, key % n], axis=1)


def config1(seed: int = 0):
    edges = random_graph(1000, 5000, seed=seed)
    xy = np.random.default_rng(seed + 1).uniform(0.0, 1.0, (1000, 2))
    g = LayoutGraph(np.arange(1000), xy, edges)
    return g, {"radius": 0.005, "ideal": IDEAL_70, "metrics": ("nc", "ma", "ml", "ec", "eca")}


def config2(seed: int = 0):
    import networkx as nx

    G = nx.barabasi_albert_graph(20000, 2, seed=seed)
    edges = np.asarray(list(G.edges()), dtype=np.int64)
    rng = np.random.default_rng(seed + 1)
    centres = rng.uniform(0.0, 1.0, (20, 2))
    labels = rng.integers(0, 20, 20000)
    xy = centres[labels] + rng.normal(0.0, 0.05, (20000, 2))
    g = LayoutGraph(np.arange(20000), xy, edges)
    return g, {"radius": 0.001, "ideal": IDEAL_70, "metrics": ("nc", "ma", "ml", "ec", "eca")}


C3_RHO = math.sqrt(1e-4 / math.pi) * 1.02


def config3(seed: int = 0):
    from scipy.spatial import cKDTree

    xy = np.random.default_rng(seed).uniform(0.0, 1.0, (100000, 2))
    pairs = cKDTree(xy).query_pairs(C3_RHO, output_type="ndarray")
    g = LayoutGraph.from_normalized(xy, _canonical(pairs, len(xy)))
    return g, {"radius": 2.5e-4, "ideal": IDEAL_70, "metrics": ("ec", "eca", "nc")}


def triangular_lattice(R: int, seed: int = 0, jitter: float = 1e-3):
    """R x R triangular lattice, spacing 1, odd rows shifted by 1/2, row pitch
    sqrt(3)/2, uniform jitter in [-jitter, jitter] per coordinate; edges to
    the three forward neighbours -> (R-1)(3R-1) edges."""
    i, j = np.divmod(np.arange(R * R, dtype=np.int64), R)
    x = j + 0.5 * (i % 2)
    y = i * (math.sqrt(3.0) / 2.0)
    xy = np.stack([x, y], axis=1) + np.random.default_rng(seed).uniform(
        -jitter, jitter, (R * R, 2))
    vid = i * R + j
    parts = [np.stack([vid[j < R - 1], vid[j < R - 1] + 1], axis=1)]  # same row
    up = i < R - 1
    even = up & (i % 2 == 0)
    odd = up & (i % 2 == 1)
    # even row (offset 0): neighbours (i+1, j-1) and (i+1, j)
    parts.append(np.stack([vid[even & (j > 0)], vid[even & (j > 0)] + R - 1], axis=1))
    parts.append(np.stack([vid[even], vid[even] + R], axis=1))
    # odd row (offset 1/2): neighbours (i+1, j) and (i+1, j+1)
    parts.append(np.stack([vid[odd], vid[odd] + R], axis=1))
    parts.append(np.stack([vid[odd & (j < R - 1)], vid[odd & (j < R - 1)] + R + 1], axis=1))
    edges = _canonical(np.concatenate(parts), R * R)
    return xy, edges


def config4(seed: int = 0, R: int = 1000):
    xy, edges = triangular_lattice(R, seed=seed)
    g = LayoutGraph.from_normalized(xy, edges)
    return g, {"radius": 0.25, "ideal": IDEAL_70, "metrics": ("nc", "ma", "ml", "ec", "eca")}


def chung_lu(n: int, m: int, gamma: float, rng: np.random.Generator, xy: np.ndarray):
    """Chung-Lu multigraph sampled by inverse-CDF endpoint draws with weights
    (i+1)^(-1/(gamma-1)); loops, duplicates and zero-length (coincident
    endpoint) pairs are dropped and the draw topped up until m unique edges
    exist; a random subset of exactly m is kept."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    keys = np.empty(0, dtype=np.int64)
    while len(keys) < m:
        k = int((m - len(keys)) * 1.1) + 1024
        u = np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), n - 1)
        v = np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), n - 1)
        lo = np.minimum(u, v).astype(np.int64)
        hi = np.maximum(u, v).astype(np.int64)
        ok = (lo != hi) & np.any(xy[lo] != xy[hi], axis=1)
        keys = np.unique(np.concatenate([keys, lo[ok] * np.int64(n) + hi[ok]]))
    keys = np.sort(rng.permutation(keys)[:m])
    return np.stack([keys // n, keys % n], axis=1)


def config5(seed: int = 5, n: int = 1_500_000, m: int = 4_000_000):
    rng = np.random.default_rng(seed)
    xy = rng.integers(0, 2**16, (n, 2)).astype(np.float64)
    edges = chung_lu(n, m, 2.3, rng, xy)
    g = LayoutGraph.from_normalized(xy, edges)
    return g, {"radius": 8.0, "ideal": IDEAL_70, "metrics": ("ec", "eca", "nc")}


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(config: int, **kw):
    return CONFIGS[int(config)](**kw)


def verify_contract(g) -> None:
    """Assert the LayoutGraph contract on a generated graph (tests)."""
    e = g.edges
    if len(e):
        assert np.all(e[:, 0] < e[:, 1])
        norm, loops, dupes = normalize_edges(e)
        assert loops == 0 and dupes == 0
        assert np.array_equal(norm, e)
        assert not np.any(np.all(g.xy[e[:, 0]] == g.xy[e[:, 1]], axis=1))
    assert np.all(np.isfinite(g.xy))


def fingerprint(g) -> str:
    """Short content hash of (xy, edges) for golden-fixture identity checks."""
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.xy, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(g.edges, dtype=np.int64).tobytes())
    return h.hexdigest()[:16]
