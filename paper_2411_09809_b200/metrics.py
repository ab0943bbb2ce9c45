"""Drop-in exact readability metrics on B200.

Same names, signatures, validation, degenerate-case returns and scalar types
as the reference's serial oracle functions
(/root/reference/pkg/src/glare/metrics/exact.py, re-exported by
metrics/__init__.py:11-25):

    node_occlusion(g, r) -> int                      exact.py:55-74
    minimum_angle(g) -> float                        exact.py:119-124
    edge_length_variation(g) -> float                exact.py:134-142
    edge_crossing(g) -> int                          exact.py:225-227
    edge_crossing_angle(g, ideal_angle=7pi/18)       exact.py:230-238
    _crossing_scan(g, ideal_angle=None)              exact.py:145-222

``g`` is this package's ``LayoutGraph``, the reference's own ``LayoutGraph``
(duck-typed on ``xy``/``edges``), or a ``DeviceGraph`` whose arrays already
live in HBM.  The arithmetic runs in the hand-written sm_100a kernels of
``libglare_b200.so``; there is no CPU path.

Each all-pairs metric takes a keyword-only ``strategy``:

* ``"dense"`` -- every tile pair of the upper triangle (the roofline-judged
  kernel; with an ideal angle the edges are put in direction order with hub
  groups, see ``CrossingRecords``);
* ``"culled"`` -- elements reordered by Morton code (vertices: position;
  edges: the 4-D code of the bbox sides, with hub groups), only tile pairs
  whose tile bounding boxes can interact are scanned (exactly the same
  result; orders of magnitude fewer pair tests on spatially local inputs,
  46% fewer on C5's long random edges);
* ``"auto"`` (default) -- culled when the candidate tile pairs are at most
  ``CULL_FRACTION`` (occlusion) / ``CROSS_CULL_FRACTION`` (crossing) of all
  tile pairs, dense otherwise.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _lib
from .model import IDEAL_ANGLE_DEFAULT, ParameterError, check_ideal_angle, check_radius

STRATEGIES = ("auto", "dense", "culled")
CULL_FRACTION = 0.25      # auto (occlusion): cull when candidates <= this share of tile pairs
# auto (crossing): a culled unit costs about as much as a dense one (the
# dense pass has the one-DADD angle in most units, the culled list does not,
# but needs no band order); C5 keeps 35% of the tile pairs as mixed units: 1.6 s vs 4.5 s
CROSS_CULL_FRACTION = 0.75
#: cost of a certified full unit (no predicate; closed form or piecewise-linear
#: sums over sorted angles) relative to a mixed one, for the auto decision and
#: balanced shards (C5: 10.3 M full units in ~15 ms, 42.7 M mixed in ~1.4 s)
FULL_UNIT_WEIGHT = 0.05
AUTO_MIN_EDGES = 20_000   # auto: below this the dense pass is microseconds
# theta order: vertices of at least this degree get their own edge group
# (glr_theta_sort_edges; 0 = the library default).  Tuning knob only.
HUB_DEGREE = int(os.environ.get("GLARE_B200_HUB_DEGREE", "0"))


class DeviceGraph:
    """Positions and normalised edge index pairs resident on a CUDA device.

    ``xy``: float64 (n, 2) contiguous; ``edges``: int64 (m, 2) contiguous,
    normalised as ``LayoutGraph`` does (small index first, unique).
    """

    __slots__ = ("xy", "edges")

    def __init__(self, xy: torch.Tensor, edges: torch.Tensor):
        if xy.dtype != torch.float64 or xy.dim() != 2 or xy.shape[1] != 2 or not xy.is_cuda:
            raise ValueError("DeviceGraph.xy must be a CUDA float64 (n, 2) tensor")
        if edges.dtype != torch.int64 or edges.dim() != 2 or edges.shape[1] != 2:
            raise ValueError("DeviceGraph.edges must be an int64 (m, 2) tensor")
        if edges.device != xy.device:
            raise ValueError("DeviceGraph tensors must share a device")
        if edges.numel():
            # the kernels index xy[edges] unchecked: one device min/max here
            lo, hi = (int(v) for v in torch.aminmax(edges))
            if lo < 0 or hi >= xy.shape[0]:
                raise ValueError(f"DeviceGraph.edges index out of range [0, {xy.shape[0]}): "
                                 f"min {lo}, max {hi}")
        self.xy = xy.contiguous()
        self.edges = edges.contiguous()

    @classmethod
    def from_graph(cls, g, device=None, pin: bool = False) -> "DeviceGraph":
        if isinstance(g, DeviceGraph):
            return g
        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        xy = torch.from_numpy(np.ascontiguousarray(g.xy, dtype=np.float64))
        ed = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64).reshape(-1, 2))
        if pin:
            xy = xy.pin_memory()
            ed = ed.pin_memory()
        return cls(xy.to(device, non_blocking=pin), ed.to(device, non_blocking=pin))

    @property
    def num_vertices(self) -> int:
        return int(self.xy.shape[0])

    @property
    def num_edges(self) -> int:
        return int(self.edges.shape[0])


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev(g) -> DeviceGraph:
    _lib.lib()  # fail loudly before any work if the CUDA library is unusable
    return DeviceGraph.from_graph(g)


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _check_strategy(strategy: str) -> str:
    if strategy not in STRATEGIES:
        raise ParameterError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
    return strategy


def _classified_candidates(buf: torch.Tensor, n: int, m: int, rows: tuple[int, int] | None = None):
    """glr_crossing_candidates_classified / _rows: ([mixed | full] list,
    sub-unit masks, mixed, full); ``rows = (rank, world)`` keeps the tile rows
    ti = rank (mod world) only."""
    L = _lib.lib()
    rank, world = rows if rows is not None else (0, 1)
    counts = (ctypes.c_uint64 * 2)()
    _lib.check(L.glr_crossing_candidates_rows(_ptr(buf), n, m, None, None, 0, counts, rank, world,
                                              _stream()),
               "glr_crossing_candidates_rows")
    mixed, full = int(counts[0]), int(counts[1])
    lst = torch.empty((max(mixed + full, 1), 2), dtype=torch.int32, device=buf.device)
    sub_dtype = {2: torch.int16, 4: torch.int32, 8: torch.int64}[L.glr_crossing_sub_mask_bytes()]
    sub = torch.zeros(max(mixed + full, 1), dtype=sub_dtype, device=buf.device)
    if mixed + full:
        _lib.check(L.glr_crossing_candidates_rows(_ptr(buf), n, m, _ptr(lst), _ptr(sub),
                                                  mixed + full, counts, rank, world, _stream()),
                   "glr_crossing_candidates_rows")
    return lst[:mixed + full], sub, mixed, full


def _global_cost(cost: float, world: int, device) -> float:
    """Sum of the ranks' plan costs (torch.distributed when initialised;
    otherwise this rank's cost times world -- single-process callers that
    walk the ranks one after the other should name the strategy instead of
    "auto", since their estimates may differ near the threshold)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == world:
        t = torch.tensor([cost], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())
    return cost * world


def _candidates(fn, *args) -> torch.Tensor:
    """Two-phase candidate list: count (synchronous), allocate, fill."""
    count = ctypes.c_uint64(0)
    _lib.check(fn(*args, None, 0, ctypes.byref(count), _stream()), fn.__name__)
    n = int(count.value)
    dev = torch.device("cuda", torch.cuda.current_device())
    lst = torch.empty((max(n, 1), 2), dtype=torch.int32, device=dev)
    if n:
        _lib.check(fn(*args, _ptr(lst), n, ctypes.byref(count), _stream()), fn.__name__)
    return lst[:n]


# ---- unit-range kernels (device results, no host sync) ----------------------


def occlusion_units(n: int) -> int:
    return int(_lib.lib().glr_occlusion_units(n))


def crossing_units(m: int) -> int:
    return int(_lib.lib().glr_crossing_units(m))


def occlusion_threshold(r: float) -> float:
    """(2r)^2 with the reference's own expression (exact.py:63)."""
    return (2.0 * r) ** 2


def occlusion_partial(dg: DeviceGraph, thr: float, unit_begin: int, unit_end: int,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """Device float64[1]: occluding pairs inside dense units [unit_begin, unit_end)."""
    L = _lib.lib()
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=dg.xy.device)
    rc = L.glr_occlusion_count(_ptr(dg.xy), dg.num_vertices, float(thr), int(unit_begin),
                               int(unit_end), _ptr(out), _stream())
    _lib.check(rc, "glr_occlusion_count")
    return out


class OcclusionPlan:
    """Node-occlusion pass for one radius.  ``culled``: vertices in Morton
    order and the candidate vertex-tile pairs whose boxes are closer than 2r;
    otherwise the dense triangle over the input order."""

    def __init__(self, dg: DeviceGraph, r: float, strategy: str = "auto"):
        L = _lib.lib()
        self.r = r
        self.thr = occlusion_threshold(r)
        self.n = dg.num_vertices
        self.dense_units = occlusion_units(self.n)
        self.list = None
        self.xy = dg.xy
        strategy = _check_strategy(strategy)
        if strategy != "dense" and self.n >= 2:
            xs = torch.empty_like(dg.xy)
            _lib.check(L.glr_spatial_sort_vertices(_ptr(dg.xy), self.n, _ptr(xs), _stream()),
                       "glr_spatial_sort_vertices")
            lst = _candidates(L.glr_occlusion_candidates, _ptr(xs), self.n, 2.0 * r)
            if strategy == "culled" or len(lst) <= CULL_FRACTION * self.dense_units:
                self.xy, self.list = xs, lst

    @property
    def culled(self) -> bool:
        return self.list is not None

    @property
    def units(self) -> int:
        return len(self.list) if self.culled else self.dense_units

    def partial(self, unit_begin: int, unit_end: int,
                out: torch.Tensor | None = None) -> torch.Tensor:
        L = _lib.lib()
        if out is None:
            out = torch.empty(1, dtype=torch.float64, device=self.xy.device)
        if self.culled:
            rc = L.glr_occlusion_count_list(_ptr(self.xy), self.n, self.thr,
                                            _ptr(self.list) if len(self.list) else None,
                                            len(self.list), int(unit_begin), int(unit_end),
                                            _ptr(out), _stream())
            _lib.check(rc, "glr_occlusion_count_list")
        else:
            rc = L.glr_occlusion_count(_ptr(self.xy), self.n, self.thr, int(unit_begin),
                                       int(unit_end), _ptr(out), _stream())
            _lib.check(rc, "glr_occlusion_count")
        return out


class CrossingRecords:
    """Prepared per-edge records (glr_crossing_prepare) kept in HBM so that
    several unit ranges / both E_c and E_ca reuse one prologue.

    ``strategy`` selects dense or culled scanning (see the module docstring);
    with culling the records hold the Morton-ordered edge list and ``list``
    the candidate tile pairs.  ``order="theta"`` makes dense records hold the
    edges ordered by direction (glr_theta_sort_edges), which lets the fused
    E_c + E_ca pass evaluate the angle deviation with one FP64 operation per
    pair in almost every unit; ``"input"`` keeps the caller's order with
    ``strategy="dense"`` (unit ranges then match the oracle's unit-range
    restatement).  When ``"auto"`` builds the culled plan and then prefers the
    dense pass, input order reuses the Morton-ordered records (one prologue);
    theta order prepares its own (the Morton order is needed to decide, the
    direction order to run).  Results never depend on the order."""

    ORDERS = ("input", "theta")

    def __init__(self, dg: DeviceGraph, strategy: str = "dense", order: str = "input",
                 rows: tuple[int, int] | None = None):
        strategy = _check_strategy(strategy)
        if order not in self.ORDERS:
            raise ParameterError(f"order must be one of {self.ORDERS}, got {order!r}")
        if rows is not None and not (rows[1] >= 1 and 0 <= rows[0] < rows[1]):
            raise ParameterError(f"rows must be (rank, world) with 0 <= rank < world, got {rows!r}")
        self.m = dg.num_edges
        self.n = dg.num_vertices
        self.list = self.sub = None
        self.n_mixed = self.n_full = 0
        #: (rank, world) when a culled plan holds only this rank's tile rows
        self.rows = None
        if strategy != "dense" and self.m >= 2 and (strategy == "culled"
                                                    or self.m >= AUTO_MIN_EDGES):
            L = _lib.lib()
            es = torch.empty_like(dg.edges)
            _lib.check(L.glr_spatial_sort_edges(_ptr(dg.xy), self.n, _ptr(dg.edges), self.m,
                                                _ptr(es), _stream()),
                       "glr_spatial_sort_edges")
            self._prepare(dg.xy, es)
            if rows is not None and rows[1] == 1:
                rows = None
            lst, sub, mixed, full = _classified_candidates(self.buf, self.n, self.m, rows)
            cost = mixed + FULL_UNIT_WEIGHT * full
            if rows is not None:
                # every rank must take the same decision: sum the ranks' costs
                cost = _global_cost(cost, rows[1], self.buf.device)
            if strategy == "culled" or cost <= CROSS_CULL_FRACTION * crossing_units(self.m):
                self.list, self.sub, self.n_mixed, self.n_full = lst, sub, mixed, full
                self.rows = rows
                return
            if order == "input":
                # auto chose the dense pass: results never depend on the edge
                # order, so the Morton-ordered records serve it as they are
                # (no second prologue)
                return
        if order == "theta" and self.m >= 2:
            es = torch.empty_like(dg.edges)
            _lib.check(_lib.lib().glr_theta_sort_edges(_ptr(dg.xy), self.n, _ptr(dg.edges),
                                                       self.m, HUB_DEGREE, _ptr(es), _stream()),
                       "glr_theta_sort_edges")
            self._prepare(dg.xy, es)
            return
        self._prepare(dg.xy, dg.edges)

    def _prepare(self, xy: torch.Tensor, edges: torch.Tensor) -> None:
        L = _lib.lib()
        nbytes = int(L.glr_crossing_records_bytes(self.n, self.m))
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=xy.device)
        rc = L.glr_crossing_prepare(_ptr(xy), self.n, _ptr(edges) if self.m else None, self.m,
                                    _ptr(self.buf), _stream())
        _lib.check(rc, "glr_crossing_prepare")

    @property
    def culled(self) -> bool:
        return self.list is not None

    @property
    def units(self) -> int:
        return len(self.list) if self.culled else crossing_units(self.m)

    #: skip the sub-unit blocks certified empty (tuning / cross-check knob)
    use_sub_masks = True

    def _sub_ptr(self):
        return _ptr(self.sub) if self.use_sub_masks and len(self.list) else None

    #: pair-kernel modes (glr_crossing_fast_path / glr_crossing_set_mode)
    MODE_GENERAL, MODE_SIGN, MODE_FILTER = 0, 1, 2

    def mode(self) -> int:
        """Pair-kernel mode of these records (synchronises the stream)."""
        mode = _lib.lib().glr_crossing_fast_path(_ptr(self.buf), _stream())
        if mode < 0:
            _lib.check(_lib.GLR_ECUDA, "glr_crossing_fast_path")
        return mode

    def set_mode(self, mode: int) -> "CrossingRecords":
        """Force a pair-kernel mode (cross-checks); 1 and 2 degrade to 0
        outside the fast window.  All modes give identical results."""
        _lib.check(_lib.lib().glr_crossing_set_mode(_ptr(self.buf), int(mode), _stream()),
                   "glr_crossing_set_mode")
        return self

    def fast_path(self) -> bool:
        """True when the input lies in the fast window (modes 1/2)."""
        return self.mode() != self.MODE_GENERAL

    def partial_interleaved(self, ideal: float | None, rank: int, world: int,
                            out: torch.Tensor | None = None) -> torch.Tensor:
        """Device float64[2]: this rank's share of the whole unit space under
        interleaved chunk ownership (glr_crossing_pairs_interleaved); the
        ranks' partials sum exactly to the full (count, dev_sum)."""
        if out is None:
            out = torch.empty(2, dtype=torch.float64, device=self.buf.device)
        if self.culled:
            if self.rows is not None:
                # the plan already holds this rank's rows only: scan all of it
                if (int(rank), int(world)) != tuple(self.rows):
                    raise ParameterError(
                        f"plan built for rows {self.rows}, asked for rank {rank} of {world}")
                rank, world = 0, 1
            if len(self.list) == 0:
                return out.zero_()
            rc = _lib.lib().glr_crossing_pairs_classified(
                _ptr(self.buf), self.n, self.m, 0 if ideal is None else 1,
                0.0 if ideal is None else float(ideal), _ptr(self.list), self._sub_ptr(),
                self.n_mixed, self.n_full, 0, len(self.list), int(rank), int(world), _ptr(out),
                _stream())
            _lib.check(rc, "glr_crossing_pairs_classified")
            return out
        rc = _lib.lib().glr_crossing_pairs_interleaved(
            _ptr(self.buf), self.n, self.m, 0 if ideal is None else 1,
            0.0 if ideal is None else float(ideal), None, 0, int(rank), int(world), _ptr(out),
            _stream())
        _lib.check(rc, "glr_crossing_pairs_interleaved")
        return out

    def tile_weights(self, beta: float | None = None) -> np.ndarray:
        """Per j-tile cost weights (glr_crossing_tile_weights), on the host."""
        from .sharding import RUN_START_BETA

        T = -(-max(self.m, 1) // _lib.lib().glr_crossing_tile())
        w = torch.empty(T, dtype=torch.float64, device=self.buf.device)
        rc = _lib.lib().glr_crossing_tile_weights(
            _ptr(self.buf), self.n, self.m, RUN_START_BETA if beta is None else float(beta),
            _ptr(w), _stream())
        _lib.check(rc, "glr_crossing_tile_weights")
        return w.cpu().numpy()

    def shard(self, rank: int, world: int, balanced: bool = True) -> tuple[int, int]:
        """This rank's contiguous unit range: equal estimated cost (balanced)
        or equal unit counts."""
        from . import sharding

        if world == 1 or not balanced or self.m < 2:
            return sharding.shard_range(self.units, rank, world)
        w = self.tile_weights()
        if not self.culled:
            return sharding.triangle_range(w, rank, world, _lib.lib().glr_crossing_band())
        lst = self.list.cpu().numpy()
        unit_w = w[lst[:, 1]] * np.where(lst[:, 0] == lst[:, 1], 0.5, 1.0)
        unit_w[self.n_mixed:] *= FULL_UNIT_WEIGHT
        return sharding.weighted_range(unit_w, rank, world)

    def partial(self, ideal: float | None, unit_begin: int, unit_end: int,
                out: torch.Tensor | None = None) -> torch.Tensor:
        """Device float64[2] = (count, dev_sum) over units [unit_begin, unit_end)."""
        if out is None:
            out = torch.empty(2, dtype=torch.float64, device=self.buf.device)
        L = _lib.lib()
        angle = 0 if ideal is None else 1
        ideal_v = 0.0 if ideal is None else float(ideal)
        if self.culled:
            rc = L.glr_crossing_pairs_classified(_ptr(self.buf), self.n, self.m, angle, ideal_v,
                                                 _ptr(self.list) if len(self.list) else None,
                                                 self._sub_ptr(), self.n_mixed, self.n_full,
                                                 int(unit_begin),
                                                 int(unit_end), 0, 1, _ptr(out), _stream())
            _lib.check(rc, "glr_crossing_pairs_classified")
        else:
            rc = L.glr_crossing_pairs(_ptr(self.buf), self.n, self.m, angle, ideal_v,
                                      int(unit_begin), int(unit_end), _ptr(out), _stream())
            _lib.check(rc, "glr_crossing_pairs")
        return out


def length_variation_device(dg: DeviceGraph, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device float64[3] = (mean length, sum (l - mean)^2, M_l)."""
    if out is None:
        out = torch.empty(3, dtype=torch.float64, device=dg.xy.device)
    rc = _lib.lib().glr_edge_length_variation(
        _ptr(dg.xy), dg.num_vertices, _ptr(dg.edges) if dg.num_edges else None,
        dg.num_edges, _ptr(out), _stream())
    _lib.check(rc, "glr_edge_length_variation")
    return out


def minimum_angle_device(dg: DeviceGraph, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device float64[3] = (sum of d_v, vertices with degree >= 1, M_a)."""
    if out is None:
        out = torch.empty(3, dtype=torch.float64, device=dg.xy.device)
    rc = _lib.lib().glr_minimum_angle(
        _ptr(dg.xy), dg.num_vertices, _ptr(dg.edges) if dg.num_edges else None,
        dg.num_edges, _ptr(out), _stream())
    _lib.check(rc, "glr_minimum_angle")
    return out


# ---- drop-in metric functions ------------------------------------------------


def _num_vertices(g) -> int:
    return int(g.num_vertices)


def _num_edges(g) -> int:
    return int(g.num_edges)


def node_occlusion(g, r: float, *, strategy: str = "auto") -> int:
    """Unordered vertex pairs with squared distance strictly below (2r)^2."""
    r = check_radius(r)
    _check_strategy(strategy)
    n = _num_vertices(g)
    if n < 2:
        return 0
    occlusion_threshold(r)  # raises OverflowError exactly where exact.py:63 does
    plan = OcclusionPlan(_dev(g), r, strategy)
    return int(plan.partial(0, plan.units).item())


def minimum_angle(g) -> float:
    """1 minus the mean normalised deviation from each vertex's ideal gap."""
    if _num_edges(g) == 0:
        return 1.0
    s, count, _ = minimum_angle_device(_dev(g)).tolist()
    return 1.0 - s / count  # exact.py:124: 1 - mean(d_v)


def edge_length_variation(g) -> float:
    """Coefficient-of-variation style spread of edge lengths, in [0, 1]."""
    m = _num_edges(g)
    if m <= 1:
        return 0.0
    mean, sq, _ = length_variation_device(_dev(g)).tolist()
    # exact.py:141-142 on the host, so degenerate inputs raise what the
    # reference raises (ZeroDivisionError when every length is 0.0)
    la = math.sqrt(sq / (m * mean * mean))
    return la / math.sqrt(m - 1)


def _crossing_scan(g, ideal_angle: float | None = None, *,
                   strategy: str = "auto") -> tuple[int, float]:
    """(crossing count, sum of |ideal - crossing angle| over crossings)."""
    _check_strategy(strategy)
    m = _num_edges(g)
    if m < 2:
        return 0, 0.0
    rec = CrossingRecords(_dev(g), strategy, "input" if ideal_angle is None else "theta")
    out = rec.partial(ideal_angle, 0, rec.units)
    count, dev = out.tolist()
    return int(count), (float(dev) if ideal_angle is not None else 0.0)


def edge_crossing(g, *, strategy: str = "auto") -> int:
    """Count of non-adjacent edge pairs that properly intersect."""
    return _crossing_scan(g, strategy=strategy)[0]


def edge_crossing_angle(g, ideal_angle: float = IDEAL_ANGLE_DEFAULT, *,
                        strategy: str = "auto") -> float:
    """1 minus the mean normalised deviation of crossing angles from ideal."""
    ideal_angle = check_ideal_angle(ideal_angle)
    total, dev_sum = _crossing_scan(g, ideal_angle, strategy=strategy)
    if total == 0:
        return 1.0
    return 1.0 - (dev_sum / ideal_angle) / total


def crossing_count_and_angle(g, ideal_angle: float = IDEAL_ANGLE_DEFAULT, *,
                             strategy: str = "auto") -> tuple[int, float]:
    """E_c and E_ca from ONE fused scan (the engine uses this when both are
    requested; the reference runs _crossing_scan twice, engine.py:85-92)."""
    ideal_angle = check_ideal_angle(ideal_angle)
    total, dev_sum = _crossing_scan(g, ideal_angle, strategy=strategy)
    eca = 1.0 if total == 0 else 1.0 - (dev_sum / ideal_angle) / total
    return total, eca


__all__ = [
    "DeviceGraph",
    "CrossingRecords",
    "OcclusionPlan",
    "STRATEGIES",
    "node_occlusion",
    "minimum_angle",
    "edge_length_variation",
    "edge_crossing",
    "edge_crossing_angle",
    "_crossing_scan",
    "crossing_count_and_angle",
    "occlusion_partial",
    "occlusion_units",
    "crossing_units",
    "occlusion_threshold",
    "length_variation_device",
    "minimum_angle_device",
]
