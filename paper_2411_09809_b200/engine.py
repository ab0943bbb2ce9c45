"""`evaluate` with a "b200" mode: the reference engine's report, GPU metrics.

Mirrors the reference's oracle dispatch (/root/reference/pkg/src/glare/
engine.py:74-94 and 140-160) and its report type (model.py:189-267): same
metric keys (nc, ma, ml, ec, eca), same canonical order, same degenerate-case
warning strings, same per-metric wall times in ``report.elapsed``.  The only
difference is that E_c and E_ca share ONE fused crossing scan when both are
requested (the reference scans twice, engine.py:85-92); the scan's time is
charged to whichever of the two comes first and the second reads ~0.

``bench`` mirrors engine.py:209-256's invariant for this path: values must
not change with the number of shards the pair space is split into
(counts exactly, reals within 1e-9 relative), which is exactly what a
multi-GPU run relies on.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

from . import metrics as M
from . import sharding
from .model import (
    METRIC_FIELDS,
    WARN_FEW_EDGES_LENGTH,
    WARN_NO_CROSSINGS,
    WARN_NO_EDGES_ANGLE,
    InvariantError,
    MetricParams,
    ParameterError,
    SchemaError,
)

MODES = ("b200", "b200-enhanced")
_DEFAULT_METRICS = ("nc", "ma", "ml", "ec", "eca")
_ENHANCED_METRICS = ("nc", "ec", "eca")  # engine.py:33


@dataclass
class ReadabilityReport:
    """Metric values, parameter echo, per-metric seconds, warnings
    (reference model.py:189-216; to_dict has the same schema)."""

    mode: str
    node_occlusion: int | None = None
    minimum_angle: float | None = None
    edge_length_variation: float | None = None
    edge_crossing: int | None = None
    edge_crossing_angle: float | None = None
    params: dict = field(default_factory=dict)
    elapsed: dict = field(default_factory=dict)
    warnings: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {
            "mode": self.mode,
            "metrics": {name: getattr(self, name) for name in METRIC_FIELDS.values()},
            "params": dict(self.params),
            "elapsed": dict(self.elapsed),
            "warnings": list(self.warnings),
        }

    def to_json(self) -> str:
        """Canonical JSON (sorted keys, indent 2, finite values only), as the
        reference's graphio.dump_report_json (graphio.py:234-239)."""
        try:
            return json.dumps(self.to_dict(), sort_keys=True, indent=2, allow_nan=False)
        except ValueError as exc:
            raise SchemaError(f"report contains a non-finite value: {exc}") from exc


def _normalize_metrics(metrics, mode: str = "b200") -> tuple:
    """engine.py:36-55: all five metrics in b200 mode; b200-enhanced (the
    reference's "enhanced" mode on the GPU) supports nc, ec, eca."""
    enhanced = mode == "b200-enhanced"
    if metrics is None:
        return _ENHANCED_METRICS if enhanced else _DEFAULT_METRICS
    seen = []
    for key in metrics:
        if key not in METRIC_FIELDS:
            raise ParameterError(f"unknown metric {key!r}; choose from {sorted(METRIC_FIELDS)}")
        if key not in seen:
            seen.append(key)
    if not seen:
        raise ParameterError("no metrics requested")
    if enhanced:
        bad = [k for k in seen if k not in _ENHANCED_METRICS]
        if bad:
            raise ParameterError(f"enhanced mode supports only {_ENHANCED_METRICS}, not {bad}")
    return tuple(seen)


def _check_mode(mode: str) -> str:
    if mode not in MODES:
        raise ParameterError(f"mode must be one of {MODES}, got {mode!r}")
    return mode


def _params_echo(params: MetricParams, world: int) -> dict:
    return {
        "radius": params.radius,
        "ideal_angle_deg": math.degrees(params.ideal_angle),
        "strip_fraction": params.strip_fraction,
        "orientation": params.orientation,
        "gpus": world,
    }


class _Evaluator:
    """Per-metric closures returning (value, warnings); E_c/E_ca share the
    fused scan (cached on first use)."""

    def __init__(self, g, params: MetricParams, rank: int, world: int):
        self.g = g
        self.p = params
        self.rank = rank
        self.world = world
        self._dg = None
        self._scan = None

    def dg(self):
        if self._dg is None:
            self._dg = M.DeviceGraph.from_graph(self.g)
        return self._dg

    def scan(self):
        if self._scan is None:
            if self.g.num_edges < 2:
                self._scan = (0, 0.0)
            elif self.world == 1:
                self._scan = M._crossing_scan(self.dg(), self.p.ideal_angle)
            else:
                out = sharding.sharded_evaluate(self.dg(), None, self.p.ideal_angle,
                                                self.rank, self.world, strategy="auto")
                c, d, _ = out.tolist()
                self._scan = (int(c), float(d))
        return self._scan

    def enhanced_entry(self, key: str):
        """engine.py:119-137 (the reference's "enhanced" mode) on the GPU."""
        from . import enhanced as E

        g, p = self.g, self.p
        if key == "nc":
            return lambda: (E.node_occlusion_grid(self.dg() if g.num_vertices >= 2 else g,
                                                  p.radius), [])
        if key == "ec":
            return lambda: (E.edge_crossing_enhanced(g, p.strip_fraction, p.orientation), [])

        def eca():
            count, dev = E.crossing_angle_stats(g, p.strip_fraction, p.ideal_angle,
                                                p.orientation)
            if count == 0:
                return 1.0, [WARN_NO_CROSSINGS]
            return 1.0 - (dev / p.ideal_angle) / count, []

        return eca

    def entry(self, key: str):
        g, p = self.g, self.p
        if key == "nc":
            if self.world == 1 or g.num_vertices < 2:
                return lambda: (M.node_occlusion(self.dg() if g.num_vertices >= 2 else g,
                                                 p.radius), [])

            def nc():
                out = sharding.sharded_evaluate(self.dg(), p.radius, None, self.rank, self.world,
                                                with_crossing=False, strategy="auto")
                return int(out[2].item()), []

            return nc
        if key == "ma":
            if g.num_edges == 0:
                return lambda: (1.0, [WARN_NO_EDGES_ANGLE])
            return lambda: (M.minimum_angle(self.dg()), [])
        if key == "ml":
            if g.num_edges <= 1:
                return lambda: (0.0, [WARN_FEW_EDGES_LENGTH])
            return lambda: (M.edge_length_variation(self.dg()), [])
        if key == "ec":
            return lambda: (self.scan()[0], [])

        def eca():
            count, dev = self.scan()
            if count == 0:
                return 1.0, [WARN_NO_CROSSINGS]
            return 1.0 - (dev / p.ideal_angle) / count, []

        return eca


def evaluate(g, mode: str = "b200", params: MetricParams | None = None, metrics=None,
             rank: int = 0, world: int = 1) -> ReadabilityReport:
    """Compute the requested metrics on the GPU and return a timed report
    (reference engine.py:140-160).  With world > 1 every rank of an
    initialised torch.distributed group calls this; the pair space is split
    across ranks and each report carries the combined values."""
    mode = _check_mode(mode)
    params = params if params is not None else MetricParams()
    params.validate()
    keys = _normalize_metrics(metrics, mode)
    ev = _Evaluator(g, params, rank, world)
    report = ReadabilityReport(mode=mode, params=_params_echo(params, world))
    for key in keys:
        name = METRIC_FIELDS[key]
        fn = ev.enhanced_entry(key) if mode == "b200-enhanced" else ev.entry(key)
        t0 = time.perf_counter()
        value, warns = fn()
        report.elapsed[name] = time.perf_counter() - t0
        setattr(report, name, value)
        report.warnings.extend(warns)
    return report


def compare(g, params: MetricParams | None = None, metrics=None) -> list:
    """Strip-sweep (b200-enhanced) vs exact (b200) values with percentage
    errors, as the reference's compare (engine.py:163-200)."""
    keys = _normalize_metrics(metrics if metrics is not None else _ENHANCED_METRICS,
                              "b200-enhanced")
    params = params if params is not None else MetricParams()
    params.validate()
    exact = evaluate(g, "b200", params, metrics=keys)
    approx = evaluate(g, "b200-enhanced", params, metrics=keys)
    rows = []
    for key in keys:
        name = METRIC_FIELDS[key]
        o, e = getattr(exact, name), getattr(approx, name)
        if o != 0:
            pct, flagged = abs(e - o) / abs(o) * 100.0, False
        elif e == 0:
            pct, flagged = 0.0, False
        else:
            pct, flagged = None, True
        rows.append({"metric": key, "oracle": o, "enhanced": e, "pct_error": pct,
                     "flagged": flagged})
    return rows


def _values_match(a, b) -> bool:
    """engine.py:203-206."""
    if isinstance(a, int) and isinstance(b, int):
        return a == b
    return abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))


def bench(g, shard_counts=(1, 2, 4, 8), params: MetricParams | None = None, metrics=None) -> list:
    """Seconds per metric when the pair space is split into 1, 2, 4, 8 unit
    ranges evaluated one after another on this GPU; values must be identical
    across shard counts (counts exactly, reals 1e-9), else InvariantError --
    the multi-GPU invariant checked on one device."""
    counts = list(shard_counts)
    if not counts or any((not isinstance(c, int)) or c < 1 for c in counts):
        raise ParameterError(f"shard counts must be integers >= 1, got {counts}")
    params = (params if params is not None else MetricParams()).validate()
    keys = _normalize_metrics(metrics if metrics is not None else ("nc", "ec", "eca"))
    dg = M.DeviceGraph.from_graph(g)
    rows = []
    base: dict = {}
    rec = M.CrossingRecords(dg, order="theta") if g.num_edges >= 2 else None
    for shards in counts:
        t0 = time.perf_counter()
        cnt = dev = 0.0
        occ = 0.0
        for r in range(shards):
            if rec is not None and ("ec" in keys or "eca" in keys):
                c, d = rec.partial(params.ideal_angle, *sharding.shard_range(rec.units, r, shards)).tolist()
                cnt += c
                dev += d
            if "nc" in keys and g.num_vertices >= 2:
                U = M.occlusion_units(g.num_vertices)
                occ += M.occlusion_partial(dg, M.occlusion_threshold(params.radius),
                                           *sharding.shard_range(U, r, shards)).item()
        seconds = time.perf_counter() - t0
        values = {"nc": int(occ), "ec": int(cnt),
                  "eca": 1.0 if cnt == 0 else 1.0 - (dev / params.ideal_angle) / cnt}
        for key in keys:
            if key not in values:
                continue
            if key not in base:
                base[key] = values[key]
            elif not _values_match(base[key], values[key]):
                raise InvariantError(
                    f"{key} changed across shard counts: {base[key]!r} at {counts[0]} "
                    f"vs {values[key]!r} at {shards}")
            rows.append({"shards": shards, "metric": key, "value": values[key],
                         "seconds": seconds})
    return rows
