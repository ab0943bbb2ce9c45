"""evaluate(g, "b200") mirrors the reference engine's oracle reports
(engine.py:74-160, tests/test_engine.py:21-187 of the reference)."""

from __future__ import annotations

import math

import pytest

import cases
from conftest import graph_from, strict_close
from paper_2411_09809_b200 import configs
from paper_2411_09809_b200.engine import _normalize_metrics, _values_match, evaluate
from paper_2411_09809_b200.model import MetricParams, ParameterError


def test_metric_key_validation():
    assert _normalize_metrics(None) == ("nc", "ma", "ml", "ec", "eca")
    assert _normalize_metrics(["ec", "nc", "ec"]) == ("ec", "nc")
    with pytest.raises(ParameterError, match="unknown metric"):
        _normalize_metrics(["xx"])
    with pytest.raises(ParameterError, match="no metrics requested"):
        _normalize_metrics([])
    with pytest.raises(ParameterError, match="mode must be one of"):
        evaluate(graph_from(cases.x_graph), mode="oracle")
    with pytest.raises(ParameterError):
        evaluate(graph_from(cases.x_graph), params=MetricParams(radius=-1.0))
    assert _values_match(3, 3) and not _values_match(3, 4)
    assert _values_match(0.5, 0.5 + 1e-12)


def test_degenerate_reports_need_no_gpu():
    g = graph_from(cases.occ_three)  # 3 vertices, no edges
    r = evaluate(g, metrics=["ma", "ml", "ec", "eca"])
    assert r.minimum_angle == 1.0 and r.edge_length_variation == 0.0
    assert r.edge_crossing == 0 and r.edge_crossing_angle == 1.0
    assert r.warnings == [
        "graph has no edges; minimum_angle reported as 1.0",
        "fewer than 2 edges; edge_length_variation reported as 0.0",
        "no crossings found; edge_crossing_angle reported as 1.0",
    ]
    d = r.to_dict()
    assert set(d) == {"mode", "metrics", "params", "elapsed", "warnings"}
    assert set(d["metrics"]) == {"node_occlusion", "minimum_angle", "edge_length_variation",
                                 "edge_crossing", "edge_crossing_angle"}


@pytest.mark.gpu
def test_x_graph_report(gpu):
    """Reference tests/test_engine.py:22-30: nc 0, ec 1, eca 5/7."""
    r = evaluate(graph_from(cases.x_graph))
    assert r.node_occlusion == 0 and r.edge_crossing == 1
    assert r.edge_crossing_angle == pytest.approx(5.0 / 7.0)
    assert r.warnings == []
    assert list(r.elapsed) == ["node_occlusion", "minimum_angle", "edge_length_variation",
                               "edge_crossing", "edge_crossing_angle"]
    assert '"edge_crossing": 1' in r.to_json()


@pytest.mark.gpu
def test_c1_report_matches_reference(gpu, golden_configs):
    g, p = configs.config1()
    want = golden_configs["configs"]["C1"]
    r = evaluate(g, params=MetricParams(radius=p["radius"], ideal_angle=p["ideal"]))
    assert r.node_occlusion == want["nc"] and r.edge_crossing == want["ec"]
    for name, key in (("minimum_angle", "ma"), ("edge_length_variation", "ml"),
                      ("edge_crossing_angle", "eca")):
        assert strict_close(getattr(r, name), want[key])
    assert r.params["ideal_angle_deg"] == pytest.approx(70.0)


@pytest.mark.gpu
def test_bench_invariant_across_shards(gpu):
    from paper_2411_09809_b200.engine import bench

    g = graph_from(cases.lattice_stress)
    rows = bench(g, shard_counts=(1, 2, 4, 8), params=MetricParams(radius=1.0))
    by = {}
    for row in rows:
        by.setdefault(row["metric"], set()).add(row["value"])
    assert by["ec"] == {4194903} and by["nc"] == {9588}
    assert len(rows) == 12
    assert all(math.isfinite(r["seconds"]) for r in rows)


def test_enhanced_mode_metric_validation():
    from paper_2411_09809_b200 import ParameterError
    from paper_2411_09809_b200.engine import _normalize_metrics, evaluate

    assert _normalize_metrics(None, "b200-enhanced") == ("nc", "ec", "eca")
    with pytest.raises(ParameterError):
        _normalize_metrics(["ma"], "b200-enhanced")
    with pytest.raises(ParameterError):
        evaluate(None, mode="enhanced")


@pytest.mark.gpu
def test_gpu_enhanced_mode_report_and_compare(gpu):
    import math

    import strip_cases
    from paper_2411_09809_b200 import (MetricParams, crossing_angle_stats,
                                       edge_crossing_enhanced, node_occlusion)
    from paper_2411_09809_b200.engine import compare, evaluate
    from paper_2411_09809_b200.model import LayoutGraph

    ids, xy, pairs = strip_cases.GRAPHS["rg_80_300"]
    g = LayoutGraph(ids, xy, pairs)
    p = MetricParams(radius=0.5, ideal_angle=math.radians(70), strip_fraction=0.1,
                     orientation="both")
    rep = evaluate(g, "b200-enhanced", p)
    assert rep.mode == "b200-enhanced"
    assert rep.edge_crossing == edge_crossing_enhanced(g, 0.1, "both")
    c, d = crossing_angle_stats(g, 0.1, p.ideal_angle, "both")
    assert rep.edge_crossing_angle == pytest.approx(1.0 - (d / p.ideal_angle) / c, rel=1e-12)
    assert rep.node_occlusion == node_occlusion(g, 0.5)
    assert rep.minimum_angle is None
    rows = compare(g, p)
    assert [r["metric"] for r in rows] == ["nc", "ec", "eca"]
    ec_row = rows[1]
    assert ec_row["enhanced"] <= ec_row["oracle"] and not ec_row["flagged"]
