"""Input contract of the drop-in functions mirrors the reference's data model
(/root/reference/pkg/src/glare/model.py:56-186; behaviour asserted by the
reference's tests/test_model.py:22-113)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2411_09809_b200.model import (
    InputError,
    LayoutGraph,
    MetricParams,
    ParameterError,
    check_ideal_angle,
    check_radius,
    normalize_edges,
)


def test_normalize_orders_dedupes_and_counts():
    e, loops, dupes = normalize_edges([(3, 1), (1, 3), (2, 2), (0, 5), (5, 0), (1, 2)])
    assert e.tolist() == [[0, 5], [1, 2], [1, 3]]
    assert loops == 1 and dupes == 2
    assert e.dtype == np.int64


def test_normalize_matches_np_unique_rows():
    rng = np.random.default_rng(0)
    pairs = rng.integers(0, 50, (2000, 2))
    e, loops, dupes = normalize_edges(pairs)
    keep = pairs[pairs[:, 0] != pairs[:, 1]]
    ref = np.unique(np.stack([keep.min(1), keep.max(1)], 1), axis=0)
    assert np.array_equal(e, ref)
    assert loops == int(np.sum(pairs[:, 0] == pairs[:, 1]))
    assert dupes == len(keep) - len(ref)


def test_normalize_empty_and_bad_shape():
    e, loops, dupes = normalize_edges([])
    assert e.shape == (0, 2) and loops == 0 and dupes == 0
    with pytest.raises(InputError):
        normalize_edges([1, 2, 3])
    e, loops, _ = normalize_edges([(4, 4)])
    assert e.shape == (0, 2) and loops == 1


def test_layout_graph_sorts_ids_and_maps_edges():
    g = LayoutGraph([10, 2, 7], [(1.0, 1.0), (2.0, 2.0), (3.0, 3.0)], [(10, 2), (7, 10)])
    assert g.ids.tolist() == [2, 7, 10]
    assert g.xy.tolist() == [[2.0, 2.0], [3.0, 3.0], [1.0, 1.0]]
    assert g.edges.tolist() == [[0, 2], [1, 2]]
    assert g.num_vertices == 3 and g.num_edges == 2


@pytest.mark.parametrize(
    "ids,xy,edges,msg",
    [
        ([0, 1], [(0.0, 0.0)], [], "positions must have shape"),
        ([], np.zeros((0, 2)), [], "graph needs at least one vertex"),
        ([0, 1], [(0.0, 0.0), (math.inf, 0.0)], [], "vertex coordinates must be finite"),
        ([0, 0], [(0.0, 0.0), (1.0, 0.0)], [], "duplicate vertex id 0"),
        ([0, 1], [(0.0, 0.0), (1.0, 0.0)], [(0, 5)], "edge endpoint 5 is not a vertex"),
        ([0, 1], [(1.0, 1.0), (1.0, 1.0)], [(0, 1)], "zero-length edge (0, 1)"),
        ([[0, 1]], [(1.0, 1.0)], [], "vertex ids must be a 1-D sequence"),
    ],
)
def test_layout_graph_rejects(ids, xy, edges, msg):
    with pytest.raises(InputError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        LayoutGraph(ids, xy, edges)


def test_isolated_vertices_kept_and_counts():
    g = LayoutGraph([0, 1, 2, 3], np.arange(8.0).reshape(4, 2), [(0, 1), (1, 0), (2, 2)])
    assert g.num_vertices == 4 and g.num_edges == 1
    assert g.loops_dropped == 1 and g.dupes_dropped == 1


def test_params_validation_messages():
    MetricParams().validate()
    with pytest.raises(ParameterError, match="radius must be finite and > 0"):
        MetricParams(radius=0.0).validate()
    with pytest.raises(ParameterError, match="ideal angle must lie in"):
        MetricParams(ideal_angle=math.pi).validate()
    with pytest.raises(ParameterError):
        check_radius(math.nan)
    with pytest.raises(ParameterError):
        check_radius(-1.0)
    with pytest.raises(ParameterError):
        check_ideal_angle(0.0)
    assert check_ideal_angle(math.pi / 2) == math.pi / 2


def test_from_positions_and_with_xy():
    g = LayoutGraph.from_positions({5: (0.0, 0.0), 3: (1.0, 1.0)}, [(5, 3)])
    assert g.ids.tolist() == [3, 5]
    g2 = g.with_xy(g.xy * 2.0)
    assert g2.xy.tolist() == [[2.0, 2.0], [0.0, 0.0]]
    assert g2.edges.tolist() == g.edges.tolist()
