"""fr_layout: the oracle restatement and the GPU
kernel against the reference's own outputs (tests/golden/layout_golden.json,
made by tests/golden/make_golden_layout.py), bit for bit."""

from __future__ import annotations

import hashlib
import json
import math
import os

import numpy as np
import pytest

import layout_cases

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def layout_golden():
    with open(os.path.join(HERE, "golden", "layout_golden.json")) as fh:
        return json.load(fh)["cases"]


def _sha(xy):
    return hashlib.sha256(np.ascontiguousarray(xy, dtype=np.float64).tobytes()).hexdigest()


def _index_edges(edges):
    from paper_2411_09809_b200.model import normalize_edges

    ids = np.unique(np.asarray(edges, dtype=np.int64))
    ne, _, _ = normalize_edges(edges)
    return ids, np.searchsorted(ids, ne[:, 0]), np.searchsorted(ids, ne[:, 1])


@pytest.mark.parametrize("name", sorted(layout_cases.CASES))
def test_oracle_fr_layout_matches_reference(layout_golden, name):
    from oracle.glare_oracle import fr_layout_positions

    edges, kw = layout_cases.CASES[name]
    want = layout_golden[name]
    ids, ei, ej = _index_edges(edges)
    xy = fr_layout_positions(len(ids), ei, ej, kw["iterations"], kw["seed"], kw["extent"])
    assert len(xy) == want["n"]
    assert _sha(xy) == want["sha256"], name


def test_layout_errors_mirror_reference():
    from paper_2411_09809_b200 import InputError, ParameterError, fr_layout, generate_layout
    from paper_2411_09809_b200 import random_layout

    e = np.array([[0, 1], [1, 2]])
    with pytest.raises(ParameterError):
        fr_layout(e, iterations=0)
    with pytest.raises(ParameterError):
        fr_layout(e, extent=math.inf)
    with pytest.raises(ParameterError):
        random_layout(e, extent=-1.0)
    with pytest.raises(InputError):
        random_layout(np.empty((0, 2), dtype=np.int64))
    with pytest.raises(ParameterError):
        generate_layout(e, kind="spring")


def test_random_layout_matches_reference_recipe():
    from paper_2411_09809_b200 import random_layout

    e = np.array([[0, 1], [5, 9]])
    g = random_layout(e, seed=0)
    assert g.ids.tolist() == [0, 1, 5, 9]
    want = np.random.default_rng(0).uniform(0.0, 100.0, size=(4, 2))
    assert np.array_equal(g.xy, want)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(layout_cases.CASES))
def test_gpu_fr_layout_bit_exact(gpu, layout_golden, name):
    from paper_2411_09809_b200 import fr_layout

    edges, kw = layout_cases.CASES[name]
    want = layout_golden[name]
    g = fr_layout(edges, **kw)
    assert g.num_vertices == want["n"] and g.num_edges == want["m"]
    if "xy_hex" in want:
        got = [v.hex() for v in g.xy.ravel().tolist()]
        assert got == want["xy_hex"]
    assert _sha(g.xy) == want["sha256"], name


@pytest.mark.gpu
def test_gpu_generate_layout_and_metrics(gpu):
    from paper_2411_09809_b200 import edge_crossing, generate_layout

    edges, kw = layout_cases.CASES["ref_test_30_60"]
    g1 = generate_layout(edges, kind="fr", **kw)
    g2 = generate_layout(edges, kind="fr", **kw)
    assert np.array_equal(g1.xy, g2.xy)
    assert g1.xy.min() >= 0.0 and g1.xy.max() <= 10.0
    rand = generate_layout(edges, kind="random", seed=8, extent=10.0)
    assert edge_crossing(g1) < edge_crossing(rand)  # test_graphio.py:169-177


@pytest.mark.gpu
def test_gpu_branch_free_division_matches_ddiv_rn(gpu):
    """The repulsion kernel's branch-free division equals __ddiv_rn (IEEE
    round-to-nearest) on 2^28 operand pairs incl. near-midpoint quotients."""
    import ctypes

    import torch

    from paper_2411_09809_b200 import _lib

    bad = ctypes.c_uint64(0)
    rc = _lib.lib().glr_selftest_division(1 << 28, 20241019, ctypes.byref(bad),
                                          torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "glr_selftest_division")
    assert bad.value == 0
