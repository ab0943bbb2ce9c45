"""The C-ABI library loads and exports every symbol include/glare_b200.h
declares; host-only entry points (tile/unit arithmetic, error strings) work
without a GPU.  No compute calls here."""

from __future__ import annotations

import os
import re
import subprocess

import pytest

from conftest import REPO
from paper_2411_09809_b200 import _lib

HEADER = os.path.join(REPO, "include", "glare_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(glr_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    return _lib.load_library()


def test_library_built_for_sm100a():
    assert os.path.exists(_lib.LIB_PATH), "run make / __graft_entry__.build()"
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_exported_and_bound(L):
    names = _declared()
    assert len(names) >= 14
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(names)


def test_host_only_entry_points(L):
    assert L.glr_version() >> 16 == 1
    tile = L.glr_crossing_tile()
    assert tile > 0 and tile % 32 == 0
    for m in (0, 1, 2, tile, tile + 1, 5000, 4_000_000):
        T = max(1, -(-m // tile))
        assert L.glr_crossing_units(m) == T * (T + 1) // 2
    vt = L.glr_occlusion_tile()
    for n in (1, 2, vt, 3 * vt + 7, 1_500_000):
        T = -(-n // vt)
        assert L.glr_occlusion_units(n) == T * (T + 1) // 2
    assert L.glr_crossing_records_bytes(500, 1000) >= 1000 * 64


def test_argument_errors_reported_without_gpu(L):
    # invalid arguments are rejected before any CUDA call
    rc = L.glr_crossing_pairs(None, 5, 10, 0, 0.0, 0, 1, None, None)
    assert rc == _lib.GLR_EARG
    assert b"invalid" in L.glr_last_error()
    rc = L.glr_occlusion_count(None, -1, 1.0, 0, 1, None, None)
    assert rc == _lib.GLR_EARG
    # edge orders (direction / 4-D bbox Morton): null buffers, > 2^31 edges
    rc = L.glr_theta_sort_edges(None, 10, None, 5, 0, None, None)
    assert rc == _lib.GLR_EARG and b"glr_theta_sort_edges" in L.glr_last_error()
    rc = L.glr_theta_sort_edges(None, 10, None, 1 << 31, 0, None, None)
    assert rc == _lib.GLR_EARG
    rc = L.glr_spatial_sort_edges(None, 10, None, 5, None, None)
    assert rc == _lib.GLR_EARG and b"glr_spatial_sort_edges" in L.glr_last_error()


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2411_09809_b200 as G
    from conftest import graph_from
    import cases

    with pytest.raises(RuntimeError, match="CUDA device"):
        G.edge_crossing(graph_from(cases.x_graph))
    # degenerate inputs return the reference's constants without touching the GPU
    assert G.edge_crossing(graph_from(cases.occ_boundary)) == 0
    assert G.minimum_angle(graph_from(cases.occ_three)) == 1.0


def test_no_oracle_on_product_path():
    """The product package never imports the oracle."""
    pkg = os.path.join(REPO, "paper_2411_09809_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f
