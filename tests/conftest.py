"""Shared test configuration.

Markers: ``gpu`` tests need a CUDA device (B200) and the built library; they
call the product path through the C ABI.  Everything else runs on CPU.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (REPO, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN_DIR = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built sm_100a library")
    config.addinivalue_line("markers", "slow: full-size configuration checks (minutes)")


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN_DIR, name)) as f:
        return json.load(f)


def rel_close(a: float, b: float, tol: float = 1e-9) -> bool:
    """The reference's own real-valued tolerance (test_acceptance.py:66-67,
    engine.py:203-206)."""
    if isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b):
        return True
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))


def strict_close(a: float, b: float, tol: float = 1e-9, floor: float = 1e-15) -> bool:
    """1e-9 RELATIVE (north-star tolerance), with an absolute floor for values
    that are pure rounding noise (e.g. M_l of equal lengths ~1e-17)."""
    if isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b):
        return True
    return abs(a - b) <= max(tol * max(abs(a), abs(b)), floor)


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("golden_small.json")


@pytest.fixture(scope="session")
def golden_configs():
    return load_golden("golden.json")


def graph_from(builder):
    """This package's LayoutGraph from a tests/cases.py builder."""
    from paper_2411_09809_b200.model import LayoutGraph

    out = builder()
    if len(out) == 2:
        pos, edges = out
        return LayoutGraph.from_positions(pos, edges)
    ids, xy, pairs = out
    return LayoutGraph(ids, xy, pairs)


def fingerprint(g) -> str:
    from paper_2411_09809_b200.configs import fingerprint as fp

    return fp(g)


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2411_09809_b200 import _lib

    return _lib.lib()

