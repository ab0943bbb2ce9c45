"""The bench.py JSON contract: one line with the driver's keys, for the
reference arm (CPU, runs here) and for our arm (B200, also under torchrun)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600, torchrun=False):
    cmd = [sys.executable]
    if torchrun:
        cmd += ["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                "--master-addr", "127.0.0.1", "--master-port", "29517"]
    out = subprocess.run(cmd + [os.path.join(REPO, "bench.py")] + args, cwd=REPO,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C5")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def _check_ours(d):
    assert BASE_KEYS <= set(d)
    assert d["unit"] == "pairs/s" and d["dtype"] == "f64" and d["data"] == "synthetic"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] <= 1 and r["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 88_000_000 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    # the three passes agree with each other (bench asserts it) and the count is C5's
    assert d["result"]["edge_crossing"] == 1844517725761
    assert d["result"]["node_occlusion"] == 207826
    assert d["crossing_culled"]["candidate_units"] < d["crossing_culled"]["dense_units"]


@pytest.mark.gpu
def test_our_arm_line(gpu):
    _check_ours(_run(["--steps", "1", "--warmup", "1", "--e2e-steps", "1", "--no-layout",
                      "--no-cpu-baseline"]))


@pytest.mark.gpu
def test_our_arm_line_under_torchrun(gpu):
    d = _run(["--gpus", "1", "--steps", "1", "--warmup", "1", "--e2e-steps", "1",
              "--no-layout", "--no-cpu-baseline"], torchrun=True)
    _check_ours(d)
    assert d["n_gpus"] == 1
