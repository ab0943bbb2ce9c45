"""The "b200" mode registered with the reference package itself
(paper_2411_09809_b200/glare_plugin.py).

The reference is imported from baseline/_ref (the pip-installed reference,
which travels to the GPU box) or, in the build container, from
/root/reference/pkg/src; the tests skip when neither exists.  CPU tests use
inputs whose metrics are degenerate (no GPU work: the drop-ins return the
reference's degenerate values before any kernel call); GPU tests evaluate
real graphs and compare with the reference's goldens.
"""

from __future__ import annotations

import asyncio
import json
import os
import sys

import numpy as np
import pytest

from conftest import REPO, load_golden, strict_close

_CANDIDATES = [os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"]


@pytest.fixture()
def glare():
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "glare")):
            if path not in sys.path:
                sys.path.insert(0, path)
            break
    else:
        pytest.skip("the reference package glare is not importable here")
    pytest.importorskip("fastapi")
    import glare as G

    from paper_2411_09809_b200 import glare_plugin

    glare_plugin.install(G)
    yield G
    glare_plugin.uninstall()


def _tiny(G, n=1):
    return G.LayoutGraph(np.arange(n), np.zeros((n, 2)) + np.arange(n)[:, None], [])


def test_mode_registered_and_restored(glare):
    from paper_2411_09809_b200 import glare_plugin

    assert "b200" in glare.model.MODES and "b200" in glare.engine.MODES
    glare_plugin.uninstall()
    assert "b200" not in glare.model.MODES
    with pytest.raises(glare.ParameterError):
        glare.evaluate(_tiny(glare), "b200")
    glare_plugin.install(glare)
    glare_plugin.install(glare)  # idempotent
    assert glare.model.MODES.count("b200") == 1


def test_degenerate_report_equals_oracle(glare):
    g = _tiny(glare)
    b = glare.evaluate(g, "b200")
    o = glare.evaluate(g, "oracle")
    assert b.mode == "b200"
    db, do = b.to_dict(), o.to_dict()
    assert db["metrics"] == do["metrics"] and db["warnings"] == do["warnings"]
    assert db["params"] == do["params"] and set(db["elapsed"]) == set(do["elapsed"])
    # the reference's own report parser accepts the b200 report (model.py:231)
    back = glare.ReadabilityReport.from_dict(json.loads(json.dumps(db)))
    assert back.mode == "b200" and back.to_dict()["metrics"] == db["metrics"]


def test_parameter_errors_are_the_references(glare):
    g = _tiny(glare)
    for kw in ({"params": glare.MetricParams(radius=-1.0)},
               {"metrics": ["nope"]}, {"metrics": []}):
        with pytest.raises(glare.ParameterError) as e_b:
            glare.evaluate(g, "b200", **kw)
        with pytest.raises(glare.ParameterError) as e_o:
            glare.evaluate(g, "oracle", **kw)
        assert str(e_b.value) == str(e_o.value)


def test_engine_bench_invariant_in_b200_mode(glare):
    rows = glare.engine.bench(_tiny(glare), "b200", thread_counts=(1, 2))
    assert {r["metric"] for r in rows} == {"nc", "ma", "ml", "ec", "eca"}
    assert all(r["speedup"] > 0 for r in rows)


def test_service_evaluate_b200(glare):
    import importlib

    import httpx

    app_mod = importlib.import_module("glare.service.app")

    async def post():
        transport = httpx.ASGITransport(app=app_mod.app)
        async with httpx.AsyncClient(transport=transport, base_url="http://t") as c:
            return await c.post("/evaluate", json={
                "graph": {"edges": [], "positions": [{"id": 0, "x": 0.0, "y": 0.0}]},
                "mode": "b200"})

    resp = asyncio.run(post())
    assert resp.status_code == 200, resp.text
    body = resp.json()
    assert body["mode"] == "b200" and body["metrics"]["edge_crossing"] == 0


def test_cli_eval_b200(glare, tmp_path, capsys):
    from glare import cli

    (tmp_path / "e.txt").write_text("0 1\n")
    (tmp_path / "l.csv").write_text("id,x,y\n0,0,0\n1,1,1\n")
    out = tmp_path / "r.json"
    rc = cli.main(["eval", "--edges", str(tmp_path / "e.txt"), "--layout",
                   str(tmp_path / "l.csv"), "--mode", "b200", "--metrics", "ml,ec,eca",
                   "--out", str(out)])
    assert rc == 0, capsys.readouterr().err
    doc = json.loads(out.read_text())
    assert doc["mode"] == "b200"
    assert doc["metrics"]["edge_crossing"] == 0
    assert doc["metrics"]["edge_length_variation"] == 0.0


@pytest.mark.gpu
def test_gpu_x_graph_and_c1(glare, gpu):
    """glare.engine.evaluate(g, "b200") on the reference's known answer and
    on config 1 against the reference's own values (tests/golden)."""
    from paper_2411_09809_b200 import configs

    x = glare.LayoutGraph.from_positions(
        {0: (0.0, 0.0), 1: (1.0, 1.0), 2: (0.0, 1.0), 3: (1.0, 0.0)}, [(0, 1), (2, 3)])
    r = glare.evaluate(x, "b200", metrics=["nc", "ec", "eca"])
    assert (r.node_occlusion, r.edge_crossing) == (0, 1)
    assert strict_close(r.edge_crossing_angle, 5.0 / 7.0)

    gold = load_golden("golden.json")["configs"]["C1"]
    g1, p = configs.make(1)
    g = glare.LayoutGraph(g1.ids, g1.xy, g1.edges)
    rep = glare.evaluate(g, "b200", glare.MetricParams(radius=p["radius"]))
    assert rep.node_occlusion == gold["nc"] and rep.edge_crossing == gold["ec"]
    for key, field in (("ma", "minimum_angle"), ("ml", "edge_length_variation"),
                       ("eca", "edge_crossing_angle")):
        assert strict_close(getattr(rep, field), gold[key], floor=0.0), key
    rows = glare.engine.bench(g, "b200", thread_counts=(1, 2), metrics=["ec", "eca"])
    assert {r["value"] for r in rows if r["metric"] == "ec"} == {gold["ec"]}
