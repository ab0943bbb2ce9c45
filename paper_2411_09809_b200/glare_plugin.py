"""Registers "b200" as an evaluation mode of the reference package itself.

``install()`` makes glare run its own engine, report, service and CLI on the
B200 kernels:

* ``glare.model.MODES`` (model.py:38) gains "b200", so ``ReadabilityReport
  .from_dict`` accepts b200 reports (model.py:231) and ``engine._check_mode``
  accepts the mode (engine.py:58-61);
* ``glare.engine.evaluate`` (engine.py:140-160) dispatches "b200" to
  ``_b200_entry`` -- the oracle's per-metric closures (engine.py:74-94) with
  this package's drop-in metrics and the same warning strings -- and every
  other mode to the original function; ``engine.compare`` / ``engine.bench``
  (engine.py:163-256) and the package-level ``glare.evaluate`` see it, so
  ``bench(g, "b200")`` checks its identical-values invariant on the GPU path;
* the service's request/response models (service/schemas.py:37,43,70) take
  "b200", and the in-process app is rebuilt with them (service/app.py);
* the CLI's ``--mode`` choices of ``eval`` and ``bench`` (cli.py:232,318)
  list "b200".

Reports keep the reference's schema (model.py:203-216) with ``mode ==
"b200"``.  When E_c and E_ca are both requested they share one fused
crossing scan (the reference scans twice, engine.py:85-92); its time is
charged to the first of the two.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib
import typing

MODE = "b200"
_saved: dict = {}


def _b200_entry(g, key, p, model, cache):
    """Per-metric closure returning (value, warnings), as engine._oracle_entry."""
    from . import metrics as M

    if key == "nc":
        return lambda: (M.node_occlusion(g, p.radius), [])
    if key == "ma":
        if g.num_edges == 0:
            return lambda: (1.0, [model.WARN_NO_EDGES_ANGLE])
        return lambda: (M.minimum_angle(g), [])
    if key == "ml":
        if g.num_edges <= 1:
            return lambda: (0.0, [model.WARN_FEW_EDGES_LENGTH])
        return lambda: (M.edge_length_variation(g), [])

    def scan():
        if "scan" not in cache:
            cache["scan"] = M._crossing_scan(g, p.ideal_angle)
        return cache["scan"]

    if key == "ec":
        return lambda: (scan()[0], [])

    def eca():
        count, dev = scan()
        if count == 0:
            return 1.0, [model.WARN_NO_CROSSINGS]
        return 1.0 - (dev / p.ideal_angle) / count, []

    return eca


def _with_mode(literal, mode=MODE):
    args = typing.get_args(literal)
    return literal if mode in args else typing.Literal[args + (mode,)]


def _patch_schemas(glare_pkg) -> None:
    try:
        schemas = importlib.import_module(glare_pkg.__name__ + ".service.schemas")
        app_mod = importlib.import_module(glare_pkg.__name__ + ".service.app")
    except ImportError:  # fastapi/pydantic absent: engine-level install only
        return
    new = {}
    for name in ("EvaluateRequest", "ReportModel", "BenchRequest"):
        base = getattr(schemas, name)
        field = base.model_fields["mode"]
        ns = {"__annotations__": {"mode": _with_mode(field.annotation)},
              "__module__": schemas.__name__, "__doc__": base.__doc__}
        if not field.is_required():
            ns["mode"] = field.default
        new[name] = type(name, (base,), ns)
    _saved["schemas"] = {n: getattr(schemas, n) for n in new}
    _saved["app"] = app_mod.app
    for name, cls in new.items():
        setattr(schemas, name, cls)
        setattr(app_mod, name, cls)
    app_mod.app = app_mod.create_app()  # routes resolve the new models
    service = importlib.import_module(glare_pkg.__name__ + ".service")
    if getattr(service, "app", None) is _saved["app"]:  # re-exported instance
        service.app = app_mod.app


def _patch_cli(glare_pkg) -> None:
    try:
        import click

        cli = importlib.import_module(glare_pkg.__name__ + ".cli")
    except ImportError:
        return
    saved = []
    for cmd in (cli.cmd_eval, cli.cmd_bench):
        for opt in cmd.params:
            if opt.name == "mode" and MODE not in opt.type.choices:
                saved.append((opt, opt.type))
                opt.type = click.Choice(list(opt.type.choices) + [MODE])
    _saved["cli"] = saved


def install(glare_pkg=None):
    """Register the b200 mode with the imported glare package (idempotent).
    Returns the glare package."""
    if glare_pkg is None:
        import glare as glare_pkg
    if _saved.get("installed") is glare_pkg:
        return glare_pkg
    model = importlib.import_module(glare_pkg.__name__ + ".model")
    engine = importlib.import_module(glare_pkg.__name__ + ".engine")
    dataflow = importlib.import_module(glare_pkg.__name__ + ".dataflow")
    _saved.update(modes=model.MODES, evaluate=engine.evaluate, pkg_evaluate=glare_pkg.evaluate)
    modes = model.MODES + ((MODE,) if MODE not in model.MODES else ())
    model.MODES = modes
    engine.MODES = modes
    original = engine.evaluate

    def evaluate(g, mode="oracle", params=None, exec_cfg=None, metrics=None):
        if mode != MODE:
            return original(g, mode, params, exec_cfg, metrics)
        engine._check_mode(mode)
        params = params if params is not None else model.MetricParams()
        params.validate()
        exec_cfg = exec_cfg if exec_cfg is not None else dataflow.ExecConfig()
        keys = engine._normalize_metrics(metrics, mode)
        cache: dict = {}
        entries = [(model.METRIC_FIELDS[k], _b200_entry(g, k, params, model, cache))
                   for k in keys]
        return model.build_report(mode, engine._params_echo(params, exec_cfg), entries)

    evaluate.__doc__ = original.__doc__
    engine.evaluate = evaluate
    glare_pkg.evaluate = evaluate
    _patch_schemas(glare_pkg)
    _patch_cli(glare_pkg)
    _saved["installed"] = glare_pkg
    return glare_pkg


def uninstall() -> None:
    """Restore the glare package's original modes, engine, service and CLI."""
    glare_pkg = _saved.pop("installed", None)
    if glare_pkg is None:
        return
    model = importlib.import_module(glare_pkg.__name__ + ".model")
    engine = importlib.import_module(glare_pkg.__name__ + ".engine")
    model.MODES = engine.MODES = _saved.pop("modes")
    engine.evaluate = _saved.pop("evaluate")
    glare_pkg.evaluate = _saved.pop("pkg_evaluate")
    if "schemas" in _saved:
        schemas = importlib.import_module(glare_pkg.__name__ + ".service.schemas")
        app_mod = importlib.import_module(glare_pkg.__name__ + ".service.app")
        for name, cls in _saved.pop("schemas").items():
            setattr(schemas, name, cls)
            setattr(app_mod, name, cls)
        service = importlib.import_module(glare_pkg.__name__ + ".service")
        if getattr(service, "app", None) is app_mod.app:
            service.app = _saved["app"]
        app_mod.app = _saved.pop("app")
    for opt, typ in _saved.pop("cli", []):
        opt.type = typ
