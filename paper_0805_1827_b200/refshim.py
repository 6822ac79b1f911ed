"""Register the B200 engine inside an installed reference package (the drop-in shim).

The reference resolves its kernel backend by NAME in every phase builder and
worker task (``get_backend``, _kernels/__init__.py:37-53; re-resolved in
boundary_iz.py:284, boundary_cmc.py:214, pricer.py:157) and rejects names it
does not know (:53), so a backend object cannot simply be passed in.
``register(bermuda)`` teaches an installed ``bermuda`` package the name
``"cuda"`` at two levels:

* **kernel backend**: ``get_backend("cuda")`` (or ``BERMUDA_BACKEND=cuda``)
  returns :mod:`paper_0805_1827_b200.backend`, which has the reference
  backend's duck-typed surface (core_backend.py:12-58).  The reference's own
  ``build_iz_boundary`` / ``build_cmc_rule`` / ``price`` then run unchanged
  with every kernel call on the GPU.  CUDA does not survive the reference's
  fork pool (engine.py:111-113): use ``Engine(workers=1)`` or
  ``pool="thread"``.
* **CLI / phase level**: ``bermuda price|bench|table --backend cuda``
  (cli.py:349-394) routes ``build_and_price`` (cli.py:142-170) to this
  package's device-resident phase builders and returns the reference's own
  result types (``PriceEstimate``, ``CmcBuildReport`` / ``IzBuildReport``).
  For this backend the worker count of ``bench`` is the number of item
  partitions (``dist.virtual_shards``), so its exit-2 determinism check
  (cli.py:303-309) compares prices across partitions of every phase.

``to_reference`` converts this package's results into the reference's
types (JSON v1 round trip for rules, field copy for estimates and reports).
Nothing here imports the reference: the caller passes its ``bermuda``.
"""

from __future__ import annotations

import argparse
import functools
import importlib
import json
import os
import time

from . import backend as _backend

__all__ = ["register", "unregister", "to_reference", "build_and_price"]

NAME = "cuda"
_PATCHED_MODULES = ("_kernels", "boundary_cmc", "boundary_iz", "pricer", "cli")


def _mod(bermuda, name: str):
    return importlib.import_module(f"{bermuda.__name__}.{name}")


def _wants_cuda(name) -> bool:
    if name is None:
        name = os.environ.get("BERMUDA_BACKEND", "auto")
    return str(name).lower() == NAME


def register(bermuda):
    """Install the ``"cuda"`` backend into the reference package ``bermuda``.

    Idempotent; returns ``bermuda``.  ``unregister`` restores the original
    functions."""
    kern = _mod(bermuda, "_kernels")
    if getattr(kern, "_brm_registered", False):
        return bermuda
    orig_get = kern.get_backend
    orig_avail = kern.available_backends

    @functools.wraps(orig_get)
    def get_backend(name=None):
        if _wants_cuda(name):
            return _backend
        return orig_get(name)

    @functools.wraps(orig_avail)
    def available_backends():
        return list(orig_avail()) + [NAME]

    saved = {}
    for modname in _PATCHED_MODULES:
        mod = _mod(bermuda, modname)
        for attr, repl in (("get_backend", get_backend), ("available_backends", available_backends)):
            if hasattr(mod, attr):
                saved[(modname, attr)] = getattr(mod, attr)
                setattr(mod, attr, repl)
    cli = _mod(bermuda, "cli")
    saved[("cli", "_parser")] = cli._parser
    saved[("cli", "build_and_price")] = cli.build_and_price
    orig_parser, orig_bap = cli._parser, cli.build_and_price

    @functools.wraps(orig_parser)
    def _parser():
        top = orig_parser()
        for act in top._actions:
            if isinstance(act, argparse._SubParsersAction):
                for sub in act.choices.values():
                    for a in sub._actions:
                        if a.dest == "backend" and a.choices is not None and NAME not in a.choices:
                            a.choices = list(a.choices) + [NAME]
        return top

    @functools.wraps(orig_bap)
    def build_and_price(cfg, engine=None):
        if str(cfg.backend).lower() != NAME:
            return orig_bap(cfg, engine)
        return _cli_build_and_price(bermuda, cfg, engine)

    # cmd_price / cmd_bench / cmd_table look both names up in the module at call time
    cli._parser = _parser
    cli.build_and_price = build_and_price
    kern._brm_registered = True
    kern._brm_saved = saved
    return bermuda


def unregister(bermuda) -> None:
    kern = _mod(bermuda, "_kernels")
    saved = getattr(kern, "_brm_saved", None)
    if not saved:
        return
    for (modname, attr), fn in saved.items():
        setattr(_mod(bermuda, modname), attr, fn)
    kern._brm_registered = False
    kern._brm_saved = None


# ------------------------------------------------------------ conversions ----
def to_reference(obj, bermuda):
    """This package's result object -> the reference's type of the same name."""
    from .boundary_cmc import CmcBuildReport, CmcRule
    from .boundary_iz import IzBoundary, IzBuildReport
    from .boosting import StumpEnsemble
    from .pricer import PriceEstimate
    if isinstance(obj, CmcRule):
        return _mod(bermuda, "boundary_cmc").CmcRule.from_json(obj.to_json())
    if isinstance(obj, IzBoundary):
        if obj.iz_space != 0:
            raise ValueError("the reference has no log-space (geometric put) boundary")
        return _mod(bermuda, "boundary_iz").IzBoundary.from_json(obj.to_json())
    if isinstance(obj, StumpEnsemble):
        return _mod(bermuda, "boosting").StumpEnsemble.from_json(json.dumps(obj.to_json_dict()))
    if isinstance(obj, PriceEstimate):
        return _mod(bermuda, "pricer").PriceEstimate(
            price=obj.price, variance=obj.variance, ci95=obj.ci95, n_paths=obj.n_paths, timings=dict(obj.timings),
            rule_kind=obj.rule_kind, unconverged_points=obj.unconverged_points)
    if isinstance(obj, CmcBuildReport):
        return _mod(bermuda, "boundary_cmc").CmcBuildReport(
            calc_seconds=obj.calc_seconds, class_seconds=obj.class_seconds, per_date=list(obj.per_date),
            one_class_dates=list(obj.one_class_dates))
    if isinstance(obj, IzBuildReport):
        return _mod(bermuda, "boundary_iz").IzBuildReport(
            glp_seconds=obj.glp_seconds, calc_seconds=obj.calc_seconds, reg_seconds=obj.reg_seconds,
            per_date=list(obj.per_date), unconverged_points=obj.unconverged_points,
            iteration_counts=list(obj.iteration_counts))
    raise TypeError(f"no reference counterpart for {type(obj).__name__}")


def build_and_price(bermuda, cfg, engine=None):
    """The reference CLI's ``build_and_price`` (cli.py:142-170) on this engine."""
    return _cli_build_and_price(bermuda, cfg, engine)


def _cli_build_and_price(bermuda, cfg, engine):
    """Same phases, seeds and outputs as cli.py:142-170; ``engine.workers``
    (else ``cfg.workers``) is the number of item partitions."""
    from . import boundary_cmc as C
    from . import boundary_iz as Z
    from . import pricer as P
    from .dist import virtual_shards
    params, spec = cfg.market(), cfg.spec()
    parts = getattr(engine, "nb_tasks", None) or getattr(engine, "workers", None) or cfg.nb_tasks or cfg.workers
    timings = {}
    report = None
    unconverged = 0
    with virtual_shards(max(int(parts), 1)):
        if cfg.method == "iz":
            t0 = time.perf_counter()
            boundary, rep = Z.build_iz_boundary(params, spec, cfg.j_points, cfg.n1, cfg.epsilon, cfg.max_iter,
                                                seed=cfg.seed, lo_mult=cfg.glp_lo_mult, hi_mult=cfg.glp_hi_mult)
            timings["build"] = time.perf_counter() - t0
            rule = P.IzRule(boundary)
            unconverged = rep.unconverged_points
            report = to_reference(rep, bermuda)
        elif cfg.method == "cmc":
            t0 = time.perf_counter()
            cmc, rep = C.build_cmc_rule(params, spec, C.CmcBuildConfig(cfg.n1, cfg.n2, cfg.boost_rounds),
                                        seed=cfg.seed)
            timings["build"] = time.perf_counter() - t0
            rule = P.CmcScoreRule(cmc)
            report = to_reference(rep, bermuda)
        else:
            rule = P.EuropeanRule()
        est = P.price(params, spec, rule, cfg.n_paths, cfg.seed, build_timings=timings,
                      unconverged_points=unconverged)
    return to_reference(est, bermuda), report
