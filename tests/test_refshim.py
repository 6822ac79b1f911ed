"""The drop-in shim from the reference side, without a GPU (registration only).

``refshim.register`` teaches the unmodified reference package (oracle/_ref)
the backend name "cuda": its registry (_kernels/__init__.py:37-53), the
per-module ``get_backend`` bindings the builders re-resolve by name, and the
CLI's ``--backend`` choices (cli.py:349-394).  The GPU runs are in
tests/test_gpu_dropin.py.
"""
import json

import pytest

R = pytest.importorskip("oracle.reference")
from paper_0805_1827_b200 import backend as BE  # noqa: E402
from paper_0805_1827_b200 import refshim  # noqa: E402


@pytest.fixture()
def B():
    mod = R.bermuda()
    refshim.register(mod)
    yield mod
    refshim.unregister(mod)


def test_registry_resolves_cuda_by_name(B, monkeypatch):
    import importlib
    kern = importlib.import_module("bermuda._kernels")
    assert kern.get_backend("cuda") is BE
    assert kern.get_backend("CUDA") is BE
    assert "cuda" in kern.available_backends()
    # the names the builders and worker tasks re-resolve (boundary_cmc.py:214, pricer.py:157)
    for name in ("boundary_cmc", "boundary_iz", "pricer", "cli"):
        assert importlib.import_module(f"bermuda.{name}").get_backend("cuda") is BE
    monkeypatch.setenv("BERMUDA_BACKEND", "cuda")
    assert kern.get_backend() is BE
    monkeypatch.setenv("BERMUDA_BACKEND", "cython")
    assert kern.get_backend().name == "cython"
    # unknown names still raise the reference's error (_kernels/__init__.py:53)
    with pytest.raises(ValueError):
        kern.get_backend("opencl")


def test_backend_surface_matches_reference(B):
    import importlib
    ref = importlib.import_module("bermuda._kernels.core_backend")
    for fn in ("raw_uint64", "normals", "stopped_sums", "iz_solve", "cmc_labels"):
        assert callable(getattr(BE, fn)), fn
        assert callable(getattr(ref, fn)), fn
    assert BE.name == "cuda"


def test_cli_accepts_backend_cuda(B):
    import importlib
    cli = importlib.import_module("bermuda.cli")
    for cmd in ("price", "bench", "table", "oracle"):
        extra = ["iz_prices"] if cmd == "table" else []
        args = cli._parser().parse_args([cmd, *extra, "--backend", "cuda"])
        assert args.backend == "cuda"


def test_unregister_restores_the_reference():
    import importlib
    mod = R.bermuda()
    kern = importlib.import_module("bermuda._kernels")
    before = kern.get_backend
    refshim.register(mod)
    refshim.register(mod)  # idempotent
    refshim.unregister(mod)
    assert kern.get_backend is before
    with pytest.raises(ValueError):
        kern.get_backend("cuda")
    with pytest.raises(SystemExit):
        importlib.import_module("bermuda.cli")._parser().parse_args(["price", "--backend", "cuda"])


def test_to_reference_round_trips_rules(B):
    """A rule built by this package becomes the reference's own type, and back."""
    import numpy as np

    import paper_0805_1827_b200 as E
    ens = E.StumpEnsemble(dim=6, rounds=(E.Stump(2, 101.5, 1.0, 0.3), E.Stump(5, float("-inf"), -1.0, 0.1)))
    rule = E.CmcRule(5, 9, True, {3: ens, 7: E.StumpEnsemble(dim=6, rounds=(), intercept=-1.0)})
    ref_rule = refshim.to_reference(rule, B)
    assert type(ref_rule).__module__ == "bermuda.boundary_cmc"
    assert json.loads(ref_rule.to_json()) == json.loads(rule.to_json())
    x = np.array([90.0, 110.0, 102.0, 95.0, 99.0])
    assert ref_rule.score(3, x) == rule.score(3, x)
    est = E.PriceEstimate(price=1.5, variance=2.0, ci95=0.1, n_paths=10, timings={"pricing": 0.1},
                          rule_kind="cmc", unconverged_points=0)
    ref_est = refshim.to_reference(est, B)
    assert type(ref_est).__module__ == "bermuda.pricer"
    assert ref_est.to_json_dict() == est.to_json_dict()
