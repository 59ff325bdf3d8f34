"""Host logic of the strategy plug-in (strategy.install()),
on the CPU: which weight table the installed `gpu` strategy asks for.

The reference is imported from baseline/_ref (installed by
tools/install_reference.sh); solve_gpu is replaced by a recorder, so no
device is needed."""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT

REF = ROOT / "baseline" / "_ref"


@pytest.fixture()
def installed(monkeypatch):
    if not (REF / "fodeabm").exists():
        pytest.skip("reference not installed at baseline/_ref")
    sys.path.insert(0, str(REF))
    import fodeabm.cli  # noqa: F401

    from paper_1611_08678_b200 import strategy

    calls = []

    def fake_solve_gpu(problem, grid, **kw):
        calls.append(kw)
        return "trajectory"

    monkeypatch.setattr(strategy, "solve_gpu", fake_solve_gpu)
    strategy.uninstall()
    fodeabm = strategy.install()
    yield fodeabm, calls
    strategy.uninstall()


def _cfg(n_steps=64):
    return type("Cfg", (), {"strategy": "gpu", "n_steps": n_steps})()


def test_install_registers_the_gpu_strategy(installed):
    fodeabm, _ = installed
    from fodeabm import bench, cli

    assert "gpu" in bench.STRATEGIES
    args = cli._build_parser().parse_args(["solve", "--strategy", "gpu"])
    assert args.strategy == "gpu"


def test_default_uses_the_reference_table(installed):
    fodeabm, calls = installed
    from fodeabm import cli
    from fodeabm.systems import rhs_linear

    problem = fodeabm.FractionalProblem(alpha=0.5, dim=1, rhs=rhs_linear(-1.0), y0=[1.0], t_end=1.0)
    assert cli.solve_with_strategy(problem, _cfg()) == "trajectory"
    # the stock seam: this package's bitwise-equal "reference" mode (plan cache kept)
    assert calls[-1]["weights"] == "reference"


def test_a_patched_seam_is_passed_through(installed, monkeypatch):
    fodeabm, calls = installed
    import fodeabm.core as rcore
    import fodeabm.serial as rserial
    from fodeabm import cli
    from fodeabm.systems import rhs_linear

    real = rcore.precompute_weights

    def zero_c(alpha, n_steps):
        t = real(alpha, n_steps)
        return rcore.WeightTable(alpha=alpha, b=t.b, a=t.a, c=np.zeros(n_steps + 1))

    monkeypatch.setattr(rserial, "precompute_weights", zero_c)
    problem = fodeabm.FractionalProblem(alpha=0.5, dim=1, rhs=rhs_linear(-1.0), y0=[1.0], t_end=1.0)
    cli.solve_with_strategy(problem, _cfg(64))
    table = calls[-1]["weights"]
    assert not isinstance(table, str)
    assert np.array_equal(table.c, np.zeros(65)) and np.array_equal(table.b, real(0.5, 64).b)


def test_uninstall_restores_the_reference(installed):
    fodeabm, _ = installed
    from fodeabm import bench, cli

    from paper_1611_08678_b200 import strategy

    strategy.uninstall()
    assert "gpu" not in bench.STRATEGIES
    with pytest.raises(SystemExit):
        cli._build_parser().parse_args(["solve", "--strategy", "gpu"])
