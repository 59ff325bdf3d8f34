"""The reference's own CLI, bench and verify harness driving the GPU engine
through the plug-in (strategy.install()), on the GPU box.

Needs the reference installed at baseline/_ref (pip --target, git-ignored,
travels to the box); skipped when it is absent."""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref_pkg():
    if not (REF / "fodeabm").exists():
        pytest.skip("reference not installed at baseline/_ref")
    sys.path.insert(0, str(REF))
    import fodeabm
    import fodeabm.cli  # noqa: F401

    from paper_1611_08678_b200 import strategy

    # the reference's own weight table (precompute_weights, core.py:134-154):
    # the 1e-12 parity mode; the default device table is more accurate and
    # differs by ~1e-13 relative, which chaotic bursting (Hindmarsh-Rose) amplifies
    strategy.install()  # default: the reference's own seam table (the 1e-12 drop-in)
    yield fodeabm
    strategy.uninstall()


def _read_csv(path):
    return np.loadtxt(path, delimiter=",", skiprows=1)


def test_cli_solve_gpu_matches_serial(ref_pkg, tmp_path):
    from fodeabm import cli

    args = ["solve", "--system", "linear", "--alpha", "0.8", "--tmax", "10", "--steps", "1000"]
    assert cli.main(args + ["--strategy", "serial", "--output", str(tmp_path / "s.csv")]) == 0
    assert cli.main(args + ["--strategy", "gpu", "--output", str(tmp_path / "g.csv")]) == 0
    s, g = _read_csv(tmp_path / "s.csv"), _read_csv(tmp_path / "g.csv")
    assert s.shape == g.shape == (1001, 2)
    assert np.array_equal(s[:, 0], g[:, 0])
    assert np.max(np.abs(g[:, 1] - s[:, 1])) <= 1e-12 * np.max(np.abs(s[:, 1]))


def test_cli_solve_hindmarsh_rose_gpu(ref_pkg, tmp_path):
    from fodeabm import cli

    args = ["solve", "--system", "hindmarsh-rose", "--alpha", "0.9", "--tmax", "20", "--steps", "2000"]
    assert cli.main(args + ["--strategy", "serial", "--output", str(tmp_path / "s.csv")]) == 0
    assert cli.main(args + ["--strategy", "gpu", "--output", str(tmp_path / "g.csv")]) == 0
    s, g = _read_csv(tmp_path / "s.csv"), _read_csv(tmp_path / "g.csv")
    scale = np.max(np.abs(s[:, 1:]), axis=0)
    assert np.max(np.abs(g[:, 1:] - s[:, 1:]) / scale) <= 1e-12


def test_bench_run_cell_gpu_is_deterministic(ref_pkg):
    from fodeabm import bench
    from fodeabm.systems import rhs_linear

    problem = ref_pkg.FractionalProblem(alpha=0.6, dim=1, rhs=rhs_linear(-1.0), y0=[1.0], t_end=5.0)
    t, stats = bench.run_cell(problem, "gpu", 20000, repetitions=3)  # raises if repetitions differ
    assert t > 0 and stats["strategy"] == "gpu" and stats["kernel_ms"] > 0


def test_reference_equivalence_check_includes_gpu(ref_pkg):
    from fodeabm import checks

    res = checks.check_strategy_equivalence(n_steps=512, n_workers=2, chunk=128)
    gpu = [r for r in res if r.name == "gpu strategy"]
    assert len(gpu) == 1 and gpu[0].passed, gpu


def test_device_table_through_the_reference_seam(ref_pkg, monkeypatch):
    """SURVEY §8c parity protocol item 2: the device ACCURATE table, injected
    into the reference's own solve_serial through its precompute_weights seam
    (serial.py:24-31), against the GPU solve with the same table: <= 1e-12."""
    import ctypes
    import math

    import fodeabm.core as rcore
    import fodeabm.serial as rserial

    from paper_1611_08678_b200 import _native as nat
    import paper_1611_08678_b200 as fabm

    alpha, N, h = 0.99, 20000, 1e-3
    lib = nat.load()
    b, a, c = (np.empty(N + 1) for _ in range(3))
    st = nat.Status()
    assert lib.fabm_weights(alpha, N, nat.WEIGHTS_ACCURATE, math.gamma(alpha + 1.0), math.gamma(alpha + 2.0),
                            nat.dptr(b), nat.dptr(a), nat.dptr(c), ctypes.byref(st)) == 0
    table = rcore.WeightTable(alpha=alpha, b=b, a=a, c=c)
    monkeypatch.setattr(rserial, "precompute_weights", lambda al, n: table)

    def lorenz(t, y):
        return (10.0 * (y[1] - y[0]), y[0] * (28.0 - y[2]) - y[1], y[0] * y[1] - 8.0 / 3.0 * y[2])

    rprob = ref_pkg.FractionalProblem(alpha=alpha, dim=3, rhs=lorenz, y0=(1.0, 1.0, 1.0), t_end=N * h)
    ref = ref_pkg.solve_serial(rprob, ref_pkg.GridSpec(n_steps=N, h=h))
    prob = fabm.FractionalProblem(alpha=alpha, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=N * h)
    gpu = fabm.solve_gpu(prob, fabm.GridSpec(n_steps=N, h=h), weights="accurate")
    scale = np.max(np.abs(ref.states), axis=0)
    assert np.max(np.abs(gpu.states - ref.states) / scale) <= 1e-12


def test_patched_seam_reaches_the_gpu_strategy(ref_pkg, monkeypatch):
    """A table patched into fodeabm.serial.precompute_weights (as the reference's
    mutation tests do) is what the installed gpu strategy integrates with."""
    import fodeabm.core as rcore
    import fodeabm.serial as rserial
    from fodeabm import cli
    from fodeabm.systems import rhs_linear

    real = rcore.precompute_weights

    def zero_c(alpha, n_steps):
        t = real(alpha, n_steps)
        return rcore.WeightTable(alpha=alpha, b=t.b, a=t.a, c=np.zeros(n_steps + 1))

    problem = ref_pkg.FractionalProblem(alpha=0.5, dim=1, rhs=rhs_linear(-1.0), y0=[1.0], t_end=1.0)
    cfg = type("Cfg", (), {"strategy": "gpu", "n_steps": 500})()
    good = cli.solve_with_strategy(problem, cfg).states
    monkeypatch.setattr(rserial, "precompute_weights", zero_c)
    bad = cli.solve_with_strategy(problem, cfg).states
    serial_bad = rserial.solve_serial(problem, problem.grid(500)).states
    assert not np.allclose(good, bad)
    assert np.max(np.abs(bad - serial_bad)) <= 1e-12 * np.max(np.abs(serial_bad))
