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
    strategy.install(weights="reference")
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
