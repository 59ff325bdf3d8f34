"""Device single-step ops vs the reference's step_predictor / step_corrector
(serial.py:74-111), restated in oracle/abm_oracle.py, on the reference's own
golden trajectories (tests/golden/)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, problem_from_golden
from oracle import abm_oracle

pytestmark = pytest.mark.gpu


class Traj:
    def __init__(self, grid, states, f_cache):
        self.grid, self.states, self.f_cache = grid, states, f_cache


def _case(name):
    import paper_1611_08678_b200 as fabm

    g = golden(name)
    problem, grid = problem_from_golden(g)
    rows = g["rows"]
    assert np.array_equal(rows, np.arange(len(rows))), "needs a contiguous prefix fixture"
    n = len(rows) - 1
    sub = fabm.GridSpec(n_steps=n, h=grid.h)
    return problem, sub, Traj(sub, g["states"], g["f_cache"]), fabm.precompute_weights(problem.alpha, n)


@pytest.mark.parametrize("name", ["c1_linear", "hindmarsh_rose", "lorenz_prefix", "financial_2048"])
def test_steps_match_oracle(name):
    from paper_1611_08678_b200 import steps

    problem, grid, traj, w = _case(name)
    N = grid.n_steps
    ns = np.unique(np.concatenate([np.arange(min(N, 40)), np.linspace(0, N - 1, 60).astype(np.int64)]))
    yp = steps.step_predictor_many(problem, w, traj, ns)
    y = steps.step_corrector_many(problem, w, traj, ns, yp)
    for i, n in enumerate(ns):
        want_p = abm_oracle.step_predictor(problem.alpha, problem.y0, grid.h, w.b, traj.f_cache, n)
        want_c = abm_oracle.step_corrector(problem.alpha, problem.y0, problem.rhs, grid.h, w.a, w.c,
                                           traj.f_cache, n, yp[i])
        np.testing.assert_allclose(yp[i], want_p, rtol=1e-12, atol=1e-14 * np.abs(want_p).max())
        np.testing.assert_allclose(y[i], want_c, rtol=1e-12, atol=1e-14 * np.abs(want_c).max())


@pytest.mark.parametrize("name", ["c1_linear", "lorenz_prefix"])
def test_trajectory_is_self_consistent(name):
    # re-running every step from the reference's stored prefix reproduces y_{n+1}
    from paper_1611_08678_b200 import steps

    problem, grid, traj, w = _case(name)
    assert steps.trajectory_residual(problem, w, traj) <= 1e-12


def test_scalar_ops_and_errors():
    import paper_1611_08678_b200 as fabm
    from paper_1611_08678_b200 import steps

    # alpha = 1, dy = 1, h = 0.1: predictor and corrector both give 0.1 (test_serial.py:59-68)
    problem = fabm.FractionalProblem(alpha=1.0, dim=1, rhs=fabm.rhs_constant([1.0]), y0=[0.0], t_end=1.0)
    grid = problem.grid(10)
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    w = fabm.precompute_weights(1.0, 10)
    yp = steps.step_predictor(problem, w, traj, 0)
    assert abs(yp[0] - 0.1) <= 1e-15
    assert abs(steps.step_corrector(problem, w, traj, 0, yp)[0] - 0.1) <= 1e-15
    with pytest.raises(fabm.SolverStepError) as ei:
        steps.step_corrector(problem, w, traj, 1, np.array([float("nan")]))
    assert ei.value.step == 1 and ei.value.t == 2 * grid.h
    for n in (-1, 10):
        with pytest.raises(ValueError):
            steps.step_predictor(problem, w, traj, n)
