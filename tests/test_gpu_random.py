"""Randomised parity sweep (seeded): random systems, orders, step counts and
initial states through the single-trajectory engine and the batch engine,
each against the C restatement of the reference solver (oracle/abm_oracle.c)
run with the same weight table.  Step counts straddle the engine's block
(128), chunk (32) and window (4 blocks) structure; horizons stay short for
the chaotic systems so the 1e-12 normwise bar measures the arithmetic, not
the Lyapunov growth of roundoff (at alpha = 1 Chen doubles roundoff every
~0.35 time units: even the NumPy and C restatements differ by 4e-13 at
T = 2.7).  FABM_RANDOM_CASES=600 ran clean on a B200."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import normwise_dev
from oracle import abm_oracle, c_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _case(fabm, rng):
    kind = rng.choice(["linear", "constant", "hindmarsh-rose", "lorenz", "chen", "rossler", "financial", "power-law"])
    alpha = float(rng.choice([1.0, rng.uniform(0.2, 1.0)]))
    N = int(rng.choice([rng.integers(1, 700), rng.integers(500, 6000),
                        128 * int(rng.integers(1, 40)) + int(rng.integers(-2, 3))]))
    N = max(N, 1)
    if kind == "linear":
        d = int(rng.integers(1, 5))
        rhs = fabm.rhs_linear(float(rng.uniform(-2.0, 0.5)))
        y0 = rng.uniform(-2, 2, d)
    elif kind == "constant":
        d = int(rng.integers(1, 5))
        rhs = fabm.rhs_constant(rng.uniform(-3, 3, d))
        y0 = rng.uniform(-1, 1, d)
    elif kind == "power-law":
        d = 1
        rhs = fabm.rhs_power_law(alpha, float(rng.uniform(alpha, 3.0)))
        y0 = np.zeros(1)
    else:
        d = 3
        rhs = {"hindmarsh-rose": fabm.rhs_hindmarsh_rose, "lorenz": fabm.rhs_lorenz, "chen": fabm.rhs_chen,
               "rossler": fabm.rhs_rossler, "financial": fabm.rhs_financial}[kind]()
        y0 = {"hindmarsh-rose": (0.1, 0.2, 0.2), "lorenz": (1.0, 1.0, 1.0), "chen": (-9.0, -5.0, 14.0),
              "rossler": (0.5, 1.5, 0.1), "financial": (2.0, 3.0, 2.0)}[kind] + rng.uniform(-0.1, 0.1, 3)
    h = 1.5 / 6000 if kind in ("lorenz", "chen", "rossler", "hindmarsh-rose", "financial") else float(rng.uniform(1e-3, 5e-3))
    problem = fabm.FractionalProblem(alpha=alpha, dim=d, rhs=rhs, y0=y0, t_end=N * h)
    return kind, problem, fabm.GridSpec(n_steps=N, h=h)


def _oracle(problem, grid, weights):
    tag = problem.rhs.device_system
    return c_oracle.solve(tag.name, tag.params, problem.alpha, problem.y0, grid.h, grid.n_steps, weights)


N_CASES = int(os.environ.get("FABM_RANDOM_CASES", "40"))


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_engine_vs_c_oracle(fabm, seed):
    rng = np.random.default_rng(1000 + seed)
    kind, problem, grid = _case(fabm, rng)
    table = fabm.precompute_weights(problem.alpha, grid.n_steps)
    try:
        ref, fref = _oracle(problem, grid, (table.b, table.a, table.c))
    except RuntimeError as exc:  # the reference blows up: same step and t on the device
        with pytest.raises(fabm.SolverStepError) as ei:
            fabm.solve_gpu(problem, grid, weights=table)
        assert (ei.value.step, ei.value.t) == (exc.step, exc.t), (kind, problem.alpha)
        return
    traj = fabm.solve_gpu(problem, grid, weights=table)
    assert normwise_dev(traj.states, ref) <= TOL, (kind, problem.alpha, grid.n_steps)
    assert normwise_dev(traj.f_cache, fref) <= TOL, (kind, problem.alpha, grid.n_steps)


@pytest.mark.parametrize("seed", range(8))
def test_random_batch_vs_c_oracle(fabm, seed):
    rng = np.random.default_rng(2000 + seed)
    T = int(rng.integers(1, 70))
    N = int(rng.integers(1, 5000))
    h = 3.0 / 6000
    rhs = fabm.rhs_financial() if seed % 2 else fabm.rhs_lorenz()
    base = np.array((2.0, 3.0, 2.0) if seed % 2 else (1.0, 1.0, 1.0))
    alphas = rng.uniform(0.5, 1.0, T)
    probs = [fabm.FractionalProblem(alpha=float(a), dim=3, rhs=rhs, y0=base + rng.uniform(-0.1, 0.1, 3), t_end=N * h)
             for a in alphas]
    grid = fabm.GridSpec(n_steps=N, h=h)
    res = fabm.solve_batch_gpu(probs, grid)
    for i in rng.choice(T, size=min(T, 6), replace=False):
        p = probs[i]
        w = abm_oracle.accurate_weights(p.alpha, N)
        ref, _ = _oracle(p, grid, w)
        assert normwise_dev(res.states[i], ref) <= TOL, (T, N, p.alpha)


@pytest.mark.parametrize("seed", range(max(4, N_CASES // 10)))
def test_random_virtual_shards_bitwise(fabm, seed):
    # the sharded protocol (one-GPU emulation, K shards) is bitwise the single-GPU solve
    rng = np.random.default_rng(3000 + seed)
    kind, problem, grid = _case(fabm, rng)
    K = int(rng.integers(2, 9))
    try:
        ref = fabm.solve_gpu(problem, grid)
    except fabm.SolverStepError:
        return
    plan = fabm.GpuPlan(problem, grid)
    try:
        plan.set_virtual_shards(K)
        plan.set_y0(problem.y0)
        plan.run()
        got = plan.download()
    finally:
        plan.close()
    assert np.array_equal(got.states, ref.states), (kind, K, grid.n_steps)
