"""GPU parity of the batched engine (BASELINE config 4: an alpha sweep of the
fractional financial system) against the CPU oracle and the single-trajectory
engine."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import normwise_dev
from oracle import abm_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def sweep(fabm, T, N, h=1e-3, y0=(2.0, 3.0, 2.0)):
    rhs = fabm.rhs_financial()
    alphas = 0.9 + 0.1 * np.arange(T) / T  # the config 4 sweep spacing
    probs = [fabm.FractionalProblem(alpha=float(a), dim=3, rhs=rhs, y0=y0, t_end=N * h) for a in alphas]
    return probs, fabm.GridSpec(n_steps=N, h=h)


def test_batch_vs_oracle(fabm):
    probs, grid = sweep(fabm, 6, 1500)
    res = fabm.solve_batch_gpu(probs, grid, f_cache=True)
    for i, p in enumerate(probs):
        w = abm_oracle.accurate_weights(p.alpha, grid.n_steps)
        ref, fref = abm_oracle.solve_serial(p.alpha, p.y0, p.rhs, grid.h, grid.n_steps, weights=w)
        assert normwise_dev(res.states[i], ref) <= TOL
        assert normwise_dev(res.f_cache[i], fref) <= TOL
    np.testing.assert_array_equal(res.y_last, res.states[:, -1])


def test_batch_vs_single_engine(fabm):
    probs, grid = sweep(fabm, 5, 3000)
    res = fabm.solve_batch_gpu(probs, grid)
    for i, p in enumerate(probs):
        single = fabm.solve_gpu(p, grid)
        assert normwise_dev(res.states[i], single.states) <= 1e-13


def test_batch_deterministic_and_order_independent(fabm):
    probs, grid = sweep(fabm, 40, 700)
    a = fabm.solve_batch_gpu(probs, grid)
    b = fabm.solve_batch_gpu(probs, grid)
    assert np.array_equal(a.states, b.states)
    # a trajectory's result does not depend on its batch neighbours
    c = fabm.solve_batch_gpu(probs[7:9], grid)
    assert np.array_equal(c.states, a.states[7:9])


@pytest.mark.parametrize("N", [1, 2, 5, 127, 128, 129, 300])
def test_batch_edge_sizes(fabm, N):
    lam = fabm.rhs_linear(-0.7)
    probs = [fabm.FractionalProblem(alpha=al, dim=2, rhs=lam, y0=(1.0, -0.5), t_end=1.0) for al in (0.3, 0.8, 1.0)]
    grid = probs[0].grid(N)
    res = fabm.solve_batch_gpu(probs, grid)
    for i, p in enumerate(probs):
        w = abm_oracle.accurate_weights(p.alpha, N)
        ref, _ = abm_oracle.solve_serial(p.alpha, p.y0, p.rhs, grid.h, N, weights=w)
        assert normwise_dev(res.states[i], ref) <= TOL


def test_batch_error_is_per_trajectory(fabm):
    ok = fabm.rhs_linear(-1.0)
    bad = fabm.rhs_linear(1e40)
    probs = [fabm.FractionalProblem(alpha=0.8, dim=1, rhs=r, y0=[1.0], t_end=1.0) for r in (ok, bad, ok, bad)]
    grid = probs[0].grid(20)
    with pytest.raises(fabm.SolverStepError) as info:
        fabm.solve_batch_gpu(probs, grid)
    assert info.value.index == 1
    assert info.value.step == 3  # same first failing step as the reference (tests/golden/errors.json)
    res = fabm.solve_batch_gpu(probs, grid, raise_on_error=False)
    assert res.error[0] == 1
    single = fabm.solve_gpu(probs[2], grid)
    np.testing.assert_allclose(res.states[2], single.states, rtol=1e-13)


def test_batch_mixed_members_rejected(fabm):
    a = fabm.FractionalProblem(alpha=0.8, dim=3, rhs=fabm.rhs_lorenz(), y0=(1, 1, 1), t_end=1.0)
    b = fabm.FractionalProblem(alpha=0.8, dim=3, rhs=fabm.rhs_chen(), y0=(1, 1, 1), t_end=1.0)
    with pytest.raises(ValueError):
        fabm.solve_batch_gpu([a, b], a.grid(10))


@pytest.mark.parametrize("kind", ["power-law", "constant4", "linear4", "hindmarsh-rose"])
def test_batch_other_systems_and_dims(fabm, kind):
    # every device rhs family through the batch engine (d = 1, 3, 4), vs the oracle
    rng = np.random.default_rng(len(kind))
    alphas = rng.uniform(0.3, 1.0, 5)
    N = 700
    probs = []
    for a in alphas:
        a = float(a)
        if kind == "power-law":
            probs.append(fabm.FractionalProblem(alpha=a, dim=1, rhs=fabm.rhs_power_law(a, 2.5), y0=[0.0], t_end=1.0))
        elif kind == "constant4":
            probs.append(fabm.FractionalProblem(alpha=a, dim=4, rhs=fabm.rhs_constant([1.0, -2.0, 0.5, 3.0]),
                                                y0=[0.0, 1.0, 2.0, 3.0], t_end=1.0))
        elif kind == "linear4":
            probs.append(fabm.FractionalProblem(alpha=a, dim=4, rhs=fabm.rhs_linear(-0.9), y0=[1.0, -1.0, 0.5, 2.0],
                                                t_end=1.0))
        else:
            probs.append(fabm.FractionalProblem(alpha=a, dim=3, rhs=fabm.rhs_hindmarsh_rose(), y0=fabm.HR_DEFAULT_Y0,
                                                t_end=7.0))
    grid = probs[0].grid(N)
    res = fabm.solve_batch_gpu(probs, grid, f_cache=True)
    for i, p in enumerate(probs):
        w = abm_oracle.accurate_weights(p.alpha, N)
        ref, fref = abm_oracle.solve_serial(p.alpha, p.y0, p.rhs, grid.h, N, weights=w)
        assert normwise_dev(res.states[i], ref) <= TOL
        assert normwise_dev(res.f_cache[i], fref) <= TOL


def test_config4_full_sweep_members_independent_of_the_batch(fabm):
    """BASELINE config 4 at its full size -- 4096 alphas, N = 1e5, T = 100 --
    then four members (first, two inner, last) re-solved as a batch of
    four: bitwise the same y_N, so every member of the full sweep is the
    trajectory the oracle-checked small batches produce (a member's pull
    segments and reduction order depend on its own block index only)."""
    probs, grid = sweep(fabm, 4096, 100_000)
    full = fabm.solve_batch_gpu(probs, grid, states=False)
    assert full.y_last.shape == (4096, 3) and np.isfinite(full.y_last).all()
    pick = [0, 1365, 2730, 4095]
    few = fabm.solve_batch_gpu([probs[i] for i in pick], grid, states=False)
    assert np.array_equal(few.y_last, full.y_last[pick])
