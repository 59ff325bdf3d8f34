"""GPU parity: the device engine (via the C ABI, libfabm.so) against the
reference's own trajectories (tests/golden/) and the CPU oracle.

Tolerance contract (BASELINE.json north_star):
  * reference weight table injected  -> <= 1e-12 normwise relative
  * device ACCURATE weights           -> <= 1e-12 vs the oracle run with the
                                         same accurate table injected
  * closed form (C1 Mittag-Leffler)  -> discretisation error bounds
Bitwise: repeat solves, and the prefix of a long run vs the short run.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import TRAJ_FIXTURES, golden, golden_errors, normwise_dev, problem_from_golden, sup_rel_dev
from oracle import abm_oracle, c_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.mark.parametrize("name", TRAJ_FIXTURES)
def test_reference_table_parity(fabm, name):
    g = golden(name)
    problem, grid = problem_from_golden(g)
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    rows = g["rows"]
    assert normwise_dev(traj.states[rows], g["states"]) <= TOL
    assert normwise_dev(traj.f_cache[rows], g["f_cache"]) <= TOL
    assert traj.states.shape == (grid.n_steps + 1, problem.dim)
    assert not traj.states.flags.writeable


def test_c2_lorenz_full_parity(fabm):
    """BASELINE config 2 (Lorenz a=0.99, T=100, N=1e5), non-chaotic: full horizon."""
    g = golden("c2_lorenz_full")
    problem, grid = problem_from_golden(g)
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    rows = g["rows"]
    assert normwise_dev(traj.states[rows], g["states"]) <= TOL
    np.testing.assert_allclose(traj.states[-1], [-8.4841261, -8.48133593, 27.00215473], rtol=1e-7)


def test_c1_mittag_leffler(fabm):
    g = golden("c1_linear")
    problem, grid = problem_from_golden(g)
    traj = fabm.solve_gpu(problem, grid)  # device ACCURATE weights
    t = grid.times()[::50]
    exact = np.array([abm_oracle.mittag_leffler(0.8, -(ti ** 0.8)) for ti in t])
    err = np.abs(traj.states[::50, 0] - exact)
    assert err.max() <= 4e-5
    assert abs(traj.states[-1, 0] - 0.042979301317701527263) <= 1e-6


@pytest.mark.parametrize("alpha", [0.3, 0.5, 0.9, 0.99, 1.0])
def test_device_weights_vs_mpmath(fabm, alpha):
    import ctypes

    from paper_1611_08678_b200 import _native as nat

    lib = nat.load()
    N = 10**6
    b = np.empty(N + 1)
    a = np.empty(N + 1)
    c = np.empty(N + 1)
    st = nat.Status()
    rc = lib.fabm_weights(alpha, N, nat.WEIGHTS_ACCURATE, math.gamma(alpha + 1.0), math.gamma(alpha + 2.0),
                          nat.dptr(b), nat.dptr(a), nat.dptr(c), ctypes.byref(st))
    assert rc == 0, st.message
    idx = np.array([0, 1, 2, 3, 4, 7, 8, 15, 16, 100, 1234, 10**4, 10**5, 10**6])
    exact = abm_oracle.exact_weights(alpha, idx)
    got = np.stack([b[idx], a[idx], c[idx]], axis=1)
    assert (np.abs(got - exact) / np.abs(exact)).max() <= 8e-15
    # the formula mode reproduces the reference expression to pow rounding
    rc = lib.fabm_weights(alpha, 2000, nat.WEIGHTS_FORMULA, math.gamma(alpha + 1.0), math.gamma(alpha + 2.0),
                          nat.dptr(b), nat.dptr(a), nat.dptr(c), ctypes.byref(st))
    assert rc == 0
    # (a and c cancel catastrophically: a 1-ulp pow difference is amplified
    # by up to ~n^2, so only the loose agreement of the same formula is checked)
    rb, ra, rc_ = abm_oracle.reference_weights(alpha, 2000)
    np.testing.assert_allclose(b[:2001], rb, rtol=1e-11)
    np.testing.assert_allclose(a[:2001], ra, rtol=1e-6)
    np.testing.assert_allclose(c[:2001], rc_, rtol=1e-6)


@pytest.mark.parametrize("name", ["lorenz_prefix", "hindmarsh_rose", "financial_4095"])
def test_accurate_weights_vs_oracle(fabm, name):
    g = golden(name)
    problem, grid = problem_from_golden(g)
    traj = fabm.solve_gpu(problem, grid, weights="accurate")
    w = abm_oracle.accurate_weights(problem.alpha, grid.n_steps)
    ref, _ = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, grid.n_steps, weights=w)
    assert normwise_dev(traj.states, ref) <= TOL


def test_determinism_bitwise(fabm):
    problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=20.0)
    grid = problem.grid(20000)
    a = fabm.solve_gpu(problem, grid)
    b = fabm.solve_gpu(problem, grid)
    assert np.array_equal(a.states, b.states)
    assert np.array_equal(a.f_cache, b.f_cache)


def test_prefix_of_long_run_is_bitwise(fabm):
    """The first M steps of an N-step run equal the M-step run."""
    lor = fabm.rhs_lorenz()
    long = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=lor, y0=(1.0, 1.0, 1.0), t_end=10.0)
    grid = fabm.GridSpec(n_steps=100000, h=1e-4)
    full = fabm.solve_gpu(long, grid)
    M = 7777
    short = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=lor, y0=(1.0, 1.0, 1.0), t_end=M * 1e-4)
    pre = fabm.solve_gpu(short, fabm.GridSpec(n_steps=M, h=1e-4))
    assert np.array_equal(full.states[: M + 1], pre.states)


def test_large_n_vs_c_oracle(fabm):
    """N = 3e4 Lorenz on the C1e-4 grid: engine vs the C oracle (same accurate table)."""
    lor = fabm.rhs_lorenz()
    N = 30000
    problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=lor, y0=(1.0, 1.0, 1.0), t_end=N * 1e-4)
    grid = fabm.GridSpec(n_steps=N, h=1e-4)
    traj = fabm.solve_gpu(problem, grid)
    w = abm_oracle.accurate_weights(problem.alpha, N)
    ref, fref = c_oracle.solve("lorenz", lor.device_system.params, problem.alpha, problem.y0, grid.h, N, w,
                               threads=c_oracle.max_threads())
    assert normwise_dev(traj.states, ref) <= TOL
    assert normwise_dev(traj.f_cache, fref) <= TOL


@pytest.mark.parametrize("name", ["overflow", "initial"])
def test_error_step_matches_reference(fabm, name):
    errs = golden_errors()
    lam, y0, N = errs[name + "_config"]
    step, t = errs[name]
    problem = fabm.FractionalProblem(alpha=0.8, dim=1, rhs=fabm.rhs_linear(lam), y0=[y0], t_end=1.0)
    with np.errstate(over="ignore", invalid="ignore"):
        with pytest.raises(fabm.SolverStepError) as info:
            fabm.solve_gpu(problem, problem.grid(N), weights="reference")
    assert info.value.step == step
    assert info.value.t == pytest.approx(t, rel=1e-15)


def test_constant_preservation_bitwise(fabm):
    # pkg/tests/test_serial.py:112-116
    problem = fabm.FractionalProblem(alpha=0.5, dim=2, rhs=fabm.rhs_constant([0.0, 0.0]), y0=(3.0, -1.5), t_end=1.0)
    traj = fabm.solve_gpu(problem, problem.grid(2000))
    assert (traj.states == np.array([3.0, -1.5])).all()
    assert (traj.f_cache == 0.0).all()


def test_alpha_one_exact(fabm):
    # pkg/tests/test_serial.py:118-123 — alpha = 1, constant rhs: y = 1 + 2.5 t
    problem = fabm.FractionalProblem(alpha=1.0, dim=1, rhs=fabm.rhs_constant([2.5]), y0=(1.0,), t_end=2.0)
    grid = problem.grid(1000)
    traj = fabm.solve_gpu(problem, grid)
    np.testing.assert_allclose(traj.states[:, 0], 1.0 + 2.5 * grid.times(), rtol=1e-12)


@pytest.mark.parametrize("N", [1, 2, 3, 5, 127, 128, 129, 383, 384, 385, 512, 641])
def test_edge_sizes(fabm, N):
    """Step counts around the block (128) and window (3 blocks) boundaries."""
    problem = fabm.FractionalProblem(alpha=0.7, dim=1, rhs=fabm.rhs_linear(-0.5), y0=[1.0], t_end=1.0)
    grid = problem.grid(N)
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    ref, fref = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, N)
    assert sup_rel_dev(traj.states, ref) <= 1e-12
    assert sup_rel_dev(traj.f_cache, fref) <= 1e-12


def test_plain_callable_rejected(fabm):
    problem = fabm.FractionalProblem(alpha=0.5, dim=1, rhs=lambda t, y: (0.0,), y0=[0.0], t_end=1.0)
    with pytest.raises(ValueError):
        fabm.solve_gpu(problem, problem.grid(10))


def test_accepts_reference_style_objects(fabm):
    """Duck-typed problem/grid objects (e.g. fodeabm's own) are accepted."""
    from types import SimpleNamespace

    rhs = fabm.rhs_linear(-1.0)
    p = SimpleNamespace(alpha=0.8, dim=1, rhs=rhs, y0=np.array([1.0]), t_end=10.0,
                        eval_rhs0=lambda: np.array([-1.0]))
    grid = fabm.GridSpec(n_steps=1000, h=0.01)
    traj = fabm.solve_gpu(p, grid, weights="reference")
    g = golden("c1_linear")
    assert normwise_dev(traj.states, g["states"]) <= TOL


@pytest.mark.parametrize("factory,y0,alpha", [
    ("rhs_lorenz", (1.0, 1.0, 1.0), 0.99),
    ("rhs_chen", (-9.0, -5.0, 14.0), 0.9),
    ("rhs_rossler", (0.5, 1.5, 0.1), 0.9),
    ("rhs_financial", (2.0, 3.0, 2.0), 0.95),
    ("rhs_hindmarsh_rose", (0.1, 0.2, 0.2), 0.9),
])
def test_device_rhs_bitwise_equals_host(fabm, factory, y0, alpha):
    """f_cache rows are device rhs outputs: they equal the host rhs bit for bit."""
    rhs = getattr(fabm, factory)()
    problem = fabm.FractionalProblem(alpha=alpha, dim=3, rhs=rhs, y0=y0, t_end=0.05)
    grid = problem.grid(500)
    traj = fabm.solve_gpu(problem, grid)
    t = grid.times()
    host = np.array([np.asarray(rhs(t[i], traj.states[i]), dtype=np.float64) for i in range(len(t))])
    assert np.array_equal(host, traj.f_cache)


def test_power_law_device_rhs_bitwise(fabm):
    rhs = fabm.rhs_power_law(0.5, 2.0)
    problem = fabm.FractionalProblem(alpha=0.5, dim=1, rhs=rhs, y0=[0.0], t_end=1.0)
    grid = problem.grid(300)
    traj = fabm.solve_gpu(problem, grid)
    host = np.array([rhs(ti, None)[0] for ti in grid.times()])
    # CUDA pow vs libm pow may differ by an ulp; the reference tolerance is 1e-14 here
    np.testing.assert_allclose(traj.f_cache[:, 0], host, rtol=2e-16 * 4, atol=0)


# ---- dim > 4: componentwise systems are solved in blocks of <= 4 components
def test_componentwise_high_dim_matches_oracle_and_1d_solves(fabm):
    rng = np.random.default_rng(5)
    d = 6
    y0 = rng.uniform(-2.0, 2.0, size=d)
    problem = fabm.FractionalProblem(alpha=0.7, dim=d, rhs=fabm.rhs_linear(-0.8), y0=y0, t_end=5.0)
    grid = problem.grid(3000)
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    ref_states, _ = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, grid.n_steps)
    assert normwise_dev(traj.states, ref_states) <= 1e-12
    # each component is exactly its own 1-D solve (the engine's arithmetic is per component)
    for i in range(d):
        p1 = fabm.FractionalProblem(alpha=0.7, dim=1, rhs=fabm.rhs_linear(-0.8), y0=[y0[i]], t_end=5.0)
        assert np.array_equal(fabm.solve_gpu(p1, grid, weights="reference").states[:, 0], traj.states[:, i])


def test_componentwise_constant_dim_20(fabm):
    vals = np.linspace(-3.0, 3.0, 20)
    problem = fabm.FractionalProblem(alpha=0.5, dim=20, rhs=fabm.rhs_constant(vals), y0=np.zeros(20), t_end=1.0)
    grid = problem.grid(500)
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    ref_states, ref_f = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, grid.n_steps)
    assert normwise_dev(traj.states, ref_states) <= 1e-12
    assert np.array_equal(traj.f_cache, ref_f)


def test_componentwise_high_dim_error_is_earliest_step(fabm):
    y0 = np.array([1.0, 1.0, 1.0, 1.0, 1e300, 1.0])
    problem = fabm.FractionalProblem(alpha=1.0, dim=6, rhs=fabm.rhs_linear(80.0), y0=y0, t_end=10.0)
    grid = problem.grid(1000)
    p1 = fabm.FractionalProblem(alpha=1.0, dim=1, rhs=fabm.rhs_linear(80.0), y0=[1e300], t_end=10.0)
    with pytest.raises(fabm.SolverStepError) as e1:
        fabm.solve_gpu(p1, grid)
    with pytest.raises(fabm.SolverStepError) as e6:
        fabm.solve_gpu(problem, grid)
    assert (e6.value.step, e6.value.t) == (e1.value.step, e1.value.t)


def test_watchdog_raises_strategy_timeout(fabm, monkeypatch):
    # dev switch 8 keeps the bulk agents idle, so the stepper waits for target
    # sums that never come: the device watchdog must fire (the reference's
    # StrategyTimeoutError, _shm.py:115-116) and leave the GPU usable
    import time

    problem = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=1.0)
    grid = problem.grid(5000)
    monkeypatch.setenv("FABM_DEBUG_MODE", "8")
    t0 = time.perf_counter()
    with pytest.raises(fabm.StrategyTimeoutError):
        fabm.solve_gpu(problem, grid, timeout_s=0.5)
    assert time.perf_counter() - t0 < 30.0
    monkeypatch.delenv("FABM_DEBUG_MODE")
    traj = fabm.solve_gpu(problem, grid, weights="reference")
    ref_states, _ = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, grid.n_steps)
    assert normwise_dev(traj.states, ref_states) <= 1e-12


def test_streamed_host_output_equals_download(fabm):
    # solve_gpu streams the trajectory into pinned host memory during the run;
    # it must equal the device-resident result copied back afterwards
    import gc

    from paper_1611_08678_b200 import solver

    problem = fabm.FractionalProblem(alpha=0.95, dim=3, rhs=fabm.rhs_chen(), y0=(-9.0, -5.0, 14.0), t_end=2.0)
    grid = problem.grid(20000)
    plan = fabm.GpuPlan(problem, grid)
    plan.set_y0(problem.y0)
    a = plan.run_to_host()
    plan.run()
    b = plan.download()
    plan.close()
    assert np.array_equal(a.states, b.states) and np.array_equal(a.f_cache, b.f_cache)
    assert not a.states.flags.writeable
    # buffers return to the pool when the trajectory dies, and are reused
    nbytes = 8 * 3 * (grid.n_steps + 1)
    solver._PINNED.keep_bytes = max(solver._PINNED.keep_bytes, solver._PINNED.kept + 2 * nbytes)
    ptrs = {a.states.ctypes.data, a.f_cache.ctypes.data}
    del a
    gc.collect()
    c = fabm.solve_gpu(problem, grid)
    assert {c.states.ctypes.data, c.f_cache.ctypes.data} == ptrs
    assert np.array_equal(c.states, b.states)


def test_parallel_strategy_entry_points(fabm):
    # fodeabm.solve_block_parallel / solve_reduction_parallel names on the engine:
    # equivalent to solve_serial (reference EQUIV_TOL 1e-10; here the 1e-12 contract)
    g = golden("hindmarsh_rose")
    problem, grid = problem_from_golden(g)
    st_b, st_r = {}, {}
    blk = fabm.solve_block_parallel(problem, grid, 4, stats=st_b)
    red = fabm.solve_reduction_parallel(problem, grid, 3, 256, stats=st_r)
    ref = g["states"]
    rows = g["rows"]
    assert normwise_dev(blk.states[rows], ref) <= 1e-12 and normwise_dev(red.states[rows], ref) <= 1e-12
    assert np.array_equal(blk.states, fabm.solve_gpu(problem, grid, weights="reference").states)
    assert st_b["plan"].n_workers == 4 and st_r["chunk"] == 256
    # the per-worker counters are "not applicable" (no host workers), not zeros
    assert st_b["idle_steps"] is None and st_r["partial_sums_sent"] is None
    assert st_b["kernel_ms"] > 0


def test_release_cached_memory(fabm):
    from paper_1611_08678_b200 import solver

    problem = fabm.FractionalProblem(alpha=0.8, dim=1, rhs=fabm.rhs_linear(-1.0), y0=[1.0], t_end=1.0)
    a = fabm.solve_gpu(problem, problem.grid(3000))
    fabm.release_cached_memory()
    assert not solver._PLAN_CACHE and solver._PINNED.kept == 0
    b = fabm.solve_gpu(problem, problem.grid(3000))  # plans and buffers come back on demand
    assert np.array_equal(a.states, b.states)
