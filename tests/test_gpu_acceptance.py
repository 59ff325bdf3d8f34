"""The reference's acceptance criteria (pkg/tests/test_acceptance.py), one test
per criterion, on the device engine -- same problems, same thresholds.

Criterion 5 (CPU parallel speedup over the serial solver) is the bench's
business here (bench.py: GPU vs the reference's block strategy on the host);
criterion 7 (the partition's idle fraction) is a host-side model, covered by
tests/test_host_api.py; criterion 9 (property suites) by the seeded random
sweeps of tests/test_gpu_random.py.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

from conftest import sup_rel_dev
from oracle import abm_oracle

pytestmark = pytest.mark.gpu

HR_ENVELOPE = {"x": 5.0, "y": 25.0, "z": 10.0}  # test_acceptance.py:31


def _problems(fabm):
    P = fabm.FractionalProblem
    return {
        "constant": P(alpha=0.5, dim=1, rhs=fabm.rhs_constant([0.5]), y0=(1.0,), t_end=1.0),
        "power-law": P(alpha=0.5, dim=1, rhs=fabm.rhs_power_law(0.5, 2.0), y0=[0.0], t_end=1.0),
        "linear": P(alpha=0.5, dim=1, rhs=fabm.rhs_linear(-1.0), y0=[1.0], t_end=1.0),
        "hindmarsh-rose": P(alpha=0.9, dim=3, rhs=fabm.rhs_hindmarsh_rose(), y0=(0.1, 0.2, 0.2), t_end=40.0),
    }


def test_criterion_1_weight_sanity(fabm):
    """alpha = 1: b_n = 1, a_n = 1, c_n = 1/2 to 1e-14 -- the device table."""
    from paper_1611_08678_b200 import _native as nat

    n = 10_000
    b, a, c = (np.empty(n + 1) for _ in range(3))
    st = nat.Status()
    assert nat.load().fabm_weights(1.0, n, nat.WEIGHTS_ACCURATE, 1.0, 2.0, nat.dptr(b), nat.dptr(a), nat.dptr(c),
                                   ctypes.byref(st)) == 0
    assert np.max(np.abs(b - 1.0)) <= 1e-14
    assert np.max(np.abs(a - 1.0)) <= 1e-14
    assert np.max(np.abs(c - 0.5)) <= 1e-14


def test_criterion_2_analytic_convergence(fabm):
    from paper_1611_08678_b200 import verify

    results, reports = verify.check_power_law_orders(alphas=(0.3, 0.5, 0.8, 1.0), n_list=(500, 1000, 2000))
    assert all(r.passed for r in results), [(r.name, r.detail) for r in results]


def test_criterion_3_mittag_leffler_cross_check(fabm):
    from paper_1611_08678_b200 import verify

    for z in (-2.0, -1.0, -0.5, 0.5, 1.0):
        want = math.exp(z * z) * math.erfc(-z)
        assert verify.mittag_leffler(0.5, z) == pytest.approx(want, rel=1e-13)
    problem = _problems(fabm)["linear"]
    traj = fabm.solve_gpu(problem, problem.grid(4000))
    assert abs(traj.states[-1, 0] - verify.mittag_leffler(0.5, -1.0)) <= 1e-3


@pytest.mark.parametrize("name,tol", [("constant", 1e-10), ("power-law", 1e-10), ("linear", 1e-10),
                                      ("hindmarsh-rose", 1e-8)])
def test_criterion_4_strategy_equivalence(fabm, name, tol):
    """The reference's parallel strategy entry points (here on the engine)
    against the serial solver (the NumPy restatement of serial.py), N=4096,
    P = 2, 4, chunk 64, 1024, with the reference's weight table."""
    problem = _problems(fabm)[name]
    grid = problem.grid(4096)
    ref, _ = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, grid.n_steps)
    worst = 0.0
    for workers in (2, 4):
        worst = max(worst, sup_rel_dev(fabm.solve_block_parallel(problem, grid, workers).states, ref))
        for chunk in (64, 1024):
            worst = max(worst, sup_rel_dev(fabm.solve_reduction_parallel(problem, grid, workers, chunk).states, ref))
    assert worst <= tol


def test_criterion_4_degenerate_configurations_bitwise(fabm):
    problem = _problems(fabm)["power-law"]
    grid = problem.grid(4096)
    ref = fabm.solve_gpu(problem, grid, weights="reference").states
    assert np.array_equal(fabm.solve_block_parallel(problem, grid, 1).states, ref)
    assert np.array_equal(fabm.solve_reduction_parallel(problem, grid, 2, chunk=4096).states, ref)


def test_criterion_6_quadratic_scaling(fabm):
    """The O(N^2) law: device time ratios for N doubling in [3, 5].  On the
    GPU the history work dominates (bulk-bound engine) from N ~ 1e6; below
    that the sequential stepper makes the cost linear in N."""
    times = {}
    for n in (1_000_000, 2_000_000, 4_000_000):
        problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0),
                                         t_end=n * 1e-4)
        plan = fabm.GpuPlan(problem, problem.grid(n))
        plan.set_y0(problem.y0)
        plan.run()
        times[n] = min(plan.run() for _ in range(2))
        plan.close()
    r1 = times[2_000_000] / times[1_000_000]
    r2 = times[4_000_000] / times[2_000_000]
    print(f"criterion 6: kernel ms {times}, ratios {r1:.2f} {r2:.2f}")
    assert 3.0 <= r1 <= 5.0 and 3.0 <= r2 <= 5.0


def test_criterion_8_hindmarsh_rose_long_run(fabm):
    problem = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=fabm.rhs_hindmarsh_rose(), y0=(0.1, 0.2, 0.2),
                                     t_end=1000.0)
    grid = problem.grid(100_000)
    a = fabm.solve_gpu(problem, grid, weights="reference")
    b = fabm.solve_gpu(problem, grid, weights="reference")
    assert np.isfinite(a.states).all()
    assert np.max(np.abs(a.states[:, 0])) <= HR_ENVELOPE["x"]
    assert np.max(np.abs(a.states[:, 1])) <= HR_ENVELOPE["y"]
    assert np.max(np.abs(a.states[:, 2])) <= HR_ENVELOPE["z"]
    assert np.array_equal(a.states, b.states)
