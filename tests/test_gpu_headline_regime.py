"""Parity in the regime the headline runs in (VERDICT r1 "what's missing" #3).

The N=1e6 headline spends its time in code that small-N tests never reach:
agents that own several target blocks and switch between them (spilling and
reloading partial sums), bulk units claimed by agents other than their owner,
and targets whose bulk sum is the fixed-order reduction of many unit
partials (engine.cuh "units").  These tests force that regime -- by capping
the bulk CTAs at small N, and by running past the threshold at N=4e5 -- and
compare the whole trajectory with the C oracle (oracle/abm_oracle.c, the
restatement of serial.py:150-170) on the SAME weight table.  They also run
the batch kernel's many-partial regime (config 4 at N=1e5: up to 25 pull
slots per block) against the oracle.

Tolerance: <= 1e-12 normwise relative (BASELINE.json north_star).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

from conftest import normwise_dev
from oracle import c_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def device_table(alpha: float, n: int, mode: str = "accurate"):
    """The exact table the engine generates on the device (fabm_weights)."""
    from paper_1611_08678_b200 import _native as nat

    lib = nat.load()
    b, a, c = (np.empty(n + 1) for _ in range(3))
    st = nat.Status()
    m = nat.WEIGHTS_ACCURATE if mode == "accurate" else nat.WEIGHTS_FORMULA
    rc = lib.fabm_weights(alpha, n, m, math.gamma(alpha + 1.0), math.gamma(alpha + 2.0),
                          nat.dptr(b), nat.dptr(a), nat.dptr(c), ctypes.byref(st))
    assert rc == 0, st.message
    return b, a, c


def lorenz(fabm, N, h):
    return fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=N * h)


@pytest.mark.parametrize("ctas", [2, 4])
def test_multi_target_agents_vs_c_oracle(fabm, ctas):
    """N=3e4 on 2 or 4 bulk CTAs: 32/64 agents own ~7/~4 target blocks each,
    fall behind the stepper and hand units to claimers; each target sums up
    to 29 unit partials.  Equal to the oracle, and bitwise equal to the run
    on all SMs (the unit partition depends on N only)."""
    N, h = 30000, 1e-4
    problem = lorenz(fabm, N, h)
    grid = fabm.GridSpec(n_steps=N, h=h)
    plan = fabm.GpuPlan(problem, grid)
    plan.set_y0(problem.y0)
    plan.set_bulk_ctas(ctas)
    plan.run()
    capped = plan.download()
    st = plan.stats()
    assert st["bulk_ctas"] == ctas
    assert st["segment"] > 1
    plan.set_bulk_ctas(None)
    plan.run()
    full = plan.download()
    plan.close()
    assert np.array_equal(capped.states, full.states)
    assert np.array_equal(capped.f_cache, full.f_cache)
    w = device_table(problem.alpha, N)
    ref, fref = c_oracle.solve("lorenz", problem.rhs.device_system.params, problem.alpha, problem.y0, h, N, w,
                               threads=c_oracle.max_threads())
    assert normwise_dev(capped.states, ref) <= TOL
    assert normwise_dev(capped.f_cache, fref) <= TOL
    if ctas == 2:
        # the owners cannot keep up on two SMs: claimers took units, and the
        # stepper went through its out-of-line wait paths (far handoffs late,
        # or the ring full behind helpers waiting for the bulk) and came back
        assert st["bulk_claims"] > 0
        assert st["leader_wait_ns"] + st["leader_throttle_ns"] > 0


def test_claims_independent_of_schedule(fabm):
    """Bulk CTA counts 1..6 and the default: bitwise the same trajectory."""
    N, h = 12000, 1e-3
    problem = lorenz(fabm, N, h)
    plan = fabm.GpuPlan(problem, fabm.GridSpec(n_steps=N, h=h))
    plan.set_y0(problem.y0)
    runs = []
    for ctas in (1, 3, 6, None):
        plan.set_bulk_ctas(ctas)
        plan.run()
        runs.append(plan.download().states)
    plan.close()
    for r in runs[1:]:
        assert np.array_equal(r, runs[0])


@pytest.mark.parametrize("weights", ["accurate", "reference"])
def test_lorenz_N4e5_full_trajectory_vs_c_oracle(fabm, weights):
    """Lorenz alpha=0.99, h=1e-4, N=4e5: past the N~3e5 point where every
    agent owns more than one target at full occupancy.  Whole trajectory vs
    the C oracle with the same table (device ACCURATE, or the reference's
    precompute_weights table injected)."""
    N, h = 400000, 1e-4
    problem = lorenz(fabm, N, h)
    grid = fabm.GridSpec(n_steps=N, h=h)
    stats = {}
    traj = fabm.solve_gpu(problem, grid, weights=weights, stats=stats)
    if weights == "accurate":
        w = device_table(problem.alpha, N)
    else:
        t = fabm.precompute_weights(problem.alpha, N)
        w = (t.b, t.a, t.c)
    ref, fref = c_oracle.solve("lorenz", problem.rhs.device_system.params, problem.alpha, problem.y0, h, N, w,
                               threads=c_oracle.max_threads())
    assert normwise_dev(traj.states, ref) <= TOL
    assert normwise_dev(traj.f_cache, fref) <= TOL
    assert stats["bulk_tiles"] > 0


def test_config4_members_full_N_vs_c_oracle(fabm):
    """Four members of the config-4 sweep (financial system), N=1e5 on a
    T=30 horizon (the financial system drifts chaotically over
    T=100 at the 1e-12 level): blocks past J=64 sum more than two pull
    partials (up to 25).  Each trajectory vs the C oracle on its own device
    ACCURATE table."""
    N, T = 100000, 30.0
    alphas = [0.9, 0.9 + 0.1 * 1365 / 4096, 0.9 + 0.1 * 2730 / 4096, 0.9 + 0.1 * 4095 / 4096]
    rhs = fabm.rhs_financial()
    problems = [fabm.FractionalProblem(alpha=a, dim=3, rhs=rhs, y0=(2.0, 3.0, 2.0), t_end=T) for a in alphas]
    grid = problems[0].grid(N)
    res = fabm.solve_batch_gpu(problems, grid, states=True)
    for i, p in enumerate(problems):
        w = device_table(p.alpha, N)
        ref, _ = c_oracle.solve("financial", rhs.device_system.params, p.alpha, p.y0, grid.h, N, w,
                                threads=c_oracle.max_threads())
        assert normwise_dev(res.states[i], ref) <= TOL, f"member {i} (alpha={p.alpha})"


@pytest.mark.skipif(not __import__("os").environ.get("FABM_LONG_PARITY"),
                    reason="~3 min of C oracle on 16 cores: FABM_LONG_PARITY=1 to run")
def test_headline_N1e6_full_trajectory_vs_c_oracle(fabm):
    """The bench workload itself -- Lorenz alpha=0.99, T=100, N=1e6, device
    ACCURATE table -- whole trajectory against the C oracle on the same table
    (opt-in: the oracle needs ~155 s on 16 host cores)."""
    N, h = 1_000_000, 1e-4
    problem = lorenz(fabm, N, h)
    grid = fabm.GridSpec(n_steps=N, h=h)
    traj = fabm.solve_gpu(problem, grid, weights="accurate")
    w = device_table(problem.alpha, N)
    ref, fref = c_oracle.solve("lorenz", problem.rhs.device_system.params, problem.alpha, problem.y0, h, N, w,
                               threads=c_oracle.max_threads())
    dev_s, dev_f = normwise_dev(traj.states, ref), normwise_dev(traj.f_cache, fref)
    print(f"N=1e6 normwise deviation: states {dev_s:.3e}, f_cache {dev_f:.3e}")
    assert dev_s <= TOL and dev_f <= TOL


@pytest.mark.parametrize("system,y0,T", [("chen", (-9.0, -5.0, 14.0), 4.0), ("rossler", (0.5, 1.5, 0.1), 20.0),
                                         ("hindmarsh-rose", (0.1, 0.2, 0.2), 1000.0)])
def test_config3_systems_multi_target_vs_c_oracle(fabm, system, y0, T):
    """Config 3's systems (Chen, Rössler; alpha = 0.9) in the multi-target
    regime: N = 2e5 on 4 bulk CTAs (64 agents owning ~25 target blocks each,
    claimed units, many-partial reductions).  Whole trajectory vs the C
    oracle on the device ACCURATE table.  Horizons: Chen's largest Lyapunov
    exponent amplifies the last-bit differences of two summation orders to
    O(1) by T = 20 (measured: 1.7 normwise), so Chen runs to T = 4 (h = 2e-5);
    Rössler to T = 20 (h = 1e-4); Hindmarsh-Rose, the paper's Table 2
    workload, to T = 1000 (h = 5e-3; at the paper's h = 0.01, T = 2000, the
    two summation orders differ by 9e-13, too close to the bound)."""
    N = 200000
    h = T / N
    rhs = {"chen": fabm.rhs_chen, "rossler": fabm.rhs_rossler, "hindmarsh-rose": fabm.rhs_hindmarsh_rose}[system]()
    problem = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=rhs, y0=y0, t_end=T)
    plan = fabm.GpuPlan(problem, fabm.GridSpec(n_steps=N, h=h))
    plan.set_y0(problem.y0)
    plan.set_bulk_ctas(4)
    plan.run()
    traj = plan.download()
    st = plan.stats()
    plan.close()
    assert st["bulk_ctas"] == 4 and st["bulk_claims"] > 0
    w = device_table(problem.alpha, N)
    ref, fref = c_oracle.solve(system, rhs.device_system.params, problem.alpha, problem.y0, h, N, w,
                               threads=c_oracle.max_threads())
    dev_s, dev_f = normwise_dev(traj.states, ref), normwise_dev(traj.f_cache, fref)
    print(f"{system} N=2e5 T={T}: normwise deviation states {dev_s:.3e}, f_cache {dev_f:.3e}")
    assert dev_s <= TOL and dev_f <= TOL


def test_config5_size_prefix_is_the_headline_bitwise(fabm):
    """Size-independent property at the largest BASELINE size: the first 1e6
    steps of the N = 1e7 config-5 trajectory (one GPU) are bitwise the
    N = 1e6 headline solve -- the weight table, the unit partition and the
    reduction order depend on the step / block index only, so the whole
    N = 1e7 regime (256-chunk units, ~30 units per late target) reproduces
    the oracle-checked headline run exactly where they overlap."""
    h = 1e-4
    big = fabm.solve_gpu(lorenz(fabm, 10_000_000, h), fabm.GridSpec(n_steps=10_000_000, h=h))
    head = fabm.solve_gpu(lorenz(fabm, 1_000_000, h), fabm.GridSpec(n_steps=1_000_000, h=h))
    assert np.array_equal(big.states[: 1_000_001], head.states)
    assert np.array_equal(big.f_cache[: 1_000_001], head.f_cache)
    assert np.isfinite(big.states).all()
