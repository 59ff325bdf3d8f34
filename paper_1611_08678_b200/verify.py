"""Verification on the device: the reference's analytic oracles and
convergence suite (verify.py, checks.py) driven through the GPU engines
(SURVEY.md §8f row 4).

* :func:`mittag_leffler` / :func:`mittag_leffler_many` — E_alpha(z) by the
  reference's series (verify.py:28-64), evaluated by a device kernel
  (``csrc/oracles.cuh``), one thread per (alpha, z); same errors
  (``ValueError``, ``ArithmeticError``, +-inf on overflow).
* :func:`convergence_sweep` — the power-law refinement study
  (checks.py:52-70) for MANY alphas at once: one batched device solve per N
  (``solve_batch_gpu``) covers every alpha, so a 64-alpha x 4-N sweep is four
  launches instead of 256 serial solves.
* :func:`run_verification_suite` — checks.py:171-177 with the GPU strategy:
  power-law orders, constant-forcing exactness, the linear problem against
  the device Mittag-Leffler, and equivalence of the three device code paths
  (the single-trajectory engine, the batch engine and the sharded-protocol
  emulation) in place of block/reduction vs serial.

Report types (``CheckResult``, ``ConvergenceReport``, ``observed_order``)
mirror the reference's so ``fodeabm verify`` style output and its CSV report
(verify.py:124-133) read the same.
"""

from __future__ import annotations

import csv
import ctypes
import io
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .core import FractionalProblem, GridSpec, SolverStepError
from .solver import GpuPlan, solve_batch_gpu, solve_gpu
from .systems import rhs_linear, rhs_power_law

__all__ = [
    "mittag_leffler",
    "mittag_leffler_many",
    "exact_power_law",
    "observed_order",
    "ConvergenceReport",
    "CheckResult",
    "convergence_sweep",
    "check_power_law_orders",
    "check_constant_forcing",
    "check_linear_mittag_leffler",
    "check_strategy_equivalence",
    "run_verification_suite",
]

# checks.py:30-37
ORDER_SLACK = 0.2
TERMINAL_TOL = 1e-2
ML_TOL = 1e-3
EQUIV_TOL = 1e-10
ROUNDOFF_FLOOR = 1e-13

ML_OK, ML_INVALID, ML_OVERFLOW, ML_NOCONV = 0, 1, 2, 3


# ---------------------------------------------------------------- oracles
def mittag_leffler_many(alpha, z, *, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """E_alpha(z) elementwise on the device; returns (values, codes).

    codes: 0 ok, 1 invalid argument, 2 overflow (value +-inf), 3 no convergence.
    """
    a, x = np.broadcast_arrays(np.asarray(alpha, dtype=np.float64), np.asarray(z, dtype=np.float64))
    shape = a.shape
    a = np.ascontiguousarray(a.reshape(-1))
    x = np.ascontiguousarray(x.reshape(-1))
    out = np.empty(a.shape[0])
    codes = np.empty(a.shape[0], dtype=np.int32)
    st = nat.Status()
    rc = nat.load().fabm_mittag_leffler(nat.dptr(a), nat.dptr(x), a.shape[0], int(device), nat.dptr(out),
                                        codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(st))
    if rc != nat.FABM_OK:
        raise RuntimeError(f"libfabm error {rc}: {st.message.decode(errors='replace')}")
    return out.reshape(shape), codes.reshape(shape)


def mittag_leffler(alpha: float, z: float, *, device: int = 0) -> float:
    """E_alpha(z) by its power series with compensated summation (verify.py:28-64)."""
    alpha = float(alpha)
    z = float(z)
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"alpha must lie in (0, 1], got {alpha!r}")
    if not math.isfinite(z) or abs(z) > 10.0:
        raise ValueError(f"|z| <= 10 required (series validity), got {z!r}")
    v, c = mittag_leffler_many(alpha, z, device=device)
    if int(c) == ML_NOCONV:
        raise ArithmeticError(f"Mittag-Leffler series did not converge in 20000 terms for alpha={alpha}, z={z}")
    return float(v)


def exact_power_law(beta: float, t: float) -> float:
    """t^beta for beta > 0, t >= 0 (verify.py:67-76)."""
    beta = float(beta)
    t = float(t)
    if beta <= 0.0:
        raise ValueError("beta must be positive")
    if t < 0.0:
        raise ValueError("t must be non-negative")
    return t ** beta


def observed_order(errors) -> float:
    """Least-squares slope of log(error) against log(h) (verify.py:79-97)."""
    if len(errors) < 2:
        raise ValueError("need at least two (N, error) pairs")
    ns = [int(n) for n, _ in errors]
    es = [float(e) for _, e in errors]
    if any(b <= a for a, b in zip(ns, ns[1:])):
        raise ValueError("N values must be strictly increasing")
    if any(not math.isfinite(e) or e <= 0.0 for e in es):
        raise ValueError("errors must be positive and finite")
    return float(np.polyfit(np.log([1.0 / n for n in ns]), np.log(es), 1)[0])


@dataclass(frozen=True)
class ConvergenceReport:
    """Grid-refinement study for one problem at one order (verify.py:100-151)."""

    alpha: float
    problem: str
    errors: tuple
    observed_order: float = field(default=float("nan"))

    @classmethod
    def from_errors(cls, alpha: float, problem: str, errors) -> "ConvergenceReport":
        errors = tuple((int(n), float(e)) for n, e in errors)
        return cls(alpha=alpha, problem=problem, errors=errors, observed_order=observed_order(list(errors)))

    def to_csv(self) -> str:
        out = io.StringIO()
        w = csv.writer(out, lineterminator="\n")
        w.writerow(["alpha", "problem", "N", "sup_error"])
        for n, e in self.errors:
            w.writerow([f"{self.alpha:.17g}", self.problem, n, f"{e:.17g}"])
        w.writerow(["observed_order", f"{self.observed_order:.17g}"])
        return out.getvalue()


@dataclass(frozen=True)
class CheckResult:
    name: str
    passed: bool
    detail: str


# ------------------------------------------------------------ sweeps
def _power_problem(alpha: float, beta: float = 2.0, t_end: float = 1.0) -> FractionalProblem:
    return FractionalProblem(alpha=alpha, dim=1, rhs=rhs_power_law(alpha, beta), y0=[0.0], t_end=t_end)


def convergence_sweep(alphas, n_list=(500, 1000, 2000), beta: float = 2.0, t_end: float = 1.0, *,
                      device: int = 0) -> tuple[list[ConvergenceReport], np.ndarray]:
    """Power-law refinement study for every alpha at once (checks.py:52-70).

    One batched device solve per N covers all alphas.  Returns the reports
    (one per alpha, sup error against the exact t^beta on every grid) and the
    terminal absolute errors on the finest grid.
    """
    alphas = [float(a) for a in alphas]
    n_list = [int(n) for n in n_list]
    errs = np.empty((len(alphas), len(n_list)))
    terminal = np.full(len(alphas), math.nan)
    problems = [_power_problem(a, beta, t_end) for a in alphas]
    for j, n in enumerate(n_list):
        grid = problems[0].grid(n)
        res = solve_batch_gpu(problems, grid, states=True)
        exact = grid.times() ** beta
        dev = np.abs(res.states[:, :, 0] - exact[None, :])
        errs[:, j] = np.maximum(dev.max(axis=1), 1e-300)
        terminal = np.abs(res.states[:, -1, 0] - t_end ** beta)
    reports = [ConvergenceReport.from_errors(a, f"power-law beta={beta:g}", list(zip(n_list, errs[i])))
               for i, a in enumerate(alphas)]
    return reports, terminal


def check_power_law_orders(alphas=(0.3, 0.5, 0.8, 1.0), n_list=(500, 1000, 2000), *, device: int = 0):
    """Observed order >= min(2, 1+alpha) - slack, terminal error <= 1e-2 (checks.py:73-107)."""
    reports, terminal = convergence_sweep(alphas, n_list, device=device)
    results = []
    for rep, term in zip(reports, terminal):
        bound = min(2.0, 1.0 + rep.alpha) - ORDER_SLACK
        exact_to_roundoff = max(e for _, e in rep.errors) <= ROUNDOFF_FLOOR
        order_ok = exact_to_roundoff or rep.observed_order >= bound
        detail = (f"order={rep.observed_order:.3f} (bound {bound:.2f}"
                  f"{', exact to roundoff' if exact_to_roundoff else ''}), terminal={term:.3e}")
        results.append(CheckResult(f"power-law order alpha={rep.alpha:g} [gpu]", order_ok and term <= TERMINAL_TOL,
                                   detail))
    return results, reports


def check_constant_forcing(alpha: float = 0.5, n_steps: int = 500, *, weights="reference",
                           device: int = 0) -> CheckResult:
    """beta = alpha: constant forcing, exact solution t^alpha (checks.py:103-119).

    ``weights``: the table the solve uses -- by default the reference's
    ``precompute_weights`` (through :data:`solver.precompute_weights`, the
    seam of serial.py:24-31), or a mode / table as for :func:`solve_gpu`.  A
    corrupted table (e.g. ``c = 0``) must fail this check
    (pkg/tests/test_verify.py:167-180)."""
    problem = _power_problem(alpha, beta=alpha)
    grid = problem.grid(n_steps)
    try:
        traj = solve_gpu(problem, grid, weights=weights, device=device)
    except SolverStepError as exc:
        return CheckResult(f"constant-forcing exactness alpha={alpha:g} [gpu]", False, f"solver failed: {exc}")
    err = float(np.max(np.abs(traj.states[:, 0] - grid.times() ** alpha)))
    return CheckResult(f"constant-forcing exactness alpha={alpha:g} [gpu]", err <= 1e-10,
                       f"sup error {err:.3e} (roundoff expected)")


def check_linear_mittag_leffler(n_steps: int = 4000, lam: float = -1.0, alpha: float = 0.5, t_end: float = 1.0,
                                *, weights="reference", device: int = 0) -> CheckResult:
    """Terminal value of the linear problem against the device series
    (checks.py:122-141).  A table with the predictor sign flipped must fail
    it (pkg/tests/test_verify.py:151-165)."""
    problem = FractionalProblem(alpha=alpha, dim=1, rhs=rhs_linear(lam), y0=[1.0], t_end=t_end)
    try:
        traj = solve_gpu(problem, problem.grid(n_steps), weights=weights, device=device)
    except SolverStepError as exc:
        return CheckResult("linear Mittag-Leffler [gpu]", False, f"solver failed: {exc}")
    exact = mittag_leffler(alpha, lam * t_end ** alpha, device=device)
    err = abs(float(traj.states[-1, 0]) - exact)
    if not math.isfinite(err):
        err = math.inf
    return CheckResult("linear Mittag-Leffler [gpu]", err <= ML_TOL,
                       f"|y_N - E_{alpha:g}({lam * t_end ** alpha:g})| = {err:.3e} (tol {ML_TOL:g})")


def _sup_rel_dev(a: np.ndarray, b: np.ndarray) -> float:
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


def _reference_solve_serial():
    """The reference's own ``solve_serial`` when the reference package is
    importable (installed next to this one, e.g. baseline/_ref), else None."""
    import importlib
    import sys
    from pathlib import Path

    try:
        return importlib.import_module("fodeabm").solve_serial
    except ImportError:
        pass
    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if (ref / "fodeabm").is_dir():
        sys.path.append(str(ref))
        try:
            return importlib.import_module("fodeabm").solve_serial
        except ImportError:
            return None
    return None


def check_strategy_equivalence(n_steps: int = 2048, n_shards: int = 2, *, device: int = 0) -> list[CheckResult]:
    """The device code paths against the serial solver and each other on the
    power-law problem (checks.py:144-168).

    * ``gpu vs solve_serial``: the engine with the reference's table against
      the reference's own ``solve_serial`` (its tolerance EQUIV_TOL), when the
      reference package is importable; the check is reported as not run
      otherwise (it does not pass silently);
    * ``step residual``: every step of the engine's trajectory re-evaluated by
      the independent single-step kernel (``steps.trajectory_residual``);
    * the batch engine (an independent kernel, same ACCURATE weights) and the
      sharded-protocol emulation (bitwise) against the engine.
    """
    from .core import precompute_weights
    from .steps import trajectory_residual

    problem = _power_problem(0.5)
    grid = problem.grid(n_steps)
    out = []
    serial = _reference_solve_serial()
    dev_ref = solve_gpu(problem, grid, weights="reference", device=device)
    if serial is not None:
        ref_traj = serial(problem, grid)
        dev = _sup_rel_dev(dev_ref.states, np.asarray(ref_traj.states))
        out.append(CheckResult("gpu vs solve_serial [gpu]", dev <= EQUIV_TOL, f"sup rel dev {dev:.3e}"))
    else:
        out.append(CheckResult("gpu vs solve_serial [gpu]", False, "not run: the reference package is not importable"))
    res = trajectory_residual(problem, precompute_weights(problem.alpha, n_steps), dev_ref, device=device)
    out.append(CheckResult("step residual [gpu]", res <= EQUIV_TOL, f"normwise residual {res:.3e}"))
    ref = solve_gpu(problem, grid, weights="accurate", device=device)
    batch = solve_batch_gpu([problem], grid, states=True, device=device)
    dev = _sup_rel_dev(batch.states[0], ref.states)
    out.append(CheckResult("batch engine [gpu]", dev <= EQUIV_TOL, f"sup rel dev {dev:.3e}"))
    plan = GpuPlan(problem, grid, weights="accurate", device=device)
    try:
        plan.set_virtual_shards(n_shards)
        plan.set_y0(problem.y0)
        plan.run()
        shard = plan.download()
    finally:
        plan.close()
    same = bool(np.array_equal(shard.states, ref.states))
    out.append(CheckResult(f"sharded protocol K={n_shards} [gpu]", same,
                           "bitwise equal" if same else f"sup rel dev {_sup_rel_dev(shard.states, ref.states):.3e}"))
    return out


def run_verification_suite(*, device: int = 0):
    """The full analytic suite on the GPU (checks.py:171-177)."""
    results, reports = check_power_law_orders(device=device)
    results.append(check_constant_forcing(device=device))
    results.append(check_linear_mittag_leffler(device=device))
    results.extend(check_strategy_equivalence(device=device))
    return results, reports
