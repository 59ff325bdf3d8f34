"""Single-step public ops on the device: ``step_predictor`` / ``step_corrector``
(reference serial.py:74-111), plus their batched forms.

The reference recomputes one PECE step from the completed prefix of a
trajectory (two ``np.dot`` over the history).  Here each requested step is
one warp of ``step_pc_kernel`` (``csrc/steps.cuh``), so many steps -- up to
every step of a trajectory -- are evaluated in one launch.  That gives an
a-posteriori consistency check of any trajectory (:func:`trajectory_residual`):
re-running step n from the stored prefix must reproduce y_{n+1}.

Errors follow the reference: an index outside ``[0, N)`` raises
``ValueError``; a non-finite predicted state or rhs output raises
``SolverStepError(step=n, t=(n+1)h)``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .core import SolverStepError
from .solver import _raise_status, _structs

__all__ = ["step_predictor", "step_corrector", "step_predictor_many", "step_corrector_many", "trajectory_residual"]

_MESSAGES = {1: "predicted state is non-finite", 2: "rhs returned a non-finite value"}


def _run(problem, weights, traj, ns, y_pred, device):
    ns = np.ascontiguousarray(np.asarray(ns, dtype=np.int64).reshape(-1))
    grid = traj.grid
    pr, gr, _ = _structs(problem, grid)
    d = int(problem.dim)
    b = np.ascontiguousarray(weights.b, dtype=np.float64)
    a = np.ascontiguousarray(weights.a, dtype=np.float64)
    c = np.ascontiguousarray(weights.c, dtype=np.float64)
    nw = min(b.shape[0], a.shape[0], c.shape[0])
    fc = np.ascontiguousarray(traj.f_cache, dtype=np.float64)
    if fc.ndim != 2 or fc.shape[1] != d:
        raise ValueError(f"f_cache must have shape (rows, {d}), got {fc.shape}")
    yq = None
    if y_pred is not None:
        yq = np.ascontiguousarray(np.asarray(y_pred, dtype=np.float64).reshape(ns.shape[0], d))
    yp = np.empty((ns.shape[0], d))
    y = np.empty((ns.shape[0], d))
    err = np.empty(ns.shape[0], dtype=np.int32)
    st = nat.Status()
    rc = nat.load().fabm_step_pc(ctypes.byref(pr), ctypes.byref(gr), nat.dptr(b), nat.dptr(a), nat.dptr(c), nw,
                                 nat.dptr(fc), fc.shape[0], ns.ctypes.data_as(nat._I64P), ns.shape[0],
                                 nat.dptr(yq), nat.dptr(yp), nat.dptr(y),
                                 err.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(device), ctypes.byref(st))
    if rc != nat.FABM_OK:
        _raise_status(st)
    return ns, yp, y, err


def _raise_first(ns, err, h):
    bad = np.flatnonzero(err)
    if bad.size:
        i = int(bad[0])
        n = int(ns[i])
        raise SolverStepError(_MESSAGES[int(err[i])], step=n, t=(n + 1) * h)


def step_predictor(problem, weights, traj, n: int, *, device: int = 0) -> np.ndarray:
    """Predicted state yP_{n+1} from the completed prefix y_0..y_n (serial.py:74-83)."""
    _, yp, _, _ = _run(problem, weights, traj, [int(n)], None, device)
    return yp[0]


def step_corrector(problem, weights, traj, n: int, y_pred, *, device: int = 0) -> np.ndarray:
    """Corrected state y_{n+1} given a predicted state for t_{n+1} (serial.py:86-111)."""
    ns, _, y, err = _run(problem, weights, traj, [int(n)], np.asarray(y_pred, dtype=np.float64), device)
    _raise_first(ns, err, float(traj.grid.h))
    return y[0]


def step_predictor_many(problem, weights, traj, ns, *, device: int = 0) -> np.ndarray:
    """step_predictor for every index in ``ns`` at once -> (len(ns), d)."""
    _, yp, _, _ = _run(problem, weights, traj, ns, None, device)
    return yp


def step_corrector_many(problem, weights, traj, ns, y_preds=None, *, device: int = 0) -> np.ndarray:
    """step_corrector for every index in ``ns`` -> (len(ns), d).

    ``y_preds`` (len(ns), d) defaults to the predictor of each step, i.e. one
    full PECE step from each prefix.  The first failing index raises.
    """
    ns, _, y, err = _run(problem, weights, traj, ns, y_preds, device)
    _raise_first(ns, err, float(traj.grid.h))
    return y


def trajectory_residual(problem, weights, traj, ns=None, *, device: int = 0) -> float:
    """max_n normwise |PECE(prefix n) - y_{n+1}| / max|y| over the steps ``ns``
    (default: all N) -- the trajectory's self-consistency under ``weights``."""
    N = int(traj.grid.n_steps)
    ns = np.arange(N) if ns is None else np.asarray(ns, dtype=np.int64)
    y = step_corrector_many(problem, weights, traj, ns, device=device)
    ref = np.asarray(traj.states)[ns + 1]
    scale = np.maximum(np.max(np.abs(np.asarray(traj.states)), axis=0), 1e-300)
    return float(np.max(np.abs(y - ref) / scale)) if len(ns) else 0.0
