"""ctypes wrapper of oracle/libabm_oracle.so — TEST INFRASTRUCTURE ONLY.

Fast CPU checker (tests/) and the timed CPU implementation of bench.py's
reference / cpu_baseline legs.  Never used by the product path.
"""

from __future__ import annotations

import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libabm_oracle.so"
_lib = None

SYSTEM_IDS = {
    "constant": 0, "power-law": 1, "linear": 2, "hindmarsh-rose": 3,
    "lorenz": 4, "chen": 5, "rossler": 6, "financial": 7,
}


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        DP = ctypes.POINTER(ctypes.c_double)
        lib.abm_oracle_solve.restype = ctypes.c_int
        lib.abm_oracle_solve.argtypes = [
            ctypes.c_int, DP, ctypes.c_int, ctypes.c_double, DP, ctypes.c_double, ctypes.c_int64,
            ctypes.c_double, ctypes.c_double, DP, DP, DP, DP, DP, ctypes.c_int,
            ctypes.POINTER(ctypes.c_int64), DP,
        ]
        lib.abm_oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(load().abm_oracle_max_threads())


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def solve(system: str, params, alpha: float, y0, h: float, n_steps: int, weights, threads: int = 1):
    """(states, f_cache) or raises RuntimeError('step n t') on non-finite rhs."""
    lib = load()
    y0 = np.ascontiguousarray(np.asarray(y0, dtype=np.float64).reshape(-1))
    d = y0.shape[0]
    N = int(n_steps)
    b, a, c = (np.ascontiguousarray(np.asarray(w, dtype=np.float64)[: N + 1]) for w in weights)
    prm = np.zeros(16)
    prm[: len(params)] = params
    Y = np.empty((N + 1, d))
    Fc = np.empty((N + 1, d))
    ha = h ** alpha
    ig = 1.0 / math.gamma(alpha + 2.0)
    es = ctypes.c_int64(0)
    et = ctypes.c_double(0.0)
    rc = lib.abm_oracle_solve(SYSTEM_IDS[system], _p(prm), d, alpha, _p(y0), h, N, ha, ig, _p(b), _p(a), _p(c),
                              _p(Y), _p(Fc), int(threads), ctypes.byref(es), ctypes.byref(et))
    if rc != 0:
        err = RuntimeError(f"non-finite rhs at step {es.value}, t={et.value!r}")
        err.step, err.t = es.value, et.value
        raise err
    return Y, Fc
