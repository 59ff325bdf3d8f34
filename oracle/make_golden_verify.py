"""Generate tests/golden/verify_reference.npz from the REFERENCE's verify/checks
modules (verify.py:28-151, checks.py:52-107), for the device oracles.

Run:  python oracle/make_golden_verify.py      (needs /root/reference)

Contents:
  ml_alpha, ml_z, ml_value, ml_abs   E_alpha(z) from the reference series on a
                                     grid of alpha in (0, 1] and z in [-10, 10],
                                     plus sum_k |term_k| (the conditioning)
  pl_alphas, pl_n, pl_err, pl_order, pl_terminal
                                     the reference's power_law_study
  report_csv                         ConvergenceReport.to_csv of alpha = 0.5
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
sys.path.insert(0, str(REF_SRC))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from fodeabm.checks import power_law_study  # noqa: E402
from fodeabm.verify import mittag_leffler  # noqa: E402


def abs_series(alpha, z):
    """sum |term_k| over the terms the reference adds (same stopping rule)."""
    if z == 0.0:
        return 1.0
    la = math.log(abs(z))
    s = 0.0
    total = 0.0
    for k in range(20000):
        try:
            term = math.exp(k * la - math.lgamma(alpha * k + 1.0))
        except OverflowError:
            return math.inf
        s += term
        total += -term if (z < 0 and k & 1) else term
        if k >= 5 and term < 1e-16 * abs(total):
            break
    return s


def main():
    alphas = np.array([0.05, 0.1, 0.25, 0.3, 0.5, 0.7, 0.8, 0.9, 0.99, 1.0])
    zs = np.concatenate([np.linspace(-10.0, 10.0, 41), [-1.0, 1.0, -(10.0 ** 0.8), -0.5, 1e-3, -1e-3]])
    A, Z = np.meshgrid(alphas, zs, indexing="ij")
    val = np.empty(A.shape)
    mag = np.empty(A.shape)
    for i in np.ndindex(A.shape):
        try:
            val[i] = mittag_leffler(A[i], Z[i])
        except ArithmeticError:
            val[i] = np.nan
        mag[i] = abs_series(A[i], Z[i])
    pl_alphas = np.array([0.3, 0.5, 0.8, 1.0])
    pl_n = np.array([500, 1000, 2000])
    errs, orders, terms = [], [], []
    report_csv = ""
    for a in pl_alphas:
        rep, term = power_law_study(float(a), tuple(int(n) for n in pl_n))
        errs.append([e for _, e in rep.errors])
        orders.append(rep.observed_order)
        terms.append(term)
        if a == 0.5:
            report_csv = rep.to_csv()
    np.savez_compressed(OUT / "verify_reference.npz", ml_alpha=A, ml_z=Z, ml_value=val, ml_abs=mag,
                        pl_alphas=pl_alphas, pl_n=pl_n, pl_err=np.array(errs), pl_order=np.array(orders),
                        pl_terminal=np.array(terms), report_csv=np.array(report_csv))
    print("verify_reference.npz", A.shape, "orders", orders)


if __name__ == "__main__":
    main()
