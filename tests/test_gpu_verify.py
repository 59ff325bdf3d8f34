"""Device oracles and the GPU verification suite vs the reference's own
verify.py / checks.py outputs (tests/golden/verify_reference.npz, made by
oracle/make_golden_verify.py)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GOLDEN


def _ref():
    with np.load(GOLDEN / "verify_reference.npz") as z:
        return {k: z[k] for k in z.files}


def test_convergence_report_csv_matches_reference():
    from paper_1611_08678_b200.verify import ConvergenceReport

    g = _ref()
    i = int(np.flatnonzero(g["pl_alphas"] == 0.5)[0])
    rep = ConvergenceReport.from_errors(0.5, "power-law beta=2", list(zip(g["pl_n"], g["pl_err"][i])))
    assert rep.to_csv() == str(g["report_csv"])
    assert rep.observed_order == g["pl_order"][i]


@pytest.mark.gpu
def test_mittag_leffler_device_vs_reference():
    from paper_1611_08678_b200.verify import mittag_leffler_many

    g = _ref()
    val, codes = mittag_leffler_many(g["ml_alpha"], g["ml_z"])
    ref = g["ml_value"]
    inf = np.isinf(ref)
    # the reference returns +-inf when a term overflows (code 2) or the sum
    # itself overflows (code 0): same cells, same sign
    assert np.array_equal(np.isinf(val), inf)
    assert np.array_equal(np.sign(val[inf]), np.sign(ref[inf]))
    assert np.all((codes[inf] == 2) | (codes[inf] == 0)) and np.all(codes[~inf] == 0)
    # finite cells: within the series' conditioning (sum |term_k| times the
    # ulp error of exp/lgamma on arguments up to ~700)
    fin = ~inf
    tol = 2e-13 * g["ml_abs"][fin] + 1e-15 * np.abs(ref[fin])
    err = np.abs(val[fin] - ref[fin])
    assert np.all(err <= tol), f"worst err/tol {np.max(err / tol):.3g}"
    # small arguments (|z| <= 1: no cancellation, exp/lgamma arguments O(1)) agree to a few ulp
    good = fin & (np.abs(g["ml_z"]) <= 1.0)
    rel = np.abs(val[good] - ref[good]) / np.abs(ref[good])
    assert np.max(rel) <= 1e-14


@pytest.mark.gpu
def test_mittag_leffler_scalar_semantics():
    from paper_1611_08678_b200.verify import mittag_leffler

    assert mittag_leffler(0.5, 0.0) == 1.0
    assert abs(mittag_leffler(1.0, 1.0) - math.e) <= 4e-16 * math.e  # E_1 = exp
    # E_{1/2}(-1) = e erfc(1) (reference test_verify.py:16-18)
    assert abs(mittag_leffler(0.5, -1.0) - math.exp(1.0) * math.erfc(1.0)) <= 1e-14
    for a, z in [(0.0, 1.0), (1.5, 1.0), (0.5, 11.0), (0.5, math.nan), (0.5, math.inf)]:
        with pytest.raises(ValueError):
            mittag_leffler(a, z)


@pytest.mark.gpu
def test_convergence_sweep_matches_reference_study():
    from paper_1611_08678_b200.verify import ROUNDOFF_FLOOR, convergence_sweep

    g = _ref()
    reports, terminal = convergence_sweep(g["pl_alphas"], g["pl_n"])
    for i, rep in enumerate(reports):
        errs = np.array([e for _, e in rep.errors])
        if g["pl_alphas"][i] == 1.0:  # exact to roundoff in both
            assert errs.max() <= ROUNDOFF_FLOOR and g["pl_err"][i].max() <= ROUNDOFF_FLOOR
            continue
        # device ACCURATE weights vs the reference's NumPy-pow table: same errors to ~1e-9
        assert np.allclose(errs, g["pl_err"][i], rtol=1e-7, atol=0)
        assert abs(rep.observed_order - g["pl_order"][i]) <= 1e-6
        assert abs(terminal[i] - g["pl_terminal"][i]) <= 1e-7 * g["pl_terminal"][i] + 1e-15


@pytest.mark.gpu
def test_wide_alpha_sweep_orders():
    # the cheap GPU sweep: 64 alphas x 4 grids in four batched launches
    from paper_1611_08678_b200.verify import ORDER_SLACK, convergence_sweep

    alphas = np.linspace(0.2, 0.98, 64)
    reports, terminal = convergence_sweep(alphas, (250, 500, 1000, 2000))
    for rep in reports:
        assert rep.observed_order >= min(2.0, 1.0 + rep.alpha) - ORDER_SLACK
    assert np.all(terminal <= 1e-2)


@pytest.mark.gpu
def test_gpu_verification_suite_passes():
    from paper_1611_08678_b200.verify import run_verification_suite

    results, reports = run_verification_suite()
    failed = [r for r in results if not r.passed]
    assert not failed, failed
    assert len(reports) == 4 and len(results) == 4 + 1 + 1 + 4


# ---- mutation detection (pkg/tests/test_verify.py:143-180): the device
# verification suite must FAIL on a sabotaged weight table, whether it comes
# through the precompute_weights seam or is passed in directly
def _sabotaged_flip_b(real):
    def fn(alpha, n_steps):
        from paper_1611_08678_b200.core import WeightTable

        table = real(alpha, n_steps)
        n = np.arange(n_steps + 1, dtype=np.float64)
        bad_b = ((n + 1.0) ** alpha + n ** alpha) / math.gamma(alpha + 1.0)  # the paper's printed "+"
        return WeightTable(alpha=alpha, b=bad_b, a=table.a, c=table.c)

    return fn


def _sabotaged_zero_c(real):
    def fn(alpha, n_steps):
        from paper_1611_08678_b200.core import WeightTable

        table = real(alpha, n_steps)
        return WeightTable(alpha=alpha, b=table.b, a=table.a, c=np.zeros(n_steps + 1))

    return fn


@pytest.mark.gpu
def test_flipped_predictor_sign_fails_verification(monkeypatch):
    from paper_1611_08678_b200 import solver, verify

    assert verify.check_linear_mittag_leffler(n_steps=500).passed
    real = solver.precompute_weights
    monkeypatch.setattr(solver, "precompute_weights", _sabotaged_flip_b(real))
    assert not verify.check_linear_mittag_leffler(n_steps=500).passed
    monkeypatch.undo()
    # the same table passed explicitly
    bad = _sabotaged_flip_b(real)(0.5, 500)
    assert not verify.check_linear_mittag_leffler(n_steps=500, weights=bad).passed
    assert verify.check_linear_mittag_leffler(n_steps=500).passed  # the seam is restored


@pytest.mark.gpu
def test_missing_first_node_term_fails_verification(monkeypatch):
    from paper_1611_08678_b200 import solver, verify

    assert verify.check_constant_forcing(n_steps=500).passed
    real = solver.precompute_weights
    monkeypatch.setattr(solver, "precompute_weights", _sabotaged_zero_c(real))
    assert not verify.check_constant_forcing(n_steps=500).passed
    monkeypatch.undo()
    bad = _sabotaged_zero_c(real)(0.5, 500)
    assert not verify.check_constant_forcing(n_steps=500, weights=bad).passed


@pytest.mark.gpu
def test_strategy_equivalence_includes_serial_oracle_row():
    from paper_1611_08678_b200 import verify

    rows = {r.name: r for r in verify.check_strategy_equivalence()}
    assert "gpu vs solve_serial [gpu]" in rows and "step residual [gpu]" in rows
    assert rows["step residual [gpu]"].passed, rows["step residual [gpu]"].detail
    # baseline/_ref travels with the repo to the GPU box: the reference is importable there
    assert rows["gpu vs solve_serial [gpu]"].passed, rows["gpu vs solve_serial [gpu]"].detail
