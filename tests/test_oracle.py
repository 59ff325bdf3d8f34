"""Pin the CPU oracle to the reference's own outputs (tests/golden/, generated
by oracle/make_golden.py from /root/reference) before trusting it."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import TRAJ_FIXTURES, golden, golden_errors, normwise_dev, problem_from_golden
from oracle import abm_oracle, c_oracle


@pytest.mark.parametrize("alpha", [0.3, 0.5, 0.77, 0.8, 0.9, 0.99, 1.0])
def test_reference_weights_bitwise(alpha):
    g = golden("weights_ref")
    b, a, c = abm_oracle.reference_weights(alpha, 500)
    assert np.array_equal(b, g[f"b_{alpha}"])
    assert np.array_equal(a, g[f"a_{alpha}"])
    assert np.array_equal(c, g[f"c_{alpha}"])


def test_reference_weight_goldens_from_reference_tests():
    # pkg/tests/test_weights.py:24-29 (30-digit mpmath values, alpha = 1/2)
    b, a, c = abm_oracle.reference_weights(0.5, 20)
    assert b[0] == pytest.approx(1.1283791670955125739, rel=1e-14)
    assert b[1] == pytest.approx(0.46738995451021813786, rel=1e-14)
    assert a[0] == pytest.approx(0.62318660601362418382, rel=1e-13)
    assert a[10] == pytest.approx(0.17019763901701524634, rel=1e-13)
    assert c[0] == pytest.approx(0.37612638903183752463, rel=1e-14)
    assert c[1] == pytest.approx(0.22032973752843147868, rel=1e-14)


@pytest.mark.parametrize("alpha", [0.1, 0.3, 0.5, 0.8, 0.9, 0.99, 1.0])
def test_accurate_weights_vs_mpmath(alpha):
    idx = np.array([0, 1, 2, 3, 4, 7, 8, 15, 16, 100, 1234, 10**4, 10**5, 10**6, 10**7])
    exact = abm_oracle.exact_weights(alpha, idx)
    got = np.stack(abm_oracle.accurate_weights_at(alpha, idx), axis=1)
    rel = np.abs(got - exact) / np.abs(exact)
    assert rel.max() <= 4e-15, rel.max()


def test_reference_weights_lose_accuracy_at_large_n():
    # the reference table is far from exact for large n, which is
    # why parity runs inject it and the device offers an accurate mode
    g = golden("weights_ref")
    idx = g["sample_index"]
    exact = abm_oracle.exact_weights(0.99, idx)
    rel_a = np.abs(g["sample_a_0.99"] - exact[:, 1]) / np.abs(exact[:, 1])
    assert rel_a[-1] > 1e-4  # n = 1e7


@pytest.mark.parametrize("name", TRAJ_FIXTURES)
def test_numpy_oracle_reproduces_reference(name):
    g = golden(name)
    problem, grid = problem_from_golden(g)
    states, f_cache = abm_oracle.solve_serial(problem.alpha, problem.y0, problem.rhs, grid.h, grid.n_steps)
    # same NumPy/BLAS calls in the same order: bitwise on the generating host,
    # within 1e-14 normwise on any other BLAS build
    assert normwise_dev(states[g["rows"]], g["states"]) <= 1e-14
    assert normwise_dev(f_cache[g["rows"]], g["f_cache"]) <= 1e-14


@pytest.mark.parametrize("name", TRAJ_FIXTURES)
@pytest.mark.parametrize("threads", [1, 3])
def test_c_oracle_matches_reference(name, threads):
    g = golden(name)
    problem, grid = problem_from_golden(g)
    tag = problem.rhs.device_system
    w = abm_oracle.reference_weights(problem.alpha, grid.n_steps)
    states, f_cache = c_oracle.solve(tag.name, tag.params, problem.alpha, problem.y0, grid.h, grid.n_steps, w,
                                     threads=threads)
    tol = 1e-12
    assert normwise_dev(states[g["rows"]], g["states"]) <= tol
    assert normwise_dev(f_cache[g["rows"]], g["f_cache"]) <= tol


def test_c_oracle_error_step_matches_reference():
    errs = golden_errors()
    for name in ("overflow", "initial"):
        lam, y0, N = errs[name + "_config"]
        step, t = errs[name]
        w = abm_oracle.reference_weights(0.8, N)
        with pytest.raises(RuntimeError) as info:
            c_oracle.solve("linear", (lam,), 0.8, [y0], 1.0 / N, N, w)
        assert info.value.step == step
        assert info.value.t == pytest.approx(t, rel=1e-15)


def test_numpy_oracle_error_step_matches_reference():
    errs = golden_errors()
    import paper_1611_08678_b200 as fabm

    for name in ("overflow", "initial"):
        lam, y0, N = errs[name + "_config"]
        step, _ = errs[name]
        with np.errstate(over="ignore", invalid="ignore"):
            with pytest.raises(abm_oracle.OracleStepError) as info:
                abm_oracle.solve_serial(0.8, [y0], fabm.rhs_linear(lam), 1.0 / N, N)
        assert info.value.step == step


def test_chunked_history_matches_dot():
    rng = np.random.default_rng(7)
    f = rng.standard_normal((3000, 3))
    w = rng.random(3001)
    for n in (0, 1, 63, 64, 65, 2999):
        want = np.dot(w[n - np.arange(n + 1)], f[: n + 1])
        got = abm_oracle.chunked_history(f, w, n, 0, 64)
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)


def test_c1_against_mittag_leffler():
    # BASELINE config 1 vs the closed form y = E_0.8(-t^0.8) (50-digit mpmath)
    g = golden("c1_linear")
    t = np.arange(int(g["n_steps"]) + 1) * float(g["h"])
    exact = np.array([abm_oracle.mittag_leffler(0.8, -(ti ** 0.8)) for ti in t[::50]])
    err = np.abs(g["states"][::50, 0] - exact)
    assert err.max() <= 4e-5
    assert abs(g["states"][-1, 0] - 0.042979301317701527263) <= 1e-6


# ---- trajectory CSV (cli.py:97-105): the oracle pinned to the reference's own files
def _csv_case(name):
    import gzip

    from conftest import GOLDEN

    with np.load(GOLDEN / "csv_inputs.npz") as z:
        states, t = z[f"{name}_states"], z[f"{name}_t"]
    return states, t, gzip.decompress((GOLDEN / f"csv_{name}.csv.gz").read_bytes())


@pytest.mark.parametrize("name", ["c1_linear", "hr", "values"])
def test_csv_oracle_matches_reference_files(name):
    from oracle import csv_oracle

    states, t, ref = _csv_case(name)
    assert csv_oracle.format_csv(states, t) == ref
