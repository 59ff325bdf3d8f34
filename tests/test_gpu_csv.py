"""GPU trajectory CSV writer vs the reference's bytes (cli.py:97-105).

The bar is bit-exact: the device formatter must produce exactly the bytes
the reference's Python loop writes (tests/golden/csv_*.csv.gz, written by the
reference itself), and exactly CPython's f"{v:.17g}" (oracle/csv_oracle.py)
for any double.
"""

from __future__ import annotations

import gzip

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import csv_oracle

pytestmark = pytest.mark.gpu


class Rows:
    def __init__(self, states, t):
        self.states = np.ascontiguousarray(states, dtype=np.float64)
        self.t = np.ascontiguousarray(t, dtype=np.float64)
        self.dim = self.states.shape[1]


def _case(name):
    with np.load(GOLDEN / "csv_inputs.npz") as z:
        states, t = z[f"{name}_states"], z[f"{name}_t"]
    return Rows(states, t), gzip.decompress((GOLDEN / f"csv_{name}.csv.gz").read_bytes())


@pytest.mark.parametrize("name", ["c1_linear", "hr", "values"])
def test_csv_matches_reference_bytes(fabm, name):
    traj, ref = _case(name)
    assert fabm.format_trajectory_csv(traj) == ref


@pytest.mark.parametrize("name", ["c1_linear", "values"])
def test_write_csv_file_matches_reference(fabm, tmp_path, name):
    traj, ref = _case(name)
    path = tmp_path / f"{name}.csv"
    fabm.write_trajectory_csv(path, traj)
    assert path.read_bytes() == ref


def _random_doubles(rng, n):
    bits = rng.integers(0, 2 ** 63, size=n, dtype=np.int64).astype(np.uint64)
    bits |= rng.integers(0, 2, size=n).astype(np.uint64) << np.uint64(63)
    return bits.view(np.float64)


@pytest.mark.parametrize("dim", [1, 3, 7, 40])
def test_csv_random_bit_patterns(fabm, dim):
    # every exponent range, both signs, nan/inf included by chance
    rng = np.random.default_rng(dim)
    n = 40000 if dim < 10 else 4000  # dim 40: 192-row tiles (shared-memory budget)
    vals = _random_doubles(rng, n * (dim + 1)).reshape(n, dim + 1)
    traj = Rows(vals[:, 1:], vals[:, 0])
    assert fabm.format_trajectory_csv(traj) == csv_oracle.format_csv(traj.states, traj.t)


def test_csv_typical_magnitudes_and_ties(fabm):
    # the fast path (1e-11 .. 1e17) and every 17th-digit tie 2^-k, k = 25..70
    rng = np.random.default_rng(7)
    v = rng.standard_normal(120000) * 10.0 ** rng.integers(-12, 18, size=120000)
    ties = np.concatenate([[2.0 ** -k, -(2.0 ** -k), 3 * 2.0 ** -k] for k in range(1, 80)])
    v = np.concatenate([v, ties, np.ldexp(rng.integers(1, 2 ** 53, size=3000).astype(np.float64), -60)])
    n = len(v) // 3 * 3
    vals = v[:n].reshape(-1, 3)
    traj = Rows(vals[:, 1:], vals[:, 0])
    assert fabm.format_trajectory_csv(traj) == csv_oracle.format_csv(traj.states, traj.t)


def test_csv_empty_and_single_row(fabm):
    traj = Rows(np.zeros((0, 2)), np.zeros(0))
    assert fabm.format_trajectory_csv(traj) == b"t,y0,y1\n"
    traj = Rows(np.array([[-0.0, 1e300]]), np.array([0.0]))
    assert fabm.format_trajectory_csv(traj) == b"t,y0,y1\n0,-0,1.0000000000000001e+300\n"


def test_csv_of_a_solve(fabm, tmp_path):
    # solve -> CSV, through the public call and straight from the plan's device states
    problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=10.0)
    grid = fabm.GridSpec(n_steps=20000, h=5e-4)
    plan = fabm.GpuPlan(problem, grid)
    plan.set_y0(problem.y0)
    plan.run()
    traj = plan.download()
    ref = csv_oracle.format_csv(traj.states, traj.t)
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    fabm.write_trajectory_csv(p1, traj)
    plan.write_csv(p2)
    plan.close()
    assert p1.read_bytes() == ref
    assert p2.read_bytes() == ref


def test_csv_large_round_trip(fabm):
    # N = 1e6 rows: size-independent checks (row count, spot rows, exact round trip of every value)
    n = 1_000_001
    rng = np.random.default_rng(11)
    states = rng.standard_normal((n, 3)) * np.array([10.0, 20.0, 30.0])
    t = np.arange(n, dtype=np.float64) * 1e-4
    data = fabm.format_trajectory_csv(Rows(states, t))
    lines = data.split(b"\n")
    assert lines[0] == b"t,y0,y1,y2" and lines[-1] == b"" and len(lines) == n + 2
    rows = np.concatenate([np.arange(50), rng.integers(0, n, 2000), np.arange(n - 50, n)])
    assert [lines[1 + r] for r in rows] == csv_oracle.format_rows(states, t, rows)
    back = np.array(b",".join(lines[1:-1]).split(b","), dtype=np.float64).reshape(n, 4)
    assert np.array_equal(back[:, 0], t) and np.array_equal(back[:, 1:], states)


def test_csv_bad_path_raises_oserror(fabm, tmp_path):
    traj = Rows(np.zeros((3, 1)), np.arange(3.0))
    with pytest.raises(FileNotFoundError):
        fabm.write_trajectory_csv(tmp_path / "missing" / "x.csv", traj)
    with pytest.raises(IsADirectoryError):
        fabm.write_trajectory_csv(tmp_path, traj)
