"""Generate tests/golden/csv_*: CSVs written by the REFERENCE's own
write_trajectory_csv (cli.py:97-105), with the inputs that produced them.

Run:  python oracle/make_golden_csv.py      (needs /root/reference)

Cases (inputs in csv_inputs.npz, output csv_<case>.csv.gz):
  c1_linear   BASELINE config 1 trajectory from solve_serial (d = 1, 1001 rows)
  hr          Hindmarsh-Rose trajectory from solve_serial (d = 3, 501 rows)
  values      synthetic rows of edge values through the same writer: ties of
              the 17th digit, powers of ten and their neighbours, subnormals,
              the largest doubles, +-0, inf, nan, and random bit patterns over
              the whole exponent range (d = 3, 4000 rows; t = random too)
"""

from __future__ import annotations

import gzip
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
sys.path.insert(0, str(REF_SRC))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from fodeabm import FractionalProblem, solve_serial  # noqa: E402
from fodeabm.cli import write_trajectory_csv  # noqa: E402
from fodeabm.systems import HR_DEFAULT_Y0, rhs_hindmarsh_rose, rhs_linear  # noqa: E402


class Rows:
    """Duck-typed trajectory (the writer reads .dim, .t, .states)."""

    def __init__(self, states, t):
        self.states = states
        self.t = t
        self.dim = states.shape[1]


def edge_values(rng) -> np.ndarray:
    v = [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
         2.225073858507201e-308, 1.7976931348623157e308, -1.7976931348623157e308, 1.0, -1.0, 0.1, 1 / 3]
    for k in range(-330, 310):  # powers of ten and both neighbours
        x = float(f"1e{k}")
        v += [x, np.nextafter(x, 0.0), np.nextafter(x, np.inf)]
    for k in range(1, 80):  # 2^-k: exact decimals ending in 5 (17th-digit ties for k = 25 ..)
        v += [2.0 ** -k, 3 * 2.0 ** -k, 2.0 ** k, 2.0 ** k + 1]
    for k in (16, 17, 18):
        v += [9.999999999999999e-5, 99999999999999999.0, 9.9999999999999992e16, 1e16 - 1, 1e17 - 16]
    bits = rng.integers(0, 2 ** 63, size=6000, dtype=np.int64).astype(np.uint64)
    bits |= rng.integers(0, 2, size=6000).astype(np.uint64) << np.uint64(63)
    v += list(bits.view(np.float64))
    v += list(rng.standard_normal(1500) * 10.0 ** rng.integers(-12, 18, size=1500))
    return np.asarray(v, dtype=np.float64)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(20261018)
    cases = {}
    p1 = FractionalProblem(alpha=0.8, dim=1, rhs=rhs_linear(-1.0), y0=[1.0], t_end=10.0)
    tr = solve_serial(p1, p1.grid(1000))
    cases["c1_linear"] = (np.array(tr.states), np.array(tr.t))
    p2 = FractionalProblem(alpha=0.9, dim=3, rhs=rhs_hindmarsh_rose(), y0=HR_DEFAULT_Y0, t_end=50.0)
    tr = solve_serial(p2, p2.grid(500))
    cases["hr"] = (np.array(tr.states), np.array(tr.t))
    vals = edge_values(rng)
    n = (len(vals) // 4) * 4
    vals = rng.permutation(vals[:n]).reshape(-1, 4)
    cases["values"] = (np.ascontiguousarray(vals[:, 1:]), np.ascontiguousarray(vals[:, 0]))
    arrays = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (states, t) in cases.items():
            path = Path(tmp) / f"{name}.csv"
            write_trajectory_csv(str(path), Rows(states, t))
            data = path.read_bytes()
            (OUT / f"csv_{name}.csv.gz").write_bytes(gzip.compress(data, compresslevel=9, mtime=0))
            arrays[f"{name}_states"] = states
            arrays[f"{name}_t"] = t
            print(f"  csv_{name}.csv.gz  rows={len(t)} dim={states.shape[1]} bytes={len(data)}")
    np.savez_compressed(OUT / "csv_inputs.npz", **arrays)


if __name__ == "__main__":
    main()
