"""A plain C host of the C ABI (tests/c/abi_smoke.c): the header compiles as
C99 and links against libfabm.so (CPU), and the program's solve and CSV agree
with the Python front end (GPU)."""

from __future__ import annotations

import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

PKG = ROOT / "paper_1611_08678_b200"
SRC = ROOT / "tests" / "c" / "abi_smoke.c"


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    if not (PKG / "libfabm.so").exists():
        pytest.skip("libfabm.so not built")
    exe = tmp_path / "abi_smoke"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"), str(SRC),
                    "-L", str(PKG), "-lfabm", f"-Wl,-rpath,{PKG}", "-o", str(exe)], check=True)
    return exe


def test_c_host_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_host_matches_python_front_end(tmp_path, fabm):
    exe = _build(tmp_path)
    n = 20000
    out = subprocess.run([str(exe), str(n), str(tmp_path)], check=True, capture_output=True,
                         text=True).stdout.split("\n")
    y_n = [float(v) for v in out[0].split()[1:]]
    csv_bytes = int(out[1].split()[1])
    problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=n * 1e-3)
    traj = fabm.solve_gpu(problem, fabm.GridSpec(n_steps=n, h=1e-3))
    # the C host leaves h^alpha and Gamma(alpha+2) to the library (libm), the
    # Python front end passes CPython's values (serial.py:135-136): a few ulp apart
    assert np.max(np.abs(np.array(y_n) - traj.states[-1]) / np.abs(traj.states[-1])) <= 1e-12
    # the C host's CSV is the reference loop's bytes for the C host's own states
    from oracle import csv_oracle

    states = np.fromfile(tmp_path / "states.bin", dtype=np.float64).reshape(n + 1, 3)
    csv = (tmp_path / "traj.csv").read_bytes()
    assert len(csv) == csv_bytes
    assert csv == csv_oracle.format_csv(states, np.arange(n + 1, dtype=np.float64) * 1e-3)
