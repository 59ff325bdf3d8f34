"""Shared test helpers.  GPU tests are marked ``@pytest.mark.gpu``; the CPU
suite (``-m "not gpu"``) runs without a device."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu on the B200 box)")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        out = {k: z[k] for k in z.files}
    if "meta" in out:
        out["meta"] = json.loads(str(out["meta"]))
    return out


def golden_errors() -> dict:
    return json.loads((GOLDEN / "errors.json").read_text())


def normwise_dev(a: np.ndarray, b: np.ndarray) -> float:
    """max |a-b| / max|b| per component (the SURVEY §8c normwise metric)."""
    scale = np.maximum(np.max(np.abs(b), axis=0), 1e-300)
    return float(np.max(np.abs(a - b) / scale))


def sup_rel_dev(a: np.ndarray, b: np.ndarray) -> float:
    """Elementwise relative deviation with a 1e-30 floor (reference conftest.py:38-40)."""
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


@pytest.fixture(scope="session")
def fabm():
    import paper_1611_08678_b200 as pkg

    return pkg


def problem_from_golden(g: dict):
    """Our FractionalProblem + GridSpec for a golden trajectory fixture."""
    import paper_1611_08678_b200 as fabm

    meta = g["meta"]
    sysname = meta["system"]
    if sysname == "linear":
        rhs = fabm.rhs_linear(*meta["params"])
    elif sysname == "power-law":
        rhs = fabm.rhs_power_law(meta["alpha"], meta["beta"])
    elif sysname == "hindmarsh-rose":
        rhs = fabm.rhs_hindmarsh_rose()
    elif sysname == "lorenz":
        rhs = fabm.rhs_lorenz(*meta["params"])
    elif sysname == "chen":
        rhs = fabm.rhs_chen(*meta["params"])
    elif sysname == "rossler":
        rhs = fabm.rhs_rossler(*meta["params"])
    elif sysname == "financial":
        rhs = fabm.rhs_financial(*meta["params"])
    else:
        raise KeyError(sysname)
    y0 = np.asarray(g["y0"], dtype=np.float64)
    problem = fabm.FractionalProblem(alpha=float(g["alpha"]), dim=len(y0), rhs=rhs, y0=y0, t_end=float(g["t_end"]))
    grid = fabm.GridSpec(n_steps=int(g["n_steps"]), h=float(g["h"]))
    return problem, grid


TRAJ_FIXTURES = (
    "c1_linear",
    "linear_d2",
    "power_law",
    "hindmarsh_rose",
    "lorenz_prefix",
    "chen_prefix",
    "rossler_prefix",
    "financial_0",
    "financial_2048",
    "financial_4095",
)
