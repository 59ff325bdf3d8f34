"""Generate tests/golden/ by running the REFERENCE (fodeabm) in this container.

Run:  python oracle/make_golden.py          (needs /root/reference; ~1 min)

The reference is pure Python, so it is imported from
/root/reference/pkg/src (read-only) — it cannot travel to the GPU box, which
is why its outputs are committed as small .npz fixtures.  Every fixture
records the call that produced it; tests/test_oracle.py pins the NumPy/C
oracle against them and the GPU parity tests compare the device engine with
the same fixtures.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"

sys.path.insert(0, str(REF_SRC))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

import fodeabm  # noqa: E402
from fodeabm import FractionalProblem, precompute_weights, solve_serial  # noqa: E402
from fodeabm import corrector_weight_a, corrector_weight_c, predictor_weight  # noqa: E402
from fodeabm.systems import rhs_hindmarsh_rose, rhs_linear, rhs_power_law  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_08678_b200 import systems as oursys  # noqa: E402  (host rhs, same expressions)


def save(name: str, **arrays):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"  {name}.npz", {k: getattr(v, "shape", v) for k, v in arrays.items()})


def run(problem, grid):
    t0 = time.perf_counter()
    traj = solve_serial(problem, grid)
    return traj, time.perf_counter() - t0


def traj_case(name, problem, n_steps=None, h=None, rows=None, meta=None):
    if h is not None:
        grid = fodeabm.GridSpec(n_steps=n_steps, h=h)
    else:
        grid = problem.grid(n_steps)
    traj, dt = run(problem, grid)
    sel = np.arange(grid.n_steps + 1) if rows is None else np.asarray(rows)
    save(
        name,
        alpha=np.float64(problem.alpha),
        y0=np.asarray(problem.y0),
        t_end=np.float64(problem.t_end),
        n_steps=np.int64(grid.n_steps),
        h=np.float64(grid.h),
        rows=sel,
        states=traj.states[sel],
        f_cache=traj.f_cache[sel],
        seconds=np.float64(dt),
        meta=np.array(json.dumps(meta or {})),
    )


def main():
    print("reference:", fodeabm.__file__, "numpy", np.__version__)
    # -- weights: bitwise tables and large-index samples (core.py:134-154)
    tables = {}
    for al in (0.3, 0.5, 0.77, 0.8, 0.9, 0.99, 1.0):
        t = precompute_weights(al, 500)
        tables[f"b_{al}"] = t.b
        tables[f"a_{al}"] = t.a
        tables[f"c_{al}"] = t.c
    idx = np.array([0, 1, 2, 3, 10, 100, 1000, 12345, 10**5, 10**6, 10**7])
    for al in (0.5, 0.99):
        tables[f"sample_b_{al}"] = np.array([predictor_weight(al, int(n)) for n in idx])
        tables[f"sample_a_{al}"] = np.array([corrector_weight_a(al, int(n)) for n in idx])
        tables[f"sample_c_{al}"] = np.array([corrector_weight_c(al, int(n)) for n in idx])
    save("weights_ref", sample_index=idx, **tables)

    # -- C1: linear D^0.8 y = -y, y0=1, T=10, N=1000 (BASELINE config 1)
    p = FractionalProblem(alpha=0.8, dim=1, rhs=rhs_linear(-1.0), y0=[1.0], t_end=10.0)
    traj_case("c1_linear", p, 1000, meta={"system": "linear", "params": [-1.0]})

    # -- linear vector problem (dim 2, alpha 0.6) and power law (alpha 0.5, beta 2)
    p = FractionalProblem(alpha=0.6, dim=2, rhs=rhs_linear(-0.5), y0=[1.0, -2.0], t_end=3.0)
    traj_case("linear_d2", p, 800, meta={"system": "linear", "params": [-0.5]})
    p = FractionalProblem(alpha=0.5, dim=1, rhs=rhs_power_law(0.5, 2.0), y0=[0.0], t_end=1.0)
    traj_case("power_law", p, 1000, meta={"system": "power-law", "alpha": 0.5, "beta": 2.0})

    # -- Hindmarsh-Rose (the paper's demonstration system)
    p = FractionalProblem(alpha=0.9, dim=3, rhs=rhs_hindmarsh_rose(), y0=(0.1, 0.2, 0.2), t_end=10.0)
    traj_case("hindmarsh_rose", p, 2000, meta={"system": "hindmarsh-rose"})

    # -- BASELINE systems through the reference solver with our host rhs
    lor = oursys.rhs_lorenz()
    p = FractionalProblem(alpha=0.99, dim=3, rhs=lor, y0=(1.0, 1.0, 1.0), t_end=3.0)
    traj_case("lorenz_prefix", p, 3000, h=1e-3, meta={"system": "lorenz", "params": list(lor.device_system.params),
                                                      "note": "C2 grid h=1e-3, first 3000 steps (prefix trick)"})
    chen = oursys.rhs_chen()
    p = FractionalProblem(alpha=0.9, dim=3, rhs=chen, y0=(-9.0, -5.0, 14.0), t_end=0.3)
    traj_case("chen_prefix", p, 3000, h=1e-4, meta={"system": "chen", "params": list(chen.device_system.params),
                                                    "note": "C3 grid h=1e-4, t<=0.3 (chaotic: short horizon)"})
    ros = oursys.rhs_rossler()
    p = FractionalProblem(alpha=0.9, dim=3, rhs=ros, y0=(0.5, 1.5, 0.1), t_end=0.3)
    traj_case("rossler_prefix", p, 3000, h=1e-4, meta={"system": "rossler", "params": list(ros.device_system.params)})
    fin = oursys.rhs_financial()
    # C4 sweep alphas = 0.9 + 0.1 * arange(4096) / 4096: first, middle, last
    for i in (0, 2048, 4095):
        al = 0.9 + 0.1 * i / 4096
        p = FractionalProblem(alpha=al, dim=3, rhs=fin, y0=(2.0, 3.0, 2.0), t_end=2.0)
        traj_case(f"financial_{i}", p, 2000, h=1e-3,
                  meta={"system": "financial", "params": list(fin.device_system.params)})

    # -- C2 full run: Lorenz alpha 0.99, y0 (1,1,1), T=100, N=1e5 (sampled rows)
    p = FractionalProblem(alpha=0.99, dim=3, rhs=lor, y0=(1.0, 1.0, 1.0), t_end=100.0)
    rows = np.concatenate([np.arange(0, 100001, 500), [99999, 100000]])
    traj_case("c2_lorenz_full", p, 100000, rows=np.unique(rows),
              meta={"system": "lorenz", "params": list(lor.device_system.params)})

    # -- error semantics: first non-finite rhs (serial.py:157-168, core.py:226-236)
    errs = {}
    for name, lam, y0, N in (("overflow", 1e40, 1.0, 20), ("initial", 1e300, 1e300, 5)):
        p = FractionalProblem(alpha=0.8, dim=1, rhs=rhs_linear(lam), y0=[y0], t_end=1.0)
        try:
            solve_serial(p, p.grid(N))
            errs[name] = (-1, float("nan"))
        except fodeabm.SolverStepError as exc:
            errs[name] = (exc.step, exc.t)
        errs[name + "_config"] = (lam, y0, N)
    (OUT / "errors.json").write_text(json.dumps(errs, indent=1))
    print("  errors.json", errs)

    meta = {
        "generated_by": "oracle/make_golden.py",
        "reference": str(REF_SRC),
        "numpy": np.__version__,
        "python": platform.python_version(),
        "machine": platform.machine(),
        "cpu": platform.processor(),
    }
    try:
        from threadpoolctl import threadpool_info

        meta["blas"] = [{k: i.get(k) for k in ("internal_api", "version", "architecture")} for i in threadpool_info()]
    except Exception:
        pass
    (OUT / "META.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
