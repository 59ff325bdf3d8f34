"""BASELINE config 3: fractional Chen and Rossler systems, N=1e6, alpha=0.9,
T=100 (h=1e-4), one B200.  Median of 3 solve_gpu calls after a warm-up."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1611_08678_b200 as fabm

cases = {
    "chen": (fabm.rhs_chen(), (-9.0, -5.0, 14.0)),
    "rossler": (fabm.rhs_rossler(), (0.5, 1.5, 0.1)),
}
peak = fabm.measure_dfma_peak(0)
for name, (rhs, y0) in cases.items():
    p = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=rhs, y0=y0, t_end=100.0)
    g = p.grid(1_000_000)
    fabm.solve_gpu(p, g)
    runs = []
    for _ in range(3):
        st = {}
        t0 = time.perf_counter()
        tr = fabm.solve_gpu(p, g, stats=st)
        runs.append((time.perf_counter() - t0, st["kernel_ms"]))
    wall, kern = sorted(runs)[1]
    fma = 3.0 * 1e12
    print(json.dumps({"system": name, "alpha": 0.9, "n_steps": 1_000_000, "t_end": 100.0, "y0": y0,
                      "solve_gpu_ms": wall * 1e3, "kernel_ms": kern, "steps_per_s": 1e6 / (kern * 1e-3),
                      "fp64_frac": fma / (kern * 1e-3) / peak, "max_abs_state": np.abs(tr.states).max(0).tolist(),
                      "y_N": tr.states[-1].tolist()}), flush=True)
