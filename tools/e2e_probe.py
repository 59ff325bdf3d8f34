"""Breakdown of the public solve_gpu call at the headline size (N=1e6)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import solver
N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
g = p.grid(N)
fabm.solve_gpu(p, g)
plan = solver._cached_plan(p, g, "accurate", 0)
for mode in ("to_host", "download", "to_host", "download"):
    t0 = time.perf_counter()
    if mode == "to_host":
        tr = plan.run_to_host()
    else:
        plan.run(); tr = plan.download()
    t1 = time.perf_counter()
    print(f"{mode:9s} {1e3*(t1-t0):8.2f} ms  kernel {plan.stats()['kernel_ms']:.2f} ms")
    del tr
for i in range(4):
    t0 = time.perf_counter(); tr = fabm.solve_gpu(p, g); t1 = time.perf_counter()
    print(f"solve_gpu {1e3*(t1-t0):8.2f} ms  kernel {plan.stats()['kernel_ms']:.2f} ms  pool kept {solver._PINNED.kept/1e6:.0f} MB")
