"""Small invocations of every device entry point (also a driver for compute-sanitizer where the pool allows it;
  compute-sanitizer --tool memcheck  python tools/sanitize.py
  compute-sanitizer --tool synccheck python tools/sanitize.py
(race detection / sanitizers on small N)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm  # noqa: E402
from paper_1611_08678_b200 import steps, verify  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
p = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=N * 1e-3)
g = fabm.GridSpec(n_steps=N, h=1e-3)
tr = fabm.solve_gpu(p, g, weights="reference", timeout_s=600)
print("engine", tr.states[-1])
plan = fabm.GpuPlan(p, g)
plan.set_virtual_shards(2)
plan.run(timeout_s=600)
print("sharded(2)", np.array_equal(plan.download().states, fabm.solve_gpu(p, g, timeout_s=600).states))
plan.close()
res = fabm.solve_batch_gpu([fabm.FractionalProblem(alpha=a, dim=3, rhs=fabm.rhs_financial(), y0=(2.0, 3.0, 2.0),
                                                   t_end=N * 1e-3) for a in (0.9, 0.95)], g)
print("batch", res.y_last)
w = fabm.precompute_weights(p.alpha, N)
print("steps", steps.trajectory_residual(p, w, tr, np.arange(0, N, 7)))
print("csv", len(fabm.format_trajectory_csv(tr)))
print("ml", verify.mittag_leffler_many([0.5, 0.9], [-1.0, 3.0])[0])
print("weights", fabm.solve_gpu(p, g, weights="formula", timeout_s=600).states[-1])
