"""Fractional Lorenz, alpha = 0.99, N = 1e6 steps on one B200 (the headline
workload), written as the reference's CSV.

    python examples/lorenz_n1e6.py [out.csv]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm  # noqa: E402

problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=100.0)
grid = problem.grid(1_000_000)
fabm.solve_gpu(problem, grid)  # first call: module load, plan and pinned buffers
stats = {}
t0 = time.perf_counter()
traj = fabm.solve_gpu(problem, grid, stats=stats)
t1 = time.perf_counter()
print(f"solve_gpu: {1e3 * (t1 - t0):.1f} ms ({stats['kernel_ms']:.1f} ms kernel), y_N = {traj.states[-1]}")
if len(sys.argv) > 1:
    st = {}
    fabm.write_trajectory_csv(sys.argv[1], traj, stats=st)
    print(f"wrote {st['bytes'] / 1e6:.1f} MB of CSV ({st['kernel_ms']:.2f} ms formatting on the GPU)")
