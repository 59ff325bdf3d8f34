"""One batch-kernel launch for ncu captures: the financial alpha sweep (BASELINE
config 4) at T trajectories (default 512: the 8-GPU share), N=1e5, T=100."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm

T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
N = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100000
rhs = fabm.rhs_financial()
probs = [fabm.FractionalProblem(alpha=0.9 + 0.1 * i / T, dim=3, rhs=rhs, y0=(2.0, 3.0, 2.0), t_end=100.0)
         for i in range(T)]
grid = fabm.GridSpec(n_steps=N, h=100.0 / N)
for _ in range(2):
    res = fabm.solve_batch_gpu(probs, grid, states=False)
print(f"T={T} N={N} batch kernel {res.kernel_ms:.1f} ms")
