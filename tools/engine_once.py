"""One device-resident engine run (for ncu captures): Lorenz alpha=0.99, T=100."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
plan = fabm.GpuPlan(p, p.grid(N))
for _ in range(2):
    ms = plan.run()
print(f"N={N} engine {ms:.2f} ms  steps/s={N/(ms*1e-3):.3e}")
