"""Per-call latency of solve_gpu on the small BASELINE configs (C1 linear N=1e3, C2 Lorenz N=1e5)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
cases = {
    "C1 linear N=1e3": (fabm.FractionalProblem(alpha=0.8, dim=1, rhs=fabm.rhs_linear(-1.0), y0=[1.0], t_end=10.0), 1000),
    "C2 Lorenz N=1e5": (fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0), 100000),
}
for name, (p, n) in cases.items():
    g = p.grid(n)
    for w in ("accurate", "reference"):
        fabm.solve_gpu(p, g, weights=w)
        ts = []
        for _ in range(5):
            st = {}
            t0 = time.perf_counter(); fabm.solve_gpu(p, g, weights=w, stats=st); ts.append(time.perf_counter() - t0)
        ts.sort()
        print(f"{name} weights={w}: solve_gpu {1e3 * ts[2]:.2f} ms (kernel {st['kernel_ms']:.2f} ms)")
