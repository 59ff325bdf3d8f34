"""Quick GPU diagnostics: parity on goldens + engine timings (dev tool)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import paper_1611_08678_b200 as fabm
from conftest import golden, problem_from_golden, normwise_dev

print("devices", fabm.device_count(), flush=True)
for name in ["c1_linear", "lorenz_prefix", "hindmarsh_rose", "chen_prefix", "c2_lorenz_full"]:
    g = golden(name)
    p, grid = problem_from_golden(g)
    st = {}
    t0 = time.perf_counter()
    tr = fabm.solve_gpu(p, grid, weights="reference", stats=st)
    dt = time.perf_counter() - t0
    print(f"{name:16s} N={grid.n_steps:7d} dev={normwise_dev(tr.states[g['rows']], g['states']):.3e} "
          f"wall={dt*1e3:.1f}ms kernel={st['kernel_ms']:.2f}ms tiles={st['bulk_tiles']} wait={st['leader_wait_ns']/1e6:.2f}ms ctas={st['bulk_ctas']}", flush=True)
print("dfma peak FMA/s", fabm.measure_dfma_peak(0), flush=True)
for N in [10**5, 3 * 10**5, 10**6]:
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    plan = fabm.GpuPlan(p, p.grid(N))
    for rep in range(2):
        ms = plan.run()
        st = plan.stats()
        print(f"lorenz N={N} rep{rep} kernel={ms:.1f}ms steps/s={N/(ms*1e-3):.3e} FMA/s={3*N*N/(ms*1e-3):.3e} "
              f"tiles={st['bulk_tiles']} wait={st["leader_wait_ns"]/1e6:.1f}ms thr={st["leader_throttle_ns"]/1e6:.1f}ms ctas={st['bulk_ctas']}", flush=True)
    print("  y_N", plan.last_state(), flush=True)
    plan.close()
