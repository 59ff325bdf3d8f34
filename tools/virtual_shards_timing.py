"""Virtual (one-GPU emulated) shards K = 1, 2, 8 of the config-5 protocol: time and bitwise y_N."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1611_08678_b200 as fabm
for N in (1_000_000, 4_000_000):
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=N * 1e-4)
    ys = {}
    for K in (1, 2, 8):
        plan = fabm.GpuPlan(p, p.grid(N))
        plan.set_y0(p.y0)
        if K > 1:
            plan.set_virtual_shards(K)
        plan.run()
        ms = min(plan.run() for _ in range(2))
        ys[K] = plan.last_state()
        print(f"N={N:.0e} K={K}: {ms:.1f} ms  y_N={ys[K].tolist()}  bitwise={np.array_equal(ys[K], ys[1])}", flush=True)
        plan.close()
