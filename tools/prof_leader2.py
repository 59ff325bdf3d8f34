import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import _native as nat
lib = nat.load()
for N in [int(x) for x in (sys.argv[1:] or ["200000"])]:
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    plan = fabm.GpuPlan(p, p.grid(N))
    plan.run(); ms = plan.run()
    b = (ctypes.c_ulonglong * 8)()
    lib.fabm_debug_prof(b)
    names = {0: "gather", 1: "chain", 2: "publish", 3: "push", 7: "rest(check+slow+loop)"}
    print(f"N={N} {ms:.2f} ms  us/step={ms*1e3/N:.4f} cyc/step={ms*1e-3*1.965e9/N:.0f} ",
          " ".join(f"{v}={b[k]/N:.1f}" for k, v in names.items()), flush=True)
