"""Leader phase profile (needs a -DFABM_PROFILE build at $FABM_LIBRARY)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import _native as nat
lib = nat.load()
for N in (3000, 100000, 1000000):
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    plan = fabm.GpuPlan(p, p.grid(N))
    ms = plan.run()
    buf = (ctypes.c_ulonglong * 8)()
    lib.fabm_debug_prof(buf)
    st = plan.stats()
    names = ["pred", "corr", "publish", "slowpath+shift", "throttle"]
    print(f"N={N} kernel={ms:.1f}ms us/step={ms*1e3/N:.3f} wait={st['leader_wait_ns']/1e6:.1f}ms",
          " ".join(f"{n}={buf[i]/N:.1f}cyc" for i, n in enumerate(names)), flush=True)
    plan.close()
