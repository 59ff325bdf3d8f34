import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import _native as nat
lib = nat.load()
import sys as _s
N = int(_s.argv[1]) if len(_s.argv) > 1 else 200000
for mode in ("1", "0"):
    os.environ["FABM_DEBUG_MODE"] = mode
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    plan = fabm.GpuPlan(p, p.grid(N))
    ms = plan.run()
    buf = (ctypes.c_ulonglong * 8)()
    if hasattr(lib, "fabm_debug_prof"):
        lib.fabm_debug_prof(buf)
    names = ["chain", "publish", "slow+shift", "latewaitcyc", "h0wait", "h0work", "latecount", "h0batch"]
    print(f"mode={mode} N={N} kernel={ms:.2f}ms us/step={ms*1e3/N:.4f}",
          " ".join(f"{n}={buf[i]/N:.2f}" for i, n in enumerate(names)), flush=True)
    plan.close()
