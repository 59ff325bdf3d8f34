"""Leader-alone cycles per step with and without the bulk agents running
(FABM_DEBUG_MODE bits: 1 leader solo, 8 no bulk agents; results invalid)."""
import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import _native as nat
lib = nat.load()
for N in [int(float(a)) for a in sys.argv[1:]] or [100000, 1000000]:
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    for mode in ("1", "9"):
        os.environ["FABM_DEBUG_MODE"] = mode
        plan = fabm.GpuPlan(p, p.grid(N))
        try:
            plan.run(timeout_s=2.0)
        except Exception as exc:  # noqa: BLE001
            pass
        buf = (ctypes.c_ulonglong * 8)()
        lib.fabm_debug_prof(buf)
        print(f"N={N:.0e} debug={mode}: leader {buf[0] / N:.1f} cyc/step", flush=True)
        plan.close()
    os.environ.pop("FABM_DEBUG_MODE")
