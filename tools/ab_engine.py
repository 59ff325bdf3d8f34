"""A/B timing of engine builds: FABM_LIBRARY=<so> python tools/ab_engine.py N...
Lorenz alpha=0.99 (T=100), median of 5 runs after 2 warm-ups; prints y_N so
builds can be compared bitwise, the leader loop's cycles per step, and (env
FABM_SOLO=1) the leader warp alone (FABM_DEBUG_MODE=1: no handoff waits, no
back-pressure; results invalid, the run ends on the watchdog)."""
import ctypes
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm  # noqa: E402
from paper_1611_08678_b200 import _native as nat  # noqa: E402

lib = nat.load()
for arg in sys.argv[1:] or ["100000"]:
    N = int(float(arg))
    if os.environ.get("FABM_AB_SYS") == "linear3":
        p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_linear(-1.0), y0=(1., 2., 3.), t_end=100.0)
    else:
        p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    plan = fabm.GpuPlan(p, p.grid(N))
    for _ in range(2):
        plan.run()
    ms = statistics.median(plan.run() for _ in range(5))
    st = plan.stats()
    buf = (ctypes.c_ulonglong * 8)()
    if hasattr(lib, "fabm_debug_prof"):
        lib.fabm_debug_prof(buf)
    print(f"N={N:.0e} {ms:9.3f} ms  {N / (ms * 1e-3):.4e} steps/s  wait={st['leader_wait_ns'] / 1e6:.1f} ms  "
          f"throttle={st['leader_throttle_ns'] / 1e6:.1f} ms  leader={buf[0] / N:.1f} cyc/step  fast={buf[1] * 8 / N:.3f}  "
          f"lag={buf[2] * 8 / N:.1f}  helper1 wait={buf[3] / N:.0f} proc={buf[7] / N:.0f} cyc/step  "
          f"seg={st.get('segment')} claims={st.get('bulk_claims')} yN={plan.last_state().tolist()}", flush=True)
    plan.close()
    if os.environ.get("FABM_SOLO"):
        os.environ["FABM_DEBUG_MODE"] = "1"
        plan = fabm.GpuPlan(p, p.grid(N))
        try:
            plan.run(timeout_s=1.0)
        except Exception as exc:  # noqa: BLE001
            print("  solo run ended:", type(exc).__name__)
        lib.fabm_debug_prof(buf)
        print(f"  solo leader: {buf[0] / N:.1f} cyc/step", flush=True)
        plan.close()
        os.environ.pop("FABM_DEBUG_MODE")
