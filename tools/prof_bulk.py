import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import _native as nat
lib = nat.load()
for N in [int(x) for x in (sys.argv[1:] or ["300000", "1000000"])]:
    p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
    plan = fabm.GpuPlan(p, p.grid(N))
    ms = plan.run()
    buf = (ctypes.c_ulonglong * 8)()
    lib.fabm_debug_prof(buf)
    st = plan.stats()
    agents = st["bulk_ctas"] * 16
    cyc = ms * 1e-3 * 1.965e9
    print(f"N={N} kernel={ms:.1f}ms steps/s={N/(ms*1e-3):.3e} wait={st['leader_wait_ns']/1e6:.1f}ms "
          f"agents={agents} tile={buf[4]/agents/cyc:.3f} idle={buf[5]/agents/cyc:.3f} switch={buf[6]/agents/cyc:.3f} (fractions of kernel time per agent)", flush=True)
    if hasattr(lib, "fabm_debug_prof2"):
        b2 = (ctypes.c_ulonglong * 8)()
        lib.fabm_debug_prof2(b2)
        n_sel, n_scan, n_spill, c_top, n_fin, c_fin, c_scan, c_spl = list(b2)
        print(f"   per agent: selections {n_sel/agents:.0f} (src_done acquire {c_top/agents/cyc:.3f} of kernel time), "
              f"cursor scans {n_scan/agents:.0f} ({c_scan/agents/cyc:.3f}), spills+reloads {n_spill/agents:.0f} "
              f"({c_spl/agents/cyc:.3f}), units finished {n_fin/agents:.0f} ({c_fin/agents/cyc:.3f}); "
              f"tiles {st['bulk_tiles']/agents:.0f}, claims {st['bulk_claims']}", flush=True)
    plan.close()
