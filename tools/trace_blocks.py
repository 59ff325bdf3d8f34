import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1611_08678_b200 as fabm
from paper_1611_08678_b200 import _native as nat
lib = nat.load()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
p = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1., 1., 1.), t_end=100.0)
plan = fabm.GpuPlan(p, p.grid(N))
ms = plan.run()
nb = (N + 127) // 128
buf = (ctypes.c_ulonglong * (4 * (nb + 1)))()
lib.fabm_debug_trace.restype = ctypes.c_int
n = lib.fabm_debug_trace(buf, 4 * (nb + 1))
t = np.array(buf[:n], dtype=np.float64).reshape(-1, 4)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us
print(f"N={N} kernel={ms:.1f} ms nb={nb}")
# for target J (>= L=4): source J-4 published -> ready[J] -> staged -> needed
L = 4
rows = []
for J in range(L, nb):
    src = t[J - L, 0]; rdy = t[J, 1]; stg = t[J, 2]; need = t[J, 3]
    rows.append((J, src, rdy, stg, need))
rows = np.array(rows)
def pr(sel, label):
    r = rows[sel]
    print(label, "n=", len(r))
    for q in (0.1, 0.5, 0.9, 0.99):
        print(f"  q{q}: ready-src={np.nanquantile(r[:,2]-r[:,1], q):8.1f}us stage-ready={np.nanquantile(r[:,3]-r[:,2], q):8.1f}us need-stage={np.nanquantile(r[:,4]-r[:,3], q):8.1f}us")
pr(slice(None), "all")
k = len(rows)
pr(slice(0, k // 4), "first quarter")
pr(slice(3 * k // 4, k), "last quarter")
# lateness: staged after needed
late = rows[:, 3] - rows[:, 4]
print("late blocks (staged after need):", int(np.nansum(late > 0)), "total late us:", float(np.nansum(np.clip(late, 0, None))))
for J, src, rdy, stg, need in rows[::max(1, k // 20)]:
    print(f"J={int(J):6d} src@{src:9.1f} ready@{rdy:9.1f} staged@{stg:9.1f} need@{need:9.1f}")
# where the stepper loses time: lateness per decile of the run
dec = np.array_split(np.arange(k), 10)
print("late us per decile of target blocks:", [round(float(np.nansum(np.clip(late[d], 0, None))) / 1e3, 2) for d in dec], "ms")
