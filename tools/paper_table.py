"""The paper's Table 2 workload on one B200: the fractional Hindmarsh-Rose
model (reference systems.py:101-123, default parameters and y0, alpha = 0.9)
at the paper's step counts (their "CUDA" column is on an
unstated ~2016 GPU).  One solve per N through solve_gpu (device-resident
weights, trajectory streamed to the host), median of 3 after a warm-up."""
import json, statistics, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm

PAPER_CUDA_S = {100000: 169.06, 500000: 1276.42, 1000000: 2670.56, 1500000: 4450.09,
                2000000: 6639.45, 2500000: 9229.66, 3000000: 12226.39}
rows = []
for n, paper_s in PAPER_CUDA_S.items():
    p = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=fabm.rhs_hindmarsh_rose(), y0=fabm.HR_DEFAULT_Y0,
                               t_end=n * 0.01)
    g = p.grid(n)
    fabm.solve_gpu(p, g)
    ts = []
    for _ in range(3):
        st = {}
        t0 = time.perf_counter()
        fabm.solve_gpu(p, g, stats=st)
        ts.append((time.perf_counter() - t0, st["kernel_ms"]))
    wall, kern = sorted(ts)[1]
    rows.append({"n_steps": n, "solve_gpu_s": wall, "kernel_ms": kern, "paper_cuda_s": paper_s,
                 "speedup_vs_paper_gpu": paper_s / wall, "fp64_fma_per_s": 3.0 * n * n / (kern * 1e-3)})
    print(json.dumps(rows[-1]), flush=True)
