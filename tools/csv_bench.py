"""Time the GPU CSV writer vs the reference's Python loop (restated in oracle/csv_oracle.py).

python tools/csv_bench.py [N ...]   (Lorenz-like random states, d = 3)
"""
import sys, time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_08678_b200 as fabm  # noqa: E402
from oracle import csv_oracle  # noqa: E402


class Rows:
    def __init__(self, states, t):
        self.states, self.t, self.dim = states, t, states.shape[1]


for n in [int(float(a)) for a in sys.argv[1:]] or [1_000_001]:
    rng = np.random.default_rng(0)
    states = rng.standard_normal((n, 3)) * np.array([10.0, 20.0, 30.0])
    t = np.arange(n, dtype=np.float64) * 1e-4
    tr = Rows(states, t)
    fabm.format_trajectory_csv(Rows(states[:1000], t[:1000]))
    st = {}
    t0 = time.perf_counter()
    data = fabm.format_trajectory_csv(tr, stats=st)
    t1 = time.perf_counter()
    path = "/tmp/fabm_csv_bench.csv"
    st2 = {}
    t2 = time.perf_counter()
    fabm.write_trajectory_csv(path, tr, stats=st2)
    t3 = time.perf_counter()
    m = min(n, 100_000)
    t4 = time.perf_counter()
    csv_oracle.format_csv(states[:m], t[:m])
    t5 = time.perf_counter()
    cpu_rows = m / (t5 - t4)
    print(f"N={n} bytes={len(data)} kernels {st['kernel_ms']:.2f} ms ({n / st['kernel_ms'] * 1e3:.3e} rows/s, "
          f"{len(data) / st['kernel_ms'] / 1e6:.1f} GB/s out) | format_trajectory_csv {1e3 * (t1 - t0):.1f} ms | "
          f"write_trajectory_csv {1e3 * (t3 - t2):.1f} ms | python loop {cpu_rows:.3e} rows/s -> "
          f"{n / cpu_rows:.1f} s projected")
