"""Per-solve cost over a long random sweep (tests/test_gpu_random.py cases),
to find state that accumulates across solves.  Prints the time of every
block of 25 solves, the pinned-pool size and buffer count; with
--release N calls release_cached_memory() every N solves."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_1611_08678_b200 as fabm  # noqa: E402
from paper_1611_08678_b200 import solver  # noqa: E402
from test_gpu_random import _case, _oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=300)
ap.add_argument("--release", type=int, default=0)
ap.add_argument("--oracle", action="store_true", help="also run the C oracle, as the test does")
ap.add_argument("--keep", action="store_true", help="keep every trajectory alive")
args = ap.parse_args()
kept = []
t0 = time.perf_counter()
tb = t0
for s in range(args.cases):
    rng = np.random.default_rng(1000 + s)
    kind, problem, grid = _case(fabm, rng)
    table = fabm.precompute_weights(problem.alpha, grid.n_steps)
    if args.oracle:
        try:
            _oracle(problem, grid, (table.b, table.a, table.c))
        except RuntimeError:
            pass
    try:
        tr = fabm.solve_gpu(problem, grid, weights=table)
        if args.keep:
            kept.append(tr)
    except fabm.SolverStepError:
        pass
    if args.release and (s + 1) % args.release == 0:
        solver.release_cached_memory()
    if (s + 1) % 25 == 0:
        now = time.perf_counter()
        nbuf = sum(len(v) for v in solver._PINNED.free.values())
        print(f"{s + 1:4d} solves  block {1e3 * (now - tb) / 25:8.2f} ms/solve  pool {solver._PINNED.kept / 2**20:8.1f} MiB"
              f" in {nbuf} bufs", flush=True)
        tb = now
print(f"total {time.perf_counter() - t0:.1f} s")
