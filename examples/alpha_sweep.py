"""BASELINE config 4: the fractional financial system swept over 4096 orders
alpha in [0.9, 1), N = 1e5, sharded over the GPUs of a node.

    python examples/alpha_sweep.py                      # one GPU
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/alpha_sweep.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1611_08678_b200 as fabm  # noqa: E402
from paper_1611_08678_b200 import parallel  # noqa: E402

T = int(os.environ.get("SWEEP", "4096"))
problems = [fabm.FractionalProblem(alpha=0.9 + 0.1 * i / T, dim=3, rhs=fabm.rhs_financial(), y0=(2.0, 3.0, 2.0),
                                   t_end=100.0) for i in range(T)]
grid = problems[0].grid(100_000)
if "WORLD_SIZE" in os.environ:
    import torch
    import torch.distributed as dist

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
t0 = time.perf_counter()
y_all, mine = parallel.solve_batch_distributed(problems, grid)
t1 = time.perf_counter()
if int(os.environ.get("RANK", "0")) == 0:
    print(f"{T} trajectories x {grid.n_steps} steps in {t1 - t0:.2f} s; "
          f"y_N(alpha=0.9) = {y_all[0]}, y_N(alpha->1) = {y_all[-1]}, finite: {bool(np.isfinite(y_all).all())}")
if "WORLD_SIZE" in os.environ:
    dist.destroy_process_group()
