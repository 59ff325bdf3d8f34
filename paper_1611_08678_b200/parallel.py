"""Multi-GPU plumbing: one process per GPU over torch.distributed (NCCL on the
B200 box, gloo for the CPU tests).

Two sharded paths:

* the batched sweep (BASELINE config 4): trajectories are independent, so each
  rank integrates a contiguous slice with no data-path collective, and the
  final states are all-gathered once (:func:`solve_batch_distributed`);
* one long trajectory (config 5, :func:`solve_sharded`): every rank hosts
  bulk agents of the same engine; rank 0 also runs the stepper.  The ranks
  exchange CUDA IPC handles of their shard arenas once, then the kernels talk
  over NVLink (f rows out of rank 0, finished target-block sums into rank 0).
  This replaces the reference's block-partitioned ParallelABM
  (parallel/block.py:44-236), whose lower workers send per-step partial sums
  to the owner: here the history of each target block is cut into fixed
  segments whose partial sums any GPU may compute, and rank 0 adds them once
  per target block in a fixed order -- one reduction per future block, not
  per step -- so the result is bitwise equal to the single-GPU solve.
"""

from __future__ import annotations

import os

import numpy as np

# the reference's fodeabm.parallel names (parallel/__init__.py), on the engine
from .strategies import (  # noqa: E402,F401
    PartitionPlan,
    idle_fraction,
    make_partition,
    owner,
    solve_block_parallel,
    solve_reduction_parallel,
)

__all__ = ["shard_bounds", "gather_rows", "solve_batch_distributed", "solve_sharded", "PartitionPlan",
           "make_partition", "owner", "idle_fraction", "solve_block_parallel", "solve_reduction_parallel"]


def shard_bounds(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of `count` items for `rank`; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    q, r = divmod(int(count), int(world))
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def gather_rows(local: np.ndarray, count: int, world: int, rank: int, group=None) -> np.ndarray:
    """All-gather the per-rank row blocks of a (count, ...) array in rank order."""
    local = np.ascontiguousarray(local)
    if world <= 1:
        return local
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    tail = local.shape[1:]
    sizes = [shard_bounds(count, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros((width, *tail), dtype=torch.float64, device=device)
    buf[: local.shape[0]] = torch.from_numpy(local).to(device)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    parts = [out[r][: hi - lo].cpu().numpy() for r, (lo, hi) in enumerate(sizes)]
    return np.concatenate(parts, axis=0)


def solve_batch_distributed(problems, grid, *, solver=None, device: int | None = None, group=None):
    """Shard a sweep over the ranks of the default process group.

    Returns (y_last of the whole sweep on every rank, this rank's BatchResult
    or None for an empty slice).  `solver` defaults to
    :func:`paper_1611_08678_b200.solve_batch_gpu`.  Collective: every rank
    reaches the gather even when its own slice is empty or its solve fails;
    a failure anywhere raises the same exception on every rank (the lowest
    failing trajectory of the sweep for a non-finite rhs, with its global
    ``index``), so no rank is left blocked in the collective.
    """
    import torch.distributed as dist

    if solver is None:
        from .solver import solve_batch_gpu as solver
    problems = list(problems)
    if not problems:
        raise ValueError("solve_batch_distributed needs at least one problem")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(len(problems), world, rank)
    kwargs = {"states": False, "raise_on_error": False}
    if device is None and "LOCAL_RANK" in os.environ:
        device = int(os.environ["LOCAL_RANK"])  # one process per GPU (torchrun)
    if device is not None:
        kwargs["device"] = device
    res, err = None, None
    d = int(problems[0].dim)
    local = np.zeros((hi - lo, d))
    if hi > lo:
        try:
            res = solver(problems[lo:hi], grid, **kwargs)
            local = np.asarray(res.y_last, dtype=np.float64).reshape(hi - lo, d)
            if getattr(res, "error", None) is not None:
                idx, exc = res.error
                exc.index = lo + int(idx)
                err = exc
        except Exception as exc:  # keep the collective sequence aligned across ranks
            err = exc
    rec = _error_record(err)
    if rec is not None and rec[0] == "step":
        rec = rec + (getattr(err, "index", None),)
    if world > 1:
        records = [None] * world
        dist.all_gather_object(records, rec, group=group)
    else:
        records = [rec]
    bad = [(r, x) for r, x in enumerate(records) if x is not None]
    if bad:
        # the lowest failing trajectory of the sweep (ranks hold ascending slices)
        r, x = bad[0]
        if x[0] == "step":
            exc = _raise_record_exc(x[:4], r)
            exc.index = x[4]
            raise exc
        _raise_record(x[:4], r)
    return gather_rows(local, len(problems), world, rank, group), res


def _error_record(exc):
    """A picklable summary of a solve error (exceptions with keyword-only
    state do not survive all_gather_object)."""
    from .core import SolverStepError, StrategyTimeoutError

    if exc is None:
        return None
    if isinstance(exc, SolverStepError):
        return ("step", str(exc), exc.step, exc.t)
    if isinstance(exc, StrategyTimeoutError):
        return ("timeout", str(exc), None, None)
    if isinstance(exc, ValueError):
        return ("value", str(exc), None, None)
    return ("runtime", f"{type(exc).__name__}: {exc}", None, None)


def _raise_record_exc(rec, rank):
    from .core import SolverStepError, StrategyTimeoutError

    kind, msg, step, t = rec
    if kind == "step":
        return SolverStepError("rhs returned a non-finite value", step=step, t=t)
    if kind == "timeout":
        return StrategyTimeoutError(f"rank {rank}: {msg}")
    if kind == "value":
        return ValueError(msg)
    return RuntimeError(f"rank {rank}: {msg}")


def _raise_record(rec, rank):
    raise _raise_record_exc(rec, rank)


def first_error(records):
    """The error every rank raises after a sharded solve: the stepper's (rank
    0) unless it was only the echo of a peer's abort, else the lowest rank's."""
    recs = [(r, rec) for r, rec in enumerate(records) if rec is not None]
    if not recs:
        return None
    for r, rec in recs:
        if "aborted by a peer shard" not in rec[1]:
            return r, rec
    return recs[0]


def solve_sharded(problem, grid, *, weights="accurate", device: int | None = None, timeout_s: float | None = None,
                  group=None, plan_cls=None, stats: dict | None = None):
    """Integrate ONE trajectory with its history sharded over the ranks of
    ``group`` (one process per GPU).  Collective: every rank calls it with the
    same problem and grid.  Rank 0 returns the :class:`Trajectory`, the others
    ``None``; an error on any rank raises the same exception on every rank.
    """
    import os

    import torch.distributed as dist

    from .solver import DEFAULT_TIMEOUT_S, GpuPlan, solve_gpu

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    timeout_s = DEFAULT_TIMEOUT_S if timeout_s is None else timeout_s
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank))
    if world == 1 and plan_cls is None:
        return solve_gpu(problem, grid, weights=weights, device=device, timeout_s=timeout_s, stats=stats)
    if plan_cls is None:
        plan_cls = GpuPlan
    if not grid.spans(problem.t_end):
        raise ValueError(f"grid (h={grid.h!r}, N={grid.n_steps}) does not span t_end={problem.t_end!r}")
    problem.eval_rhs0()
    err = None
    plan = None
    try:
        plan = plan_cls(problem, grid, weights=weights, device=device)
        plan.set_y0(problem.y0)
        handle = plan.ipc_handle()
    except Exception as exc:  # keep the collective sequence aligned across ranks
        err, handle = exc, None
    handles = [None] * world
    dist.all_gather_object(handles, handle, group=group)
    if err is None and any(h is None for h in handles):
        err = RuntimeError("a peer rank failed to create its shard")
    if err is None:
        try:
            plan.attach_shards(world, rank, b"".join(handles))
            plan.reset()
        except Exception as exc:
            err = exc
    oks = [None] * world
    dist.all_gather_object(oks, err is None, group=group)  # doubles as the pre-launch barrier
    if err is None and not all(oks):
        err = RuntimeError("a peer rank failed to attach its shard")
    if err is None:
        try:
            plan.run(timeout_s)
            if stats is not None:
                stats.update(plan.stats())  # this rank's engine counters (kernel_ms: its own launch)
        except Exception as exc:
            err = exc
    records = [None] * world
    dist.all_gather_object(records, _error_record(err), group=group)
    picked = first_error(records)
    traj = None
    if picked is None and rank == 0:
        traj = plan.download()
    # an arena must outlive the peers' mappings of it: detach, barrier, free
    if plan is not None:
        try:
            plan.detach_shards()
        except Exception:
            pass
    dist.barrier(group=group)
    if plan is not None:
        plan.close()
    if picked is not None:
        _raise_record(picked[1], picked[0])
    return traj
