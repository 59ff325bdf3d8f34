"""Multi-GPU plumbing: one process per GPU over torch.distributed (NCCL on the
B200 box, gloo for the CPU tests).

Only the batched sweep shards (BASELINE config 4): trajectories are
independent, so each rank integrates a contiguous slice with no data-path
collective, and the final states are all-gathered once.  The single headline
trajectory does not shard in this round (replicas only).
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_bounds", "gather_rows", "solve_batch_distributed"]


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

    Returns (y_last of the whole sweep on every rank, this rank's BatchResult).
    `solver` defaults to :func:`paper_1611_08678_b200.solve_batch_gpu`.
    """
    import torch.distributed as dist

    if solver is None:
        from .solver import solve_batch_gpu as solver
    problems = list(problems)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(len(problems), world, rank)
    kwargs = {"states": False}
    if device is not None:
        kwargs["device"] = device
    res = solver(problems[lo:hi], grid, **kwargs)
    return gather_rows(res.y_last, len(problems), world, rank, group), res
