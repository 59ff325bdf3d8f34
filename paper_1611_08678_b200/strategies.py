"""The reference's parallel strategy entry points on the device engine.

``fodeabm.parallel`` exposes ``solve_block_parallel`` (parallel/block.py:
44-236: P forked workers own contiguous step blocks and push per-step partial
sums to the owner) and ``solve_reduction_parallel`` (parallel/reduction.py:
139-355: chunked history reductions over P processes), plus the partition
model ``make_partition`` (parallel/partition.py:54-74).  Both solvers are
"equivalent to solve_serial" with the reference's weight table.  Here they
keep their signatures, argument validation and ``stats`` keys so callers of
the reference switch unchanged, and run on the one-launch GPU engine, which
supersedes both decompositions: the bulk Toeplitz tiles play
the senders' partial sums, the stepper the owner.  ``n_workers`` and
``chunk`` are validated as in the reference; the worker counters in
``stats`` are None (no host workers exist: "not applicable") and the
engine's own counters are added.
"""

from __future__ import annotations

from dataclasses import dataclass


from .solver import solve_gpu

__all__ = ["PartitionPlan", "make_partition", "owner", "idle_fraction", "solve_block_parallel",
           "solve_reduction_parallel"]

DEFAULT_WATCHDOG_S = 60.0  # parallel/_shm.py:35


@dataclass(frozen=True)
class PartitionPlan:
    """Contiguous step blocks of ceil(N/P) steps (parallel/partition.py:20-51)."""

    n_steps: int
    n_workers: int
    block_size: int
    blocks: tuple


def make_partition(n_steps: int, n_workers: int) -> PartitionPlan:
    """Split N steps into P contiguous blocks of ceil(N/P) steps (partition.py:54-74)."""
    n_steps = int(n_steps)
    n_workers = int(n_workers)
    if n_steps < 1:
        raise ValueError("n_steps must be >= 1")
    if n_workers < 1:
        raise ValueError("n_workers must be >= 1")
    if n_workers > n_steps:
        raise ValueError(f"n_workers={n_workers} exceeds n_steps={n_steps}; each worker needs at least one step")
    block = -(-n_steps // n_workers)
    blocks = tuple((min(p * block, n_steps), min((p + 1) * block, n_steps)) for p in range(n_workers))
    return PartitionPlan(n_steps=n_steps, n_workers=n_workers, block_size=block, blocks=blocks)


def owner(plan: PartitionPlan, n: int) -> int:
    """Index of the worker whose block contains step n (partition.py:76-80)."""
    if not 0 <= n < plan.n_steps:
        raise IndexError(f"step index {n} outside [0, {plan.n_steps})")
    return min(n // plan.block_size, plan.n_workers - 1)


def idle_fraction(plan: PartitionPlan, worker: int) -> float:
    """Fraction of steps before the iteration reaches a worker's block (partition.py:83-93)."""
    if not 0 <= worker < plan.n_workers:
        raise IndexError(f"worker index {worker} outside [0, {plan.n_workers})")
    return min(worker * plan.block_size, plan.n_steps) / plan.n_steps


def _not_applicable(stats: dict) -> None:
    # the reference's per-worker counters (block.py:230-231, reduction.py:
    # 348-349) describe host workers that do not exist here: present, None
    # ("not applicable"), with the engine's own counters beside them
    stats["idle_steps"] = None
    stats["partial_sums_sent"] = None
    stats["worker_counters"] = ("not applicable: no host workers; the engine reports bulk_tiles, "
                                "bulk_claims, leader_wait_ns instead")


def _check_grid(problem, grid):
    N = grid.n_steps
    if not grid.spans(problem.t_end):
        raise ValueError(f"grid (h={grid.h!r}, N={N}) does not span t_end={problem.t_end!r}")


def solve_block_parallel(problem, grid, n_workers: int, *, watchdog_s: float = DEFAULT_WATCHDOG_S,
                         stats: dict | None = None, device: int = 0):
    """Drop-in for ``fodeabm.solve_block_parallel`` (block.py:44-236) on the GPU."""
    _check_grid(problem, grid)
    plan = make_partition(grid.n_steps, n_workers)
    eng: dict = {}
    traj = solve_gpu(problem, grid, weights="reference", device=device, timeout_s=watchdog_s, stats=eng)
    if stats is not None:
        stats.update(eng)
        _not_applicable(stats)
        stats["plan"] = plan
    return traj


def solve_reduction_parallel(problem, grid, n_workers: int, chunk: int = 1024, *,
                             watchdog_s: float = DEFAULT_WATCHDOG_S, stats: dict | None = None, device: int = 0):
    """Drop-in for ``fodeabm.solve_reduction_parallel`` (reduction.py:139-355) on the GPU."""
    _check_grid(problem, grid)
    N = grid.n_steps
    n_workers = int(n_workers)
    if not 1 <= n_workers <= N:
        raise ValueError(f"n_workers must lie in [1, {N}], got {n_workers}")
    chunk = int(chunk)
    if chunk < 1:
        raise ValueError(f"chunk must be >= 1, got {chunk}")
    eng: dict = {}
    traj = solve_gpu(problem, grid, weights="reference", device=device, timeout_s=watchdog_s, stats=eng)
    if stats is not None:
        stats.update(eng)
        _not_applicable(stats)
        stats["chunk"] = chunk
    return traj
