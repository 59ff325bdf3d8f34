"""The sharded single-trajectory engine (BASELINE config 5) on one GPU.

Only one GPU is available to the tests, so the n-shard protocol runs in its
one-GPU emulation (``GpuPlan.set_virtual_shards``): every shard gets its own
f-history copy (filled by the stepper's fan-out writes), its own control
block (src_done released into it, abort propagated to it) and its own
accumulator scratch, and agent CTA b serves shard (b-1) % n.  The IPC
mapping layer between processes is exercised by tests/test_gpu_sharded_ipc.py
(two processes on one GPU) and its host protocol by
tests/test_parallel_host.py (gloo, world 2).

The bulk units (engine.cuh "units") and the fixed-order reduction of their
partials depend on the block index only, so the sharded result is bitwise
equal to the single-GPU one whichever shard computed a unit.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import normwise_dev
from oracle import abm_oracle

pytestmark = pytest.mark.gpu


def lorenz(fabm, N, h=1e-3):
    prob = fabm.FractionalProblem(alpha=0.99, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=N * h)
    return prob, fabm.GridSpec(n_steps=N, h=h)


def run_plan(fabm, prob, grid, shards):
    plan = fabm.GpuPlan(prob, grid)
    try:
        if shards > 1:
            plan.set_virtual_shards(shards)
        plan.run()
        return plan.download(), plan.stats()
    finally:
        plan.close()


@pytest.mark.parametrize("N", [3000, 40000, 200000, 2000000])
def test_virtual_shards_bitwise_equal_single(fabm, N):
    prob, grid = lorenz(fabm, N)
    ref, st1 = run_plan(fabm, prob, grid, 1)
    for shards in (2, 3, 8):
        got, st = run_plan(fabm, prob, grid, shards)
        assert np.array_equal(got.states, ref.states), shards
        assert np.array_equal(got.f_cache, ref.f_cache), shards
        assert st["bulk_tiles"] == st1["bulk_tiles"]


def test_virtual_shards_vs_oracle(fabm):
    prob, grid = lorenz(fabm, 20000)
    got, _ = run_plan(fabm, prob, grid, 4)
    w = abm_oracle.accurate_weights(prob.alpha, grid.n_steps)
    ref, _ = abm_oracle.solve_serial(prob.alpha, prob.y0, prob.rhs, grid.h, grid.n_steps, weights=w)
    # chaotic system: compare over the first 2000 steps (short horizon)
    assert normwise_dev(got.states[:2000], ref[:2000]) <= 1e-12


def test_virtual_shards_error_step(fabm):
    # y' = 60 y overflows after a few thousand steps: the failing step must be
    # the single-GPU (= reference) one
    prob = fabm.FractionalProblem(alpha=0.9, dim=1, rhs=fabm.rhs_linear(60.0), y0=[1.0], t_end=40.0)
    grid = prob.grid(40000)
    with pytest.raises(fabm.SolverStepError) as one:
        run_plan(fabm, prob, grid, 1)
    with pytest.raises(fabm.SolverStepError) as many:
        run_plan(fabm, prob, grid, 5)
    assert one.value.step > 1000
    assert (many.value.step, many.value.t) == (one.value.step, one.value.t)


def test_detach_restores_single_gpu_plan(fabm):
    prob, grid = lorenz(fabm, 5000)
    plan = fabm.GpuPlan(prob, grid)
    try:
        plan.run()
        a = plan.download().states
        plan.set_virtual_shards(3)
        plan.run()
        b = plan.download().states
        plan.detach_shards()
        plan.run()
        c = plan.download().states
    finally:
        plan.close()
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_virtual_shards_rejects_bad_counts(fabm):
    prob, grid = lorenz(fabm, 1000)
    plan = fabm.GpuPlan(prob, grid)
    try:
        for bad in (0, 9):
            with pytest.raises(ValueError):
                plan.set_virtual_shards(bad)
    finally:
        plan.close()
