"""Multi-process host logic of the sharded sweep (gloo, world_size 2, CPU)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1611_08678_b200.parallel import gather_rows, shard_bounds


def test_shard_bounds_cover_exactly_once():
    for count in (1, 5, 4096, 4097):
        for world in (1, 2, 3, 8):
            if world > count:
                continue
            spans = [shard_bounds(count, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1611_08678_b200.parallel import solve_batch_distributed

        class FakeResult:
            def __init__(self, y):
                self.y_last = y

        def fake_solver(problems, grid, **kw):
            # a stand-in for solve_batch_gpu: y_N = (alpha, index) per member
            return FakeResult(np.array([[p[0], p[1]] for p in problems], dtype=np.float64))

        problems = [(0.9 + 0.1 * i / 7, float(i)) for i in range(7)]
        y_all, _ = solve_batch_distributed(problems, None, solver=fake_solver)
        q.put((rank, y_all.tolist()))
    finally:
        dist.destroy_process_group()


def test_sharded_sweep_gathers_in_order_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [[0.9 + 0.1 * i / 7, float(i)] for i in range(7)]
    for rank in (0, 1):
        np.testing.assert_allclose(results[rank], want)


def test_gather_rows_single_process_identity():
    a = np.arange(6.0).reshape(3, 2)
    assert np.array_equal(gather_rows(a, 3, 1, 0), a)
