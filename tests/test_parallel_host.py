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


class FakeProblem:
    def __init__(self, alpha, idx):
        self.alpha, self.idx, self.dim = alpha, idx, 2


class FakeResult:
    def __init__(self, y, error=None):
        self.y_last = y
        self.error = error


def _fake_solver(problems, grid, **kw):
    # a stand-in for solve_batch_gpu: y_N = (alpha, index) per member; the
    # member with idx == grid["fail"] has a non-finite rhs (raise_on_error
    # False: reported, not raised), idx == grid["crash"] raises outright
    from paper_1611_08678_b200.core import SolverStepError

    assert kw.get("raise_on_error") is False
    err = None
    for i, p in enumerate(problems):
        if grid and p.idx == grid.get("crash"):
            raise RuntimeError("device lost")
        if grid and p.idx == grid.get("fail") and err is None:
            err = (i, SolverStepError("rhs returned a non-finite value", step=17, t=0.018))
    return FakeResult(np.array([[p.alpha, p.idx] for p in problems], dtype=np.float64), err)


def _worker(rank, world, port, q, count, grid):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1611_08678_b200.parallel import solve_batch_distributed

        problems = [FakeProblem(0.9 + 0.1 * i / 7, float(i)) for i in range(count)]
        try:
            y_all, _ = solve_batch_distributed(problems, grid, solver=_fake_solver)
            q.put((rank, ("ok", y_all.tolist())))
        except Exception as exc:  # noqa: BLE001
            q.put((rank, ("raised", type(exc).__name__, getattr(exc, "step", None), getattr(exc, "index", None))))
    finally:
        dist.destroy_process_group()


def _run_world2(count, grid=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, count, grid)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def test_sharded_sweep_gathers_in_order_gloo():
    results = _run_world2(7)
    want = [[0.9 + 0.1 * i / 7, float(i)] for i in range(7)]
    for rank in (0, 1):
        assert results[rank][0] == "ok"
        np.testing.assert_allclose(results[rank][1], want)


def test_sharded_sweep_empty_slice_does_not_hang_gloo():
    # one trajectory over two ranks: rank 1's slice is empty
    results = _run_world2(1)
    for rank in (0, 1):
        assert results[rank] == ("ok", [[0.9, 0.0]])


def test_sharded_sweep_error_raised_on_every_rank_gloo():
    # member 5 (rank 1's slice) has a non-finite rhs: both ranks raise the
    # same SolverStepError, with the global index of the failing member
    results = _run_world2(7, {"fail": 5.0})
    for rank in (0, 1):
        assert results[rank] == ("raised", "SolverStepError", 17, 5)
    # a solver crash on rank 0 does not leave rank 1 blocked in the gather
    results = _run_world2(7, {"crash": 1.0})
    for rank in (0, 1):
        assert results[rank][:2] == ("raised", "RuntimeError")


def test_gather_rows_single_process_identity():
    a = np.arange(6.0).reshape(3, 2)
    assert np.array_equal(gather_rows(a, 3, 1, 0), a)


# ---------------------------------------------------------------- config 5
def _sharded_worker(rank, world, port, q, fail):
    """solve_sharded's collective sequence with a stand-in plan: the IPC
    handles reach every rank in rank order, every rank resets before the
    launch barrier, only rank 0 downloads, and an error on any rank raises
    the same exception everywhere."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    log = []
    try:
        import paper_1611_08678_b200 as fabm
        from paper_1611_08678_b200.parallel import solve_sharded

        class FakePlan:
            def __init__(self, problem, grid, *, weights, device):
                log.append(("create", device))
                self.grid = grid

            def set_y0(self, y0):
                log.append(("y0", list(y0)))

            def ipc_handle(self):
                return bytes([rank]) * 64

            def attach_shards(self, n, r, handles):
                log.append(("attach", n, r, [handles[64 * i] for i in range(n)]))

            def reset(self):
                log.append(("reset",))

            def run(self, timeout_s):
                log.append(("run",))
                if fail == "step" and rank == 0:
                    raise fabm.SolverStepError("rhs returned a non-finite value", step=3, t=0.2)
                if fail == "timeout" and rank == 1:
                    raise fabm.StrategyTimeoutError("device watchdog expired")
                if fail == "timeout" and rank == 0:
                    raise fabm.StrategyTimeoutError("aborted by a peer shard")

            def download(self):
                log.append(("download",))
                return "trajectory"

            def detach_shards(self):
                log.append(("detach",))

            def close(self):
                log.append(("close",))

        prob = fabm.FractionalProblem(alpha=0.8, dim=1, rhs=fabm.rhs_linear(-1.0), y0=[1.0], t_end=1.0)
        try:
            out = solve_sharded(prob, prob.grid(1000), plan_cls=FakePlan)
            q.put((rank, ("ok", out, log)))
        except Exception as exc:  # noqa: BLE001
            q.put((rank, (type(exc).__name__, getattr(exc, "step", None), log)))
    finally:
        dist.destroy_process_group()


def _run_sharded(fail):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, fail)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def test_solve_sharded_protocol_gloo():
    res = _run_sharded(None)
    for rank in (0, 1):
        tag, out, log = res[rank]
        assert tag == "ok"
        assert out == ("trajectory" if rank == 0 else None)
        names = [e[0] for e in log]
        assert names == ["create", "y0", "attach", "reset", "run"] + (["download"] if rank == 0 else []) + [
            "detach", "close"]
        assert log[0] == ("create", rank)
        assert log[2] == ("attach", 2, rank, [0, 1])  # handles in rank order


def test_solve_sharded_errors_agree_gloo():
    res = _run_sharded("step")
    for rank in (0, 1):
        assert res[rank][:2] == ("SolverStepError", 3)
        assert "download" not in [e[0] for e in res[rank][2]]
    # rank 0 only saw the echo of rank 1's watchdog: the peer's error wins
    res = _run_sharded("timeout")
    for rank in (0, 1):
        assert res[rank][0] == "StrategyTimeoutError"


def test_first_error_prefers_the_cause():
    from paper_1611_08678_b200.parallel import first_error

    assert first_error([None, None]) is None
    echo = ("timeout", "aborted by a peer shard", None, None)
    cause = ("timeout", "device watchdog expired", None, None)
    assert first_error([echo, cause]) == (1, cause)
    step = ("step", "x", 3, 0.2)
    assert first_error([step, echo]) == (0, step)
