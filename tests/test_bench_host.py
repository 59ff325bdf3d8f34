"""Host logic of bench.py on the CPU: the reference arm's prefix projection,
the sub-records' collective error handling (world 1 and a gloo world of 2),
and the reference arm's rank handling under torchrun."""

from __future__ import annotations

import os
import socket
import types

import pytest

import bench


class FakeClock:
    """time.perf_counter stand-in: each solve(M) advances it by a*M + c*M^2."""

    def __init__(self, a: float, c: float):
        self.a, self.c, self.t = a, c, 0.0

    def __call__(self) -> float:
        return self.t

    def solve(self, problem, grid):
        m = grid.n_steps
        self.t += self.a * m + self.c * m * m


def _fake_fodeabm():
    return types.SimpleNamespace(
        FractionalProblem=lambda **kw: types.SimpleNamespace(**kw),
        GridSpec=lambda n_steps, h: types.SimpleNamespace(n_steps=n_steps, h=h),
    )


def test_projection_recovers_the_quadratic_law(monkeypatch):
    clock = FakeClock(a=2e-6, c=3e-10)
    monkeypatch.setattr(bench.time, "perf_counter", clock)
    out = bench.project_reference(_fake_fodeabm(), clock.solve, (50_000, 100_000), 1_000_000)
    want = 2e-6 * 1e6 + 3e-10 * 1e12
    assert out["projected_seconds"] == pytest.approx(want, rel=1e-9)
    assert [m for m, _ in out["prefixes"]] == [50_000, 100_000]


def test_projection_falls_back_when_overheads_dominate(monkeypatch):
    # per-step cost falling with M (c < 0 in the two-point fit): a pure
    # quadratic through the longer prefix, never a negative time
    clock = FakeClock(a=1e-5, c=-1e-11)
    monkeypatch.setattr(bench.time, "perf_counter", clock)
    out = bench.project_reference(_fake_fodeabm(), clock.solve, (50_000, 100_000), 1_000_000)
    t2 = 1e-5 * 1e5 - 1e-11 * 1e10
    assert out["projected_seconds"] == pytest.approx(t2 / 1e10 * 1e12, rel=1e-9)
    assert out["projected_seconds"] > 0


def test_guarded_world_1():
    assert bench._guarded(1, lambda: {"value": 3}) == {"value": 3}

    def boom():
        raise RuntimeError("no device")

    assert bench._guarded(1, boom) == {"error": "RuntimeError: no device"}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _guarded_rank(rank, world, port, q):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def body():
        if rank == 1:
            raise ValueError("shard attach failed")
        return {"value": 1.0}

    q.put((rank, bench._guarded(world, body)))
    dist.barrier()
    dist.destroy_process_group()


def test_guarded_world_2_reports_the_error_on_every_rank():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_guarded_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == {"error": "ValueError: shard attach failed"}


def test_reference_arm_runs_on_rank_0_only(monkeypatch):
    called = []
    monkeypatch.setattr(bench, "reference_block_projection_clean", lambda n: called.append(n))
    monkeypatch.setattr(bench, "cpu_port_time", lambda *a, **k: called.append(a))
    args = types.SimpleNamespace(n=1_000_000, cpu_seconds=1.0, steps=1, warmup=0)
    assert bench.run_reference(args, world=2, rank=1) is None
    assert called == []


def test_default_invocation_is_one_gpu_and_valid_timing(monkeypatch):
    monkeypatch.setattr(bench.sys, "argv", ["bench.py"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    args = bench.parse()
    assert args.gpus == 1 and args.warmup >= 3 and args.steps >= 1
    assert args.impl != "reference"
    assert int(os.environ.get("WORLD_SIZE", "1")) == 1
