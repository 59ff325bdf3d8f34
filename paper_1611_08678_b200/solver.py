"""GPU strategy: the drop-in replacement for ``fodeabm.serial.solve_serial``.

``solve_gpu(problem, grid)`` keeps the reference call (serial.py:114-176):
same arguments, same ``Trajectory`` result (fresh read-only host arrays),
same errors — ``ValueError`` for configuration problems, ``SolverStepError``
with the failing loop index and t=(n+1)h for non-finite rhs output,
``StrategyTimeoutError`` when the device watchdog fires.  The whole O(N^2)
loop runs in one cooperative kernel on the device (csrc/engine.cuh); the
host only validates, launches and copies the trajectory back.

Weights (the ``precompute_weights`` seam, serial.py:130):
  * ``"accurate"`` (default) — generated on the device, cancellation-free;
  * ``"formula"``  — generated on the device with the reference expression;
  * ``"reference"`` — this package's ``precompute_weights`` (bitwise equal
    to the reference table), uploaded; the 1e-12 parity mode;
  * any object with ``.b .a .c`` arrays of length >= N+1 (a ``WeightTable``).
"""

from __future__ import annotations

import ctypes
import math
import os
from collections import OrderedDict

import numpy as np

from . import _native as nat
from .core import GridSpec, SolverStepError, StrategyTimeoutError, Trajectory, precompute_weights
from .systems import device_system_of

__all__ = ["solve_gpu", "solve_batch_gpu", "BatchResult", "GpuPlan", "device_count", "measure_dfma_peak",
           "release_cached_memory", "STRATEGY_NAME"]

STRATEGY_NAME = "gpu"
# the reference watchdog default (_shm.py:35); FABM_TIMEOUT_S overrides it
DEFAULT_TIMEOUT_S = float(os.environ.get("FABM_TIMEOUT_S", "60"))


def device_count() -> int:
    return int(nat.load().fabm_device_count())


def measure_dfma_peak(device: int = 0) -> float:
    """Measured FP64 FMA/s of a DFMA-bound microbenchmark on ``device``."""
    return float(nat.load().fabm_measure_dfma_peak(int(device)))


def _raise_status(st: nat.Status, h: float | None = None):
    msg = st.message.decode(errors="replace")
    if st.code == nat.FABM_ERR_NONFINITE:
        if st.kind == 1:
            exc = SolverStepError("rhs returned a non-finite value", step=0, t=0.0)
        else:
            exc = SolverStepError("rhs returned a non-finite value", step=int(st.step), t=float(st.t))
        exc.kind = int(st.kind)
        raise exc
    if st.code == nat.FABM_ERR_TIMEOUT:
        raise StrategyTimeoutError(msg or "device watchdog expired")
    if st.code == nat.FABM_ERR_CONFIG:
        raise ValueError(msg)
    raise RuntimeError(f"libfabm error {st.code}: {msg}")


def _structs(problem, grid):
    tag = device_system_of(problem.rhs)
    dim = int(problem.dim)
    if tag.dim is not None and tag.dim != dim:
        raise ValueError(f"rhs {tag.name!r} has dimension {tag.dim}, problem has dim {dim}")
    if dim > nat.MAX_DIM:
        raise ValueError(f"the device engine supports dim <= {nat.MAX_DIM} for {tag.name!r} (solve_gpu splits "
                         f"the componentwise constant/linear systems of any dim), got {dim}")
    alpha = float(problem.alpha)
    pr = nat.Problem()
    pr.alpha = alpha
    pr.dim = dim
    pr.system = tag.system_id
    for i, v in enumerate(tag.params[: nat.MAX_PARAMS]):
        pr.params[i] = v
    y0 = np.asarray(problem.y0, dtype=np.float64).reshape(-1)
    for i in range(dim):
        pr.y0[i] = float(y0[i])
    gr = nat.Grid()
    gr.n_steps = int(grid.n_steps)
    gr.h = float(grid.h)
    # the scalars of serial.py:135-136 / core.py:146-147, computed by CPython
    gr.h_alpha = float(grid.h) ** alpha
    gr.gamma1 = math.gamma(alpha + 1.0)
    gr.gamma2 = math.gamma(alpha + 2.0)
    gr.inv_gamma2 = 1.0 / math.gamma(alpha + 2.0)
    return pr, gr, tag


def _weight_arrays(weights, alpha: float, n_steps: int):
    if isinstance(weights, str):
        if weights == "accurate":
            return nat.WEIGHTS_ACCURATE, None
        if weights == "formula":
            return nat.WEIGHTS_FORMULA, None
        if weights == "reference":
            table = precompute_weights(alpha, n_steps)
        else:
            raise ValueError(f"unknown weights mode {weights!r}")
    else:
        table = weights
    arrs = []
    for name in ("b", "a", "c"):
        arr = np.ascontiguousarray(np.asarray(getattr(table, name), dtype=np.float64))
        if arr.ndim != 1 or arr.shape[0] < n_steps + 1:
            raise ValueError(f"weight table {name!r} needs at least {n_steps + 1} entries")
        arrs.append(arr[: n_steps + 1].copy())
    return nat.WEIGHTS_HOST, arrs


def _weights_key(weights, alpha: float, n_steps: int):
    """Identity of the table ``weights`` resolves to, or None if unknown (a
    caller's table object may be mutated between calls: always re-upload)."""
    if not isinstance(weights, str):
        return None
    if weights == "reference":
        # the seam: a monkeypatched precompute_weights is a different table
        return ("reference", precompute_weights, alpha, n_steps)
    return (weights, alpha, n_steps)


class GpuPlan:
    """Device-resident buffers for one (problem, grid) on one GPU.

    Re-running a plan reuses the allocation and the device weight table;
    ``run()`` times the engine kernel with CUDA events on the plan stream.
    """

    def __init__(self, problem, grid, *, weights="accurate", device: int = 0):
        lib = nat.load()
        self.problem = problem
        self.grid = grid
        self.device = int(device)
        self._pr, self._gr, self.tag = _structs(problem, grid)
        st = nat.Status()
        handle = lib.fabm_plan_create(ctypes_ref(self._pr), ctypes_ref(self._gr), self.device, ctypes_ref(st))
        if not handle:
            _raise_status(st)
        self._h = handle
        self._lib = lib
        self.weights_mode = None
        self.set_weights(weights)

    # -- configuration -------------------------------------------------
    def set_weights(self, weights):
        # the device table only changes with its inputs: a plan re-used for the
        # same (mode or table source, alpha, N) keeps it (no host table, no
        # upload, no regeneration)
        key = _weights_key(weights, float(self.problem.alpha), int(self.grid.n_steps))
        if key is not None and key == getattr(self, "_weights_key", None):
            return
        self._weights_key = None
        mode, arrs = _weight_arrays(weights, float(self.problem.alpha), int(self.grid.n_steps))
        st = nat.Status()
        ptrs = [nat.dptr(a) for a in arrs] if arrs else [None, None, None]
        rc = self._lib.fabm_plan_set_weights(self._h, mode, *ptrs, ctypes_ref(st))
        if rc != nat.FABM_OK:
            _raise_status(st)
        self.weights_mode = weights if isinstance(weights, str) else "table"
        self._weights_key = key

    def set_y0(self, y0):
        y0 = np.ascontiguousarray(np.asarray(y0, dtype=np.float64).reshape(-1))
        st = nat.Status()
        if self._lib.fabm_plan_set_y0(self._h, nat.dptr(y0), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    def set_bulk_ctas(self, n_ctas: int | None):
        """Cap the CTAs that run bulk agents (None: one per SM besides the
        stepper).  The result does not depend on it: the bulk units and the
        reduction order are fixed by n_steps."""
        st = nat.Status()
        if self._lib.fabm_plan_set_bulk_ctas(self._h, int(n_ctas or 0), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    # -- sharding (config 5) ------------------------------
    def ipc_handle(self) -> bytes:
        """CUDA IPC handle of this plan's shard arena (exchanged between ranks)."""
        buf = ctypes.create_string_buffer(nat.IPC_HANDLE_BYTES)
        st = nat.Status()
        if self._lib.fabm_plan_ipc_handle(self._h, buf, ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)
        return buf.raw

    def attach_shards(self, n_shards: int, rank: int, handles: bytes):
        """Map the arenas of all ranks (handles in rank order, IPC_HANDLE_BYTES each)."""
        if len(handles) != n_shards * nat.IPC_HANDLE_BYTES:
            raise ValueError(f"expected {n_shards} IPC handles")
        st = nat.Status()
        if self._lib.fabm_plan_attach_shards(self._h, int(n_shards), int(rank), handles, ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    def set_virtual_shards(self, n_shards: int):
        """Emulate an n-shard run on this one GPU (same protocol, local buffers)."""
        st = nat.Status()
        if self._lib.fabm_plan_set_virtual_shards(self._h, int(n_shards), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    def emulate_shards(self, on: bool = True):
        """Rank 0 of an attached plan: serve every shard from this one launch,
        through the peers' IPC mappings (the sharded protocol across processes
        where one GPU must host all ranks)."""
        st = nat.Status()
        if self._lib.fabm_plan_emulate_shards(self._h, int(bool(on)), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    def shard_counters(self) -> tuple[int, int]:
        """(src_done, bulk_tiles) of this plan's own control block."""
        a, b = ctypes.c_int64(0), ctypes.c_int64(0)
        st = nat.Status()
        if self._lib.fabm_plan_shard_counters(self._h, ctypes.byref(a), ctypes.byref(b), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)
        return int(a.value), int(b.value)

    def detach_shards(self):
        """Close the peer mappings and return to a single-GPU plan."""
        st = nat.Status()
        if self._lib.fabm_plan_detach_shards(self._h, ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    def reset(self):
        """Zero the run flags (sharded plans: on every rank, before the barrier)."""
        st = nat.Status()
        if self._lib.fabm_plan_reset(self._h, ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)

    # -- execution -----------------------------------------------------
    def run(self, timeout_s: float = DEFAULT_TIMEOUT_S) -> float:
        """Run the engine; returns the kernel time in ms (CUDA events)."""
        st = nat.Status()
        if self._lib.fabm_plan_run(self._h, float(timeout_s), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st, self.grid.h)
        return self.stats()["kernel_ms"]

    def set_host_output(self, states: np.ndarray | None, f_cache: np.ndarray | None):
        """Stream the next run's trajectory into these mapped pinned arrays (None: off)."""
        st = nat.Status()
        rc = self._lib.fabm_plan_set_host_output(self._h, nat.dptr(states), nat.dptr(f_cache), ctypes_ref(st))
        if rc != nat.FABM_OK:
            _raise_status(st)

    def run_to_host(self, timeout_s: float = DEFAULT_TIMEOUT_S) -> Trajectory:
        """Run with the trajectory streamed to fresh pinned host arrays during the
        kernel (no D2H afterwards); falls back to run() + download() if pinned
        memory is unavailable."""
        N, d = int(self.grid.n_steps), int(self.problem.dim)
        states = _PINNED.array(N + 1, d)
        f_cache = _PINNED.array(N + 1, d) if states is not None else None
        if f_cache is None:
            self.run(timeout_s)
            return self.download()
        self.set_host_output(states, f_cache)
        try:
            self.run(timeout_s)
        finally:
            self.set_host_output(None, None)
        grid = self.grid if isinstance(self.grid, GridSpec) else GridSpec(self.grid.n_steps, self.grid.h)
        return Trajectory(grid=grid, states=states, f_cache=f_cache)

    def download(self) -> Trajectory:
        N, d = int(self.grid.n_steps), int(self.problem.dim)
        states = np.empty((N + 1, d))
        f_cache = np.empty((N + 1, d))
        st = nat.Status()
        if self._lib.fabm_plan_download(self._h, nat.dptr(states), nat.dptr(f_cache), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)
        grid = self.grid if isinstance(self.grid, GridSpec) else GridSpec(self.grid.n_steps, self.grid.h)
        return Trajectory(grid=grid, states=states, f_cache=f_cache)

    def last_state(self) -> np.ndarray:
        out = np.empty(int(self.problem.dim))
        st = nat.Status()
        if self._lib.fabm_plan_download_last(self._h, nat.dptr(out), ctypes_ref(st)) != nat.FABM_OK:
            _raise_status(st)
        return out

    def write_csv(self, path, *, stats: dict | None = None) -> None:
        """The last run's trajectory as the reference CSV (cli.py:97-105), formatted on the device."""
        from .output import plan_write_csv

        plan_write_csv(self, path, stats=stats)

    def stats(self) -> dict:
        s = nat.Stats()
        self._lib.fabm_plan_stats(self._h, ctypes_ref(s))
        return s.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fabm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _PinnedPool:
    """Mapped pinned host buffers that the engine streams a trajectory into
    during the run (``fabm_plan_set_host_output``), so ``solve_gpu`` needs no
    D2H copy after the kernel.  Each solve takes fresh buffers; a buffer
    returns to the pool when every array viewing it has been garbage
    collected, so a returned ``Trajectory`` owns its memory as in the
    reference (serial.py:55-56)."""

    def __init__(self, keep_bytes: int = 1 << 31):
        import collections
        import threading

        self.keep_bytes = keep_bytes
        self.free: dict[int, list[int]] = {}
        self.kept = 0
        self.lock = threading.Lock()
        # buffers handed back by finalizers.  A finalizer runs whenever the
        # garbage collector does -- possibly inside take() on this thread,
        # with the lock held -- so it only appends here (atomic, no lock);
        # take() and drain() move the entries into the free lists.
        self.returned: "collections.deque[tuple[int, int]]" = collections.deque()

    def _drain_locked(self) -> list[int]:
        excess = []
        while self.returned:
            nbytes, ptr = self.returned.popleft()
            if self.kept + nbytes <= self.keep_bytes:
                self.free.setdefault(nbytes, []).append(ptr)
                self.kept += nbytes
            else:
                excess.append(ptr)
        return excess

    def take(self, nbytes: int) -> int | None:
        with self.lock:
            excess = self._drain_locked()
            lst = self.free.get(nbytes)
            ptr = lst.pop() if lst else None
            if ptr is not None:
                self.kept -= nbytes
        lib = nat.load()
        for p in excess:
            lib.fabm_host_free(p)
        if ptr is not None:
            return ptr
        ptr = lib.fabm_host_alloc(nbytes)
        return int(ptr) if ptr else None

    def give(self, nbytes: int, ptr: int):
        self.returned.append((nbytes, ptr))

    def drain(self) -> list[int]:
        """Empty the pool; returns the pointers for the caller to free."""
        with self.lock:
            excess = self._drain_locked()
            free, self.free, self.kept = self.free, {}, 0
        return excess + [p for ptrs in free.values() for p in ptrs]

    def array(self, rows: int, cols: int) -> np.ndarray | None:
        import weakref

        nbytes = 8 * rows * cols
        ptr = self.take(nbytes)
        if ptr is None:
            return None
        buf = (ctypes.c_double * (rows * cols)).from_address(ptr)
        weakref.finalize(buf, self.give, nbytes, ptr).atexit = False  # process exit releases pinned memory
        return np.ctypeslib.as_array(buf).reshape(rows, cols)


_PINNED = _PinnedPool()


def ctypes_ref(obj):
    import ctypes

    return ctypes.byref(obj)


_PLAN_CACHE: "OrderedDict[tuple, GpuPlan]" = OrderedDict()
_PLAN_CACHE_SIZE = 2


def _cached_plan(problem, grid, weights, device) -> GpuPlan:
    tag = device_system_of(problem.rhs)
    wkey = weights if isinstance(weights, str) else id(weights)
    key = (device, tag, int(problem.dim), float(problem.alpha), int(grid.n_steps), float(grid.h), wkey)
    plan = _PLAN_CACHE.get(key)
    if plan is not None and isinstance(weights, str):
        _PLAN_CACHE.move_to_end(key)
        plan.problem = problem
        plan.set_weights(weights)  # a no-op unless the table source changed (e.g. a patched seam)
        return plan
    plan = GpuPlan(problem, grid, weights=weights, device=device)
    if isinstance(weights, str):
        _PLAN_CACHE[key] = plan
        while len(_PLAN_CACHE) > _PLAN_CACHE_SIZE:
            _PLAN_CACHE.popitem(last=False)[1].close()
    return plan


def release_cached_memory(device: int | None = None) -> None:
    """Free what the solvers keep between calls: the cached plans (device
    buffers of the last problem sizes), the pooled pinned output buffers
    (trajectories still alive keep theirs) and the device memory pool the
    batch solver allocates from (on ``device``, default: every device)."""
    while _PLAN_CACHE:
        _PLAN_CACHE.popitem(last=False)[1].close()
    lib = nat.load()
    for ptr in _PINNED.drain():
        lib.fabm_host_free(ptr)
    for dev in ([device] if device is not None else range(int(lib.fabm_device_count()))):
        lib.fabm_trim_memory(int(dev))


def solve_gpu(
    problem,
    grid,
    *,
    weights="accurate",
    device: int = 0,
    timeout_s: float = DEFAULT_TIMEOUT_S,
    stats: dict | None = None,
) -> Trajectory:
    """Integrate ``problem`` over ``grid`` on the GPU (drop-in for solve_serial).

    Deterministic: identical inputs give bitwise-identical trajectories.
    """
    N = int(grid.n_steps)
    if not grid.spans(problem.t_end):
        raise ValueError(f"grid (h={grid.h!r}, N={N}) does not span t_end={problem.t_end!r}")
    tag = device_system_of(problem.rhs)
    # shape and finiteness of f(0, y0), exactly as the reference validates it
    problem.eval_rhs0()
    if int(problem.dim) > nat.MAX_DIM and tag.name in COMPONENTWISE:
        return _solve_by_components(problem, grid, tag, weights=weights, device=device, timeout_s=timeout_s,
                                    stats=stats)
    plan = _cached_plan(problem, grid, weights, device)
    plan.set_y0(problem.y0)
    traj = plan.run_to_host(timeout_s)
    if stats is not None:
        stats.update(plan.stats())
        stats["strategy"] = STRATEGY_NAME
    return traj


# systems whose components evolve independently: f_i depends on y_i only
# (constant: f = value, systems.py:26-36; linear: f = lam * y, :64-73)
COMPONENTWISE = ("constant", "linear")


def _component_problem(problem, tag, lo: int, hi: int):
    from .core import FractionalProblem
    from .systems import rhs_constant, rhs_linear

    rhs = rhs_constant(tag.params[lo:hi]) if tag.name == "constant" else rhs_linear(tag.params[0])
    return FractionalProblem(alpha=problem.alpha, dim=hi - lo, rhs=rhs, y0=problem.y0[lo:hi], t_end=problem.t_end)


def _solve_by_components(problem, grid, tag, **kw) -> Trajectory:
    """dim > MAX_DIM for a componentwise rhs: solve blocks of <= MAX_DIM
    components with the engine and join them.  Every component's arithmetic
    is independent of the others (history sums, assembly and rhs are all
    per component), so this is the d-dimensional solve; a non-finite value
    raises at the earliest failing step over all blocks, as the reference's
    whole-vector check does (serial.py:157,167)."""
    dim = int(problem.dim)
    stats = kw.pop("stats", None)
    states, f_cache, first = [], [], None
    kernel_ms = 0.0
    for lo in range(0, dim, nat.MAX_DIM):
        hi = min(dim, lo + nat.MAX_DIM)
        sub = {}
        try:
            tr = solve_gpu(_component_problem(problem, tag, lo, hi), grid, stats=sub, **kw)
        except SolverStepError as exc:
            key = (exc.step, getattr(exc, "kind", 3))
            if first is None or key < (first.step, getattr(first, "kind", 3)):
                first = exc
            continue
        kernel_ms += sub.get("kernel_ms", 0.0)
        states.append(tr.states)
        f_cache.append(tr.f_cache)
    if first is not None:
        raise first
    if stats is not None:
        stats.update(kernel_ms=kernel_ms, strategy=STRATEGY_NAME, component_blocks=len(states))
    g = grid if isinstance(grid, GridSpec) else GridSpec(grid.n_steps, grid.h)
    return Trajectory(grid=g, states=np.concatenate(states, axis=1), f_cache=np.concatenate(f_cache, axis=1))


class BatchResult:
    """Outputs of :func:`solve_batch_gpu` (trajectory-major arrays, read-only)."""

    def __init__(self, grid, states, f_cache, y_last, kernel_ms, error):
        self.grid = grid
        self.states = states
        self.f_cache = f_cache
        self.y_last = y_last
        self.kernel_ms = kernel_ms
        self.error = error  # None or (index, SolverStepError)
        for arr in (states, f_cache, y_last):
            if arr is not None:
                arr.setflags(write=False)

    def trajectory(self, i: int) -> Trajectory:
        if self.states is None or self.f_cache is None:
            raise ValueError("solve_batch_gpu was called without states/f_cache")
        return Trajectory(grid=self.grid, states=self.states[i].copy(), f_cache=self.f_cache[i].copy())


def solve_batch_gpu(
    problems,
    grid,
    *,
    states: bool = True,
    f_cache: bool = False,
    device: int = 0,
    raise_on_error: bool = True,
) -> BatchResult:
    """Integrate many independent problems on one GPU (BASELINE config 4).

    Equivalent to ``[solve_serial(p, grid) for p in problems]`` (serial.py:
    114-176) with device-generated ACCURATE weights per problem.  All
    problems must share the rhs system, dim, horizon and grid; alpha, y0 and
    the rhs parameters may differ.  A non-finite rhs stops only its own
    trajectory; with ``raise_on_error`` the lowest failing index is raised as
    :class:`SolverStepError` (its ``index`` attribute names the trajectory).
    """
    problems = list(problems)
    if not problems:
        raise ValueError("solve_batch_gpu needs at least one problem")
    N = int(grid.n_steps)
    for p in problems:
        if not grid.spans(p.t_end):
            raise ValueError(f"grid (h={grid.h!r}, N={N}) does not span t_end={p.t_end!r}")
    structs = [_structs(p, grid) for p in problems]
    d = int(problems[0].dim)
    T = len(problems)
    probs = (nat.Problem * T)(*[s[0] for s in structs])
    grids = (nat.Grid * T)(*[s[1] for s in structs])
    st_arr = np.empty((T, N + 1, d)) if states else None
    fc_arr = np.empty((T, N + 1, d)) if f_cache else None
    y_last = np.empty((T, d))
    ms = ctypes_double()
    st = nat.Status()
    rc = nat.load().fabm_solve_batch(probs, grids, T, int(device), nat.dptr(st_arr), nat.dptr(fc_arr),
                                     nat.dptr(y_last), ctypes_ptr(ms), ctypes_ref(st))
    error = None
    if rc == nat.FABM_ERR_NONFINITE:
        t = float(st.t)
        exc = SolverStepError(f"trajectory {st.index}: rhs returned a non-finite value", step=int(st.step), t=t)
        exc.index = int(st.index)
        if raise_on_error:
            raise exc
        error = (int(st.index), exc)
    elif rc != nat.FABM_OK:
        _raise_status(st)
    g = grid if isinstance(grid, GridSpec) else GridSpec(grid.n_steps, grid.h)
    return BatchResult(g, st_arr, fc_arr, y_last, float(ms.value), error)


def ctypes_double():
    import ctypes

    return ctypes.c_double(0.0)


def ctypes_ptr(obj):
    import ctypes

    return ctypes.pointer(obj)
