"""Register the GPU engine as a strategy of the reference package itself.

``install()`` patches a loaded ``fodeabm`` in place so that its own harness
drives the B200 engine under the name ``"gpu"``:

* ``fodeabm.bench.STRATEGIES`` gains ``"gpu"`` (bench.py:26)
* ``fodeabm.bench._solve_once`` dispatches ``"gpu"`` to :func:`solve_gpu`
  (bench.py:43-51), so ``run_cell`` / ``run_sweep`` time it beside serial,
  block and reduction, with their bitwise repeat check (bench.py:80-87)
* ``fodeabm.cli.solve_with_strategy`` does the same (cli.py:86-94) and the
  ``--strategy`` flag accepts ``gpu`` (cli.py:171)
* ``fodeabm.cli.write_trajectory_csv`` (cli.py:97-105) is replaced by the
  device formatter (:func:`paper_1611_08678_b200.output.write_trajectory_csv`,
  byte-identical output), so ``fodeabm run`` writes its CSV from the GPU for
  every strategy
* ``fodeabm.checks.check_strategy_equivalence`` (checks.py:144-168) also
  checks ``gpu`` against ``solve_serial`` on its power-law problem, so
  ``fodeabm verify`` covers the GPU strategy with the reference's tolerance

Problems built with the reference's own rhs factories run unchanged (see
:func:`paper_1611_08678_b200.systems.adopt_reference_rhs`).  ``uninstall()``
restores the originals.
"""

from __future__ import annotations

import importlib

from .output import write_trajectory_csv
from .solver import STRATEGY_NAME, solve_gpu

__all__ = ["install", "uninstall"]

_SAVED: dict = {}


def install(weights="reference"):
    """Patch the imported ``fodeabm`` (bench and cli modules); returns it.

    ``weights="reference"`` (default): the ``gpu`` strategy integrates with
    the table of the reference's own seam ``fodeabm.serial.precompute_weights``
    (serial.py:24-31, 130), so it is a drop-in for ``solve_serial`` to the
    1e-12 contract -- and a table patched into that seam (as the reference's
    mutation tests do, pkg/tests/test_verify.py:143-180) reaches the GPU too.
    ``"accurate"`` opts into the cancellation-free device table (DESIGN.md
    §2), which differs from the reference's NumPy-pow table by up to ~4e-5
    relative in a_n at n = 1e6: trajectories then differ from
    ``solve_serial`` by more than 1e-12 at large N.
    """
    fodeabm = importlib.import_module("fodeabm")
    bench = importlib.import_module("fodeabm.bench")
    cli = importlib.import_module("fodeabm.cli")
    checks = importlib.import_module("fodeabm.checks")
    if _SAVED:
        return fodeabm
    _SAVED["STRATEGIES"] = bench.STRATEGIES
    _SAVED["_solve_once"] = bench._solve_once
    _SAVED["solve_with_strategy"] = cli.solve_with_strategy
    _SAVED["_build_parser"] = cli._build_parser
    _SAVED["write_trajectory_csv"] = cli.write_trajectory_csv
    _SAVED["check_strategy_equivalence"] = checks.check_strategy_equivalence
    orig_equiv = checks.check_strategy_equivalence
    orig_once = bench._solve_once
    orig_solve = cli.solve_with_strategy
    orig_parser = cli._build_parser

    serial = importlib.import_module("fodeabm.serial")

    stock = importlib.import_module("fodeabm.core").precompute_weights

    def _table(problem, n_steps):
        # the reference seam, looked up per call (it may be monkeypatched);
        # the stock function's table is bitwise this package's "reference"
        # mode (tests/test_oracle.py), which keeps the plan cache
        if weights == "reference" and serial.precompute_weights is not stock:
            return serial.precompute_weights(problem.alpha, n_steps)
        return weights

    def _solve_once(problem, strategy, n_steps, workers, chunk, stats=None):
        if strategy == STRATEGY_NAME:
            return solve_gpu(problem, problem.grid(n_steps), weights=_table(problem, n_steps), stats=stats)
        return orig_once(problem, strategy, n_steps, workers, chunk, stats)

    def solve_with_strategy(problem, cfg):
        if cfg.strategy == STRATEGY_NAME:
            return solve_gpu(problem, problem.grid(cfg.n_steps), weights=_table(problem, cfg.n_steps))
        return orig_solve(problem, cfg)

    def _build_parser():
        parser = orig_parser()
        for action in _walk_actions(parser):
            if action.dest == "strategy" and action.choices is not None and STRATEGY_NAME not in action.choices:
                action.choices = (*action.choices, STRATEGY_NAME)
        return parser

    def check_strategy_equivalence(n_steps=2048, n_workers=2, chunk=1024):
        out = orig_equiv(n_steps, n_workers, chunk)
        problem = checks._power_problem(0.5)
        grid = problem.grid(n_steps)
        ref = checks.solve_serial(problem, grid)
        dev = checks._sup_rel_dev(solve_gpu(problem, grid, weights=_table(problem, n_steps)), ref)
        out.append(checks.CheckResult(f"{STRATEGY_NAME} strategy", dev <= checks.EQUIV_TOL, f"sup rel dev {dev:.3e}"))
        return out

    bench.STRATEGIES = (*bench.STRATEGIES, STRATEGY_NAME)
    bench._solve_once = _solve_once
    cli.solve_with_strategy = solve_with_strategy
    cli._build_parser = _build_parser
    cli.write_trajectory_csv = write_trajectory_csv
    checks.check_strategy_equivalence = check_strategy_equivalence
    return fodeabm


def uninstall():
    if not _SAVED:
        return
    bench = importlib.import_module("fodeabm.bench")
    cli = importlib.import_module("fodeabm.cli")
    bench.STRATEGIES = _SAVED["STRATEGIES"]
    bench._solve_once = _SAVED["_solve_once"]
    cli.solve_with_strategy = _SAVED["solve_with_strategy"]
    cli._build_parser = _SAVED["_build_parser"]
    cli.write_trajectory_csv = _SAVED["write_trajectory_csv"]
    importlib.import_module("fodeabm.checks").check_strategy_equivalence = _SAVED["check_strategy_equivalence"]
    _SAVED.clear()


def _walk_actions(parser):
    import argparse

    for action in parser._actions:
        yield action
        if isinstance(action, argparse._SubParsersAction):
            for sub in action.choices.values():
                yield from _walk_actions(sub)
