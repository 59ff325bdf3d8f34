"""CPU restatement of the reference's trajectory CSV writer — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, as the checker; the product path (paper_1611_08678_b200.output)
formats on the GPU and never calls it.

Restates ``write_trajectory_csv`` (reference cli.py:97-105) line for line:
header ``t,y0,..,y{d-1}``, then per row ``f"{t:.17g}"`` followed by
``f"{v:.17g}"`` for every state component, comma separated, "\\n" line ends.
The formatting is CPython's own (dtoa, correctly rounded), so this oracle is
pinned by construction; tests/test_oracle.py also checks it byte for byte
against CSVs the reference itself wrote (tests/golden/csv_*.csv.gz, made by
oracle/make_golden_csv.py).
"""

from __future__ import annotations

import io

import numpy as np


def format_csv(states, t) -> bytes:
    """The bytes write_trajectory_csv(path, traj) writes for traj.states / traj.t."""
    states = np.asarray(states)
    d = states.shape[1]
    out = io.StringIO(newline="\n")
    out.write("t," + ",".join(f"y{i}" for i in range(d)) + "\n")  # cli.py:101
    for row in range(len(t)):  # cli.py:102-104
        vals = ",".join(f"{v:.17g}" for v in states[row])
        out.write(f"{t[row]:.17g},{vals}\n")
    return out.getvalue().encode("utf-8")


def format_rows(states, t, rows) -> list[bytes]:
    """Selected data lines (no newline), for size-independent spot checks."""
    states = np.asarray(states)
    return [(f"{t[r]:.17g}," + ",".join(f"{v:.17g}" for v in states[r])).encode() for r in rows]


def write_trajectory_csv(path, traj) -> None:
    with open(path, "wb") as fh:
        fh.write(format_csv(traj.states, traj.t))
