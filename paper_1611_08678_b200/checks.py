"""The reference's ``fodeabm.checks`` names (checks.py:1-177) on the GPU:
the verification suite of :mod:`paper_1611_08678_b200.verify` under the
module name the reference uses."""

from .verify import (  # noqa: F401
    EQUIV_TOL,
    ML_TOL,
    ORDER_SLACK,
    ROUNDOFF_FLOOR,
    TERMINAL_TOL,
    CheckResult,
    check_constant_forcing,
    check_linear_mittag_leffler,
    check_power_law_orders,
    check_strategy_equivalence,
    convergence_sweep,
    run_verification_suite,
)

__all__ = ["CheckResult", "check_power_law_orders", "check_constant_forcing", "check_linear_mittag_leffler",
           "check_strategy_equivalence", "convergence_sweep", "run_verification_suite"]
