"""B200-native fractional Adams–Bashforth–Moulton history engine.

Drop-in GPU strategy for the hot path of ``fodeabm`` (arXiv 1611.08678): the
O(N^2) hereditary history sums of the PECE solver.  The public names mirror
``fodeabm/__init__.py:41-71`` for the solver path; ``solve_gpu`` replaces
``solve_serial`` and the rhs factories carry device tags.
"""

from .core import (
    FractionalProblem,
    GridSpec,
    SolverStepError,
    StrategyTimeoutError,
    Trajectory,
    WeightTable,
    corrector_weight_a,
    corrector_weight_c,
    gamma,
    precompute_weights,
    predictor_weight,
)
from .systems import (
    HR_DEFAULT_Y0,
    SYSTEM_NAMES,
    HindmarshRoseParams,
    rhs_chen,
    rhs_constant,
    rhs_financial,
    rhs_hindmarsh_rose,
    rhs_linear,
    rhs_lorenz,
    rhs_power_law,
    rhs_rossler,
)
from .output import format_trajectory_csv, write_trajectory_csv, write_trajectory_npz
from .steps import step_corrector, step_predictor
from .strategies import (
    PartitionPlan,
    idle_fraction,
    make_partition,
    owner,
    solve_block_parallel,
    solve_reduction_parallel,
)
from .verify import ConvergenceReport, exact_power_law, mittag_leffler, observed_order
from .solver import (
    BatchResult,
    GpuPlan,
    device_count,
    measure_dfma_peak,
    release_cached_memory,
    solve_batch_gpu,
    solve_gpu,
)

__version__ = "0.1.0"

__all__ = [
    "FractionalProblem",
    "GridSpec",
    "WeightTable",
    "Trajectory",
    "SolverStepError",
    "StrategyTimeoutError",
    "gamma",
    "predictor_weight",
    "corrector_weight_a",
    "corrector_weight_c",
    "precompute_weights",
    "solve_gpu",
    "solve_batch_gpu",
    "solve_block_parallel",
    "solve_reduction_parallel",
    "make_partition",
    "PartitionPlan",
    "owner",
    "idle_fraction",
    "step_predictor",
    "step_corrector",
    "ConvergenceReport",
    "mittag_leffler",
    "exact_power_law",
    "observed_order",
    "BatchResult",
    "GpuPlan",
    "device_count",
    "measure_dfma_peak",
    "release_cached_memory",
    "write_trajectory_csv",
    "format_trajectory_csv",
    "write_trajectory_npz",
    "HindmarshRoseParams",
    "HR_DEFAULT_Y0",
    "SYSTEM_NAMES",
    "rhs_constant",
    "rhs_power_law",
    "rhs_linear",
    "rhs_hindmarsh_rose",
    "rhs_lorenz",
    "rhs_chen",
    "rhs_rossler",
    "rhs_financial",
]
