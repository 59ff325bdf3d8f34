#!/bin/bash
# The engine's invariant-checked build (-DFABM_CHECKED: bounds of every unit,
# weight window and f row an agent touches; each unit computed by its
# claimant and finished exactly once; reduction counters in range; batch
# slot bounds and per-parity pull counts), then the seeded random sweeps and
# the headline-regime parity tests against it.  Substitute for
# compute-sanitizer, which is closed on this GPU pool.  Usage (GPU box):
#   bash tools/checked_sweep.sh [cases]
set -e
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -DFABM_CHECKED -I include -o paper_1611_08678_b200/libfabm_checked.so \
  paper_1611_08678_b200/csrc/fabm_api.cu
FABM_LIBRARY=paper_1611_08678_b200/libfabm_checked.so FABM_RANDOM_CASES=${1:-200} \
  python -m pytest tests/test_gpu_random.py tests/test_gpu_headline_regime.py tests/test_gpu_sharded.py \
  tests/test_gpu_batch.py -q -x
# positive control: a deliberately failed check must surface as an error
FABM_LIBRARY=paper_1611_08678_b200/libfabm_checked.so FABM_DEBUG_MODE=16 python - <<'PY'
import paper_1611_08678_b200 as fabm
p = fabm.FractionalProblem(alpha=0.9, dim=3, rhs=fabm.rhs_lorenz(), y0=(1.0, 1.0, 1.0), t_end=2.0)
try:
    fabm.solve_gpu(p, p.grid(2000))
except ValueError as exc:
    assert "FABM_CHECKED" in str(exc), exc
    print("positive control:", exc)
else:
    raise SystemExit("the checked build did not report the deliberate violation")
PY
