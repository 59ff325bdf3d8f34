"""Run the reference package's own CLI with the GPU strategy plugged in.

    python examples/reference_cli_gpu.py solve --system hindmarsh-rose --alpha 0.9 \\
        --tmax 500 --steps 500000 --strategy gpu --output hr.csv

Needs `fodeabm` importable (e.g. installed at baseline/_ref).
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
from paper_1611_08678_b200 import strategy  # noqa: E402

strategy.install()
import fodeabm.cli  # noqa: E402

sys.exit(fodeabm.cli.main(sys.argv[1:]))
