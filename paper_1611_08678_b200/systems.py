"""Right-hand sides with device tags.

Each factory returns a plain ``f(t, y)`` host callable — the same contract as
the reference factories (systems.py:26-123) — and attaches
``f.device_system = DeviceSystem(system_id, dim, params)``, which tells the
GPU engine which compiled rhs to run (csrc/device_common.cuh ``Rhs<...>``).
The host expression and the device expression use the same operator order,
so f(t, y) agrees bit for bit between them (checked on the GPU by
tests/test_gpu_parity.py::test_device_rhs_bitwise_equals_host).

``rhs_lorenz``/``rhs_chen``/``rhs_rossler``/``rhs_financial`` add the four
BASELINE.json systems, which the reference does not ship.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "DeviceSystem",
    "HindmarshRoseParams",
    "SYSTEM_IDS",
    "SYSTEM_NAMES",
    "HR_DEFAULT_Y0",
    "rhs_constant",
    "rhs_power_law",
    "rhs_linear",
    "rhs_hindmarsh_rose",
    "rhs_lorenz",
    "rhs_chen",
    "rhs_rossler",
    "rhs_financial",
    "device_system_of",
    "adopt_reference_rhs",
]

# must match FABM_SYS_* in include/fabm.h
SYSTEM_IDS = {
    "constant": 0,
    "power-law": 1,
    "linear": 2,
    "hindmarsh-rose": 3,
    "lorenz": 4,
    "chen": 5,
    "rossler": 6,
    "financial": 7,
}
SYSTEM_NAMES = tuple(SYSTEM_IDS)
HR_DEFAULT_Y0 = (0.1, 0.2, 0.2)  # reference systems.py:131


@dataclass(frozen=True)
class DeviceSystem:
    """Tag naming the compiled device rhs. ``dim`` None = any dimension."""

    name: str
    dim: int | None
    params: tuple

    @property
    def system_id(self) -> int:
        return SYSTEM_IDS[self.name]


def _tag(fn, name: str, dim, params):
    fn.device_system = DeviceSystem(name, dim, tuple(float(p) for p in params))
    return fn


def _closure_vars(fn) -> dict:
    code = getattr(fn, "__code__", None)
    cells = getattr(fn, "__closure__", None) or ()
    if code is None:
        return {}
    return {name: cell.cell_contents for name, cell in zip(code.co_freevars, cells)}


def adopt_reference_rhs(fn) -> DeviceSystem | None:
    """Device tag for an rhs built by the reference's own factories.

    ``fodeabm.systems.rhs_constant/rhs_power_law/rhs_linear/rhs_hindmarsh_rose``
    (systems.py:26-123) return closures; their qualified name and captured
    constants identify the system exactly, so problems built with the
    reference API run on the device unchanged.  Anything else returns None.
    """
    if getattr(fn, "__module__", None) != "fodeabm.systems":
        return None
    qual = getattr(fn, "__qualname__", "")
    env = _closure_vars(fn)
    try:
        if qual == "rhs_constant.<locals>.f":
            vec = np.asarray(env["vec"], dtype=np.float64).reshape(-1)
            return DeviceSystem("constant", len(vec), tuple(float(v) for v in vec))
        if qual == "rhs_power_law.<locals>.f":
            return DeviceSystem("power-law", 1, (float(env["coef"]), float(env["expo"])))
        if qual == "rhs_linear.<locals>.f":
            return DeviceSystem("linear", None, (float(env["lam"]),))
        if qual == "rhs_hindmarsh_rose.<locals>.f":
            names = ("a", "b", "c", "d", "r", "s", "x_rest", "i_ext")
            return DeviceSystem("hindmarsh-rose", 3, tuple(float(env[n]) for n in names))
    except (KeyError, TypeError, ValueError):
        return None
    return None


def device_system_of(rhs) -> DeviceSystem:
    """The device tag of ``rhs``; plain callables have none (no CPU fallback)."""
    tag = getattr(rhs, "device_system", None)
    if isinstance(tag, DeviceSystem):
        return tag
    tag = adopt_reference_rhs(rhs)
    if tag is not None:
        return tag
    raise ValueError(
        "the GPU engine needs a device rhs: build it with one of the "
        "paper_1611_08678_b200.systems factories or the reference's own "
        "fodeabm.systems factories (arbitrary Python callables cannot run on "
        "the device)"
    )


def rhs_constant(value):
    """f(t, y) = value (systems.py:26-36)."""
    vec = np.array(value, dtype=np.float64).reshape(-1)
    if not np.isfinite(vec).all():
        raise ValueError("constant rhs value must be finite")
    vec.setflags(write=False)

    def f(t, y):
        return vec

    return _tag(f, "constant", len(vec), vec)


def rhs_power_law(alpha: float, beta: float):
    """Forcing with exact solution t^beta for y0 = 0 (systems.py:39-61)."""
    alpha = float(alpha)
    beta = float(beta)
    if beta < alpha:
        raise ValueError(f"power-law forcing needs beta >= alpha, got beta={beta}, alpha={alpha}")
    coef = math.gamma(beta + 1.0) / math.gamma(beta + 1.0 - alpha)
    expo = beta - alpha
    if expo == 0.0:
        return rhs_constant([coef])

    def f(t, y):
        return (coef * t ** expo if t > 0.0 else 0.0,)

    return _tag(f, "power-law", 1, (coef, expo))


def rhs_linear(lam: float):
    """f(t, y) = lam * y (systems.py:64-73); any dimension."""
    lam = float(lam)
    if not math.isfinite(lam):
        raise ValueError("lam must be finite")

    def f(t, y):
        return lam * y

    return _tag(f, "linear", None, (lam,))


@dataclass(frozen=True)
class HindmarshRoseParams:
    """Hindmarsh–Rose constants (systems.py:76-98)."""

    a: float = 1.0
    b: float = 3.0
    c: float = 1.0
    d: float = 5.0
    r: float = 0.006
    s: float = 4.0
    x_rest: float = -1.6
    i_ext: float = 3.25

    def __post_init__(self):
        vals = (self.a, self.b, self.c, self.d, self.r, self.s, self.x_rest, self.i_ext)
        if not all(math.isfinite(v) for v in vals):
            raise ValueError("Hindmarsh-Rose parameters must be finite")
        if self.r <= 0.0:
            raise ValueError("r must be positive")


def rhs_hindmarsh_rose(params: HindmarshRoseParams | None = None):
    """Hindmarsh–Rose neuron (systems.py:101-123), same operator order."""
    p = params or HindmarshRoseParams()
    a, b, c, d = p.a, p.b, p.c, p.d
    r, s, x_rest, i_ext = p.r, p.s, p.x_rest, p.i_ext

    def f(t, state):
        x, y, z = state
        x2 = x * x
        return (
            y - a * x2 * x + b * x2 - z + i_ext,
            c - d * x2 - y,
            r * (s * (x - x_rest) - z),
        )

    return _tag(f, "hindmarsh-rose", 3, (a, b, c, d, r, s, x_rest, i_ext))


def _finite_params(*vals):
    if not all(math.isfinite(float(v)) for v in vals):
        raise ValueError("system parameters must be finite")


def rhs_lorenz(sigma: float = 10.0, rho: float = 28.0, beta: float = 8.0 / 3.0):
    """Fractional Lorenz: (sigma(y-x), x(rho-z) - y, xy - beta z)."""
    _finite_params(sigma, rho, beta)
    sigma, rho, beta = float(sigma), float(rho), float(beta)

    def f(t, s):
        x, y, z = s
        return (sigma * (y - x), x * (rho - z) - y, x * y - beta * z)

    return _tag(f, "lorenz", 3, (sigma, rho, beta))


def rhs_chen(a: float = 35.0, b: float = 3.0, c: float = 28.0):
    """Fractional Chen: (a(y-x), (c-a)x - xz + cy, xy - bz)."""
    _finite_params(a, b, c)
    a, b, c = float(a), float(b), float(c)

    def f(t, s):
        x, y, z = s
        return (a * (y - x), (c - a) * x - x * z + c * y, x * y - b * z)

    return _tag(f, "chen", 3, (a, b, c))


def rhs_rossler(a: float = 0.5, b: float = 0.2, c: float = 10.0):
    """Fractional Rössler: (-y - z, x + ay, b + z(x - c))."""
    _finite_params(a, b, c)
    a, b, c = float(a), float(b), float(c)

    def f(t, s):
        x, y, z = s
        return (-y - z, x + a * y, b + z * (x - c))

    return _tag(f, "rossler", 3, (a, b, c))


def rhs_financial(a: float = 3.0, b: float = 0.1, c: float = 1.0):
    """Fractional financial system: (z + (y - a)x, 1 - by - x^2, -x - cz)."""
    _finite_params(a, b, c)
    a, b, c = float(a), float(b), float(c)

    def f(t, s):
        x, y, z = s
        return (z + (y - a) * x, 1.0 - b * y - x * x, -x - c * z)

    return _tag(f, "financial", 3, (a, b, c))
