"""ctypes binding of libfabm.so (include/fabm.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a)
into this package directory.  There is no fallback: if the shared object is
missing or no sm_100 device is present, the solvers raise.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libfabm.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

MAX_DIM = 4
MAX_PARAMS = 16

FABM_OK = 0
FABM_ERR_NONFINITE = 1
FABM_ERR_CONFIG = 2
FABM_ERR_TIMEOUT = 3
FABM_ERR_CUDA = 4
FABM_ERR_NODEVICE = 5
FABM_ERR_IO = 6

WEIGHTS_ACCURATE = 0
WEIGHTS_FORMULA = 1
WEIGHTS_HOST = 2

IPC_HANDLE_BYTES = 64
MAX_SHARDS = 8

KIND_NAMES = {0: "none", 1: "initial", 2: "predictor", 3: "corrector"}

# every symbol include/fabm.h declares (tests/test_native_abi.py checks them)
EXPORTED_SYMBOLS = (
    "fabm_version",
    "fabm_device_count",
    "fabm_weights",
    "fabm_solve",
    "fabm_plan_create",
    "fabm_plan_set_weights",
    "fabm_plan_set_y0",
    "fabm_plan_run",
    "fabm_plan_download",
    "fabm_plan_download_last",
    "fabm_plan_stats",
    "fabm_plan_destroy",
    "fabm_plan_reset",
    "fabm_plan_set_bulk_ctas",
    "fabm_plan_ipc_handle",
    "fabm_plan_attach_shards",
    "fabm_plan_set_virtual_shards",
    "fabm_plan_emulate_shards",
    "fabm_plan_shard_counters",
    "fabm_plan_detach_shards",
    "fabm_solve_batch",
    "fabm_measure_dfma_peak",
    "fabm_format_csv",
    "fabm_write_csv",
    "fabm_plan_write_csv",
    "fabm_mittag_leffler",
    "fabm_step_pc",
    "fabm_plan_set_host_output",
    "fabm_host_alloc",
    "fabm_host_free",
    "fabm_trim_memory",
)


class Problem(ctypes.Structure):
    _fields_ = [
        ("alpha", ctypes.c_double),
        ("dim", ctypes.c_int32),
        ("system", ctypes.c_int32),
        ("params", ctypes.c_double * MAX_PARAMS),
        ("y0", ctypes.c_double * MAX_DIM),
    ]


class Grid(ctypes.Structure):
    _fields_ = [
        ("n_steps", ctypes.c_int64),
        ("h", ctypes.c_double),
        ("h_alpha", ctypes.c_double),
        ("inv_gamma2", ctypes.c_double),
        ("gamma1", ctypes.c_double),
        ("gamma2", ctypes.c_double),
    ]


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("step", ctypes.c_int64),
        ("t", ctypes.c_double),
        ("index", ctypes.c_int64),
        ("message", ctypes.c_char * 240),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("kernel_ms", ctypes.c_double),
        ("weights_ms", ctypes.c_double),
        ("steps", ctypes.c_int64),
        ("history_fma", ctypes.c_int64),
        ("bulk_tiles", ctypes.c_int64),
        ("leader_wait_ns", ctypes.c_int64),
        ("leader_throttle_ns", ctypes.c_int64),
        ("bulk_ctas", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("window_blocks", ctypes.c_int32),
        ("segment", ctypes.c_int32),
        ("bulk_claims", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_DP = ctypes.POINTER(ctypes.c_double)
_I64P = ctypes.POINTER(ctypes.c_int64)
_lib = None


def _declare(lib):
    P, G, S, St = ctypes.POINTER(Problem), ctypes.POINTER(Grid), ctypes.POINTER(Status), ctypes.POINTER(Stats)
    plan = ctypes.c_void_p
    sig = {
        "fabm_version": (ctypes.c_char_p, []),
        "fabm_device_count": (ctypes.c_int, []),
        "fabm_weights": (ctypes.c_int, [ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, _DP, _DP, _DP, S]),
        "fabm_solve": (ctypes.c_int, [P, G, ctypes.c_int, _DP, _DP, _DP, _DP, _DP, S]),
        "fabm_plan_create": (plan, [P, G, ctypes.c_int, S]),
        "fabm_plan_set_weights": (ctypes.c_int, [plan, ctypes.c_int, _DP, _DP, _DP, S]),
        "fabm_plan_set_y0": (ctypes.c_int, [plan, _DP, S]),
        "fabm_plan_run": (ctypes.c_int, [plan, ctypes.c_double, S]),
        "fabm_plan_download": (ctypes.c_int, [plan, _DP, _DP, S]),
        "fabm_plan_download_last": (ctypes.c_int, [plan, _DP, S]),
        "fabm_plan_stats": (ctypes.c_int, [plan, St]),
        "fabm_plan_destroy": (None, [plan]),
        "fabm_plan_reset": (ctypes.c_int, [plan, S]),
        "fabm_plan_set_bulk_ctas": (ctypes.c_int, [plan, ctypes.c_int, S]),
        "fabm_plan_ipc_handle": (ctypes.c_int, [plan, ctypes.c_void_p, S]),
        "fabm_plan_attach_shards": (ctypes.c_int, [plan, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, S]),
        "fabm_plan_set_virtual_shards": (ctypes.c_int, [plan, ctypes.c_int, S]),
        "fabm_plan_emulate_shards": (ctypes.c_int, [plan, ctypes.c_int, S]),
        "fabm_plan_shard_counters": (ctypes.c_int, [plan, _I64P, _I64P, S]),
        "fabm_plan_detach_shards": (ctypes.c_int, [plan, S]),
        "fabm_solve_batch": (ctypes.c_int, [P, G, ctypes.c_int64, ctypes.c_int, _DP, _DP, _DP, _DP, S]),
        "fabm_measure_dfma_peak": (ctypes.c_double, [ctypes.c_int]),
        "fabm_format_csv": (ctypes.c_int, [_DP, _DP, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int,
                                           ctypes.c_char_p, ctypes.c_int64, _I64P, _DP, S]),
        "fabm_write_csv": (ctypes.c_int, [ctypes.c_char_p, _DP, _DP, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                          ctypes.c_int, _I64P, _DP, S]),
        "fabm_plan_write_csv": (ctypes.c_int, [plan, ctypes.c_char_p, _I64P, _DP, S]),
        "fabm_plan_set_host_output": (ctypes.c_int, [plan, _DP, _DP, S]),
        "fabm_host_alloc": (ctypes.c_void_p, [ctypes.c_int64]),
        "fabm_host_free": (None, [ctypes.c_void_p]),
        "fabm_trim_memory": (ctypes.c_int, [ctypes.c_int]),
        "fabm_step_pc": (ctypes.c_int, [P, G, _DP, _DP, _DP, ctypes.c_int64, _DP, ctypes.c_int64, _I64P,
                                        ctypes.c_int64, _DP, _DP, _DP, ctypes.POINTER(ctypes.c_int32), ctypes.c_int,
                                        S]),
        "fabm_mittag_leffler": (ctypes.c_int, [_DP, _DP, ctypes.c_int64, ctypes.c_int, _DP,
                                               ctypes.POINTER(ctypes.c_int32), S]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            if os.environ.get("FABM_LIBRARY"):  # dev A/B against an older build (tools/ab_engine.py)
                continue
            raise RuntimeError(f"libfabm is missing the entry point {name} (stale build?)")
        fn.restype = res
        fn.argtypes = args


def library_path() -> Path:
    override = os.environ.get("FABM_LIBRARY")
    return Path(override) if override else LIB_PATH


def load():
    """Load libfabm.so once; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        path = library_path()
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build the CUDA engine first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(str(path))
        _declare(lib)
        _lib = lib
    return _lib


def dptr(arr: np.ndarray | None):
    if arr is None:
        return None
    assert arr.dtype == np.float64 and arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(_DP)
