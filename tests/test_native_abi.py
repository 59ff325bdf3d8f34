"""The C ABI boundary: libfabm.so builds for sm_100a, loads without a GPU and
exports every symbol include/fabm.h declares (no compute calls here)."""

from __future__ import annotations

import ctypes
import re
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_1611_08678_b200 import _native, build

    build.build()
    return _native.load()


def header_functions() -> set[str]:
    text = (ROOT / "include" / "fabm.h").read_text()
    return set(re.findall(r"\b(fabm_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_bound_symbols():
    from paper_1611_08678_b200 import _native

    assert header_functions() == set(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_1611_08678_b200" / "libfabm.so")],
                         capture_output=True, text=True, check=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(ROOT / "paper_1611_08678_b200" / "libfabm.so")],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_version_and_no_device_is_reported(lib):
    assert b"sm_100a" in lib.fabm_version()
    assert lib.fabm_device_count() >= 0


def test_struct_layout_matches_header():
    from paper_1611_08678_b200 import _native

    # fabm_problem: double + 2*int32 + 16 doubles + 4 doubles
    assert ctypes.sizeof(_native.Problem) == 8 + 8 + 8 * 16 + 8 * 4
    assert ctypes.sizeof(_native.Grid) == 8 * 6
    assert ctypes.sizeof(_native.Status) == 4 + 4 + 8 + 8 + 8 + 240


def test_config_errors_need_no_device(lib):
    from paper_1611_08678_b200 import _native

    st = _native.Status()
    b = (ctypes.c_double * 4)()
    rc = lib.fabm_weights(1.5, 3, 0, 0.0, 0.0, b, b, b, ctypes.byref(st))
    assert rc == _native.FABM_ERR_CONFIG
    assert b"alpha" in st.message


def test_new_entry_points_validate_before_any_device_work(lib):
    # argument errors are reported as FABM_ERR_CONFIG (the reference's
    # ValueError) before any CUDA call, so they behave the same without a GPU
    from paper_1611_08678_b200 import _native

    st = _native.Status()
    one = (ctypes.c_double * 4)(1.0, 2.0, 3.0, 4.0)
    n = ctypes.c_int64(0)
    # CSV: dim 0
    rc = lib.fabm_format_csv(one, None, 1, 0, 0.1, 0, None, 0, ctypes.byref(n), None, ctypes.byref(st))
    assert rc == _native.FABM_ERR_CONFIG
    # Mittag-Leffler: negative count
    rc = lib.fabm_mittag_leffler(one, one, -1, 0, one, None, ctypes.byref(st))
    assert rc == _native.FABM_ERR_CONFIG
    # step ops: index outside [0, N)
    pr, gr = _native.Problem(), _native.Grid()
    pr.alpha, pr.dim, pr.system = 0.5, 1, 2
    pr.params[0] = -1.0
    gr.n_steps, gr.h = 3, 0.1
    ns = (ctypes.c_int64 * 1)(3)
    err = (ctypes.c_int32 * 1)()
    rc = lib.fabm_step_pc(ctypes.byref(pr), ctypes.byref(gr), one, one, one, 4, one, 4, ns, 1, None, one, one, err, 0,
                          ctypes.byref(st))
    assert rc == _native.FABM_ERR_CONFIG and b"outside" in st.message
    # a null plan
    assert lib.fabm_plan_set_host_output(None, None, None, ctypes.byref(st)) == _native.FABM_ERR_CONFIG
    assert lib.fabm_plan_write_csv(None, b"x.csv", None, None, ctypes.byref(st)) == _native.FABM_ERR_CONFIG
