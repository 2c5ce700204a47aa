"""The drop-in boundary without a GPU: libfmgsr_cuda.so loads, exports every
symbol include/fmgsr_cuda.h declares, and reports argument errors through
its return codes and fmgsr_last_error() (no CUDA call is reached)."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmgsr_cuda.h")


@pytest.fixture(scope="module")
def native():
    from paper_1207_6720_b200 import _native

    if not os.path.exists(_native.LIB_PATH):  # fresh checkout: build in-tree (nvcc, sm_100a)
        subprocess.run(["make", "-s", "-C", _native.CSRC], check=True)
    _native.lib()
    return _native


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(fmgsr_\w+)\s*\(", txt, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("fmgsr_gs_sweep_f64", "fmgsr_kaczmarz_sweep_f64", "fmgsr_smooth_patches_f64",
                 "fmgsr_plan_create", "fmgsr_plan_solve", "fmgsr_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(native):
    lib = C.CDLL(native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # and the Python binding table covers exactly the header
    assert sorted(native.exported_symbols()) == declared_symbols()


def test_library_is_sm100a_code(native):
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_error_reporting(native):
    lib = native.lib()
    assert lib.fmgsr_abi_version() == 1
    d = native.PlanDesc()
    d.m0, d.m, d.n_sr, d.ns = 1, 6, 0, 1  # m0 < 2: rejected before any CUDA call
    d.geom_mode, d.dtype, d.P, d.b, d.B, d.ld = 2, 0, 4, 2, 1, 1
    h = C.c_void_p()
    rc = lib.fmgsr_plan_create(C.byref(d), C.byref(h))
    assert rc == -1
    assert b"m0 must be >= 2" in lib.fmgsr_last_error()
    d.m0, d.n_sr = 3, 3  # n_sr > m - m0 - 1
    assert lib.fmgsr_plan_create(C.byref(d), C.byref(h)) == -1
    assert b"n_sr" in lib.fmgsr_last_error()
    with pytest.raises(ValueError):
        native.check(lib.fmgsr_plan_create(C.byref(d), C.byref(h)), "plan_create")


def test_op_argument_checks_return_codes(native):
    lib = native.lib()
    # window outside the level -> -1 before launch
    rc = lib.fmgsr_gs_sweep_f64(None, None, 8, 1, 1, 64.0, 0, 9, 1, 1.0, None)
    assert rc == -1 and b"window" in lib.fmgsr_last_error()
    rc = lib.fmgsr_prolong_fmg_f64(None, None, 2, 1, 1, None)
    assert rc == -1 and b">= 4" in lib.fmgsr_last_error()
    rc = lib.fmgsr_smooth_patches_f64(None, None, None, 8, 1, 1, 63.0, None, None, None, None, 1,
                                      1, 1.0, 0, None, 0.5, None, None, 0, None)
    assert rc == -1 and b"inv_h2" in lib.fmgsr_last_error()
