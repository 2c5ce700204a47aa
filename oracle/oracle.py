"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C oracle.

``liboracle.so`` (built from ``fmgsr_oracle.c`` by ``oracle/Makefile``) is a
CPU restatement of the reference's FMG-FAS-SR path.  It is the parity checker
for the CUDA product path and the CPU baseline of ``bench.py``.  The product
package ``paper_1207_6720_b200`` never imports this module.

All functions take and return 1-D float64 numpy arrays (one right-hand side);
``fmg_solve_batch`` takes a ``(B, N)`` array and runs rows on ``nthreads``
POSIX threads.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

GEOM_HALO, GEOM_GLOBAL, GEOM_PATCHES = 0, 1, 2

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


class OrcCfg(C.Structure):
    _fields_ = [
        ("m0", C.c_int),
        ("m", C.c_int),
        ("n_sr", C.c_int),
        ("ns", C.c_int),
        ("mode", C.c_int),
        ("P", _i64),
        ("b", _i64),
        ("omega", C.c_double),
        ("nonlin", C.c_int),
    ]


def build() -> str:
    """Compile liboracle.so in place (gcc, -ffp-contract=off)."""
    src = os.path.join(_HERE, "fmgsr_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_gs_sweep.argtypes = [_dp, _dp, _i64, C.c_double, _i64, _i64, C.c_int, C.c_double]
        _lib.orc_kaczmarz_sweep.argtypes = [_dp, _dp, _i64, _i64, C.c_int, C.c_double]
        _lib.orc_smooth_patches.argtypes = [
            _dp, _dp, _dp, _i64, C.c_double, _ip, _ip, _ip, _ip, _i64, _i64,
            C.c_double, C.c_int, _dp, C.c_double, _dp,
        ]
        _lib.orc_apply_operator.argtypes = [_dp, _dp, _i64]
        _lib.orc_restrict.argtypes = [_dp, _dp, _i64]
        _lib.orc_prolong_correction.argtypes = [_dp, _dp, _i64]
        _lib.orc_prolong_fmg.argtypes = [_dp, _dp, _i64]
        _lib.orc_tau_correction.argtypes = [_dp, _dp, _i64, _dp]
        _lib.orc_coarse_rhs.argtypes = [_dp, _dp, _dp, _i64, _dp]
        _lib.orc_direct_solve.argtypes = [_dp, _dp, _i64, _dp]
        _lib.orc_banded_lu_solve.argtypes = [_dp, _dp, _i64, _dp]
        _lib.orc_banded_lu_solve.restype = C.c_int
        _lib.orc_fmg_solve.argtypes = [C.POINTER(OrcCfg), _dp, _dp]
        _lib.orc_fmg_solve_batch.argtypes = [C.POINTER(OrcCfg), _dp, _dp, _i64, C.c_int]
        _lib.orc_level_geometry.argtypes = [_i64, C.c_int, _i64, _i64, _ip, _ip]
        _lib.orc_gs_sweep_nl.argtypes = [_dp, _dp, _i64, C.c_double, _i64, _i64, C.c_int,
                                         C.c_double]
        _lib.orc_apply_nonlinear.argtypes = [_dp, _dp, _i64]
        _lib.orc_coarse_rhs_nl.argtypes = [_dp, _dp, _dp, _i64, _dp]
        _lib.orc_direct_solve_nl.argtypes = [_dp, _dp, _i64, _dp]
        _lib.orc_smooth_patches_nl.argtypes = _lib.orc_smooth_patches.argtypes
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def gs_sweep(u, f, inv_h2, start, stop, forward, omega=1.0):
    out = _f64(u).copy()
    f = _f64(f)
    lib().orc_gs_sweep(_d(out), _d(f), len(out), float(inv_h2), start, stop, int(forward), omega)
    return out


def kaczmarz_sweep(u, uc, start, stop, forward=True, proj_diag=0.5):
    out = _f64(u).copy()
    uc = _f64(uc)
    lib().orc_kaczmarz_sweep(_d(out), _d(uc), start, stop, int(forward), proj_diag)
    return out


def smooth_patches(u, f, inv_h2, olo, ohi, elo, ehi, ns, omega=1.0, uc=None, proj_diag=0.5):
    u = _f64(u)
    f = _f64(f)
    n = len(u)
    out = np.empty(n)
    scratch = np.empty(n)
    arr = [np.ascontiguousarray(a, dtype=np.int64) for a in (olo, ohi, elo, ehi)]
    ucv = _f64(uc) if uc is not None else np.zeros(1)
    lib().orc_smooth_patches(
        _d(u), _d(f), _d(out), n, float(inv_h2), *[_i(a) for a in arr], len(arr[0]),
        ns, omega, int(uc is not None), _d(ucv), proj_diag, _d(scratch),
    )
    return out


def apply_operator(u):
    u = _f64(u)
    out = np.empty_like(u)
    lib().orc_apply_operator(_d(u), _d(out), len(u))
    return out


def restrict(u):
    u = _f64(u)
    out = np.empty(len(u) // 2)
    lib().orc_restrict(_d(u), _d(out), len(u))
    return out


def prolong_correction(c):
    c = _f64(c)
    out = np.empty(2 * len(c))
    lib().orc_prolong_correction(_d(c), _d(out), len(c))
    return out


def prolong_fmg(c):
    c = _f64(c)
    out = np.empty(2 * len(c))
    lib().orc_prolong_fmg(_d(c), _d(out), len(c))
    return out


def tau_correction(u):
    u = _f64(u)
    out = np.empty(len(u) // 2)
    work = np.empty(3 * len(u) + 8)
    lib().orc_tau_correction(_d(u), _d(out), len(u), _d(work))
    return out


def coarse_rhs(f, u):
    u = _f64(u)
    f = _f64(f)
    out = np.empty(len(u) // 2)
    work = np.empty(3 * len(u) + 8)
    lib().orc_coarse_rhs(_d(f), _d(u), _d(out), len(u), _d(work))
    return out


def direct_solve(f):
    f = _f64(f)
    out = np.empty_like(f)
    work = np.empty(2 * len(f) + 2)
    lib().orc_direct_solve(_d(f), _d(out), len(f), _d(work))
    return out


def banded_lu_solve(f):
    """problem.py:61-77 direct_fine_solve (LAPACK dgbsv order)."""
    f = _f64(f)
    out = np.empty_like(f)
    work = np.empty(2 * len(f) + 2)
    if lib().orc_banded_lu_solve(_d(f), _d(out), len(f), _d(work)):
        raise RuntimeError("banded LU: the pivot search would swap rows")
    return out


def level_geometry(n, mode, P=1, b=0):
    W = np.zeros(1, dtype=np.int64)
    bb = np.zeros(1, dtype=np.int64)
    lib().orc_level_geometry(n, mode, P, b, _i(W), _i(bb))
    return int(W[0]), int(bb[0])


def make_cfg(m0, m, n_sr=0, ns=1, mode=GEOM_PATCHES, P=1, b=0, omega=1.0, nonlin=False):
    return OrcCfg(m0, m, n_sr, ns, mode, P, b, omega, int(nonlin))


# ---- nonlinear FAS restatement (-u'' + u^3 = f; see fmgsr_oracle.c) -------------------------
def gs_sweep_nl(u, f, inv_h2, start, stop, forward, omega=1.0):
    out = _f64(u).copy()
    f = _f64(f)
    lib().orc_gs_sweep_nl(_d(out), _d(f), len(out), float(inv_h2), start, stop, int(forward),
                          omega)
    return out


def apply_nonlinear(u):
    u = _f64(u)
    out = np.empty_like(u)
    lib().orc_apply_nonlinear(_d(u), _d(out), len(u))
    return out


def coarse_rhs_nl(f, u):
    u = _f64(u)
    f = _f64(f)
    out = np.empty(len(u) // 2)
    work = np.empty(3 * len(u) + 8)
    lib().orc_coarse_rhs_nl(_d(f), _d(u), _d(out), len(u), _d(work))
    return out


def direct_solve_nl(f):
    f = _f64(f)
    out = np.empty_like(f)
    work = np.empty(5 * len(f) + 8)
    lib().orc_direct_solve_nl(_d(f), _d(out), len(f), _d(work))
    return out


def smooth_patches_nl(u, f, inv_h2, olo, ohi, elo, ehi, ns, omega=1.0, uc=None, proj_diag=0.5):
    u = _f64(u)
    f = _f64(f)
    n = len(u)
    out = np.empty(n)
    scratch = np.empty(n)
    arr = [np.ascontiguousarray(a, dtype=np.int64) for a in (olo, ohi, elo, ehi)]
    ucv = _f64(uc) if uc is not None else np.zeros(1)
    lib().orc_smooth_patches_nl(
        _d(u), _d(f), _d(out), n, float(inv_h2), *[_i(a) for a in arr], len(arr[0]),
        ns, omega, int(uc is not None), _d(ucv), proj_diag, _d(scratch),
    )
    return out


def fmg_solve(cfg: OrcCfg, forcing):
    forcing = _f64(forcing)
    out = np.empty_like(forcing)
    lib().orc_fmg_solve(C.byref(cfg), _d(forcing), _d(out))
    return out


def fmg_solve_batch(cfg: OrcCfg, forcing_rows, nthreads=1):
    """forcing_rows: (B, N) float64; returns (B, N)."""
    fr = _f64(forcing_rows)
    out = np.empty_like(fr)
    lib().orc_fmg_solve_batch(C.byref(cfg), _d(fr), _d(out), fr.shape[0], int(nthreads))
    return out
