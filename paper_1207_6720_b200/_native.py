"""Loader of ``libfmgsr_cuda.so`` (the sm_100a kernels behind the C ABI of
``include/fmgsr_cuda.h``).

There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises.  ``lib()`` binds ctypes signatures once; ``call`` turns a
negative return code into ``ValueError`` (bad argument, mirroring the
reference's argument checks) or ``RuntimeError`` (CUDA failure).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FMGSR_LIB: an alternative in-tree build of the library (A/B experiments)
LIB_PATH = os.environ.get("FMGSR_LIB") or os.path.join(_HERE, "libfmgsr_cuda.so")
CSRC = os.path.join(_HERE, "csrc")

_i64 = C.c_int64
_i32 = C.c_int32
_vp = C.c_void_p
_d = C.c_double


class PlanDesc(C.Structure):
    _fields_ = [
        ("m0", _i32), ("m", _i32), ("n_sr", _i32), ("ns", _i32),
        ("geom_mode", _i32), ("dtype", _i32),
        ("P", _i64), ("b", _i64), ("B", _i64), ("ld", _i64),
        ("omega", _d), ("fused", _i32), ("use_graph", _i32), ("coarse", _i32),
        ("nonlinear", _i32),
    ]


class CommRec(C.Structure):  # fmgsr_comm_rec
    _fields_ = [
        ("step", C.c_int32),
        ("step_kind", C.c_int32),
        ("level", C.c_int32),
        ("array_level", C.c_int32),
        ("pad", C.c_int32),
        ("kind", C.c_int32),
        ("peer", C.c_int32),
        ("tag", C.c_int32),
        ("bytes", C.c_int64),
        ("addr", C.c_uint64),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("workspace_bytes", _i64), ("launches_per_solve", _i64),
        ("visits_per_solve", _i64), ("alg_bytes_per_solve", _d),
        ("finest_visit_alg_bytes", _d), ("coarse_cutoff", _i32), ("coarse_columns", _i32),
    ]


_SIGS = {
    "fmgsr_abi_version": (C.c_int, []),
    "fmgsr_last_error": (C.c_char_p, []),
    "fmgsr_gs_sweep": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _d, _i64, _i64, C.c_int, _d, _vp]),
    "fmgsr_kaczmarz_sweep": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, C.c_int, _d, _vp]),
    "fmgsr_smooth_patches": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _d, _vp, _vp, _vp, _vp,
                                       _i64, _i64, _d, C.c_int, _vp, _d, _vp, _vp, _i64, _vp]),
    "fmgsr_smooth_uniform": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _d,
                                       _vp, _d, _vp, _i64, _vp]),
    "fmgsr_smooth_uniform_nl": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _d,
                                          _vp, _d, _vp, _i64, _vp]),
    "fmgsr_coarse_rhs_nl": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_direct_solve_nl": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_apply_operator": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_restrict": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_prolong_correction": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_prolong_fmg": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_tau_correction": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_coarse_rhs": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_fas_correct": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_visit_workspace_bytes": (_i64, [_i64, _i64, _i64, _i32]),
    "fmgsr_visit_top": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _d,
                                  _vp, _vp]),
    "fmgsr_visit_down": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _d,
                                   _vp, _vp]),
    "fmgsr_visit_up": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i32, _d,
                                 _vp]),
    "fmgsr_f_cascade": (C.c_int, [_vp, _i64, _i64, _i64, _i32, C.POINTER(_vp), _vp]),
    "fmgsr_direct_solve": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "fmgsr_direct_solve_ws": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "fmgsr_banded_lu_solve": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "fmgsr_fourier_rhs": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, _vp, _vp]),
    "fmgsr_nonlinear_rhs": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "fmgsr_smooth_scratch_rows": (_i64, [_i64, _i64, _i64]),
    "fmgsr_div_check": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fmgsr_manufactured_rhs_f64": (C.c_int, [_i64, _i64, _vp, _vp, _vp]),
    "fmgsr_plan_create": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(_vp)]),
    "fmgsr_plan_destroy": (C.c_int, [_vp]),
    "fmgsr_plan_set_debug": (C.c_int, [_vp, _i32]),
    "fmgsr_plan_check_guards": (C.c_int, [_vp, C.POINTER(_i64)]),
    "fmgsr_plan_get_info": (C.c_int, [_vp, C.POINTER(PlanInfo)]),
    "fmgsr_plan_probe_ms": (C.c_int, [_vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "fmgsr_plan_solve": (C.c_int, [_vp, _vp, _vp, _vp]),
    "fmgsr_plan_solve_host": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "fmgsr_plan_solve_host_ex": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _vp]),
    "fmgsr_plan_solve_functional": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "fmgsr_plan_solve_timed": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                         C.POINTER(_i64)]),
    "fmgsr_nccl_unique_id": (C.c_int, [_vp]),
    "fmgsr_shard_plan_create": (C.c_int, [C.POINTER(PlanDesc), _i32, _i32, _vp, C.POINTER(_vp)]),
    "fmgsr_shard_group_create": (C.c_int, [C.POINTER(PlanDesc), _i32, C.POINTER(_vp)]),
    "fmgsr_shard_group_solve": (C.c_int, [_vp, _vp, _vp, _vp]),
    "fmgsr_shard_group_cutoff": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i64)]),
    "fmgsr_shard_group_destroy": (C.c_int, [_vp]),
    "fmgsr_shard_plan_forcing_slab": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_i64)]),
    "fmgsr_shard_plan_create_local": (C.c_int, [C.POINTER(PlanDesc), _i32, _i32, C.POINTER(_vp)]),
    "fmgsr_shard_plan_create_p2p": (C.c_int, [C.POINTER(PlanDesc), _i32, _i32, C.POINTER(_vp)]),
    "fmgsr_shard_p2p_export": (C.c_int, [_vp, _vp, _i64, C.POINTER(_i64)]),
    "fmgsr_shard_p2p_import": (C.c_int, [_vp, _vp, _i64]),
    "fmgsr_shard_p2p_status": (C.c_int, [_vp, C.POINTER(_i32)]),
    "fmgsr_shard_schedule": (C.c_int, [C.POINTER(PlanDesc), _i32, _i32, _vp, _i64,
                                       C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64)]),
}
_TYPED = {"fmgsr_gs_sweep", "fmgsr_kaczmarz_sweep", "fmgsr_smooth_patches", "fmgsr_smooth_uniform",
          "fmgsr_apply_operator", "fmgsr_restrict", "fmgsr_prolong_correction",
          "fmgsr_prolong_fmg", "fmgsr_tau_correction", "fmgsr_coarse_rhs", "fmgsr_fas_correct",
          "fmgsr_direct_solve", "fmgsr_direct_solve_ws", "fmgsr_banded_lu_solve",
          "fmgsr_fourier_rhs", "fmgsr_nonlinear_rhs", "fmgsr_smooth_uniform_nl", "fmgsr_coarse_rhs_nl",
          "fmgsr_direct_solve_nl", "fmgsr_div_check", "fmgsr_visit_top", "fmgsr_visit_down",
          "fmgsr_visit_up", "fmgsr_f_cascade"}

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile the extension in-tree with nvcc for sm_100a (csrc/Makefile)."""
    args = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(args + ["clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


def exported_symbols() -> list[str]:
    """Every C symbol the header declares (for the ABI export test)."""
    out = []
    for name in _SIGS:
        if name in _TYPED:
            out += [name + "_f64", name + "_f32"]
        else:
            out.append(name)
    return out


def lib():
    """The loaded library with bound signatures (raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libfmgsr_cuda.so not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        h = C.CDLL(LIB_PATH)
        for name in exported_symbols():
            base = name[:-4] if name.endswith(("_f64", "_f32")) and name[:-4] in _TYPED else name
            restype, argtypes = _SIGS[base]
            fn = getattr(h, name)
            fn.restype = restype
            fn.argtypes = argtypes
        _lib = h
    return _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("fmgsr_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")


def fn(name: str, dtype: torch.dtype | None = None):
    L = lib()
    if dtype is None:
        return getattr(L, name)
    suffix = {torch.float64: "_f64", torch.float32: "_f32"}.get(dtype)
    if suffix is None:
        raise ValueError(f"unsupported dtype {dtype}; use float64 or float32")
    return getattr(L, name + suffix)


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = lib().fmgsr_last_error().decode(errors="replace")
    if rc == -1:
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def call(name: str, dtype, *args) -> None:
    check(fn(name, dtype)(*args), name)


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream
