"""Fused level visits and the f cascade, one call per visit
(``fmgsr_visit_{top,down,up}_*`` and ``fmgsr_f_cascade_*`` in
include/fmgsr_cuda.h).

These are the kernels the native plan strings together, exposed for a driver
that runs the FMG schedule itself -- e.g. the reference's own loop
(cycles.py:95-222) with its operator calls replaced by one fused visit per
level: a visit streams each field once instead of once per operator.  V(1,1)
(one forward sweep), uniform patches (owned width ``W``, ``b``-cell buffer).

Each function returns the same fields (bit for bit, float64) as the operator
composition named in its docstring; fields follow the package convention
((n,) or (n, B), numpy or torch; see _fields.py).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _fields as F
from . import _native as N
from .stencils import level_of

_work: dict = {}


def _workspace(n: int, W: int, B: int, dt: torch.dtype, dev) -> torch.Tensor:
    """Zero-filled edge-record / counter workspace, one per (n, W, B, dtype,
    device, stream): the counters return to their start state after every
    visit, so visits queued on one stream may share it; two visits running at
    the same time on different streams must not (their arrivals would mix on
    the same counters), hence the stream in the key."""
    key = (n, W, B, dt, dev, N.stream_ptr())
    w = _work.get(key)
    if w is None:
        nbytes = N.lib().fmgsr_visit_workspace_bytes(n, W, B, 0 if dt == torch.float64 else 1)
        if nbytes <= 0:
            raise ValueError(f"no visit workspace for n={n}, W={W}, B={B}")
        w = _work[key] = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    return w


def _geometry(n: int, W: int, b: int, epi: bool) -> None:
    if W < 2 or W % 2 or n % W:
        raise ValueError(f"owned width W={W} must be even and divide n={n}")
    if epi and W < 4:
        raise ValueError("the fused restriction epilogue needs an owned width >= 4")
    if b < 0:
        raise ValueError("buffer must be >= 0")


def visit_top(u_coarse, f, W: int, b: int, omega: float = 1.0, store_u: bool = True):
    """Top of FMG step t (cycles.py:188-197 with 101-102; the paper's fused
    lines 1-5): ``u = S(prolong_fmg(u_coarse))`` (no CR), then
    ``(restrict(u), coarse_rhs(f, u))``.  Returns ``(u or None, u_coarse_new,
    f_coarse)``; ``store_u=False`` is the SR level, where u is never stored."""
    k = level_of(f)
    n = 2 ** k
    _geometry(n, W, b, True)
    if n < 8:
        raise ValueError("prolong_fmg needs a coarse field of >= 4 cells")
    dt = F.pick_dtype(u_coarse, f)
    H, Fl = F.to_field(u_coarse, dt), F.to_field(f, dt)
    if H.n != n // 2:
        raise ValueError(f"u_coarse must have {n // 2} cells, got {H.n}")
    F.same_batch(H, Fl)
    u = F.empty_like_rows(Fl, n) if store_u else None
    uH, fH = F.empty_like_rows(Fl, n // 2), F.empty_like_rows(Fl, n // 2)
    N.call("fmgsr_visit_top", dt, H.ptr(), Fl.ptr(), u.data_ptr() if u is not None else None,
           uH.data_ptr(), fH.data_ptr(), n, Fl.B, Fl.ld, W, b, float(omega),
           _workspace(n, W, Fl.B, dt, Fl.t.device).data_ptr(), N.stream_ptr())
    return (F.out(u, Fl) if u is not None else None), F.out(uH, Fl), F.out(fH, Fl)


def visit_down(u, f, W: int, b: int, omega: float = 1.0, restrict_u: bool = True):
    """Down-leg visit (cycles.py:99-105): ``u_new = S(u)``, then
    ``(restrict(u_new), coarse_rhs(f, u_new))``.  Returns ``(u_new,
    u_coarse or None, f_coarse)``."""
    k = level_of(u)
    n = 2 ** k
    _geometry(n, W, b, True)
    dt = F.pick_dtype(u, f)
    U, Fl = F.to_field(u, dt), F.to_field(f, dt)
    if Fl.n != n:
        raise ValueError("u and f must be on the same level")
    F.same_batch(U, Fl)
    out = F.empty_like_rows(U, n)
    uH = F.empty_like_rows(U, n // 2) if restrict_u else None
    fH = F.empty_like_rows(U, n // 2)
    N.call("fmgsr_visit_down", dt, U.ptr(), Fl.ptr(), out.data_ptr(),
           uH.data_ptr() if uH is not None else None, fH.data_ptr(), n, U.B, U.ld, W, b,
           float(omega), _workspace(n, W, U.B, dt, U.t.device).data_ptr(), N.stream_ptr())
    return F.out(out, U), (F.out(uH, U) if uH is not None else None), F.out(fH, U)


def visit_up(u, u_coarse, f, W: int, b: int, sr: bool = False, omega: float = 1.0):
    """Up-leg visit (cycles.py:109-134): non-SR ``S(u + prolong_correction(
    u_coarse - restrict(u)))``; SR ``S(prolong_fmg(u_coarse))`` with the
    Kaczmarz CR step onto ``u_coarse`` (``u`` unused, may be None)."""
    k = level_of(f)
    n = 2 ** k
    _geometry(n, W, b, False)
    dt = F.pick_dtype(u_coarse, f) if sr else F.pick_dtype(u, u_coarse, f)
    H, Fl = F.to_field(u_coarse, dt), F.to_field(f, dt)
    if H.n != n // 2:
        raise ValueError(f"u_coarse must have {n // 2} cells, got {H.n}")
    F.same_batch(H, Fl)
    U = None
    if not sr:
        U = F.to_field(u, dt)
        if U.n != n:
            raise ValueError("u and f must be on the same level")
        F.same_batch(U, Fl)
    out = F.empty_like_rows(Fl, n)
    N.call("fmgsr_visit_up", dt, U.ptr() if U is not None else None, H.ptr(), Fl.ptr(),
           out.data_ptr(), n, Fl.B, Fl.ld, W, b, int(bool(sr)), float(omega), N.stream_ptr())
    return F.out(out, Fl)


def f_cascade(f, levels: int):
    """Restrictions of the forcing to the next ``levels`` coarser levels in
    one stream over ``f`` (cycles.py:178-180): ``[restrict(f),
    restrict(restrict(f)), ...]``."""
    k = level_of(f)
    if not 1 <= levels <= k:
        raise ValueError(f"levels must be in 1..{k}")
    dt = F.pick_dtype(f)
    Fl = F.to_field(f, dt)
    outs = [F.empty_like_rows(Fl, Fl.n >> (j + 1)) for j in range(levels)]
    ptrs = (C.c_void_p * levels)(*[o.data_ptr() for o in outs])
    N.call("fmgsr_f_cascade", dt, Fl.ptr(), Fl.n, Fl.B, Fl.ld, levels, ptrs, N.stream_ptr())
    return [F.out(o, Fl) for o in outs]
