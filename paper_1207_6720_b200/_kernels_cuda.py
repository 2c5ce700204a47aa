"""The ``cuda`` kernel lane: the reference lane contract on sm_100a kernels.

Same three callables and argument meaning as the reference's
``_kernels_numba`` / ``_kernels_numpy`` (reference _kernels_numba.py:15-92),
backed by ``libfmgsr_cuda.so`` (``fmgsr_gs_sweep_*``, ``fmgsr_kaczmarz_sweep_*``,
``fmgsr_smooth_patches_*``).  Fields may be numpy arrays (uploaded, and for the
in-place sweeps written back into the caller's array) or CUDA tensors of shape
(n,) or (n, B).  Results are bit-identical to the numba lane in float64.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _fields as F
from . import _native as N


def _writeback(u, fld: F.Field) -> None:
    if isinstance(u, np.ndarray):
        u[...] = F.out(fld.t, fld)
    elif fld.t.data_ptr() != u.data_ptr():
        u.copy_(fld.t[:, 0] if fld.one_d else fld.t)


def gs_sweep(u, f, inv_h2, start, stop, forward, omega) -> None:
    """One Gauss-Seidel pass over [start, stop), in place on ``u``."""
    dt = F.pick_dtype(u, f)
    U = F.to_field(u, dt)
    Fd = F.to_field(f, dt)
    F.same_batch(U, Fd)
    N.call("fmgsr_gs_sweep", dt, U.ptr(), Fd.ptr(), U.n, U.B, U.ld, float(inv_h2), int(start),
           int(stop), int(bool(forward)), float(omega), N.stream_ptr())
    _writeback(u, U)


def kaczmarz_sweep(u, u_coarse, start, stop, forward, proj_diag) -> None:
    """Kaczmarz projections onto the pair averages over [start//2, stop//2), in place."""
    dt = F.pick_dtype(u, u_coarse)
    U = F.to_field(u, dt)
    C = F.to_field(u_coarse, dt)
    F.same_batch(U, C)
    N.call("fmgsr_kaczmarz_sweep", dt, U.ptr(), C.ptr(), U.n, U.B, U.ld, int(start), int(stop),
           int(bool(forward)), float(proj_diag), N.stream_ptr())
    _writeback(u, U)


def _dev_i64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.int64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64)).to("cuda")


def smooth_patches(u_in, f, inv_h2, owned_lo, owned_hi, ext_lo, ext_hi, ns, omega, use_cr,
                   u_coarse, proj_diag):
    """Additive patch smoother over explicit patch arrays; returns a new field."""
    dt = F.pick_dtype(u_in, f)
    U = F.to_field(u_in, dt)
    Fd = F.to_field(f, dt)
    F.same_batch(U, Fd)
    olo, ohi, elo, ehi = (_dev_i64(a) for a in (owned_lo, owned_hi, ext_lo, ext_hi))
    P = int(olo.numel())
    out = torch.empty_like(U.t)
    uc_ptr = 0
    if use_cr:
        C = F.to_field(u_coarse, dt)
        F.same_batch(U, C)
        uc_ptr = C.ptr()
    scratch_ptr = off_ptr = 0
    sld = 0
    keep = []
    if ns >= 2 and P > 0:
        lo = torch.clamp(elo - 1, min=0)
        hi = torch.clamp(ehi + 1, max=U.n)
        rows = hi - lo
        soff = torch.cumsum(rows, 0) - rows
        total = int(rows.sum().item())
        sld = ((U.B + 31) // 32) * 32
        scratch = torch.empty((max(total, 1), sld), dtype=dt, device=U.t.device)
        keep = [scratch, soff]
        scratch_ptr, off_ptr = scratch.data_ptr(), soff.data_ptr()
    N.call("fmgsr_smooth_patches", dt, U.ptr(), Fd.ptr(), out.data_ptr(), U.n, U.B, U.ld,
           float(inv_h2), olo.data_ptr(), ohi.data_ptr(), elo.data_ptr(), ehi.data_ptr(), P,
           int(ns), float(omega), int(bool(use_cr)), uc_ptr, float(proj_diag), scratch_ptr,
           off_ptr, sld, N.stream_ptr())
    del keep
    return F.out(out, U)


def smooth_uniform(u_in, f, W, b, ns, omega, u_coarse=None, proj_diag=0.5, nonlinear=False):
    """Additive patch smoother over the uniform partition (W owned, b buffer)."""
    dt = F.pick_dtype(u_in, f)
    U = F.to_field(u_in, dt)
    Fd = F.to_field(f, dt)
    F.same_batch(U, Fd)
    out = torch.empty_like(U.t)
    uc_ptr = 0
    if u_coarse is not None:
        C = F.to_field(u_coarse, dt)
        F.same_batch(U, C)
        uc_ptr = C.ptr()
    scratch = None
    sld = 0
    if ns >= 2 or W % 2 or nonlinear:
        rows = int(N.lib().fmgsr_smooth_scratch_rows(U.n, W, b))
        sld = ((U.B + 31) // 32) * 32
        scratch = torch.empty((max(rows, 1), sld), dtype=dt, device=U.t.device)
    N.call("fmgsr_smooth_uniform_nl" if nonlinear else "fmgsr_smooth_uniform", dt, U.ptr(),
           Fd.ptr(), out.data_ptr(), U.n, U.B, U.ld, int(W),
           int(b), int(ns), float(omega), uc_ptr, float(proj_diag),
           scratch.data_ptr() if scratch is not None else 0, sld, N.stream_ptr())
    return F.out(out, U)
