"""Matrix-free level operators on the device (reference stencils.py:18-125).

Each function validates like the reference, runs one sm_100a kernel over all
right-hand sides of the field, and returns a new field.  Operation order is
the reference's, so float64 results are bit-identical.
"""

from __future__ import annotations

import torch

from . import _fields as F
from . import _native as N


def level_of(values) -> int:
    """Level exponent of a field, validating the power-of-two length (stencils.py:18-24)."""
    n = F.length(values)
    k = max(n, 1).bit_length() - 1
    if n < 2 or 2 ** k != n:
        raise ValueError(f"field length must be a power of two >= 2, got {n}")
    return k


def _unary(name: str, x, out_rows) -> object:
    dt = F.pick_dtype(x)
    X = F.to_field(x, dt)
    out = F.empty_like_rows(X, out_rows(X.n))
    # every unary entry point takes the INPUT length (n, n_fine or n_coarse)
    N.call(name, dt, X.ptr(), out.data_ptr(), X.n, X.B, X.ld, N.stream_ptr())
    return F.out(out, X)


def apply_operator(u):
    """L_k u: rows (1/h^2)[-1, 2, -1], boundary rows (1/h^2)[3, -1] (stencils.py:27-36)."""
    level_of(u)
    return _unary("fmgsr_apply_operator", u, lambda n: n)


def restrict(u_fine):
    """Pair average 0.5 (u[2j] + u[2j+1]) (stencils.py:39-47)."""
    level_of(u_fine)
    return _unary("fmgsr_restrict", u_fine, lambda n: n // 2)


def prolong_correction(c_coarse):
    """1/4 [1, 3, 3, 1] with half-weight end rows (stencils.py:50-64)."""
    level_of(c_coarse)
    return _unary("fmgsr_prolong_correction", c_coarse, lambda n: 2 * n)


def prolong_fmg(c_coarse):
    """4th-order FMG prolongation with 4 special rows per end (stencils.py:67-105)."""
    level_of(c_coarse)
    n = F.length(c_coarse)
    if n < 4:
        raise ValueError(f"prolong_fmg needs a coarse field of >= 4 cells, got {n}")
    return _unary("fmgsr_prolong_fmg", c_coarse, lambda n: 2 * n)


def tau_correction(u_fine):
    """L_H(R u) - R(L_h u) (stencils.py:108-116)."""
    level_of(u_fine)
    level_of(range(F.length(u_fine) // 2))
    return _unary("fmgsr_tau_correction", u_fine, lambda n: n // 2)


def coarse_rhs(f_fine, u_fine, nonlinear: bool = False):
    """R f + tau(u) (stencils.py:119-125); ``nonlinear``: tau of N(u) = L u + u^3."""
    if F.length(f_fine) != F.length(u_fine):
        raise ValueError(
            f"forcing and solution sizes differ: {F.length(f_fine)} vs {F.length(u_fine)}")
    level_of(u_fine)
    level_of(range(F.length(u_fine) // 2))
    dt = F.pick_dtype(f_fine, u_fine)
    Fd = F.to_field(f_fine, dt)
    U = F.to_field(u_fine, dt)
    F.same_batch(Fd, U)
    out = F.empty_like_rows(U, U.n // 2)
    N.call("fmgsr_coarse_rhs_nl" if nonlinear else "fmgsr_coarse_rhs", dt, Fd.ptr(), U.ptr(),
           out.data_ptr(), U.n, U.B, U.ld, N.stream_ptr())
    return F.out(out, U)


def fas_correct(u_fine, u_coarse):
    """u + prolong_correction(u_H - restrict(u)), the FAS correction update
    of the up leg (cycles.py:120-121), in one kernel."""
    if 2 * F.length(u_coarse) != F.length(u_fine):
        raise ValueError("coarse field does not parent the fine field")
    level_of(u_fine)
    dt = F.pick_dtype(u_fine, u_coarse)
    U = F.to_field(u_fine, dt)
    C = F.to_field(u_coarse, dt)
    F.same_batch(U, C)
    out = torch.empty_like(U.t)
    N.call("fmgsr_fas_correct", dt, U.ptr(), C.ptr(), out.data_ptr(), U.n, U.B, U.ld,
           N.stream_ptr())
    return F.out(out, U)
