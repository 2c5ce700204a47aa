"""Model problems and synthetic right-hand sides (reference problem.py:13-77,
plus the seeded generators of the BASELINE configurations).

The reference's manufactured problem (odd sine modes with 1/j weights) is
kept for API parity.  The BASELINE workloads use seeded Fourier forcings
(SURVEY 8(d)): per RHS r, a_k = N(0,1)/k^2 from numpy's
``default_rng([seed, r])``, k = 1..32, f = sum a_k sin(k pi x), with exact
continuum solution u* = sum a_k sin(k pi x)/(k pi)^2 at cell centres
x_i = (i + 1/2)/N.  Large batches are generated on the device directly in
the [cells][RHS] layout (``fmgsr_fourier_rhs_*``), outside any timed region.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _fields as F
from . import _native as N
from .smoothers import direct_solve
from .stencils import level_of


def default_nmodes(n: int) -> int:
    return max(1, n // 16)


def cell_centers(n: int) -> np.ndarray:
    """x_i = (i + 1/2)/n (problem.py:18-20)."""
    return (np.arange(n) + 0.5) / n


def manufactured_rhs(n: int, nmodes: int | None = None) -> np.ndarray:
    """sum over odd j <= nmodes of sin(j pi x)/j (problem.py:23-33); host numpy."""
    if nmodes is None:
        nmodes = default_nmodes(n)
    if nmodes < 1:
        raise ValueError(f"nmodes must be >= 1, got {nmodes}")
    x = cell_centers(n)
    f = np.zeros(n)
    for j in range(1, nmodes + 1, 2):
        f += np.sin(j * np.pi * x) / j
    return f


def exact_solution(n: int, nmodes: int | None = None) -> np.ndarray:
    """Continuum solution of the manufactured problem (problem.py:36-46)."""
    if nmodes is None:
        nmodes = default_nmodes(n)
    if nmodes < 1:
        raise ValueError(f"nmodes must be >= 1, got {nmodes}")
    x = cell_centers(n)
    u = np.zeros(n)
    for j in range(1, nmodes + 1, 2):
        u += np.sin(j * np.pi * x) / (j * (j * np.pi) ** 2)
    return u


def rel_l2_error(u, u_ref) -> float:
    """Plain relative 2-norm error (problem.py:49-58); max over RHS for a batch."""
    if F.length(u) != F.length(u_ref):
        raise ValueError(f"field sizes differ: {F.length(u)} vs {F.length(u_ref)}")
    if not isinstance(u, torch.Tensor) and not isinstance(u_ref, torch.Tensor) \
            and np.ndim(u) == 1 and np.ndim(u_ref) == 1:
        # host vectors: numpy's norm, the reference's exact reduction
        a1 = np.asarray(u, dtype=np.float64)
        b1 = np.asarray(u_ref, dtype=np.float64)
        den1 = float(np.linalg.norm(b1))
        if den1 == 0.0:
            raise ValueError("reference field has zero norm")
        return float(np.linalg.norm(a1 - b1)) / den1
    a = torch.as_tensor(np.asarray(u) if not isinstance(u, torch.Tensor) else u,
                        dtype=torch.float64)
    b = torch.as_tensor(np.asarray(u_ref) if not isinstance(u_ref, torch.Tensor) else u_ref,
                        dtype=torch.float64).to(a.device)
    a = a.reshape(a.shape[0], -1)
    b = b.reshape(b.shape[0], -1)
    den = torch.linalg.vector_norm(b, dim=0)
    if bool((den == 0).any()):
        raise ValueError("reference field has zero norm")
    return float((torch.linalg.vector_norm(a - b, dim=0) / den).max())


def direct_fine_solve(forcing):
    """Exact solve of the level operator at the forcing's level (problem.py:61-77).

    Like the reference, an algorithm independent of the coarse solve
    (smoothers.direct_solve, L D L^T in LAPACK ?ptsv order): the general
    banded LU of scipy's solve_banded((1, 1)) -> LAPACK dgbsv (dgbtf2 + dgbtrs)
    in that operation order on the device (fmgsr_banded_lu_solve), one thread
    per right-hand side, so the two can cross-check each other."""
    level_of(forcing)
    dt = F.pick_dtype(forcing)
    Fd = F.to_field(forcing, dt)
    out = torch.empty_like(Fd.t)
    ws = torch.empty(2 * Fd.n, dtype=dt, device=Fd.t.device)
    piv = torch.zeros(1, dtype=torch.int32, device=Fd.t.device)
    N.call("fmgsr_banded_lu_solve", dt, Fd.ptr(), out.data_ptr(), Fd.n, Fd.B, Fd.ld,
           ws.data_ptr(), piv.data_ptr(), N.stream_ptr())
    if int(piv.item()):
        raise RuntimeError("direct_fine_solve: the pivot search would swap rows "
                           "(not the reference's operator)")
    return F.out(out, Fd)


# ---- BASELINE generators --------------------------------------------------------------

def fourier_coefficients(B: int, seed: int = 0, K: int = 32) -> np.ndarray:
    """a[r, k-1] = N(0,1)/k^2 from default_rng([seed, r])."""
    a = np.empty((B, K))
    kk = np.arange(1, K + 1, dtype=np.float64) ** 2
    for r in range(B):
        a[r] = np.random.default_rng([seed, r]).standard_normal(K) / kk
    return a


def fourier_batch(n: int, coef: np.ndarray, dtype: torch.dtype = torch.float64,
                  with_exact: bool = True):
    """(f, u*) of shape (n, B) on the device for coefficient rows coef[B, K]."""
    N.require_cuda()
    B, K = coef.shape
    c = torch.as_tensor(np.ascontiguousarray(coef, dtype=np.float64), device="cuda")
    f = torch.empty((n, B), dtype=dtype, device="cuda")
    u = torch.empty((n, B), dtype=dtype, device="cuda") if with_exact else None
    N.call("fmgsr_fourier_rhs", dtype, c.data_ptr(), int(K), n, B, B, f.data_ptr(),
           u.data_ptr() if u is not None else 0, N.stream_ptr())
    return f, u


def sine_problem(n: int, B: int = 1, dtype: torch.dtype = torch.float64):
    """Config 1: f = pi^2 sin(pi x), u* = sin(pi x)."""
    coef = np.full((B, 1), np.pi ** 2)
    return fourier_batch(n, coef, dtype)


def nonlinear_scales(B: int, seed: int = 0) -> np.ndarray:
    """Config 3 amplitudes s_r ~ U[0.5, 2] from default_rng([seed, r])."""
    return np.array([np.random.default_rng([seed, r]).uniform(0.5, 2.0) for r in range(B)])


def nonlinear_batch(n: int, scales: np.ndarray, dtype: torch.dtype = torch.float64):
    """Config 3: u = s x(1-x)e^x, f = -u'' + u^3 = s x(x+3)e^x + u^3, (n, B) on device."""
    N.require_cuda()
    B = len(scales)
    s = torch.as_tensor(np.asarray(scales, dtype=np.float64), device="cuda")
    f = torch.empty((n, B), dtype=dtype, device="cuda")
    u = torch.empty((n, B), dtype=dtype, device="cuda")
    N.call("fmgsr_nonlinear_rhs", dtype, s.data_ptr(), n, B, B, f.data_ptr(), u.data_ptr(),
           N.stream_ptr())
    return f, u
