"""Patch smoothers on the device (reference smoothers.py:22-225).

``smooth_level`` keeps the reference contract -- additive block-Jacobi over
the level's patches, ``ns`` repetitions of {Kaczmarz if CR, Gauss-Seidel}
with the direction flipped per repetition, owned write-back, direct solve at
the coarsest level -- and dispatches through the active kernel lane
(``backends.active()``, reference smoothers.py:194-207).  ``SmootherConfig``
adds the BASELINE geometry knobs: ``n_patches`` (P) and ``buffer`` (b).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Literal, Sequence

import numpy as np
import torch

from . import _fields as F
from . import _native as N
from . import backends, stencils
from .mesh import HaloMode, LevelGeometry, Patch, level_geometry, patch_arrays

Direction = Literal["forward", "backward"]


@dataclass(frozen=True)
class SmootherConfig:
    """Smoother parameters (reference smoothers.py:22-37).

    ns: inner sweeps per application (the nu of V(nu, nu)); halo_mode: the
    reference partition; omega: relaxation weight (1.0 in every study).
    n_patches / buffer: the P-patch geometry W_l = max(2, n_l/P) with a
    b-cell buffer; when n_patches is None the reference partition is used.
    nonlinear: solve -u'' + u^3 = f (BASELINE config 3) instead of -u'' = f;
    the reference is linear only, the restatement is oracle/fmgsr_oracle.c.
    """

    ns: int = 1
    halo_mode: HaloMode = HaloMode.HALO2
    omega: float = 1.0
    n_patches: int | None = None
    buffer: int | None = None
    nonlinear: bool = False  # -u'' + u^3 = f: Newton-GS smoother, Newton coarse solve

    def __post_init__(self) -> None:
        if self.ns < 1:
            raise ValueError(f"ns must be >= 1, got {self.ns}")
        if self.n_patches is not None:
            P = self.n_patches
            if P < 1 or P & (P - 1):
                raise ValueError(f"n_patches must be a power of two >= 1, got {P}")
        if self.buffer is not None and self.buffer < 0:
            raise ValueError(f"buffer must be >= 0, got {self.buffer}")

    def geometry(self, n: int) -> LevelGeometry:
        return level_geometry(n, self.halo_mode, self.n_patches, self.buffer)


@dataclass(frozen=True)
class CrContext:
    """Compatible-relaxation context (reference smoothers.py:40-53)."""

    u_coarse: object
    proj_diag: float = 0.5
    restrict_op: Callable = field(default=stencils.restrict, repr=False)


def _check_window(window, n):
    start, stop = window
    if not (0 <= start < stop <= n):
        raise ValueError(f"window {window} outside [0, {n})")
    return start, stop


def _check_direction(direction: str) -> bool:
    if direction not in ("forward", "backward"):
        raise ValueError(f"direction must be forward or backward, got {direction!r}")
    return direction == "forward"


def _copy(u, dt):
    if isinstance(u, torch.Tensor):
        return u.to(device="cuda", dtype=dt).clone()
    return np.array(u, dtype=np.float64, copy=True)


def patch_gs_sweep(u, f, window, direction: Direction = "forward"):
    """One Gauss-Seidel pass over ``window`` on a copy of ``u`` (smoothers.py:69-96)."""
    k = stencils.level_of(u)
    if F.length(f) != F.length(u):
        raise ValueError(f"field sizes differ: {F.length(u)} vs {F.length(f)}")
    start, stop = _check_window(window, F.length(u))
    forward = _check_direction(direction)
    out = _copy(u, F.pick_dtype(u, f))
    backends.active().gs_sweep(out, f, float(4 ** k), start, stop, forward, 1.0)
    return out


def kaczmarz_pass(u, cr: CrContext, window, direction: Direction = "forward"):
    """Project ``u`` onto the pair averages under ``window`` (smoothers.py:99-126)."""
    stencils.level_of(u)
    start, stop = _check_window(window, F.length(u))
    if start % 2 or stop % 2:
        raise ValueError(f"window {window} not aligned to coarse-cell pairs")
    forward = _check_direction(direction)
    out = _copy(u, F.pick_dtype(u, cr.u_coarse))
    backends.active().kaczmarz_sweep(out, cr.u_coarse, start, stop, forward, cr.proj_diag)
    return out


def smooth_level(u, f, cfg: SmootherConfig, m0: int, cr: CrContext | None = None,
                 patches: Sequence[Patch] | None = None):
    """Additive patch smoother on one level, direct solve at m0 (smoothers.py:129-207)."""
    k = stencils.level_of(u)
    if F.length(f) != F.length(u):
        raise ValueError(f"field sizes differ: {F.length(u)} vs {F.length(f)}")
    if k < m0:
        raise ValueError(f"level {k} below the coarsest level {m0}")
    if k == m0:
        return direct_solve(f, nonlinear=cfg.nonlinear)
    n = F.length(u)
    if cr is not None:
        if 2 * F.length(cr.u_coarse) != n:
            raise ValueError(
                f"coarse context size {F.length(cr.u_coarse)} does not parent {n}")
    lane = backends.active()
    if patches is None:
        g = cfg.geometry(n)
        return lane.smooth_uniform(u, f, g.W, g.b, cfg.ns, cfg.omega,
                                   cr.u_coarse if cr is not None else None,
                                   cr.proj_diag if cr is not None else 1.0,
                                   nonlinear=cfg.nonlinear)
    if cfg.nonlinear:
        raise ValueError("explicit patch lists are not supported for the nonlinear smoother")
    owned_lo, owned_hi, ext_lo, ext_hi = patch_arrays(list(patches))
    order = np.argsort(owned_lo)
    covered = np.all(owned_lo[order][1:] == owned_hi[order][:-1])
    if not (covered and owned_lo[order][0] == 0 and owned_hi[order][-1] == n):
        raise ValueError("explicit patch list does not tile the level")
    return lane.smooth_patches(u, f, float(4 ** k), owned_lo, owned_hi, ext_lo, ext_hi, cfg.ns,
                               cfg.omega, cr is not None,
                               cr.u_coarse if cr is not None else None,
                               cr.proj_diag if cr is not None else 1.0)


def direct_solve(f, nonlinear: bool = False):
    """Exact solve of the level operator (smoothers.py:210-225; LAPACK ?ptsv order).
    ``nonlinear``: Newton solve of L u + u^3 = f (n <= 64)."""
    stencils.level_of(f)
    dt = F.pick_dtype(f)
    Fd = F.to_field(f, dt)
    out = torch.empty_like(Fd.t)
    if nonlinear:
        if Fd.n > 64:
            raise ValueError(f"nonlinear direct solve supports at most 64 cells, got {Fd.n}")
        N.call("fmgsr_direct_solve_nl", dt, Fd.ptr(), out.data_ptr(), Fd.n, Fd.B, Fd.ld,
               N.stream_ptr())
    elif Fd.n <= 2048:
        N.call("fmgsr_direct_solve", dt, Fd.ptr(), out.data_ptr(), Fd.n, Fd.B, Fd.ld,
               N.stream_ptr())
    else:
        ws = torch.empty(2 * Fd.n, dtype=dt, device=Fd.t.device)
        N.call("fmgsr_direct_solve_ws", dt, Fd.ptr(), out.data_ptr(), Fd.n, Fd.B, Fd.ld,
               ws.data_ptr(), N.stream_ptr())
    return F.out(out, Fd)
