"""The full-multigrid FAS driver with segmental refinement (reference
cycles.py:31-253), on the device.

Two execution paths produce bit-identical results:

* the **native plan** (``plan.FmgPlan``): the level-visit schedule runs in
  C++, one fused sm_100a kernel per level visit, captured in a CUDA graph.
  ``fmg_solve`` takes it whenever no per-level state is requested;
* the **operator path** below: the reference's control flow verbatim
  (``down_leg``, ``up_leg``, ``expand_sr``), each operator one device kernel.
  It serves ``keep_state``, ``debug_sr`` and ``collect_diagnostics``, and the
  public ``down_leg`` / ``up_leg`` API.

Fields are CUDA tensors of shape (n,) or (n, B) ([cells][RHS]); numpy
forcing is accepted and the solution returned as numpy.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from . import _fields as F
from .mesh import Hierarchy
from .plan import get_plan, key_from_config
from .smoothers import CrContext, SmootherConfig, direct_solve, smooth_level
from .stencils import apply_operator, coarse_rhs, fas_correct, prolong_fmg, restrict


@dataclass(frozen=True)
class SolverConfig:
    """Hierarchy, SR depth and smoother (reference cycles.py:31-53)."""

    hierarchy: Hierarchy
    n_sr: int = 0
    smoother: SmootherConfig = field(default_factory=SmootherConfig)

    def __post_init__(self) -> None:
        m0, m = self.hierarchy.m0, self.hierarchy.m
        if m0 < 2:
            raise ValueError(
                f"m0 must be >= 2 (the high-order prolongation needs a coarse "
                f"field of >= 4 cells), got {m0}")
        if not 0 <= self.n_sr <= m - m0 - 1:
            raise ValueError(f"n_sr={self.n_sr} outside [0, {m - m0 - 1}] for m0={m0}, m={m}")

    def is_sr_level(self, level: int) -> bool:
        """True when ``level`` receives full updates (cycles.py:51-53)."""
        return level > self.hierarchy.m - self.n_sr


@dataclass
class CycleState:
    """Per-level device fields of one solve (cycles.py:56-67)."""

    u: dict
    f_work: dict
    f_orig: dict


@dataclass(frozen=True)
class LevelDiagnostics:
    level: int
    error_after_prolong: float
    error_after_cycle: float
    gamma: float
    residual_after_cycle: float


@dataclass
class Diagnostics:
    levels: list = field(default_factory=list)
    rel_error: float | None = None
    state: CycleState | None = None


def down_leg(k: int, state: CycleState, cfg: SolverConfig) -> CycleState:
    """Restrict, build the tau-corrected RHS, smooth, down to m0 (cycles.py:95-106)."""
    m0 = cfg.hierarchy.m0
    for l in range(k, m0, -1):
        u_fine = state.u[l]
        state.u[l - 1] = restrict(u_fine)
        state.f_work[l - 1] = coarse_rhs(state.f_work[l], u_fine, cfg.smoother.nonlinear)
        state.u[l - 1] = smooth_level(state.u[l - 1], state.f_work[l - 1], cfg.smoother, m0)
    return state


def up_leg(k: int, state: CycleState, cfg: SolverConfig) -> CycleState:
    """Correction update (non-SR) or full update + CR (SR), smooth (cycles.py:109-134)."""
    m0 = cfg.hierarchy.m0
    for l in range(m0, k):
        if not cfg.is_sr_level(l + 1):
            state.u[l + 1] = fas_correct(state.u[l + 1], state.u[l])
            state.u[l + 1] = smooth_level(state.u[l + 1], state.f_work[l + 1], cfg.smoother, m0)
        else:
            state.u[l + 1] = prolong_fmg(state.u[l])
            state.u[l + 1] = smooth_level(state.u[l + 1], state.f_work[l + 1], cfg.smoother, m0,
                                          cr=CrContext(u_coarse=state.u[l]))
    return state


def _norm_cols(x: torch.Tensor) -> torch.Tensor:
    return torch.linalg.vector_norm(x, dim=0)


def _algebraic_error(u, f) -> float:
    """Relative error against the exact discrete solve (cycles.py:247-253);
    the maximum over right-hand sides for a batch."""
    u_star = direct_solve(f)
    den = _norm_cols(u_star)
    num = _norm_cols(u - u_star)
    rel = torch.where(den == 0, _norm_cols(u), num / torch.where(den == 0, 1, den))
    return float(rel.max())


def _operator_path(cfg, forcing, collect_diagnostics, debug_sr):
    m0, m = cfg.hierarchy.m0, cfg.hierarchy.m
    f_orig = {m: forcing}
    for k in range(m - 1, m0 - 1, -1):
        f_orig[k] = restrict(f_orig[k + 1])
    state = CycleState(u={}, f_work={}, f_orig=f_orig)
    state.u[m0] = direct_solve(f_orig[m0], nonlinear=cfg.smoother.nonlinear)
    state.f_work[m0] = f_orig[m0]
    diag = Diagnostics()
    for k in range(m0, m):
        state.u[k + 1] = prolong_fmg(state.u[k])
        state.f_work[k + 1] = f_orig[k + 1]
        err_pre = _algebraic_error(state.u[k + 1], f_orig[k + 1]) if collect_diagnostics else 0.0
        state.u[k + 1] = smooth_level(state.u[k + 1], state.f_work[k + 1], cfg.smoother, m0)
        down_leg(k + 1, state, cfg)
        up_leg(k + 1, state, cfg)
        if collect_diagnostics:
            err_post = _algebraic_error(state.u[k + 1], f_orig[k + 1])
            res = f_orig[k + 1] - apply_operator(state.u[k + 1])
            resid = float(_norm_cols(res).max())
            gamma = err_post / err_pre if err_pre > 0.0 else math.nan
            diag.levels.append(LevelDiagnostics(k + 1, err_pre, err_post, gamma, resid))
        if debug_sr:
            for l in range(m0, k + 1):
                if cfg.is_sr_level(l):
                    state.u[l] = torch.full_like(state.u[l], math.nan)
    return state.u[m], diag, state


def fmg_solve(cfg: SolverConfig, forcing, exact=None, collect_diagnostics: bool = False,
              debug_sr: bool = False, keep_state: bool = False, fused: bool = True,
              coarse: int = -1, arith=None):
    """One full-multigrid pass (cycles.py:137-222) for one or B right-hand sides.

    ``forcing`` is (2**m,) or (2**m, B).  Returns (solution, Diagnostics).
    ``diag.rel_error`` is the plain relative L2 error against ``exact`` (the
    maximum over right-hand sides for a batch).  ``fused`` / ``coarse`` select
    the native plan's kernels (fused level visits; on-chip coarse hierarchy
    with automatic cutoff (-1), off (0) or cutoff level ``coarse - 1``); all
    choices give bit-identical results.  ``arith=torch.float64`` with a
    float32 forcing keeps every level field in fp32 and computes in fp64
    (native plan only).
    """
    m = cfg.hierarchy.m
    if F.length(forcing) != 2 ** m:
        raise ValueError(f"forcing has {F.length(forcing)} cells, expected {2 ** m}")
    dt = F.pick_dtype(forcing)
    Fd = F.to_field(forcing, dt)
    f = Fd.t
    if collect_diagnostics or debug_sr or keep_state:
        if arith is not None and arith != dt:
            raise ValueError("arith differs from the field dtype: native plan only "
                             "(no diagnostics / debug_sr / keep_state)")
        sol, diag, state = _operator_path(cfg, f, collect_diagnostics, debug_sr)
        if keep_state:
            diag.state = state
    else:
        plan = get_plan(key_from_config(cfg, Fd.B, dt, fused=fused, coarse=coarse, arith=arith))
        sol = plan.solve(f)
        diag = Diagnostics()
    if exact is not None:
        E = F.to_field(exact, dt).t
        diag.rel_error = float((_norm_cols(sol - E) / _norm_cols(E)).max())
    return F.out(sol, Fd), diag


def expand_sr(state: CycleState, cfg: SolverConfig):
    """Rebuild the finest field from the coarsest non-SR level (cycles.py:225-244)."""
    m0, m = cfg.hierarchy.m0, cfg.hierarchy.m
    v = state.u[m - cfg.n_sr]
    for l in range(m - cfg.n_sr, m):
        v_next = prolong_fmg(v)
        v = smooth_level(v_next, state.f_work[l + 1], cfg.smoother, m0, cr=CrContext(u_coarse=v))
    return v
