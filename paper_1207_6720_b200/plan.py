"""Native solve plan: one FMG-FAS(-SR) pass per call, scheduled in C++ and
replayed as a CUDA graph (``fmgsr_plan_*`` in include/fmgsr_cuda.h).

The plan owns its per-level device workspace (allocated once), fuses each
level visit of the reference driver (cycles.py:137-222) into one kernel where
eligible, and captures the whole cycle on first use for each (forcing,
solution) buffer pair.  ``FmgPlan.solve`` is what ``cycles.fmg_solve`` calls
on its fast path and what ``bench.py`` times.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import torch

from . import _native as N

GEOM_HALO, GEOM_GLOBAL, GEOM_PATCHES = 0, 1, 2


@dataclass(frozen=True)
class PlanKey:
    m0: int
    m: int
    n_sr: int
    ns: int
    geom_mode: int
    P: int
    b: int
    B: int
    dtype: torch.dtype
    omega: float
    fused: bool = True
    use_graph: bool = True
    coarse: int = -1  # on-chip coarse hierarchy: -1 auto, 0 off, k > 0 cutoff level k - 1
    nonlinear: bool = False  # -u'' + u^3 = f
    # arithmetic type (None: the field dtype); float32 fields with float64
    # arithmetic store every level in fp32 and compute in fp64 (dtype code 2)
    arith: torch.dtype | None = None


def dtype_code(key: "PlanKey") -> int:
    """The C ABI's dtype: 0 = f64, 1 = f32, 2 = f32 fields with f64 arithmetic."""
    if key.dtype == torch.float64:
        if key.arith not in (None, torch.float64):
            raise ValueError("float64 fields need float64 arithmetic")
        return 0
    if key.dtype != torch.float32:
        raise ValueError(f"unsupported field dtype {key.dtype}")
    if key.arith in (None, torch.float32):
        return 1
    if key.arith == torch.float64:
        return 2
    raise ValueError(f"unsupported arithmetic dtype {key.arith}")


def key_from_config(cfg, B: int, dtype: torch.dtype, fused: bool = True,
                    use_graph: bool = True, coarse: int = -1,
                    arith: torch.dtype | None = None) -> PlanKey:
    """PlanKey of a ``cycles.SolverConfig`` for a batch of B right-hand sides."""
    from .mesh import HaloMode

    sm = cfg.smoother
    if sm.n_patches is not None:
        mode, P = GEOM_PATCHES, sm.n_patches
        b = sm.buffer if sm.buffer is not None else (sm.halo_mode.halo or 0)
    elif sm.halo_mode is HaloMode.GLOBAL:
        mode, P, b = GEOM_GLOBAL, 1, 0
    else:
        mode, P = GEOM_HALO, 1
        b = sm.buffer if sm.buffer is not None else sm.halo_mode.halo
    return PlanKey(cfg.hierarchy.m0, cfg.hierarchy.m, cfg.n_sr, sm.ns, mode, int(P), int(b),
                   int(B), dtype, float(sm.omega), fused, use_graph, coarse, bool(sm.nonlinear),
                   None if arith == dtype else arith)


class FmgPlan:
    def __init__(self, key: PlanKey):
        N.require_cuda()
        self.key = key
        d = N.PlanDesc()
        d.m0, d.m, d.n_sr, d.ns = key.m0, key.m, key.n_sr, key.ns
        d.geom_mode = key.geom_mode
        d.dtype = dtype_code(key)
        d.P, d.b, d.B, d.ld = key.P, key.b, key.B, key.B
        d.omega = key.omega
        d.fused = int(key.fused)
        d.use_graph = int(key.use_graph)
        d.coarse = int(key.coarse)
        d.nonlinear = int(key.nonlinear)
        h = C.c_void_p()
        N.check(N.lib().fmgsr_plan_create(C.byref(d), C.byref(h)), "plan_create")
        self._h = h
        self.N = 2 ** key.m
        self.device = torch.cuda.current_device()
        # host-side plan state (graph map, level ping-pong) is not thread-safe
        self._lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().fmgsr_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def _check_io(self, forcing: torch.Tensor, out: torch.Tensor) -> None:
        k = self.key
        for name, t in (("forcing", forcing), ("solution", out)):
            if not t.is_cuda or t.dtype != k.dtype or tuple(t.shape) != (self.N, k.B) \
                    or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous {k.dtype} CUDA tensor of shape "
                                 f"({self.N}, {k.B})")
            if t.device.index != self.device:
                raise ValueError(f"{name} is on cuda:{t.device.index}, the plan on "
                                 f"cuda:{self.device}")

    def solve(self, forcing: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """One FMG pass for the (2**m, B) forcing; returns the (2**m, B) solution."""
        if out is None:
            out = torch.empty_like(forcing)
        self._check_io(forcing, out)
        with self._lock:
            N.check(N.lib().fmgsr_plan_solve(self._h, forcing.data_ptr(), out.data_ptr(),
                                             N.stream_ptr()), "plan_solve")
        return out

    def solve_functional(self, forcing: torch.Tensor, weights: torch.Tensor | None = None,
                         out: torch.Tensor | None = None) -> torch.Tensor:
        """One FMG pass that returns, per right-hand side, J = sum_i w_i u_i
        (``weights`` (2**m, B); None: the midpoint integral h * sum_i u_i)
        without ever storing the finest solution (fmgsr_plan_solve_functional)."""
        k = self.key
        if out is None:
            out = torch.empty(k.B, dtype=k.dtype, device=forcing.device)
        self._check_io(forcing, forcing)
        if weights is not None:
            self._check_io(weights, weights)
        if not out.is_cuda or out.dtype != k.dtype or out.numel() != k.B or not out.is_contiguous():
            raise ValueError(f"functional output must be a contiguous {k.dtype} CUDA tensor of {k.B}")
        with self._lock:
            N.check(N.lib().fmgsr_plan_solve_functional(
                self._h, forcing.data_ptr(), weights.data_ptr() if weights is not None else None,
                out.data_ptr(), N.stream_ptr()), "plan_solve_functional")
        return out

    def solve_host(self, forcing: torch.Tensor, out: torch.Tensor, chunks: int,
                   inputs_ready: bool = False) -> torch.Tensor:
        """End-to-end solve from HOST memory: ``forcing`` / ``out`` are pinned CPU
        tensors of shape (2**m, chunks * B); chunks of B right-hand sides are
        pipelined H2D / solve / D2H on separate streams.  Returns ``out`` once
        the current stream has reached the end of the pipeline.  With
        ``inputs_ready`` the host forcing is taken as ready at call time, so
        consecutive calls stream (FMGSR_HOST_INPUTS_READY)."""
        k = self.key
        for name, t in (("forcing", forcing), ("solution", out)):
            if t.is_cuda or t.dtype != k.dtype or tuple(t.shape) != (self.N, chunks * k.B) \
                    or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous host {k.dtype} tensor of shape "
                                 f"({self.N}, {chunks * k.B})")
        with self._lock:
            N.check(N.lib().fmgsr_plan_solve_host_ex(self._h, forcing.data_ptr(), out.data_ptr(),
                                                     chunks * k.B, chunks, int(bool(inputs_ready)),
                                                     N.stream_ptr()),
                    "plan_solve_host")
        return out

    def solve_timed(self, forcing: torch.Tensor, out: torch.Tensor):
        """Launch op by op with CUDA events per level visit; returns
        [(kind, level, ms)] with kind in top/down/up/direct."""
        self._check_io(forcing, out)
        cap = 8192
        ms = (C.c_float * cap)()
        lvl = (C.c_int32 * cap)()
        kind = (C.c_int32 * cap)()
        nv = C.c_int64()
        with self._lock:
            N.check(N.lib().fmgsr_plan_solve_timed(self._h, forcing.data_ptr(), out.data_ptr(),
                                                   N.stream_ptr(), ms, lvl, kind, cap,
                                                   C.byref(nv)), "plan_solve_timed")
        names = {0: "top", 1: "down", 2: "up", 3: "direct", 4: "cascade", 5: "coarse"}
        return [(names[kind[i]], lvl[i], ms[i]) for i in range(min(nv.value, cap))]

    def probe_ms(self) -> tuple[float, float]:
        """CUDA-event durations (ms) of the finest top / up visits of the last
        completed solve -- measured inside the replayed graph (-1: the finest
        level ran inside the on-chip coarse kernel).  Synchronise first."""
        t, u = C.c_float(), C.c_float()
        with self._lock:
            N.check(N.lib().fmgsr_plan_probe_ms(self._h, C.byref(t), C.byref(u)), "plan_probe_ms")
        return t.value, u.value

    def set_debug(self, poison: bool = True) -> None:
        """NaN-poison mode (fmgsr_plan_set_debug FMGSR_DEBUG_POISON): every solve
        fills the workspace fields with NaN first and the SR levels below each
        finished FMG step after it (the reference's debug_sr); results of a
        correct plan are unchanged."""
        with self._lock:
            N.check(N.lib().fmgsr_plan_set_debug(self._h, 1 if poison else 0), "plan_set_debug")

    def check_guards(self) -> int:
        """Changed guard bytes around the workspace arrays (plans created with
        FMGSR_GUARDS=1; -1 without guards)."""
        bad = C.c_int64()
        with self._lock:
            N.check(N.lib().fmgsr_plan_check_guards(self._h, C.byref(bad)), "plan_check_guards")
        return bad.value

    def info(self) -> dict:
        inf = N.PlanInfo()
        with self._lock:
            N.check(N.lib().fmgsr_plan_get_info(self._h, C.byref(inf)), "plan_get_info")
        return {
            "workspace_bytes": inf.workspace_bytes,
            "launches_per_solve": inf.launches_per_solve,
            "visits_per_solve": inf.visits_per_solve,
            "alg_bytes_per_solve": inf.alg_bytes_per_solve,
            "finest_visit_alg_bytes": inf.finest_visit_alg_bytes,
            "coarse_cutoff": inf.coarse_cutoff,
            "coarse_columns": inf.coarse_columns,
        }


_cache: dict[tuple, FmgPlan] = {}
_cache_lock = threading.Lock()


def get_plan(key: PlanKey) -> FmgPlan:
    """The cached plan for ``key`` on the current device and stream.  A plan's
    workspace, capture stream and graphs belong to the device that was current
    when it was built, and its per-solve state (level ping-pong, edge counters)
    is mutated by every solve, so plans are cached per (device, stream):
    solves queued on one stream are ordered, two streams never share a plan."""
    ck = (key, torch.cuda.current_device(), N.stream_ptr())
    with _cache_lock:
        p = _cache.get(ck)
        if p is None:
            if len(_cache) >= 8:
                _cache.pop(next(iter(_cache)))
            p = _cache[ck] = FmgPlan(key)
        return p
