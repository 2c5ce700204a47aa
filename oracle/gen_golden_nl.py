"""TEST INFRASTRUCTURE ONLY -- nonlinear FAS (BASELINE config 3) fixtures from
the reference's OWN driver.

The reference is linear only, so no reference output exists for
-u'' + u^3 = f.  This script pins the nonlinear path to the reference's
machinery instead: the UNMODIFIED reference package runs its own FMG driver
(cycles.fmg_solve / down_leg / up_leg, cycles.py:95-222), its own additive
patch assembly order, Kaczmarz pass and direction flips, with only the three
pointwise pieces swapped through the reference's injection points:

* a kernel lane ``numba_nl`` registered in ``fmgsr.backends._backends``
  (backends.py:22-47) with the lane's three callables; its ``gs_sweep`` is the
  pointwise Newton-GS step the builder's restatement defines
  (oracle/fmgsr_oracle.c orc_gs_sweep_nl):
      r = f_i - (inv_h2 * s_i + (u_i * u_i) * u_i),  J = diag_i + 3 (u_i * u_i),
      u_i += omega * r / J
  with s_i / diag_i exactly the reference's rows (_kernels_numba.py:15-36);
  ``kaczmarz_sweep`` and ``smooth_patches`` are the reference's own algorithm
  (_kernels_numba.py:39-92) calling that sweep;
* ``coarse_rhs`` (imported by name into cycles, cycles.py:22-28) with N(u) =
  L u + u^3 in the tau correction (stencils.py:108-125 with N for L);
* ``direct_solve`` (cycles.py and smoothers.py:210-225) by a Newton solve of
  N(u) = f from the reference's own linear solve, 10 steps, each a tridiagonal
  L + diag(3 u^2) solve in LAPACK ?ptsv order (dpttrf + dptts2).

Cases (tests/golden/nonlinear.npz):
* reduced sizes with the manufactured forcing f_s = s x(x+3)e^x +
  s^3 (x(1-x)e^x)^3 stored in the fixture (V(1,1) and V(2,2), SR depths 0-2,
  odd buffers);
* the full config-3 geometry (N = 2^20, 256 patches, b = 4, V(2,2), n_sr = 1)
  with a forcing every machine regenerates bit for bit (gen_golden_full.hash_rhs
  scaled by 64): only the SHA-256 of the solution is stored.

    python oracle/gen_golden_nl.py
"""

from __future__ import annotations

import hashlib
import os
import types

import numba as nb
import numpy as np

from gen_golden import _import_reference, patch_rule
from gen_golden_full import hash_rhs

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "nonlinear.npz")
NL_NEWTON = 10
HASH_SCALE = 64.0

_jit = {"nogil": True, "cache": False}


@nb.njit(**_jit)
def gs_sweep(u, f, inv_h2, start, stop, forward, omega):
    """Newton-GS pass over [start, stop): the reference's sweep order and rows
    (_kernels_numba.py:15-36), one pointwise Newton step per cell."""
    n = u.shape[0]
    if forward:
        i = start
        step = 1
    else:
        i = stop - 1
        step = -1
    for _ in range(stop - start):
        if i == 0:
            s = 3.0 * u[0] - u[1]
            diag = 3.0 * inv_h2
        elif i == n - 1:
            s = 3.0 * u[i] - u[i - 1]
            diag = 3.0 * inv_h2
        else:
            s = 2.0 * u[i] - u[i - 1] - u[i + 1]
            diag = 2.0 * inv_h2
        uu = u[i] * u[i]
        r = f[i] - (inv_h2 * s + uu * u[i])
        J = diag + 3.0 * uu
        u[i] += omega * r / J
        i += step


def _make_lane(ref_numba):
    """The lane module: Newton-GS sweep + the reference's Kaczmarz pass and patch
    assembly (same loop structure as _kernels_numba.smooth_patches)."""
    kaczmarz_sweep = ref_numba.kaczmarz_sweep

    @nb.njit(**_jit)
    def smooth_patches(u_in, f, inv_h2, owned_lo, owned_hi, ext_lo, ext_hi, ns, omega, use_cr,
                       u_coarse, proj_diag):
        n = u_in.shape[0]
        u_out = np.empty_like(u_in)
        scratch = u_in.copy()
        for p in range(owned_lo.shape[0]):
            ws = ext_lo[p]
            we = ext_hi[p]
            lo = ws - 1 if ws > 0 else 0
            hi = we + 1 if we < n else n
            scratch[lo:hi] = u_in[lo:hi]
            forward = True
            for _ in range(ns):
                if use_cr:
                    kaczmarz_sweep(scratch, u_coarse, ws, we, forward, proj_diag)
                gs_sweep(scratch, f, inv_h2, ws, we, forward, omega)
                forward = not forward
            u_out[owned_lo[p]:owned_hi[p]] = scratch[owned_lo[p]:owned_hi[p]]
        return u_out

    lane = types.ModuleType("fmgsr_lane_numba_nl")
    lane.gs_sweep = gs_sweep
    lane.kaczmarz_sweep = kaczmarz_sweep
    lane.smooth_patches = smooth_patches
    return lane


def install(fmgsr):
    """Swap the three pointwise pieces through the reference's injection points."""
    from fmgsr import _kernels_numba, backends, cycles, smoothers, stencils

    backends._backends["numba_nl"] = _make_lane(_kernels_numba)
    backends.set_backend("numba_nl")
    lin_direct = smoothers.direct_solve

    def apply_nonlinear(u):
        u = np.asarray(u, dtype=np.float64)
        return stencils.apply_operator(u) + (u * u) * u

    def coarse_rhs_nl(f_fine, u_fine):
        uc = stencils.restrict(u_fine)
        tau = apply_nonlinear(uc) - stencils.restrict(apply_nonlinear(u_fine))
        return stencils.restrict(f_fine) + tau

    def direct_solve_nl(f):
        f = np.asarray(f, dtype=np.float64)
        n = len(f)
        inv_h2 = float(4 ** stencils.level_of(f))
        u = lin_direct(f)  # the reference's own linear solve as the initial guess
        for _ in range(NL_NEWTON):
            r = f - apply_nonlinear(u)
            d = 2.0 * inv_h2 + 3.0 * (u * u)
            d[0] = 3.0 * inv_h2 + 3.0 * (u[0] * u[0])
            d[-1] = 3.0 * inv_h2 + 3.0 * (u[-1] * u[-1])
            e = np.full(n - 1, -inv_h2)
            for i in range(n - 1):  # dpttrf
                ei = e[i]
                e[i] = ei / d[i]
                d[i + 1] = d[i + 1] - e[i] * ei
            for i in range(1, n):  # dptts2
                r[i] = r[i] - r[i - 1] * e[i - 1]
            r[n - 1] = r[n - 1] / d[n - 1]
            for i in range(n - 2, -1, -1):
                r[i] = r[i] / d[i] - r[i + 1] * e[i]
            u = u + r
        return u

    cycles.coarse_rhs = coarse_rhs_nl
    cycles.direct_solve = direct_solve_nl
    smoothers.direct_solve = direct_solve_nl


def manufactured_nl(n, s):
    """f_s = s x(x+3)e^x + s^3 (x(1-x)e^x)^3 at cell centres."""
    x = (np.arange(n) + 0.5) / n
    ex = np.exp(x)
    u = x * (1.0 - x) * ex
    return s * x * (x + 3.0) * ex + s ** 3 * u ** 3


def main():
    fmgsr = _import_reference()
    install(fmgsr)
    from fmgsr import cycles, smoothers
    from fmgsr.mesh import HaloMode, build_hierarchy

    orig = smoothers._cached_patch_arrays

    def solve(m0, m, n_sr, ns, P, b, f):
        smoothers._cached_patch_arrays = lambda nn, _mode, P=P, b=b: patch_rule(nn, P, b)
        try:
            cfg = cycles.SolverConfig(hierarchy=build_hierarchy(m0, m), n_sr=n_sr,
                                      smoother=smoothers.SmootherConfig(ns=ns,
                                                                        halo_mode=HaloMode.HALO2))
            sol, _ = cycles.fmg_solve(cfg, f)
        finally:
            smoothers._cached_patch_arrays = orig
        return sol

    g = {}
    cases = [  # name, m0, m, n_sr, ns, P, b, s
        ("nl_c3small", 3, 12, 1, 2, 16, 4, 1.25),   # config-3 shape at reduced N
        ("nl_v11", 3, 11, 1, 1, 8, 2, 0.5),
        ("nl_sr0_oddb", 3, 12, 0, 2, 32, 3, 2.0),
        ("nl_sr2", 3, 12, 2, 2, 64, 1, 1.7),
        ("nl_v33", 3, 10, 1, 3, 8, 2, 1.0),
    ]
    for name, m0, m, n_sr, ns, P, b, s in cases:
        f = manufactured_nl(2 ** m, s)
        sol = solve(m0, m, n_sr, ns, P, b, f)
        g[f"{name}/params"] = np.array([m0, m, n_sr, ns, 2, P, b], dtype=np.int64)
        g[f"{name}/forcing"] = f
        g[f"{name}/solution"] = sol
        print(name, "solved", float(np.max(np.abs(sol))))
    g["cases"] = np.array([c[0] for c in cases])
    # the full config-3 geometry: N = 2^20, 256 patches, b = 4, V(2,2), one SR level
    hcases = [("h_c3", 3, 20, 1, 2, 256, 4, 11)]
    for name, m0, m, n_sr, ns, P, b, salt in hcases:
        f = HASH_SCALE * hash_rhs(2 ** m, salt)
        sol = solve(m0, m, n_sr, ns, P, b, f)
        g[f"{name}/params"] = np.array([m0, m, n_sr, ns, 2, P, b, salt], dtype=np.int64)
        g[f"{name}/scale"] = np.array(HASH_SCALE)
        g[f"{name}/sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(sol, dtype=np.float64).tobytes()).digest(),
            dtype=np.uint8)
        g[f"{name}/head"] = sol[:64].copy()
        print(name, "solved; sha256", hashlib.sha256(sol.tobytes()).hexdigest()[:16])
    g["hash_cases"] = np.array([c[0] for c in hcases])
    np.savez_compressed(OUT, **g)
    print("wrote", os.path.normpath(OUT), os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
