"""TEST INFRASTRUCTURE ONLY -- generate golden vectors from the real reference.

Runs the UNMODIFIED reference package ``fmgsr`` (``/root/reference/pkg/src``,
default numba lane) on seeded inputs and writes ``tests/golden/golden.npz``.
The oracle (``oracle/fmgsr_oracle.c``) and, through it, the CUDA path are
pinned to these vectors bit for bit.  ``/root/reference`` only exists in the
build container, so the fixtures are committed; this script documents how
they were made:

    python oracle/gen_golden.py

The generalised (P patches, b-cell buffer) geometry is installed with the
shim SURVEY.md section 8(c) describes: ``fmgsr.smoothers._cached_patch_arrays``
is replaced by a function returning the patch arrays of the rule
W_l = max(2, n_l / P) (``smooth_level`` looks the name up at call time,
reference smoothers.py:172-175).
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "golden.npz")


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_cache_"))
    sys.path.insert(0, REF)
    import fmgsr  # noqa: F401
    from fmgsr import backends

    backends.set_backend("numba")
    return fmgsr


def patch_rule(n, P, b):
    """W = max(2, n/P) owned cells per patch, b-cell buffer clamped to [0, n)."""
    W = max(2, n // P)
    os_ = np.arange(0, n, W, dtype=np.int64)
    oe = os_ + W
    return os_, oe, np.maximum(0, os_ - b), np.minimum(n, oe + b)


def fourier_rhs(n, seed, r, K=32):
    """a_k = N(0,1)/k^2 from default_rng([seed, r]); f = sum a_k sin(k pi x)."""
    rng = np.random.default_rng([seed, r])
    a = rng.standard_normal(K) / np.arange(1, K + 1) ** 2
    x = (np.arange(n) + 0.5) / n
    f = np.zeros(n)
    for k in range(1, K + 1):
        f += a[k - 1] * np.sin(k * np.pi * x)
    return f


def main():
    fmgsr = _import_reference()
    from fmgsr import cycles, smoothers, stencils
    from fmgsr.mesh import HaloMode, build_hierarchy, partition, patch_arrays

    orig_cached = smoothers._cached_patch_arrays
    g = {}
    rng = np.random.default_rng(20260)

    def put(name, **arrays):
        for k, v in arrays.items():
            g[f"{name}/{k}"] = np.asarray(v)

    # --- stencils (stencils.py:27-125) --------------------------------------
    for n in (4, 8, 64):
        u = rng.standard_normal(n)
        f = rng.standard_normal(n)
        put(f"stencil_n{n}", u=u, f=f,
            apply_operator=stencils.apply_operator(u),
            restrict=stencils.restrict(u),
            prolong_correction=stencils.prolong_correction(u),
            prolong_fmg=stencils.prolong_fmg(u) if n >= 4 else np.zeros(0),
            tau=stencils.tau_correction(u),
            coarse_rhs=stencils.coarse_rhs(f, u))

    # --- direct solve (smoothers.py:210-225) ----------------------------------
    for n in (4, 8, 16, 64):
        fs = rng.standard_normal((16, n)) * 10.0 ** rng.uniform(-3, 3, size=(16, 1))
        put(f"direct_n{n}", f=fs, u=np.stack([smoothers.direct_solve(f) for f in fs]))

    # --- sweeps (_kernels_numba.py:15-57) -------------------------------------
    kern = fmgsr.backends.active()
    n = 32
    u = rng.standard_normal(n)
    f = rng.standard_normal(n)
    uc = rng.standard_normal(n // 2)
    inv_h2 = float(4 ** 5)
    windows = [(0, 32), (2, 30), (5, 27), (1, 5), (0, 1), (31, 32), (7, 8)]
    gs_out, kz_out = [], []
    for (a, b) in windows:
        for fw in (True, False):
            x = u.copy()
            kern.gs_sweep(x, f, inv_h2, a, b, fw, 1.0)
            gs_out.append(x)
            y = u.copy()
            kern.kaczmarz_sweep(y, uc, a, b, fw, 0.5)
            kz_out.append(y)
    put("sweeps", u=u, f=f, uc=uc, inv_h2=inv_h2, windows=np.array(windows),
        gs=np.stack(gs_out), kaczmarz=np.stack(kz_out))

    # --- smooth_patches via smooth_level (smoothers.py:129-207) ---------------
    n = 64
    u = rng.standard_normal(n)
    f = rng.standard_normal(n)
    uc = stencils.restrict(u) + 0.1 * rng.standard_normal(n // 2)
    cases = []
    outs = []
    for mode in ("2", "4", "global"):
        for ns in (1, 2, 3):
            for cr in (0, 1):
                cfg = smoothers.SmootherConfig(ns=ns, halo_mode=HaloMode(mode))
                ctx = smoothers.CrContext(uc) if cr else None
                outs.append(smoothers.smooth_level(u, f, cfg, 2, cr=ctx))
                cases.append(("halo", mode, 0, 0, ns, cr))
    # generalised geometry, including odd buffers (numba semantics, SURVEY trap 1)
    for P in (2, 4, 8, 32):
        for b in (0, 1, 2, 3, 4, 8):
            for ns in (1, 2):
                for cr in (0, 1):
                    olo, ohi, elo, ehi = patch_rule(n, P, b)
                    outs.append(kern.smooth_patches(
                        u, f, float(4 ** 6), olo, ohi, elo, ehi, ns, 1.0, bool(cr),
                        uc if cr else np.empty(0), 0.5))
                    cases.append(("patches", "", P, b, ns, cr))
    put("smooth", u=u, f=f, uc=uc,
        cases=np.array([[0 if c[0] == "halo" else 1,
                         {"2": 2, "4": 4, "global": -1, "": 0}[c[1]], c[2], c[3], c[4], c[5]]
                        for c in cases], dtype=np.int64),
        out=np.stack(outs))

    # --- whole FMG solves (cycles.py:137-222) ----------------------------------
    fmg_cases = []

    def run(name, m0, m, n_sr, ns, geom, forcing):
        kind, P, b, mode = geom
        if kind == "patches":
            smoothers._cached_patch_arrays = lambda nn, _mode: patch_rule(nn, P, b)
            hm = HaloMode.HALO2
        else:
            smoothers._cached_patch_arrays = orig_cached
            hm = HaloMode(mode)
        try:
            cfg = cycles.SolverConfig(
                hierarchy=build_hierarchy(m0, m), n_sr=n_sr,
                smoother=smoothers.SmootherConfig(ns=ns, halo_mode=hm))
            sol, _ = cycles.fmg_solve(cfg, forcing)
        finally:
            smoothers._cached_patch_arrays = orig_cached
        put(name, forcing=forcing, solution=sol,
            params=np.array([m0, m, n_sr, ns,
                             {"patches": 2, "halo": 0, "global": 1}[kind], P, b], dtype=np.int64))
        fmg_cases.append(name)

    from fmgsr.problem import manufactured_rhs
    # the reference's own dense-replay configurations (test_cycles.py:297-351)
    for i, (mode, ns, n_sr) in enumerate([("2", 1, 0), ("2", 2, 2), ("4", 1, 1), ("global", 2, 0)]):
        kind = "global" if mode == "global" else "halo"
        run(f"fmg_ref{i}", 2, 5, n_sr, ns, (kind, 0, int(mode) if kind == "halo" else 0, mode),
            manufactured_rhs(32))
    # config 1 (BASELINE.json configs[0]): N=2^10, m0=3, 4 patches, b=2, n_sr=1, V(1,1)
    x = (np.arange(1024) + 0.5) / 1024
    run("fmg_config1", 3, 10, 1, 1, ("patches", 4, 2, ""), np.pi ** 2 * np.sin(np.pi * x))
    # config-2 geometry (P=64, b=4) at reduced N, Fourier RHS
    for n_sr in (0, 1, 2):
        run(f"fmg_c2_m12_sr{n_sr}", 3, 12, n_sr, 1, ("patches", 64, 4, ""), fourier_rhs(4096, 0, n_sr))
    # config-5 geometry sweep at reduced N (odd buffer included)
    for P, b in ((16, 1), (16, 8), (64, 2), (256, 4), (1024, 8)):
        run(f"fmg_c5_m12_P{P}_b{b}", 3, 12, 1, 1, ("patches", P, b, ""), fourier_rhs(4096, 5, P + b))
    # V(2,2)
    run("fmg_ns2_m10", 3, 10, 1, 2, ("patches", 16, 4, ""), fourier_rhs(1024, 3, 0))
    run("fmg_ns2_m10_sr0", 3, 10, 0, 2, ("patches", 8, 3, ""), fourier_rhs(1024, 3, 1))
    # config-4 geometry (P=4096, b=8) at N=2^14
    run("fmg_c4_m14", 3, 14, 1, 1, ("patches", 4096, 8, ""), fourier_rhs(16384, 4, 0))
    g["fmg_cases"] = np.array(fmg_cases)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {len(g)} arrays to {os.path.normpath(OUT)}")


if __name__ == "__main__":
    main()
