"""TEST INFRASTRUCTURE ONLY -- reference-generated fixtures at FULL BASELINE
sizes, for single right-hand sides: the unmodified reference (numba lane,
geometry shim of gen_golden.py) solves one seeded RHS of config 2
(N = 2^16, 64 patches, b = 4, the bench workload's geometry), and
tests/golden/full_size.npz keeps the forcing and the SHA-256 of the solution
bytes; plus, at the full sizes of configs 2, 5 (three geometries) and 4
(N = 2^24), the SHA-256 of the reference's solution for a forcing every
machine regenerates bit for bit (hash_rhs), so no forcing is stored.

    python oracle/gen_golden_full.py
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from gen_golden import _import_reference, fourier_rhs, patch_rule

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "full_size.npz")


def hash_rhs(n, salt):
    """A forcing every machine generates bit for bit: an integer hash of the
    cell index mapped exactly onto [-0.5, 0.5) (no libm involved), so only the
    SHA-256 of the reference's solution needs committing at any size."""
    i = np.arange(n, dtype=np.uint64)
    h = (i * np.uint64(2654435761) + np.uint64(salt)) % np.uint64(1 << 32)
    return h.astype(np.float64) / float(1 << 32) - 0.5


def main(only=()):
    """Solve every case (or only the named hash cases, merged into the existing
    fixture file)."""
    _import_reference()
    from fmgsr import cycles, smoothers
    from fmgsr.mesh import HaloMode, build_hierarchy

    orig = smoothers._cached_patch_arrays
    g = {}
    cases = [("c2", 3, 16, 1, 1, 64, 4, 0)]
    if only:
        old = np.load(OUT)
        g.update({k: old[k] for k in old.files})
        cases = []
    for name, m0, m, n_sr, ns, P, b, seed in cases:
        smoothers._cached_patch_arrays = lambda nn, _mode, P=P, b=b: patch_rule(nn, P, b)
        try:
            cfg = cycles.SolverConfig(hierarchy=build_hierarchy(m0, m), n_sr=n_sr,
                                      smoother=smoothers.SmootherConfig(ns=ns,
                                                                        halo_mode=HaloMode.HALO2))
            f = fourier_rhs(2 ** m, seed, 0)
            sol, _ = cycles.fmg_solve(cfg, f)
        finally:
            smoothers._cached_patch_arrays = orig
        g[f"{name}/forcing"] = f
        g[f"{name}/params"] = np.array([m0, m, n_sr, ns, 2, P, b], dtype=np.int64)
        g[f"{name}/sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(sol, dtype=np.float64).tobytes()).digest(),
            dtype=np.uint8)
        g[f"{name}/head"] = sol[:64].copy()
        print(name, "solved; sha256", hashlib.sha256(sol.tobytes()).hexdigest()[:16])
    # full BASELINE sizes with the hash forcing: configs 2, 5 (three geometries) and 4
    hcases = [("h_c2", 3, 16, 1, 1, 64, 4, 1), ("h_c5_P256_b4", 3, 20, 1, 1, 256, 4, 2),
              ("h_c5_P16_b1", 3, 20, 1, 1, 16, 1, 3), ("h_c5_P1024_b8", 3, 20, 1, 1, 1024, 8, 4),
              ("h_c4", 3, 24, 1, 1, 4096, 8, 5),
              # config-3 geometry with the reference's (linear) operator, V(2,2)
              ("h_c3lin", 3, 20, 1, 2, 256, 4, 6),
              # config 2 at other SR depths
              ("h_c2_sr0", 3, 16, 0, 1, 64, 4, 7), ("h_c2_sr2", 3, 16, 2, 1, 64, 4, 8),
              # two more config-5 cells (round 2)
              ("h_c5_P64_b1", 3, 20, 1, 1, 64, 1, 9), ("h_c5_P16_b8", 3, 20, 1, 1, 16, 8, 10)]
    for name, m0, m, n_sr, ns, P, b, salt in hcases:
        if only and name not in only:
            continue
        smoothers._cached_patch_arrays = lambda nn, _mode, P=P, b=b: patch_rule(nn, P, b)
        try:
            cfg = cycles.SolverConfig(hierarchy=build_hierarchy(m0, m), n_sr=n_sr,
                                      smoother=smoothers.SmootherConfig(ns=ns,
                                                                        halo_mode=HaloMode.HALO2))
            sol, _ = cycles.fmg_solve(cfg, hash_rhs(2 ** m, salt))
        finally:
            smoothers._cached_patch_arrays = orig
        g[f"{name}/params"] = np.array([m0, m, n_sr, ns, 2, P, b, salt], dtype=np.int64)
        g[f"{name}/sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(sol, dtype=np.float64).tobytes()).digest(),
            dtype=np.uint8)
        g[f"{name}/head"] = sol[:64].copy()
        print(name, "solved; sha256", hashlib.sha256(sol.tobytes()).hexdigest()[:16])
    g["hash_cases"] = np.array([c[0] for c in hcases])
    np.savez_compressed(OUT, **g)
    print("wrote", os.path.normpath(OUT), os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    import sys

    main(tuple(sys.argv[1:]))
