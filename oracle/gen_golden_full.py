"""TEST INFRASTRUCTURE ONLY -- reference-generated fixtures at FULL BASELINE
sizes, for single right-hand sides: the unmodified reference (numba lane,
geometry shim of gen_golden.py) solves one seeded RHS of config 2
(N = 2^16, 64 patches, b = 4, the bench workload's geometry), and
tests/golden/full_size.npz keeps the forcing and the SHA-256 of the solution
bytes.  (A config-5 RHS at N = 2^20 would add 6 MB of forcing to the
repository; config 5 is pinned through the oracle at full size instead.)

    python oracle/gen_golden_full.py
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from gen_golden import _import_reference, fourier_rhs, patch_rule

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "full_size.npz")


def main():
    _import_reference()
    from fmgsr import cycles, smoothers
    from fmgsr.mesh import HaloMode, build_hierarchy

    orig = smoothers._cached_patch_arrays
    g = {}
    cases = [("c2", 3, 16, 1, 1, 64, 4, 0)]
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
    np.savez_compressed(OUT, **g)
    print("wrote", os.path.normpath(OUT), os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
