"""Randomised parity sweep (test infrastructure): N seeded random
configurations of the whole solve -- geometry (P, odd/even buffers up to 12),
V(ns,ns) with ns 1..3, SR depth, linear / nonlinear, batch shapes (scalar
lanes, two-column lanes, ragged), coarse-level placement -- each checked bit
for bit against the C oracle on every column.  Prints one line per failure
and a summary; exit code 1 if anything differs.

    python tools/fuzz_parity.py [--n 400] [--seed 7]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1207_6720_b200 as fm  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=400)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--fp32", action="store_true",
                    help="fp32: two-column-lane batches (B = 64k) against the same columns "
                         "solved in 32-column batches (scalar lanes), bitwise")
    a = ap.parse_args()
    O.build()
    rng = np.random.default_rng(a.seed)
    bad = tested = 0
    for i in range(a.n):
        m0 = int(rng.integers(2, 4))
        m = int(rng.integers(m0 + 2, 13))
        P = int(2 ** rng.integers(0, m - 1))
        b = int(rng.integers(0, 13))
        ns = int(rng.choice([1, 1, 2, 3]))
        n_sr = int(rng.integers(0, m - m0))
        B = int(rng.choice([1, 2, 31, 32, 64, 65, 127, 128, 192, 256]))
        coarse = int(rng.choice([-1, -1, 0, m0 + 1, m - 1, m, m + 1]))
        nl = bool(rng.integers(0, 4) == 0)
        fused = bool(rng.integers(0, 5) != 0)
        try:
            cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr,
                                  smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b,
                                                             nonlinear=nl))
        except ValueError:
            continue
        tested += 1
        if nl:
            f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=i))
        else:
            f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=i))
        if a.fp32:
            import torch

            B2 = 64 * max(1, B // 64)
            f = (f if f.shape[1] >= B2 else f.repeat(1, B2 // f.shape[1] + 1))[:, :B2]
            f = f.float().contiguous()
            got = fm.fmg_solve(cfg, f, coarse=coarse, fused=fused)[0].cpu().numpy()
            want = torch.cat([fm.fmg_solve(cfg, f[:, c:c + 32].contiguous(), coarse=coarse,
                                           fused=fused)[0] for c in range(0, B2, 32)],
                             dim=1).cpu().numpy()
        else:
            oc = O.make_cfg(m0, m, n_sr, ns, O.GEOM_PATCHES, P, b, nonlin=nl)
            want = O.fmg_solve_batch(oc, np.ascontiguousarray(f.cpu().numpy().T), nthreads=16).T
            got = fm.fmg_solve(cfg, f, coarse=coarse, fused=fused)[0].cpu().numpy()
        if not np.array_equal(got, want, equal_nan=True):
            bad += 1
            cols = np.where((got != want).any(axis=0))[0]
            print(f"MISMATCH case {i}: m0={m0} m={m} P={P} b={b} ns={ns} n_sr={n_sr} B={B} "
                  f"coarse={coarse} nl={nl} fused={fused} columns={cols[:8].tolist()}", flush=True)
    print(f"fuzz_parity: {tested} valid configurations of {a.n} drawn, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
