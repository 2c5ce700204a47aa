"""BASELINE config 5 benchmark table: every (P, b) cell of the patch-geometry
sweep in fp64 and fp32 (N = 2^20, B = 256 seeded Fourier RHS, V(1,1), one SR
level): ms per cycle (CUDA events, graph replay, inputs resident), unknowns/s,
the finest-visit roofline fraction (T_20 + U_20 timed by event nodes inside the
replayed graph, 2.5 algorithmic words per cell each) and the whole-cycle
fraction (29 words per fine unknown), both of MEASURED_PEAKS.json hbm_gbs.

    python tools/config5_table.py [--steps 10] [--json out.json] [--md out.md]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1207_6720_b200 as fm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--json", default="")
ap.add_argument("--md", default="")
a = ap.parse_args()
peak, peak_src = bench.measured_peak()
m, B = 20, 256
n = 2 ** m
rows = []
for dt in (torch.float64, torch.float32):
    esz = 8 if dt == torch.float64 else 4
    f64, _ = fm.fourier_batch(n, fm.fourier_coefficients(B, seed=5), torch.float64,
                              with_exact=False)
    f = f64.to(dt)
    del f64
    sol = torch.empty_like(f)
    for P in (16, 64, 256, 1024):
        for b in (1, 2, 4, 8):
            cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                                  smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))
            plan = fm.FmgPlan(fm.key_from_config(cfg, B, dt))
            for _ in range(3):
                plan.solve(f, sol)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                plan.solve(f, sol)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            probes = []
            for _ in range(3):
                plan.solve(f, sol)
                torch.cuda.synchronize()
                probes.append(plan.probe_ms())
            t_ms = sum(p[0] for p in probes) / len(probes)
            u_ms = sum(p[1] for p in probes) / len(probes)
            alg_visit = 2.5 * n * B * esz
            info = plan.info()
            r = {"dtype": "f64" if esz == 8 else "f32", "P": P, "b": b, "ms_per_cycle": ms,
                 "unknowns_per_s": B * n / (ms / 1e3), "T_ms": t_ms, "U_ms": u_ms,
                 "finest_frac": 2 * alg_visit / ((t_ms + u_ms) / 1e3) / 1e9 / peak,
                 "T_frac": alg_visit / (t_ms / 1e3) / 1e9 / peak,
                 "U_frac": alg_visit / (u_ms / 1e3) / 1e9 / peak,
                 "whole_cycle_frac": info["alg_bytes_per_solve"] / (ms / 1e3) / 1e9 / peak,
                 "chains": P * B, "chain_cells": n // P + 2 * b}
            rows.append(r)
            print(json.dumps(r), flush=True)
            del plan
            torch.cuda.empty_cache()
    del f, sol
if a.json:
    with open(a.json, "w") as fh:
        json.dump({"peak_gbs": peak, "peak_source": peak_src, "rows": rows}, fh, indent=1)
if a.md:
    with open(a.md, "w") as fh:
        fh.write(f"# Config 5 sweep (N = 2^20, B = 256, V(1,1), n_sr = 1), B200\n\n"
                 f"Fractions of {peak:.1f} GB/s ({peak_src}); finest = T_20 + U_20 timed inside "
                 f"the replayed graph (2.5 words per cell each), whole = 29 words per unknown.\n\n"
                 "| dtype | P | b | ms/cycle | unknowns/s | T_20 ms | U_20 ms | finest frac | "
                 "whole frac | chains (P x B) | cells per chain |\n"
                 "|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            fh.write(f"| {r['dtype']} | {r['P']} | {r['b']} | {r['ms_per_cycle']:.2f} | "
                     f"{r['unknowns_per_s']:.3e} | {r['T_ms']:.3f} | {r['U_ms']:.3f} | "
                     f"{r['finest_frac']:.2f} | {r['whole_cycle_frac']:.2f} | {r['chains']} | "
                     f"{r['chain_cells']} |\n")
