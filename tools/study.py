"""The reference's convergence study (harness.run_full_study) on the GPU at
large N: every (halo, ns, n_sr) curve of the 24-configuration grid from
m_min to m_max, CSV in the reference schema plus each curve's observed order.

    python tools/study.py [--m-min 4] [--m-max 20] [--out study.csv]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import logging  # noqa: E402

from paper_1207_6720_b200 import harness  # noqa: E402

logging.basicConfig(level=logging.INFO, format="%(asctime)s %(message)s")

ap = argparse.ArgumentParser()
ap.add_argument("--m-min", type=int, default=4)
ap.add_argument("--m-max", type=int, default=20)
ap.add_argument("--out", default="study.csv")
a = ap.parse_args()
t0 = time.perf_counter()
recs = harness.run_full_study(a.m_min, a.m_max)
wall = time.perf_counter() - t0
harness.emit_csv(recs, a.out)
curves = {}
for r in recs:
    curves.setdefault((r.halo_mode.label, r.ns, r.n_sr), []).append(r)
print(f"{len(recs)} solves in {wall:.1f} s wall; device time {sum(r.runtime_ms for r in recs):.1f} ms")
for (halo, ns, n_sr), rs in curves.items():
    if len(rs) >= 3:
        print(f"halo={halo:6s} ns={ns} n_sr={n_sr}: order {harness.observed_order(rs):.3f}, "
              f"error at n={rs[-1].n}: {rs[-1].rel_error:.3e} (quad_ref {rs[-1].quad_ref:.3e})")
