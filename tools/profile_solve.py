"""Run a few FMG solves of a bench workload op by op (no CUDA graph) for ncu:
every level visit is its own launch in a deterministic order, so
``ncu -k regex:<kernel> --launch-skip K -c 1`` picks one visit.

    python tools/profile_solve.py [--workload config2] [--solves 1] [--graph] [--unfused]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1207_6720_b200 as fm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config2")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--unfused", action="store_true")
ap.add_argument("--P", type=int, default=0, help="override the patch count")
ap.add_argument("--b", type=int, default=-1, help="override the buffer")
ap.add_argument("--shards", type=int, default=0, help="run shard --rank of an S-way split")
ap.add_argument("--rank", type=int, default=0)
a = ap.parse_args()
w = dict(bench.WORKLOADS[a.workload])
if a.P:
    w["P"] = a.P
if a.b >= 0:
    w["b"] = a.b
dt = torch.float64 if w["dtype"] == "f64" else torch.float32
nl = bool(w.get("nonlinear", False))
cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], w["m"]), n_sr=w["n_sr"],
                      smoother=fm.SmootherConfig(ns=w["ns"], n_patches=w["P"], buffer=w["b"],
                                                 nonlinear=nl))
if not a.shards:
    plan = fm.get_plan(fm.key_from_config(cfg, w["B"], dt, fused=not a.unfused, arith=bench._arith(w),
                                          use_graph=a.graph))
if nl:
    f, _ = fm.nonlinear_batch(2 ** w["m"], fm.nonlinear_scales(w["B"]), dt)
else:
    f, _ = fm.fourier_batch(2 ** w["m"], fm.fourier_coefficients(w["B"]), dt, with_exact=False)
if a.shards:  # one shard's local plan (transfers stubbed), op by op unless --graph
    from paper_1207_6720_b200.shard import LocalShardPlan

    plan = LocalShardPlan(cfg, w["B"], a.shards, a.rank, dt, use_graph=a.graph)
    rows = 2 ** w["m"] // a.shards
    f = f[a.rank * rows:(a.rank + 1) * rows].contiguous()
sol = torch.empty_like(f)
for _ in range(a.solves):
    plan.solve(f, sol)
torch.cuda.synchronize()
print("solves done", a.workload, a.solves, plan.info())
