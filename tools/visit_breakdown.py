"""Per-level-visit device times of one FMG pass (op-by-op launches with CUDA
events on the launching stream), summed by level and kind.

    python tools/visit_breakdown.py [--workload config2] [--reps 3] [--unfused] [--B 128]
        [--P 16 --b 1] [--shards 8 --rank 4]   # one shard's plan (no transport, timing only)
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1207_6720_b200 as fm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--unfused", action="store_true")
ap.add_argument("--B", type=int, default=0, help="override the workload's batch size")
ap.add_argument("--P", type=int, default=0, help="override the patch count")
ap.add_argument("--b", type=int, default=-1, help="override the buffer")
ap.add_argument("--shards", type=int, default=0, help="time shard --rank of an S-way split")
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--total", action="store_true", help="also time the graph-replayed cycle")
a = ap.parse_args()
w = dict(bench.WORKLOADS[a.workload])
if a.B:
    w["B"] = a.B
if a.P:
    w["P"] = a.P
if a.b >= 0:
    w["b"] = a.b
dt = torch.float64 if w["dtype"] == "f64" else torch.float32
nl = bool(w.get("nonlinear", False))
cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], w["m"]), n_sr=w["n_sr"],
                      smoother=fm.SmootherConfig(ns=w["ns"], n_patches=w["P"], buffer=w["b"],
                                                 nonlinear=nl))
if nl:
    f, _ = fm.nonlinear_batch(2 ** w["m"], fm.nonlinear_scales(w["B"]), dt)
else:
    f, _ = fm.fourier_batch(2 ** w["m"], fm.fourier_coefficients(w["B"]), dt, with_exact=False)
if a.shards:
    from paper_1207_6720_b200.shard import LocalShardPlan

    plan = LocalShardPlan(cfg, w["B"], a.shards, a.rank, dt)
    rows = 2 ** w["m"] // a.shards
    f = f[a.rank * rows:(a.rank + 1) * rows].contiguous()
else:
    plan = fm.get_plan(fm.key_from_config(cfg, w["B"], dt, fused=not a.unfused,
                                          arith=bench._arith(w)))
sol = torch.empty_like(f)
for _ in range(2):
    plan.solve(f, sol)
torch.cuda.synchronize()
acc = collections.defaultdict(float)
cnt = collections.defaultdict(int)
for _ in range(a.reps):
    for kind, lvl, ms in plan.solve_timed(f, sol):
        acc[(lvl, kind)] += ms / a.reps
        cnt[(lvl, kind)] += 1
tot = sum(acc.values())
print(f"workload {a.workload} fused={not a.unfused}: sum of visit times {tot:.3f} ms")
for (lvl, kind) in sorted(acc, key=lambda k: (-k[0], k[1])):
    n = cnt[(lvl, kind)] // a.reps
    print(f"  level {lvl:2d} {kind:7s} x{n:3d}  {acc[(lvl, kind)]:8.3f} ms  {100*acc[(lvl, kind)]/tot:5.1f}%"
          f"  per-visit {acc[(lvl, kind)]/max(n,1)*1e3:8.1f} us")
if a.total:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        plan.solve(f, sol)
    e1.record()
    torch.cuda.synchronize()
    print(f"graph-replayed cycle: {e0.elapsed_time(e1) / 5:.3f} ms")
print(json.dumps(plan.info()))
