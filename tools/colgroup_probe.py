"""Probe: does splitting the RHS batch into G independent column groups, each
solved by its own plan on its own stream (staggered start), hide the
latency-bound coarse levels of one group under the streaming visits of the
others?  Prints ms per whole-batch solve for each variant.

    python tools/colgroup_probe.py [--workload config2] [--reps 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1207_6720_b200 as fm  # noqa: E402
from paper_1207_6720_b200.plan import FmgPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config2")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
dt = torch.float64 if w["dtype"] == "f64" else torch.float32
cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], w["m"]), n_sr=w["n_sr"],
                      smoother=fm.SmootherConfig(ns=w["ns"], n_patches=w["P"], buffer=w["b"]))
Bt = w["B"]
n = 2 ** w["m"]
f_all, _ = fm.fourier_batch(n, fm.fourier_coefficients(Bt), dt, with_exact=False)


def run_variant(G, sleep_cycles):
    Bg = Bt // G
    plans = [FmgPlan(fm.key_from_config(cfg, Bg, dt)) for _ in range(G)]
    fs = [f_all[:, g * Bg:(g + 1) * Bg].contiguous() for g in range(G)]
    outs = [torch.empty_like(x) for x in fs]
    streams = [torch.cuda.Stream() for _ in range(G)]
    main = torch.cuda.current_stream()

    def step():
        ev = torch.cuda.Event()
        ev.record(main)
        for g in range(G):
            with torch.cuda.stream(streams[g]):
                streams[g].wait_event(ev)
                if g and sleep_cycles:
                    torch.cuda._sleep(sleep_cycles * g)
                plans[g].solve(fs[g], outs[g])
        for g in range(G):
            e = torch.cuda.Event()
            e.record(streams[g])
            main.wait_event(e)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for _ in range(a.reps):
        step()
    t1.record(main)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.reps
    # correctness vs the one-plan solve
    ref = fm.get_plan(fm.key_from_config(cfg, Bt, dt)).solve(f_all)
    got = torch.cat(outs, dim=1)
    same = bool(torch.equal(ref, got))
    print(f"G={G} sleep={sleep_cycles:7d}: {ms:7.3f} ms/solve  bitwise-equal={same}", flush=True)
    del plans
    torch.cuda.empty_cache()


run_variant(1, 0)
for G in (2, 4):
    for sl in (0, 50000, 150000, 300000):
        run_variant(G, sl)
