"""Virtual-shard overhead on one GPU: the sharded schedule of one problem (all
S shards in lockstep on one device) against the unsharded plan.  Bit-equality
is checked; the time difference is the redundant replicated levels plus the
halo / edge-record / cutoff-gather copies (which NCCL carries on real GPUs)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1207_6720_b200 as fm  # noqa: E402
from paper_1207_6720_b200.shard import ShardGroup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config4")
ap.add_argument("--shards", type=int, nargs="+", default=[2, 4, 8])
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], w["m"]), n_sr=w["n_sr"],
                      smoother=fm.SmootherConfig(ns=1, n_patches=w["P"], buffer=w["b"]))
f, _ = fm.fourier_batch(2 ** w["m"], fm.fourier_coefficients(w["B"]), with_exact=False)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


plan = fm.get_plan(fm.key_from_config(cfg, w["B"], torch.float64))
ref = torch.empty_like(f)
t0 = timeit(lambda: plan.solve(f, ref))
print(f"{a.workload}: unsharded {t0:.2f} ms")
for S in a.shards:
    g = ShardGroup(cfg, w["B"], S)
    out = torch.empty_like(f)
    t = timeit(lambda: g.solve(f, out))
    print(f"  S={S}: cutoff L_r={g.cutoff}, halo {g.halo} rows, all shards on one GPU {t:.2f} ms, "
          f"bit-identical={torch.equal(out, ref)}")
    del g
