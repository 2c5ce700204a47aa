"""One shard's share of a patch-sharded solve, timed on ONE GPU.

For S shards, shard r runs exactly the kernels of rank r of an S-GPU solve --
its slab of every level above the replication cutoff, the replicated levels
below it, the slab-edge fix-ups -- with no transport (LocalShardPlan: halos are
never exchanged, so the numbers are timing only).  The slowest shard's time
T_S bounds an S-GPU cycle from below (NCCL exchanges come on top), so
T_1 / (S * T_S) is the predicted strong-scaling efficiency before transport.

    python tools/shard_timing.py [--workload config4] [--shards 2 4 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1207_6720_b200 as fm  # noqa: E402
from paper_1207_6720_b200.shard import LocalShardPlan, ShardedPlan, comm_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="config4")
ap.add_argument("--shards", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--json", default="")
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
cfg = bench._solver_cfg(fm, w)
B, n = w["B"], 2 ** w["m"]


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


f = bench._forcing(fm, w, torch.float64, 0)
plan = fm.get_plan(fm.key_from_config(cfg, B, torch.float64))
sol = torch.empty_like(f)
t1 = timeit(lambda: plan.solve(f, sol), a.reps)
res = {"workload": a.workload, "t1_ms": t1, "shards": {}}
print(f"{a.workload}: unsharded {t1:.3f} ms/cycle")
del plan, sol
fm.plan._cache.clear()
torch.cuda.empty_cache()
for S in a.shards:
    rows = n // S
    per = {}
    for r in sorted({0, S // 2, S - 1}):
        p = LocalShardPlan(cfg, B, S, r)
        fs = p.forcing_slab()  # resident in the plan's own slab: no copy per solve
        fs.copy_(f[r * rows:(r + 1) * rows])
        out = torch.empty_like(fs)
        per[r] = timeit(lambda: p.solve(fs, out), a.reps)
        del p, fs, out
        torch.cuda.empty_cache()
    # the same shard with the peer-memory transport mapped onto itself
    # (FMGSR_P2P_SELF_PROBE): its exchange kernels' cost -- launch, fence,
    # counter poll, copy from HBM instead of over NVLink -- on top of T_S
    os.environ["FMGSR_P2P_SELF_PROBE"] = "1"
    r = S // 2
    p = ShardedPlan(cfg, B, S, r, dtype=torch.float64, transport="p2p",
                    exchange=lambda blob: [blob] * S)
    fs = p.forcing_slab()
    fs.copy_(f[r * rows:(r + 1) * rows])
    out = torch.empty_like(fs)
    t_p2p = timeit(lambda: p.solve(fs, out), a.reps)
    del p, fs, out
    os.environ.pop("FMGSR_P2P_SELF_PROBE")
    torch.cuda.empty_cache()
    recs, cut, halo = comm_schedule(cfg, B, S, S // 2)
    rounds = len({x["step"] for x in recs if x["kind"] in ("send", "recv")})
    gathers = sum(1 for x in recs if x["kind"] == "allgather")
    tS = max(per.values())
    eff = t1 / (S * tS)
    t_x = t_p2p - per[r]  # transport overhead of the middle shard
    eff_x = t1 / (S * (tS + t_x))
    res["shards"][S] = {"ms_per_rank": per, "t_shard_ms": tS, "cutoff": cut, "halo_rows": halo,
                        "p2p_rounds": rounds, "allgathers": gathers,
                        "predicted_efficiency_before_transport": eff,
                        "p2p_self_probe_ms": t_p2p, "p2p_overhead_ms": t_x,
                        "predicted_efficiency_with_p2p_overhead": eff_x}
    print(f"  S={S}: cutoff L_r={cut}, per-shard ms {dict((k, round(v, 3)) for k, v in per.items())}"
          f" -> T1/(S*T_S) = {eff:.3f} before transport ({rounds} exchange rounds, {gathers} "
          f"gathers); p2p transport kernels +{t_x:.3f} ms (self-mapped probe) -> {eff_x:.3f}")
if a.json:
    with open(a.json, "w") as fh:
        json.dump(res, fh, indent=1)
