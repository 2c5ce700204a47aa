"""Benchmark of one FMG-FAS-SR cycle (BASELINE.json metric: fine-grid
unknowns solved per second for one cycle, and % of the HBM roofline).

    python bench.py [--gpus N --steps K --warmup W] [--workload config2]
    python bench.py --impl reference ...      # the CPU reference path (oracle port)

A step is one ``fmg_solve`` of a batch of B right-hand sides (one FMG pass:
one V-cycle per level) through the native plan (CUDA graph of fused level
visits).  Under torchrun every rank solves its own batch of B independent
right-hand sides (independent objects, no data-path collective, weak
scaling); the time is the max over ranks.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the metric's configuration (fits one GPU)
    "config2": dict(m0=3, m=16, P=64, b=4, ns=1, n_sr=1, B=1024, dtype="f64"),
    "config1": dict(m0=3, m=10, P=4, b=2, ns=1, n_sr=1, B=1, dtype="f64"),
    "config4": dict(m0=3, m=24, P=4096, b=8, ns=1, n_sr=1, B=64, dtype="f64"),
    "config5": dict(m0=3, m=20, P=256, b=4, ns=1, n_sr=1, B=256, dtype="f64"),
    "config5_f32": dict(m0=3, m=20, P=256, b=4, ns=1, n_sr=1, B=256, dtype="f32"),
    # BASELINE config 3: -u'' + u^3 = f, V(2,2), manufactured RHS scaled per RHS
    "config3": dict(m0=3, m=20, P=256, b=4, ns=2, n_sr=1, B=256, dtype="f64", nonlinear=True),
}
METRIC = "fine-grid unknowns solved/sec (one FMG-FAS-SR cycle)"
UNIT = "unknowns/s"


def throughput(world: int, B: int, n: int, ms_step: float) -> float:
    """Whole-job fine-grid unknowns per second: every rank solves B RHS of n cells."""
    return world * B * n / (ms_step / 1e3)


def reduce_max(x: float, world: int, device: str = "cuda") -> float:
    """Max over ranks (the step time the job is charged with)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "gloo":
        device = "cpu"

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_seed(rank: int) -> int:
    """Seed of the rank's RHS batch: independent problems per rank."""
    return 1000 * rank


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------
# CPU reference path: the oracle port (C restatement of the reference algorithm)
# ---------------------------------------------------------------------------------------
def cpu_rate(w, budget_s: float, nthreads: int, seed: int = 1):
    """Solve a bounded sample of the workload's RHS on the host; returns
    (unknowns/s, n_rhs, seconds).  Test infrastructure: oracle/liboracle.so."""
    from oracle import oracle as O

    n = 2 ** w["m"]
    cfg = O.make_cfg(w["m0"], w["m"], w["n_sr"], w["ns"], O.GEOM_PATCHES, w["P"], w["b"],
                     nonlin=bool(w.get("nonlinear", False)))
    x = (np.arange(n) + 0.5) / n

    def rhs(k):
        # 4 distinct seeded Fourier rows, tiled (the solve time does not depend on values)
        base = np.zeros((4, n))
        a = np.random.default_rng(seed).standard_normal((4, 32)) / np.arange(1, 33) ** 2
        for j in range(1, 33):
            base += a[:, j - 1:j] * np.sin(j * np.pi * x)[None, :]
        return np.ascontiguousarray(np.tile(base, (k // 4 + 1, 1))[:k])

    t0 = time.perf_counter()
    O.fmg_solve_batch(cfg, rhs(1), 1)  # calibrate on one RHS, one thread
    t1 = time.perf_counter() - t0
    k = max(nthreads, int(budget_s * nthreads / max(t1, 1e-6)))
    k = min(k, w["B"] * 64)
    f = rhs(k)
    t0 = time.perf_counter()
    O.fmg_solve_batch(cfg, f, nthreads)
    dt = time.perf_counter() - t0
    return k * n / dt, k, dt


def run_reference(args, w):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    nthreads = os.cpu_count() or 1
    n = 2 ** w["m"]
    vals = []
    sample = None
    for i in range(args.warmup + args.steps):
        v, k, dt = cpu_rate(w, args.ref_step_s, nthreads, seed=i)
        if i >= args.warmup:
            vals.append((v, k, dt))
        sample = f"{k} seeded RHS of N={n} (P={w['P']}, b={w['b']}) per step, {dt:.1f} s"
    tot_unk = sum(v[1] for v in vals) * n
    tot_t = sum(v[2] for v in vals)
    value = tot_unk / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / len(vals), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
        "config": workload_config(args.workload, w, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name, w, world):
    return {
        "workload": f"{name}: 1D {'-u\'\'+u^3=f' if w.get('nonlinear') else 'Poisson'} "
                    f"FMG-FAS-SR, N=2^{w['m']} fine cells, m0={w['m0']}, "
                    f"{w['P']} patches, {w['b']}-cell buffer, V({w['ns']},{w['ns']}), "
                    f"n_sr={w['n_sr']}, batch {w['B']} seeded Fourier RHS per GPU",
        "N": 2 ** w["m"], "batch_per_gpu": w["B"], "global_batch": w["B"] * world,
        "patches": w["P"], "buffer": w["b"], "ns": w["ns"], "n_sr": w["n_sr"], "m0": w["m0"],
        "parallelism": f"dp{world} (independent RHS batches per GPU)",
        "l2": "inputs larger than L2: every field of the finest level is "
              f"{2 ** w['m'] * w['B'] * (8 if w['dtype'] == 'f64' else 4) / 2**20:.0f} MiB; no flush",
    }


# ---------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------
class ClockSampler:
    """Polls SM clock and clock-event (throttle) reasons through NVML on a
    background thread every ~2 ms while the timed region runs."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, gpu_index: int):
        import threading

        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                        bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in self.REASONS.items():
                            if bits & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(0.002)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: report it
            self.err = str(e)

    def stop(self):
        if self._t is None:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": [f"nvml unavailable: {getattr(self, 'err', '?')}"]}
        self._stop.set()
        self._t.join(timeout=2)
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------------------------
# GPU path
# ---------------------------------------------------------------------------------------
def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(workload)
    except Exception:
        return None


def run_gpu(args, w):
    import torch
    import torch.distributed as dist

    import paper_1207_6720_b200 as fm

    world, rank, local = dist_env()
    # FMGSR_BENCH_BACKEND=gloo: functional check of the multi-rank plumbing with
    # several ranks on fewer GPUs (never a reported measurement: ranks share SMs)
    backend = os.environ.get("FMGSR_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dtype = torch.float64 if w["dtype"] == "f64" else torch.float32
    m, B = w["m"], w["B"]
    n = 2 ** m
    nl = bool(w.get("nonlinear", False))
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], m), n_sr=w["n_sr"],
                          smoother=fm.SmootherConfig(ns=w["ns"], n_patches=w["P"], buffer=w["b"],
                                                     nonlinear=nl))
    plan = fm.get_plan(fm.key_from_config(cfg, B, dtype))
    if nl:
        f, _ = fm.nonlinear_batch(n, fm.nonlinear_scales(B, seed=rank_seed(rank)), dtype)
    else:
        coef = fm.fourier_coefficients(B, seed=rank_seed(rank))
        f, _ = fm.fourier_batch(n, coef, dtype, with_exact=False)
    sol = torch.empty_like(f)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        plan.solve(f, sol)
    torch.cuda.synchronize()
    info = plan.info()

    # ---- device-resident throughput (value) --------------------------------------
    clk = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.solve(f, sol)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms_max = reduce_max(e0.elapsed_time(e1), world)
    ms_step = ms_max / args.steps
    value = throughput(world, B, n, ms_step)
    # finest T_m / U_m durations of the last solve of the timed region, from CUDA
    # events recorded inside the replayed graph around those two kernels, plus
    # the same probe over a few more replays (each synchronised) for the mean
    probes = [plan.probe_ms()]
    for _ in range(4):
        plan.solve(f, sol)
        torch.cuda.synchronize()
        probes.append(plan.probe_ms())

    # ---- end to end through the public API with host buffers ----------------------
    # fmgsr_plan_solve_host: pinned host forcing in, pinned host solution out;
    # the batch is pipelined in chunks (H2D / solve / D2H overlap)
    hf = f.cpu().pin_memory()
    hs = torch.empty_like(hf).pin_memory()
    chunks = args.e2e_chunks if B % args.e2e_chunks == 0 else 1
    cplan = fm.get_plan(fm.key_from_config(cfg, B // chunks, dtype))

    def e2e_step():  # consecutive batches stream: host inputs are ready at call time
        cplan.solve_host(hf, hs, chunks, inputs_ready=True)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = reduce_max(e0.elapsed_time(e1), world) / args.steps
    e2e_val = throughput(world, B, n, e2e_ms)
    nbytes = n * B * (8 if dtype == torch.float64 else 4)

    # ---- per-visit kernel times (CUDA events on the launching stream) -------------
    visits = []
    for _ in range(max(1, min(args.steps, 5))):
        visits += plan.solve_timed(f, sol)
    finest = [(k, ms_) for (k, lvl, ms_) in visits if lvl == m and k in ("top", "up")]
    by_level = {}
    for (k, lvl, ms_) in visits:
        by_level[lvl] = by_level.get(lvl, 0.0) + ms_
    tot = sum(by_level.values())
    esz = 8 if dtype == torch.float64 else 4
    # algorithmic words per cell of the finest visits: T_m and U_m
    sr_m = cfg.is_sr_level(m)
    words = {"top": 2.5 + (0.0 if sr_m else 1.0), "up": 2.5 + (0.0 if sr_m else 1.0)}
    alg = sum(words[k] * n * B * esz for k, _ in finest)
    dur = sum(ms_ for _, ms_ in finest) / 1e3
    achieved_op = alg / dur / 1e9 if dur > 0 else None
    # primary: in-graph probe (the kernels as timed in the step)
    pv = [(t, u_) for t, u_ in probes if t > 0 and u_ > 0]
    if pv:
        alg_pair = (words["top"] + words["up"]) * n * B * esz
        probe_s = sum(t + u_ for t, u_ in pv) / len(pv) / 1e3
        achieved = alg_pair / probe_s / 1e9
        probe_launches = 2 * len(pv)
    else:
        achieved, probe_launches = achieved_op, 0
    # ---- functional-only output: u_m never stored --------------------
    jout = torch.empty(B, dtype=dtype, device="cuda")
    for _ in range(2):
        plan.solve_functional(f, out=jout)
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        plan.solve_functional(f, out=jout)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    fun_ms = reduce_max(e0.elapsed_time(e1), world) / args.steps

    peak, peak_src = measured_peak()
    share = sum(ms_ for _, ms_ in finest) / tot if tot else None
    traffic = committed_traffic(args.workload)
    whole_alg = info["alg_bytes_per_solve"]

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            v, k, dt = cpu_rate(w, args.cpu_budget_s, os.cpu_count() or 1)
            cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                   "sample": f"{k} seeded RHS of N={n} (P={w['P']}, b={w['b']}) on "
                             f"{os.cpu_count()} host threads, {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": w["dtype"], "data": ("synthetic (seeded manufactured nonlinear RHS, s ~ U[0.5, 2])" if nl else "synthetic (seeded Fourier RHS, SURVEY 8(d))"),
            "config": workload_config(args.workload, w, world),
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None,
                # ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of the
                # finest visits (committed capture, profiles/traffic.json)
                "traffic": traffic.get("bytes_per_launch") if traffic else None,
                "traffic_unit": "bytes per launch",
                "traffic_detail": traffic,
                "kernel": "visit_kernel at the finest level (T_m: FMG prolongation + "
                          "patch GS + restriction/tau; U_m: FMG prolongation + Kaczmarz CR + "
                          "patch GS)",
                "alg_bytes_per_launch": alg / max(1, len(finest)),
                "achieved_source": ("CUDA events recorded inside the replayed graph around "
                                    "T_m and U_m: the last step of the timed region + 4 replays"
                                    if probe_launches else "op-by-op CUDA events"),
                "launches_measured": probe_launches or len(finest),
                "achieved_op_by_op": achieved_op,
                "probe_ms_last_timed_step": probes[0],
                "share_of_step": share, "peak_source": peak_src,
                "whole_cycle_alg_bytes": whole_alg,
                "whole_cycle_frac": whole_alg / (ms_step / 1e3) / 1e9 / peak,
            },
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "ms_per_step": e2e_ms,
                    "api": "fmgsr_plan_solve_host_ex (pinned host buffers, FMGSR_HOST_INPUTS_READY: "
                           "consecutive batches stream)", "chunks": chunks},
            "gpu_launches": info["launches_per_solve"] * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "functional_only": {
                "value": throughput(world, B, n, fun_ms), "unit": UNIT, "ms_per_step": fun_ms,
                "api": "fmgsr_plan_solve_functional (J_r = h sum_i u_i per RHS; the finest "
                       "solution is never stored)"},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_gpu_sharded(args, w):
    """One problem split across the ranks by patch slabs: strong
    scaling (total work fixed), halos / tau edge records over NCCL send/recv,
    the replication cutoff level over NCCL all-gather."""
    import torch
    import torch.distributed as dist

    import paper_1207_6720_b200 as fm
    from paper_1207_6720_b200.shard import ShardedPlan, nccl_unique_id, slab

    world, rank, local = dist_env()
    if world == 1:
        return run_gpu(args, w)
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dtype = torch.float64 if w["dtype"] == "f64" else torch.float32
    m, B = w["m"], w["B"]
    n = 2 ** m
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], m), n_sr=w["n_sr"],
                          smoother=fm.SmootherConfig(ns=w["ns"], n_patches=w["P"], buffer=w["b"]))
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    plan = ShardedPlan(cfg, B, world, rank, bytes(uid.cpu().numpy().tobytes()), dtype)
    f, _ = fm.fourier_batch(n, fm.fourier_coefficients(B, seed=0), dtype, with_exact=False)
    c0, c1 = slab(n, world, rank)
    fs = f[c0:c1].contiguous()
    del f
    sol = torch.empty_like(fs)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        plan.solve(fs, sol)
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.solve(fs, sol)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = clk.stop()
    ms_step = reduce_max(e0.elapsed_time(e1), world) / args.steps
    value = B * n / (ms_step / 1e3)  # the whole problem, solved by all ranks together
    # end to end: this rank's slab from / to pinned host memory
    hf = fs.cpu().pin_memory()
    hs = torch.empty_like(hf).pin_memory()
    dfi = torch.empty_like(fs)

    def e2e_step():
        dfi.copy_(hf, non_blocking=True)
        plan.solve(dfi, sol)
        hs.copy_(sol, non_blocking=True)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    e2e_ms = reduce_max(e0.elapsed_time(e1), world) / args.steps
    esz = 8 if dtype == torch.float64 else 4
    peak, peak_src = measured_peak()
    # per-GPU share of the whole cycle's algorithmic bytes (29 words / unknown)
    alg = 29.0 * n * B * esz
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": w["dtype"], "data": "synthetic (seeded Fourier RHS, SURVEY 8(d))",
            "config": dict(workload_config(args.workload, w, 1),
                           parallelism=f"patch slabs x{world} (NCCL halos, replicated coarse)"),
            "roofline": {"bound": "hbm", "achieved": alg / world / (ms_step / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s",
                         "frac": alg / world / (ms_step / 1e3) / 1e9 / peak, "traffic": None,
                         "kernel": "whole cycle per GPU (29 algorithmic words / unknown)",
                         "peak_source": peak_src},
            "e2e": {"value": B * n / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": (c1 - c0) * B * esz * world,
                    "d2h_bytes_per_step": (c1 - c0) * B * esz * world, "ms_per_step": e2e_ms},
            "clocks": clocks, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4)
    ap.add_argument("--shard", default="rhs", choices=["rhs", "patches"],
                    help="multi-GPU split: independent RHS batches per rank (weak), or "
                         "patch slabs of one problem (strong, SURVEY 8(e))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)
    if args.shard == "patches":
        return run_gpu_sharded(args, w)
    return run_gpu(args, w)


if __name__ == "__main__":
    sys.exit(main())
