"""Benchmark of one FMG-FAS-SR cycle (BASELINE.json metric: fine-grid
unknowns solved per second for one cycle, and % of the HBM roofline).

    python bench.py [--gpus N --steps K --warmup W] [--workload config4]
    python bench.py --impl reference ...      # the CPU reference path (oracle port)

A step is one ``fmg_solve`` of a batch of B right-hand sides (one FMG pass:
one V-cycle per level) through the native plan (CUDA graph of fused level
visits).  The default workload is BASELINE config 4 (N = 2^24, 4096 patches,
8-cell buffer, B = 64, fp64): the largest configuration that fits one GPU,
and the one BASELINE.json names for the 1/2/4/8-GPU sweep.

* N = 1: the unsharded plan.  Extra keys carry the config-2 line (BASELINE
  configs[1]) measured in the same process.
* N > 1 (one process per GPU, torchrun; ``--gpus N`` without torchrun spawns
  it): the ONE config-4 problem is split into N patch slabs:
  strong scaling, halos, tau edge records and the replication-cutoff level
  pulled from the peers' workspaces over peer memory (``--transport p2p``,
  default) or moved by NCCL send/recv + all-gather (``--transport nccl``),
  levels below the cutoff replicated.  The sharded result is compared bit for
  bit with the unsharded plan on the same forcing (``sharded_bit_exact_...``).  The
  independent-RHS-batch split (every rank its own config-4 batch, weak
  scaling, no data-path collective) is reported beside it as a control.
  ``--shard rhs`` makes the control the headline instead.

Time is the max over ranks of CUDA-event time on the launching stream; rank 0
prints one JSON line.
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
    # BASELINE.json configs[3]: the largest single-GPU configuration (headline)
    "config4": dict(m0=3, m=24, P=4096, b=8, ns=1, n_sr=1, B=64, dtype="f64", e2e_chunks=2),
    # BASELINE.json configs[1]
    "config2": dict(m0=3, m=16, P=64, b=4, ns=1, n_sr=1, B=1024, dtype="f64"),
    "config1": dict(m0=3, m=10, P=4, b=2, ns=1, n_sr=1, B=1, dtype="f64"),
    "config5": dict(m0=3, m=20, P=256, b=4, ns=1, n_sr=1, B=256, dtype="f64"),
    "config5_f32": dict(m0=3, m=20, P=256, b=4, ns=1, n_sr=1, B=256, dtype="f32"),
    # the same fp32 fields (same HBM bytes) with fp64 arithmetic
    "config5_f32f64": dict(m0=3, m=20, P=256, b=4, ns=1, n_sr=1, B=256, dtype="f32",
                           arith="f64"),
    # BASELINE config 3: -u'' + u^3 = f, V(2,2), manufactured RHS scaled per RHS
    "config3": dict(m0=3, m=20, P=256, b=4, ns=2, n_sr=1, B=256, dtype="f64", nonlinear=True),
}
DEFAULT_WORKLOAD = "config4"
METRIC = "fine-grid unknowns solved/sec (one FMG-FAS-SR cycle)"
UNIT = "unknowns/s"


def _arith(w):
    """Arithmetic dtype of a workload (None: the field dtype)."""
    import torch

    return torch.float64 if w.get("arith") == "f64" else None


def dtype_label(w) -> str:
    """The JSON line's dtype: the arithmetic type (and the storage when narrower)."""
    return "f64 (f32 fields)" if w.get("arith") == "f64" else w["dtype"]


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


def host_cores() -> dict:
    """Host threads the CPU legs use, and the physical core count (lscpu)."""
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    phys = None
    try:
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True,
                             timeout=10).stdout
        phys = len({ln for ln in out.splitlines() if ln and not ln.startswith("#")})
    except Exception:
        pass
    return {"threads": int(threads or 1), "physical_cores": phys}


def check_world(gpus: int, world: int) -> None:
    """``--gpus`` is authoritative: a launch whose world size differs is an error."""
    if gpus != world:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}; launch one process "
                         f"per GPU (torchrun --nproc-per-node {gpus}) or run without torchrun "
                         f"and let bench.py spawn the ranks")


def spawn_cmd(gpus: int, argv: list[str], port: int) -> list[str]:
    """torchrun command that re-runs this script with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1",
            "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


# ---------------------------------------------------------------------------------------
# CPU reference path: the oracle port (C restatement of the reference algorithm)
# ---------------------------------------------------------------------------------------
def _cpu_cfg(w):
    from oracle import oracle as O

    return O.make_cfg(w["m0"], w["m"], w["n_sr"], w["ns"], O.GEOM_PATCHES, w["P"], w["b"],
                      nonlin=bool(w.get("nonlinear", False)))


def _cpu_rhs(n, k, seed):
    """k seeded Fourier rows of n cells (4 distinct rows tiled: the solve time
    does not depend on the values)."""
    x = (np.arange(n) + 0.5) / n
    base = np.zeros((4, n))
    a = np.random.default_rng(seed).standard_normal((4, 32)) / np.arange(1, 33) ** 2
    for j in range(1, 33):
        base += a[:, j - 1:j] * np.sin(j * np.pi * x)[None, :]
    return np.ascontiguousarray(np.tile(base, (k // 4 + 1, 1))[:k])


def cpu_calibrate(w):
    """Seconds for one RHS of the workload on one host thread."""
    from oracle import oracle as O

    n = 2 ** w["m"]
    f = _cpu_rhs(n, 1, 0)
    t0 = time.perf_counter()
    O.fmg_solve_batch(_cpu_cfg(w), f, 1)
    return time.perf_counter() - t0


def cpu_rate(w, budget_s: float, nthreads: int, seed: int = 1, t1: float | None = None,
             mem_cap: float = 4e9):
    """Solve a bounded sample of the workload's RHS on the host; returns
    (unknowns/s, n_rhs, seconds).  Rounds of at most ``nthreads`` RHS (and
    ``mem_cap`` bytes of forcing + solution) until ``budget_s`` is spent.
    Test infrastructure: oracle/liboracle.so."""
    from oracle import oracle as O

    n = 2 ** w["m"]
    cfg = _cpu_cfg(w)
    if t1 is None:
        t1 = cpu_calibrate(w)
    per = max(1, min(int(mem_cap // (16 * n)), nthreads * max(1, int(budget_s / max(t1, 1e-6)))))
    f = _cpu_rhs(n, per, seed)
    done, dt = 0, 0.0
    while True:
        t0 = time.perf_counter()
        O.fmg_solve_batch(cfg, f, nthreads)
        dt += time.perf_counter() - t0
        done += per
        if dt >= 0.5 * budget_s or done >= w["B"] * 64:
            break
    return done * n / dt, done, dt


def run_reference(args, w):
    world, rank, _ = dist_env()
    check_world(args.gpus, world)
    if rank != 0:
        return 0
    hc = host_cores()
    nthreads = hc["threads"]
    n = 2 ** w["m"]
    t1 = cpu_calibrate(w)
    vals = []
    sample = None
    for i in range(args.warmup + args.steps):
        v, k, dt = cpu_rate(w, args.ref_step_s, nthreads, seed=i, t1=t1)
        if i >= args.warmup:
            vals.append((v, k, dt))
        sample = (f"{k} seeded RHS of N={n} (P={w['P']}, b={w['b']}) per step on {nthreads} "
                  f"host threads ({hc['physical_cores']} physical cores), {dt:.1f} s")
    tot_unk = sum(v[1] for v in vals) * n
    tot_t = sum(v[2] for v in vals)
    value = tot_unk / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / len(vals), "higher_is_better": True,
        "scaling": "strong" if world > 1 and args.shard == "patches" else "weak",
        "vs_baseline": None, "dtype": dtype_label(w), "data": "synthetic",
        "config": workload_config(args.workload, w, world, args.shard),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "physical_cores": hc["physical_cores"], "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


TRANSPORTS = {
    "p2p": "halos / tau edge records / cutoff-level chunks pulled from the peers' "
           "workspaces over peer memory (CUDA IPC, NVLink), device-side counters",
    "nccl": "NCCL send/recv halos / tau edge records, NCCL all-gather at the cutoff",
}


def workload_config(name, w, world, shard="patches", transport="p2p"):
    esz = 8 if w["dtype"] == "f64" else 4
    sharded = world > 1 and shard == "patches"
    par = (f"patch slabs x{world} of one problem ({TRANSPORTS[transport]}; coarse levels "
           "replicated)" if sharded else f"dp{world} (independent RHS batches per GPU)")
    return {
        "workload": f"{name}: 1D {'-u\'\'+u^3=f' if w.get('nonlinear') else 'Poisson'} "
                    f"FMG-FAS-SR, N=2^{w['m']} fine cells, m0={w['m0']}, "
                    f"{w['P']} patches, {w['b']}-cell buffer, V({w['ns']},{w['ns']}), "
                    f"n_sr={w['n_sr']}, batch {w['B']} seeded "
                    f"{'manufactured' if w.get('nonlinear') else 'Fourier'} RHS"
                    f"{'' if sharded else ' per GPU'}",
        "N": 2 ** w["m"], "batch_per_gpu": w["B"] if not sharded else None,
        "global_batch": w["B"] * (1 if sharded else world),
        "patches": w["P"], "buffer": w["b"], "ns": w["ns"], "n_sr": w["n_sr"], "m0": w["m0"],
        "parallelism": par,
        "l2": "inputs larger than L2: every field of the finest level is "
              f"{2 ** w['m'] * w['B'] * esz / 2**20 / (world if sharded else 1):.0f} MiB "
              "per GPU; no flush",
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


def _solver_cfg(fm, w):
    nl = bool(w.get("nonlinear", False))
    return fm.SolverConfig(hierarchy=fm.build_hierarchy(w["m0"], w["m"]), n_sr=w["n_sr"],
                           smoother=fm.SmootherConfig(ns=w["ns"], n_patches=w["P"],
                                                      buffer=w["b"], nonlinear=nl))


def _forcing(fm, w, dtype, seed):
    n, B = 2 ** w["m"], w["B"]
    if w.get("nonlinear"):
        return fm.nonlinear_batch(n, fm.nonlinear_scales(B, seed=seed), dtype)[0]
    return fm.fourier_batch(n, fm.fourier_coefficients(B, seed=seed), dtype, with_exact=False)[0]


def _timed(fn, steps, world, stream, barrier):
    """CUDA-event ms per step of ``steps`` calls of fn, max over ranks."""
    import torch

    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    return reduce_max(e0.elapsed_time(e1), world) / steps


def _finest_roofline(plan, cfg, w, f, sol, steps, ms_step, dtype, workload):
    """Roofline of the dominant kernel (finest T_m / U_m visit_kernel)."""
    import torch

    m, B, n = w["m"], w["B"], 2 ** w["m"]
    esz = 8 if dtype == torch.float64 else 4
    # finest T_m / U_m durations of the last solve of the timed region, from CUDA
    # events recorded inside the replayed graph around those two kernels, plus
    # the same probe over a few more replays (each synchronised) for the mean
    probes = [plan.probe_ms()]
    for _ in range(4):
        plan.solve(f, sol)
        torch.cuda.synchronize()
        probes.append(plan.probe_ms())
    visits = []
    for _ in range(max(1, min(steps, 3))):
        visits += plan.solve_timed(f, sol)
    finest = [(k, ms_) for (k, lvl, ms_) in visits if lvl == m and k in ("top", "up")]
    tot = sum(ms_ for (_, _, ms_) in visits)
    sr_m = cfg.is_sr_level(m)
    words = {"top": 2.5 + (0.0 if sr_m else 1.0), "up": 2.5 + (0.0 if sr_m else 1.0)}
    alg = sum(words[k] * n * B * esz for k, _ in finest)
    dur = sum(ms_ for _, ms_ in finest) / 1e3
    achieved_op = alg / dur / 1e9 if dur > 0 else None
    pv = [(t, u_) for t, u_ in probes if t > 0 and u_ > 0]
    if pv:
        alg_pair = (words["top"] + words["up"]) * n * B * esz
        probe_s = sum(t + u_ for t, u_ in pv) / len(pv) / 1e3
        achieved = alg_pair / probe_s / 1e9
        probe_launches = 2 * len(pv)
    else:
        achieved, probe_launches = achieved_op, 0
    peak, peak_src = measured_peak()
    traffic = committed_traffic(workload)
    whole_alg = plan.info()["alg_bytes_per_solve"]
    return {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if achieved else None,
        # ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of the
        # finest visits (committed capture, profiles/traffic.json)
        "traffic": traffic.get("bytes_per_launch") if traffic else None,
        "traffic_unit": "bytes per launch",
        "traffic_detail": traffic,
        "kernel": "visit_kernel at the finest level (T_m: FMG prolongation + patch GS + "
                  "restriction/tau; U_m: FMG prolongation + Kaczmarz CR + patch GS)",
        "alg_bytes_per_launch": alg / max(1, len(finest)),
        "achieved_source": ("CUDA events recorded inside the replayed graph around T_m and "
                            "U_m: the last step of the timed region + 4 replays"
                            if probe_launches else "op-by-op CUDA events"),
        "launches_measured": probe_launches or len(finest),
        "achieved_op_by_op": achieved_op,
        "probe_ms_last_timed_step": probes[0],
        "share_of_step": (dur * 1e3 / tot) if tot else None, "peak_source": peak_src,
        "whole_cycle_alg_bytes": whole_alg,
        "whole_cycle_frac": whole_alg / (ms_step / 1e3) / 1e9 / peak,
    }


def _init_dist(world, local, backend="nccl"):
    import torch
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)


def all_ok(ok: bool, world: int, device: str = "cuda") -> bool:
    """True iff ``ok`` holds on every rank (MIN over ranks)."""
    if world <= 1:
        return bool(ok)
    import torch
    import torch.distributed as dist

    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def run_gpu(args, w, note=None):
    """N = 1 (and the ``--shard rhs`` control at N > 1): every rank solves its own batch.
    ``note``: extra keys for the JSON line (the sharded path's failure, if it fell back)."""
    import torch
    import torch.distributed as dist

    import paper_1207_6720_b200 as fm

    world, rank, local = dist_env()
    check_world(args.gpus, world)
    # FMGSR_BENCH_BACKEND=gloo: functional check of the multi-rank plumbing with
    # several ranks on fewer GPUs (never a reported measurement: ranks share SMs)
    backend = os.environ.get("FMGSR_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    _init_dist(world, local, backend)
    dtype = torch.float64 if w["dtype"] == "f64" else torch.float32
    m, B = w["m"], w["B"]
    n = 2 ** m
    cfg = _solver_cfg(fm, w)
    plan = fm.get_plan(fm.key_from_config(cfg, B, dtype, arith=_arith(w)))
    f = _forcing(fm, w, dtype, rank_seed(rank))
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
    ms_step = _timed(lambda: plan.solve(f, sol), args.steps, world, stream, barrier)
    clocks = clk.stop()
    value = throughput(world, B, n, ms_step)
    roof = _finest_roofline(plan, cfg, w, f, sol, args.steps, ms_step, dtype, args.workload)

    # ---- functional-only output: u_m never stored --------------------
    fun_ms = None  # (not offered with fp64 arithmetic on fp32 fields)
    if _arith(w) is None:
        jout = torch.empty(B, dtype=dtype, device="cuda")
        for _ in range(2):
            plan.solve_functional(f, out=jout)
        torch.cuda.synchronize()
        fun_ms = _timed(lambda: plan.solve_functional(f, out=jout), args.steps, world, stream,
                        barrier)

    # ---- end to end through the public API with host buffers ----------------------
    # fmgsr_plan_solve_host: pinned host forcing in, pinned host solution out;
    # the batch is pipelined in chunks (H2D / solve / D2H overlap)
    esz = 8 if dtype == torch.float64 else 4
    hf = torch.empty(f.shape, dtype=dtype, pin_memory=True)
    hf.copy_(f)
    hs = torch.empty_like(hf).pin_memory()
    del sol
    chunks = args.e2e_chunks or w.get("e2e_chunks", 4)
    chunks = chunks if B % chunks == 0 else 1
    cplan = fm.get_plan(fm.key_from_config(cfg, B // chunks, dtype, arith=_arith(w)))

    def e2e_step():  # consecutive batches stream: host inputs are ready at call time
        cplan.solve_host(hf, hs, chunks, inputs_ready=True)

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    torch.cuda.synchronize()
    e2e_steps = args.e2e_steps or args.steps
    e2e_ms = _timed(e2e_step, e2e_steps, world, stream, barrier)
    e2e_val = throughput(world, B, n, e2e_ms)
    nbytes = n * B * esz
    del cplan, hf, hs, f
    fm.plan._cache.clear()
    torch.cuda.empty_cache()

    # ---- BASELINE configs[1] (config 2) beside the headline ------------------------
    extra = None
    if args.workload != "config2" and not args.no_extra:
        w2 = WORKLOADS["config2"]
        cfg2 = _solver_cfg(fm, w2)
        p2 = fm.get_plan(fm.key_from_config(cfg2, w2["B"], torch.float64))
        f2 = _forcing(fm, w2, torch.float64, rank_seed(rank))
        s2 = torch.empty_like(f2)
        for _ in range(args.warmup):
            p2.solve(f2, s2)
        torch.cuda.synchronize()
        ms2 = _timed(lambda: p2.solve(f2, s2), args.steps, world, stream, barrier)
        r2 = _finest_roofline(p2, cfg2, w2, f2, s2, args.steps, ms2, torch.float64, "config2")
        extra = {"workload": workload_config("config2", w2, world, "rhs")["workload"],
                 "value": throughput(world, w2["B"], 2 ** w2["m"], ms2), "unit": UNIT,
                 "ms_per_step": ms2, "roofline_frac": r2["frac"],
                 "whole_cycle_frac": r2["whole_cycle_frac"], "traffic": r2["traffic"]}
        del p2, f2, s2
        fm.plan._cache.clear()
        torch.cuda.empty_cache()

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            hc = host_cores()
            v, k, dt = cpu_rate(w, args.cpu_budget_s, hc["threads"])
            cpu = {"value": v, "unit": UNIT, "cores": hc["threads"], "kind": "port",
                   "physical_cores": hc["physical_cores"],
                   "sample": f"{k} seeded RHS of N={n} (P={w['P']}, b={w['b']}) on "
                             f"{hc['threads']} host threads, {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype_label(w),
            "data": ("synthetic (seeded manufactured nonlinear RHS, s ~ U[0.5, 2])"
                     if w.get("nonlinear") else "synthetic (seeded Fourier RHS, SURVEY 8(d))"),
            "config": workload_config(args.workload, w, world, "rhs"),
            "roofline": roof,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "ms_per_step": e2e_ms, "steps": e2e_steps,
                    "api": "fmgsr_plan_solve_host_ex (pinned host buffers, "
                           "FMGSR_HOST_INPUTS_READY: consecutive batches stream)",
                    "chunks": chunks},
            "gpu_launches": info["launches_per_solve"] * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if fun_ms is not None:
            line["functional_only"] = {
                "value": throughput(world, B, n, fun_ms), "unit": UNIT, "ms_per_step": fun_ms,
                "api": "fmgsr_plan_solve_functional (J_r = h sum_i u_i per RHS; the finest "
                       "solution is never stored)"}
        if extra:
            line["config2"] = extra
        if note:
            line.update(note)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def broadcast_uid(uid: bytes | None, rank: int, device: str = "cuda") -> bytes:
    """Rank 0's 128-byte NCCL unique id, broadcast to every rank."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def run_gpu_sharded(args, w):
    """One problem split across the ranks by patch slabs: strong
    scaling (total work fixed), halos / tau edge records over NCCL send/recv,
    the replication cutoff level over NCCL all-gather.  The RHS-batch split is
    measured afterwards as a control."""
    import torch
    import torch.distributed as dist

    import paper_1207_6720_b200 as fm
    from paper_1207_6720_b200.shard import ShardedPlan, nccl_unique_id, slab

    world, rank, local = dist_env()
    check_world(args.gpus, world)
    if world == 1:
        return run_gpu(args, w)
    # FMGSR_BENCH_BACKEND=gloo: functional check of the plumbing with several
    # ranks on one GPU (the sharded plan's own NCCL communicator then refuses
    # the shared device, which exercises the fall-back; never a measurement)
    backend = os.environ.get("FMGSR_BENCH_BACKEND", "nccl")
    cdev = "cuda" if backend == "nccl" else "cpu"
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    _init_dist(world, local, backend)
    dtype = torch.float64 if w["dtype"] == "f64" else torch.float32
    m, B = w["m"], w["B"]
    n = 2 ** m
    cfg = _solver_cfg(fm, w)
    c0, c1 = slab(n, world, rank)
    stream = torch.cuda.current_stream()
    # Build the sharded plan and run the warm-ups; if that fails on any rank
    # (no NCCL library, a geometry the split cannot take, a CUDA or NCCL
    # error), every rank falls back to the independent-RHS split and the line
    # says why.  (A failure here is raised by the NCCL calls, not hung: every
    # send has its matching receive, tests/test_shard_schedule.py.)
    plan, fs, sol, err = None, None, None, None
    try:
        if args.transport == "nccl":
            uid = broadcast_uid(nccl_unique_id() if rank == 0 else None, rank, device=cdev)
            plan = ShardedPlan(cfg, B, world, rank, uid, dtype)
        else:
            plan = ShardedPlan(cfg, B, world, rank, dtype=dtype, transport="p2p")
        f = _forcing(fm, w, dtype, 0)  # the one problem (same seed on every rank)
        # resident input: this rank's rows written into the plan's own forcing
        # slab, so a solve reads them in place (no slab copy into the plan)
        fs = plan.forcing_slab()
        fs.copy_(f[c0:c1])
        del f
        sol = torch.empty_like(fs)
        for _ in range(args.warmup):
            plan.solve(fs, sol)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001 -- reported in the line, never hidden
        err = f"{type(e).__name__}: {e}"
    if not all_ok(err is None, world, device=cdev):
        del plan, fs, sol
        torch.cuda.empty_cache()
        return run_gpu(args, w, note={
            "sharded_error": err or "failed on another rank",
            "sharded_fallback": "patch-slab split unavailable; independent RHS batches per GPU"})
    clk = ClockSampler(local)
    ms_step = _timed(lambda: plan.solve(fs, sol), args.steps, world, stream, dist.barrier)
    clocks = clk.stop()
    value = B * n / (ms_step / 1e3)  # the whole problem, solved by all ranks together
    # end to end: this rank's slab from / to pinned host memory
    hf = fs.cpu().pin_memory()
    hs = torch.empty_like(hf).pin_memory()

    def e2e_step():  # H2D straight into the plan's forcing slab
        fs.copy_(hf, non_blocking=True)
        plan.solve(fs, sol)
        hs.copy_(sol, non_blocking=True)

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = _timed(e2e_step, args.steps, world, stream, dist.barrier)
    info = plan.info()
    plan.solve(fs, sol)  # the timed solves' result, kept for the parity check
    xerr = plan.status() if args.transport == "p2p" else 0  # a peer wait timed out?
    sol_keep = sol
    del hf, hs, fs, plan
    torch.cuda.empty_cache()
    esz = 8 if dtype == torch.float64 else 4
    peak, peak_src = measured_peak()
    alg = info["alg_bytes_per_solve"]  # whole problem (29 words / unknown)

    # ---- control: every rank its own batch (weak scaling, no data-path collective) --
    # plus the parity check of the split: the unsharded plan on the same forcing,
    # this rank's rows compared bit for bit with its slab of the sharded solve
    control, eq_local = None, None
    if not args.no_extra:
        try:
            p1 = fm.get_plan(fm.key_from_config(cfg, B, dtype, arith=_arith(w)))
            f1 = _forcing(fm, w, dtype, 0)
            s1 = torch.empty_like(f1)
            p1.solve(f1, s1)
            torch.cuda.synchronize()
            eq_local = bool(torch.equal(s1[c0:c1], sol_keep))
            del f1, s1
            f1 = _forcing(fm, w, dtype, rank_seed(rank))
            s1 = torch.empty_like(f1)
            for _ in range(args.warmup):
                p1.solve(f1, s1)
            torch.cuda.synchronize()
            msc = _timed(lambda: p1.solve(f1, s1), args.steps, world, stream, dist.barrier)
            control = {"parallelism": f"dp{world} (independent RHS batches per GPU)",
                       "scaling": "weak", "value": throughput(world, B, n, msc), "unit": UNIT,
                       "ms_per_step": msc}
            del p1, f1, s1
        except Exception as e:  # the control never hides the headline
            control = {"error": str(e)}
    exact = None if args.no_extra else all_ok(bool(eq_local), world, device=cdev)
    del sol_keep
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype_label(w), "data": "synthetic (seeded Fourier RHS, SURVEY 8(d))",
            "config": workload_config(args.workload, w, world, "patches", args.transport),
            "roofline": {"bound": "hbm", "achieved": alg / world / (ms_step / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s",
                         "frac": alg / world / (ms_step / 1e3) / 1e9 / peak, "traffic": None,
                         "kernel": "whole cycle per GPU (algorithmic words / unknown / shards)",
                         "peak_source": peak_src},
            "e2e": {"value": B * n / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": (c1 - c0) * B * esz * world,
                    "d2h_bytes_per_step": (c1 - c0) * B * esz * world, "ms_per_step": e2e_ms,
                    "api": "ShardedPlan.solve (fmgsr_plan_solve) on each rank's slab, "
                           "pinned host copies in the timed region"},
            "gpu_launches": info["launches_per_solve"] * args.steps,
            "clocks": clocks, "cpu_baseline": None,
            "control_rhs_batch": control,
            "sharded_bit_exact_vs_unsharded": exact,
            "transport": args.transport, "transport_timeouts": xerr,
            "forcing": "resident in the plan's own slab (fmgsr_shard_plan_forcing_slab): "
                       "no slab copy per solve",
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the config-2 line (N=1) / the RHS-batch control (N>1)")
    ap.add_argument("--e2e-chunks", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="exchanges of the patch-slab split: peer-memory pulls (default) or NCCL")
    ap.add_argument("--shard", default="patches", choices=["rhs", "patches"],
                    help="multi-GPU split: patch slabs of one problem (strong, SURVEY 8(e), "
                         "default) or independent RHS batches per rank (weak control)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    return args


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # --gpus is authoritative: one process per GPU under torchrun
        port = 29500 + os.getpid() % 2000
        return subprocess.call(spawn_cmd(args.gpus, argv, port))
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)
    if args.shard == "patches" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_gpu_sharded(args, w)
    return run_gpu(args, w)


if __name__ == "__main__":
    sys.exit(main())
