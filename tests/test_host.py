"""Host-side logic without a GPU: patch geometry, configuration validation,
the lane registry (reference backends.py semantics), plan keys, the bench
harness helpers, and the multi-rank (weak-scaling) aggregation over a gloo
process group of world size 2."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1207_6720_b200 as fm
from paper_1207_6720_b200 import mesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- geometry (reference mesh.py:102-147) -----------------------------------------------
def test_partition_matches_reference_rule():
    for mode, halo in ((fm.HaloMode.HALO2, 2), (fm.HaloMode.HALO4, 4)):
        pts = fm.partition(16, mode)
        assert len(pts) == 8
        for k, p in enumerate(pts):
            s = 2 * k
            assert p.owned == (s, s + 2)
            assert p.extended == (max(0, s - halo), min(16, s + 2 + halo))
    assert fm.partition(32, fm.HaloMode.GLOBAL) == [fm.Patch((0, 32), (0, 32))]
    with pytest.raises(ValueError):
        fm.partition(2, fm.HaloMode.HALO2)
    with pytest.raises(ValueError):
        fm.partition(7, fm.HaloMode.HALO2)


def test_p_patch_geometry():
    g = fm.level_geometry(2 ** 16, n_patches=64, buffer=4)
    assert (g.W, g.b, g.n_patches) == (1024, 4, 64)
    g = fm.level_geometry(64, n_patches=64, buffer=4)  # n/P < 2: the reference HALO partition
    assert (g.W, g.b) == (2, 4)
    assert g.patches() == fm.partition(64, fm.HaloMode.HALO4)
    arr = mesh.patch_arrays(fm.level_geometry(32, n_patches=4, buffer=3).patches())
    assert [a.tolist() for a in arr] == [[0, 8, 16, 24], [8, 16, 24, 32], [0, 5, 13, 21],
                                         [11, 19, 27, 32]]


def test_patch_validation():
    with pytest.raises(ValueError):
        fm.Patch((2, 4), (3, 8))


# ---- configuration (reference cycles.py:31-53, smoothers.py:22-37, mesh.py:48-76) ---------
def test_config_validation():
    with pytest.raises(ValueError):
        fm.SmootherConfig(ns=0)
    with pytest.raises(ValueError):
        fm.SmootherConfig(n_patches=3)
    with pytest.raises(ValueError):
        fm.SmootherConfig(buffer=-1)
    with pytest.raises(ValueError):
        fm.build_hierarchy(3, 3)
    with pytest.raises(ValueError):
        fm.SolverConfig(hierarchy=fm.build_hierarchy(1, 6))
    with pytest.raises(ValueError):
        fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6), n_sr=4)
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6), n_sr=2)
    assert not cfg.is_sr_level(4) and cfg.is_sr_level(5) and cfg.is_sr_level(6)


def test_plan_key_from_config():
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, 16), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    k = fm.key_from_config(cfg, 1024, torch.float64)
    assert (k.m0, k.m, k.n_sr, k.ns, k.geom_mode, k.P, k.b, k.B) == (3, 16, 1, 1, 2, 64, 4, 1024)
    k = fm.key_from_config(fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6)), 1, torch.float32)
    assert (k.geom_mode, k.b, k.dtype) == (0, 2, torch.float32)
    glob = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6),
                           smoother=fm.SmootherConfig(halo_mode=fm.HaloMode.GLOBAL))
    assert fm.key_from_config(glob, 1, torch.float64).geom_mode == 1


# ---- lane registry (reference backends.py:20-63) -------------------------------------------
def test_backend_registry():
    assert fm.available_backends() == ("cuda",)
    with pytest.raises(ValueError):
        fm.set_backend("numba")  # no CPU lane exists: unknown names raise
    fm.set_backend("cuda")
    assert fm.get_backend() == "cuda"


@pytest.mark.parametrize("value,expect", [("cuda", "cuda"), ("", "cuda"), ("numpy", "rejected")])
def test_env_var_selects_or_rejects(value, expect):
    code = ("import paper_1207_6720_b200.backends as b\n"
            "try:\n    print(b.get_backend())\nexcept ValueError:\n    print('rejected')\n")
    env = dict(os.environ, FMGSR_BACKEND=value, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == expect


def test_device_entry_points_fail_loudly_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        fm.restrict(np.ones(8))


# ---- bench helpers ------------------------------------------------------------------------------
def test_bench_throughput_and_config():
    import bench

    assert bench.throughput(2, 1024, 65536, 4.0) == pytest.approx(2 * 1024 * 65536 / 4e-3)
    cfg = bench.workload_config("config2", bench.WORKLOADS["config2"], 8, "rhs")
    assert cfg["global_batch"] == 8 * 1024 and cfg["N"] == 2 ** 16
    assert "L2" in cfg["l2"] or "inputs larger" in cfg["l2"]


def test_bench_cpu_baseline_sample():
    import bench

    v, k, dt = bench.cpu_rate(bench.WORKLOADS["config1"], 0.2, 2)
    assert v > 0 and k >= 2 and dt > 0


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    ms = 3.0 + rank  # ranks finish at different times
    worst = bench.reduce_max(ms, world, device="cpu")
    q.put((rank, worst, bench.rank_seed(rank), bench.throughput(world, 1024, 2 ** 16, worst)))
    dist.destroy_process_group()


def test_multirank_aggregation_gloo():
    """Weak scaling: each rank solves its own batch (distinct seeds); the job
    is charged the slowest rank's time."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [4.0, 4.0]
    assert res[0][2] != res[1][2]
    assert res[0][3] == pytest.approx(2 * 1024 * 2 ** 16 / 4e-3)


# ---- multi-GPU host plumbing of bench.py (gloo, CPU) ---------------------------------------------
def test_bench_gpus_is_authoritative():
    import bench

    bench.check_world(4, 4)
    with pytest.raises(SystemExit, match="--gpus 8 but WORLD_SIZE=1"):
        bench.check_world(8, 1)
    cmd = bench.spawn_cmd(8, ["--gpus", "8", "--steps", "3"], 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "8", "--steps", "3"]
    a = bench.parse_args(["--gpus", "2"])
    assert a.workload == "config4" and a.shard == "patches" and a.warmup >= 3


def test_bench_sharded_config_line():
    import bench

    c = bench.workload_config("config4", bench.WORKLOADS["config4"], 8, "patches")
    assert c["global_batch"] == 64 and "patch slabs x8" in c["parallelism"]
    c1 = bench.workload_config("config4", bench.WORKLOADS["config4"], 8, "rhs")
    assert c1["global_batch"] == 8 * 64 and c1["parallelism"].startswith("dp8")


def _shard_rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1207_6720_b200.shard import slab

    uid = bytes(range(128)) if rank == 0 else None  # stands in for ncclGetUniqueId
    got = bench.broadcast_uid(uid, rank, device="cpu")
    n = 2 ** 24
    # the fall-back vote of run_gpu_sharded: one failing rank moves every rank
    votes = (bench.all_ok(True, world, device="cpu"), bench.all_ok(rank != world - 1, world, device="cpu"))
    q.put((rank, got, slab(n, world, rank), votes))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_host_side_gloo(world):
    """run_gpu_sharded's host side: rank 0's NCCL id reaches every rank, the
    slabs tile the finest level exactly once, and a failure on one rank makes
    every rank take the fall-back (all_ok is a MIN over ranks)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 500) + world
    procs = [ctx.Process(target=_shard_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == bytes(range(128)) for r in res)
    assert all(r[3] == (True, False) for r in res)
    spans = [r[2] for r in res]
    assert spans[0][0] == 0 and spans[-1][1] == 2 ** 24
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
