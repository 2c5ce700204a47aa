"""The sharded plan across PROCESSES: S ranks (one process each, gloo for the
one-time host exchange) run ``ShardedPlan(transport="p2p")`` -- halos, tau
edge records and the cutoff gather pulled from the peers' workspaces over CUDA
IPC with device-side release / acquire counters, no collective library -- and
their slabs must give the unsharded solve bit for bit.  On the one-GPU pool
every rank maps the same device (the contexts time-slice); across GPUs the same
mappings go over NVLink peer access."""

import multiprocessing as mp
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # m, P, b, n_sr, B, shards, coarse, dtype
    (12, 64, 4, 1, 64, 2, -1, "f64"),
    (13, 256, 8, 1, 64, 4, 6, "f64"),   # config-4 style buffer, cutoff forced low: many rounds
    (12, 32, 3, 0, 96, 2, 6, "f64"),    # odd buffer, no SR, B not a multiple of 64
    (13, 256, 8, 2, 64, 8, 6, "f64"),   # 8 ranks, two SR levels
    (12, 64, 4, 1, 64, 4, 6, "f32"),    # fp32 fields
]


def _cfg(fm, m, P, b, n_sr):
    return fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                           smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))


def _rank_main(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), FMGSR_P2P_TIMEOUT_S="60")
    try:
        import torch
        import torch.distributed as dist

        import paper_1207_6720_b200 as fm
        from paper_1207_6720_b200.shard import ShardedPlan, slab

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        m, P, b, n_sr, B, S, coarse, dt = case
        dtype = torch.float64 if dt == "f64" else torch.float32
        cfg = _cfg(fm, m, P, b, n_sr)
        f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + S), dtype)
        c0, c1 = slab(2 ** m, S, rank)
        plan = ShardedPlan(cfg, B, S, rank, dtype=dtype, coarse=coarse, transport="p2p")
        fs = f[c0:c1].contiguous()
        out = plan.solve(fs)
        torch.cuda.synchronize()
        first = out.cpu().numpy().copy()
        out2 = plan.solve(fs)  # graph replay: the epoch advances on the device
        second = out2.cpu().numpy().copy()
        # the forcing written into the plan's own slab: solved in place (no slab copy)
        own = plan.forcing_slab()
        assert tuple(own.shape) == tuple(fs.shape) and own.dtype == fs.dtype
        own.copy_(fs)
        out3 = plan.solve(own)
        out3 = plan.solve(own)  # and its graph replayed
        err = plan.status()
        q.put((rank, first, second, out3.cpu().numpy(), err, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent, never a hang
        q.put((rank, None, None, None, -1, f"{type(e).__name__}: {e}"))


@pytest.mark.parametrize("case", CASES)
def test_p2p_sharded_processes_match_unsharded(fm, case):
    import torch

    m, P, b, n_sr, B, S, coarse, dt = case
    dtype = torch.float64 if dt == "f64" else torch.float32
    want = fm.fmg_solve(_cfg(fm, m, P, b, n_sr),
                        fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + S),
                                         dtype)[0],
                        coarse=coarse)[0]
    torch.cuda.synchronize()
    want = want.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import socket

    with socket.socket() as sk:  # a free port for this group's rendezvous
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = [ctx.Process(target=_rank_main, args=(r, S, port, case, q)) for r in range(S)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, a, a2, a3, err, msg = q.get(timeout=240)
            res[r] = (a, a2, a3, err, msg)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(S):
        a, a2, a3, err, msg = res[r]
        assert msg is None, f"rank {r}: {msg}"
        assert err == 0, f"rank {r}: a peer wait timed out"
        rows = 2 ** m // S
        assert np.array_equal(a, want[r * rows:(r + 1) * rows]), f"rank {r} differs"
        assert np.array_equal(a2, a), f"rank {r}: graph replay differs"
        assert np.array_equal(a3, a), f"rank {r}: in-place forcing slab differs"
