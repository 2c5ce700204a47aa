"""Patch-slab sharding of one FMG-FAS-SR solve.

The finest levels are split into S contiguous slabs of patches (the additive
smoother makes patches independent; only stencil halos and the tau edge
records at slab boundaries couple neighbours); levels at or below the
replication cutoff are all-gathered once per V-cycle and solved redundantly
by every shard.  Two drivers run the same sharded schedule:

* ``ShardGroup``: S virtual shards on the current device, in lockstep on one
  stream, transfers as device copies -- bit-identical to the unsharded plan
  (``tests/test_gpu_shard.py``);
* ``ShardedPlan``: one shard per GPU (one process per GPU, torchrun), halos
  and edge records over NCCL send/recv and the cutoff level over NCCL
  all-gather -- or, ``transport="p2p"``, pulled straight from the peers'
  workspaces over peer memory with device-side counters -- all captured in
  the plan's CUDA graph.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .plan import PlanKey, dtype_code, key_from_config


def _desc(key: PlanKey) -> N.PlanDesc:
    d = N.PlanDesc()
    d.m0, d.m, d.n_sr, d.ns = key.m0, key.m, key.n_sr, key.ns
    d.geom_mode = key.geom_mode
    d.dtype = dtype_code(key)
    d.P, d.b, d.B, d.ld = key.P, key.b, key.B, key.B
    d.omega = key.omega
    d.fused = int(key.fused)
    d.use_graph = int(key.use_graph)
    d.coarse = int(key.coarse)
    d.nonlinear = int(key.nonlinear)
    return d


def slab(n: int, shards: int, rank: int) -> tuple[int, int]:
    """Rows [c0, c1) of an n-cell level owned by ``rank``."""
    w = n // shards
    return rank * w, (rank + 1) * w


class ShardGroup:
    """All ``shards`` slabs of one problem on this device (virtual shards)."""

    def __init__(self, cfg, B: int, shards: int, dtype=torch.float64, coarse: int = -1,
                 use_graph: bool = True):
        N.require_cuda()
        self.key = key_from_config(cfg, B, dtype, use_graph=use_graph, coarse=coarse)
        d = _desc(self.key)
        h = C.c_void_p()
        N.check(N.lib().fmgsr_shard_group_create(C.byref(d), int(shards), C.byref(h)),
                "shard_group_create")
        self._h = h
        self.shards = shards
        self.N = 2 ** self.key.m
        cut, halo = C.c_int32(), C.c_int64()
        N.check(N.lib().fmgsr_shard_group_cutoff(h, C.byref(cut), C.byref(halo)), "cutoff")
        self.cutoff, self.halo = cut.value, halo.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().fmgsr_shard_group_destroy(h)
            except Exception:
                pass
            self._h = None

    def solve(self, forcing: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(forcing)
        k = self.key
        for t in (forcing, out):
            if not t.is_cuda or t.dtype != k.dtype or tuple(t.shape) != (self.N, k.B) \
                    or not t.is_contiguous():
                raise ValueError(f"expected a contiguous CUDA {k.dtype} tensor ({self.N}, {k.B})")
        N.check(N.lib().fmgsr_shard_group_solve(self._h, forcing.data_ptr(), out.data_ptr(),
                                                N.stream_ptr()), "shard_group_solve")
        return out


class _DeviceView:
    """A device array owned by a plan, exposed through __cuda_array_interface__
    (the tensor made from it keeps this object, and so the plan, alive)."""

    def __init__(self, ptr: int, shape, dtype, owner):
        self._owner = owner
        typestr = {torch.float64: "<f8", torch.float32: "<f4"}[dtype]
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": None}


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.check(N.lib().fmgsr_nccl_unique_id(buf), "nccl_unique_id")
    return bytes(buf)


def _allgather_bytes(blob: bytes) -> list[bytes]:
    """Every rank's blob in rank order over the default torch.distributed group."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, blob)
    return out


class ShardedPlan:
    """This rank's shard of one problem, one GPU per rank.

    ``transport="nccl"``: halos, edge records and the cutoff gather over NCCL
    send / recv / all-gather; ``uid`` is the 128-byte id from
    ``nccl_unique_id()`` on rank 0, broadcast to every rank (e.g. with
    torch.distributed).
    ``transport="p2p"``: no collective library -- every rank maps its peers'
    plan workspaces (CUDA IPC, NVLink peer access) and pulls what it needs with
    device-side release / acquire counters (fmgsr_shard_plan_create_p2p);
    ``exchange(blob) -> [blob of rank 0, ..., blob of rank S-1]`` is any host
    all-gather (default: torch.distributed.all_gather_object), used once.  It
    also runs with several ranks on ONE GPU (the one-GPU multi-process tests).
    ``solve`` takes and returns the rank's slab: (2**m / shards, B) rows
    [c0, c1) of the global arrays."""

    def __init__(self, cfg, B: int, shards: int, rank: int, uid: bytes | None = None,
                 dtype=torch.float64, coarse: int = -1, use_graph: bool = True,
                 transport: str = "nccl", exchange=None):
        N.require_cuda()
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport must be 'nccl' or 'p2p', got {transport!r}")
        self.key = key_from_config(cfg, B, dtype, use_graph=use_graph, coarse=coarse)
        d = _desc(self.key)
        h = C.c_void_p()
        if transport == "nccl":
            if uid is None:
                raise ValueError("the NCCL transport needs the rank-0 unique id (uid)")
            idbuf = (C.c_uint8 * 128).from_buffer_copy(uid)
            N.check(N.lib().fmgsr_shard_plan_create(C.byref(d), int(shards), int(rank), idbuf,
                                                    C.byref(h)), "shard_plan_create")
        else:
            N.check(N.lib().fmgsr_shard_plan_create_p2p(C.byref(d), int(shards), int(rank),
                                                        C.byref(h)), "shard_plan_create_p2p")
        self._h = h
        self.shards, self.rank, self.transport = shards, rank, transport
        self.rows = 2 ** self.key.m // shards
        if transport == "p2p":
            n = C.c_int64()
            N.check(N.lib().fmgsr_shard_p2p_export(h, None, 0, C.byref(n)), "shard_p2p_export")
            buf = (C.c_uint8 * n.value)()
            N.check(N.lib().fmgsr_shard_p2p_export(h, buf, n.value, C.byref(n)),
                    "shard_p2p_export")
            blobs = (exchange or _allgather_bytes)(bytes(buf))
            if len(blobs) != shards or any(len(b) != n.value for b in blobs):
                raise ValueError("p2p exchange: expected one blob per rank of equal size")
            allb = (C.c_uint8 * (n.value * shards)).from_buffer_copy(b"".join(blobs))
            N.check(N.lib().fmgsr_shard_p2p_import(h, allb, n.value), "shard_p2p_import")

    def forcing_slab(self) -> torch.Tensor:
        """The plan's own finest-level forcing slab as a (rows, B) CUDA tensor
        (fmgsr_shard_plan_forcing_slab).  Fill it and pass it to ``solve``: the
        solve then reads the forcing where it lies instead of first copying the
        caller's slab into the plan (2 x the slab bytes of HBM traffic)."""
        ptr, rows = C.c_void_p(), C.c_int64()
        N.check(N.lib().fmgsr_shard_plan_forcing_slab(self._h, C.byref(ptr), C.byref(rows)),
                "shard_plan_forcing_slab")
        k = self.key
        return torch.as_tensor(_DeviceView(ptr.value, (rows.value, k.B), k.dtype, self),
                               device="cuda")

    def status(self) -> int:
        """p2p transport: synchronise and return 0, or non-zero if a peer wait timed out."""
        err = C.c_int32()
        N.check(N.lib().fmgsr_shard_p2p_status(self._h, C.byref(err)), "shard_p2p_status")
        return err.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().fmgsr_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def solve(self, forcing_slab: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(forcing_slab)
        k = self.key
        for name, t in (("forcing slab", forcing_slab), ("solution slab", out)):
            if not t.is_cuda or t.dtype != k.dtype or tuple(t.shape) != (self.rows, k.B) \
                    or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous {k.dtype} CUDA tensor of shape "
                                 f"({self.rows}, {k.B})")
        if forcing_slab.data_ptr() == out.data_ptr():
            raise ValueError("the solution slab must not alias the forcing slab")
        N.check(N.lib().fmgsr_plan_solve(self._h, forcing_slab.data_ptr(), out.data_ptr(),
                                         N.stream_ptr()), "plan_solve")
        return out

    def solve_timed(self, forcing_slab: torch.Tensor, out: torch.Tensor):
        """Op by op with CUDA events per level visit: [(kind, level, ms)]."""
        cap = 8192
        ms = (C.c_float * cap)()
        lvl = (C.c_int32 * cap)()
        kind = (C.c_int32 * cap)()
        nv = C.c_int64()
        N.check(N.lib().fmgsr_plan_solve_timed(self._h, forcing_slab.data_ptr(), out.data_ptr(),
                                               N.stream_ptr(), ms, lvl, kind, cap,
                                               C.byref(nv)), "plan_solve_timed")
        names = {0: "top", 1: "down", 2: "up", 3: "direct", 4: "cascade", 5: "coarse"}
        return [(names[kind[i]], lvl[i], ms[i]) for i in range(min(nv.value, cap))]

    def info(self) -> dict:
        inf = N.PlanInfo()
        N.check(N.lib().fmgsr_plan_get_info(self._h, C.byref(inf)), "plan_get_info")
        return {"workspace_bytes": inf.workspace_bytes,
                "launches_per_solve": inf.launches_per_solve,
                "alg_bytes_per_solve": inf.alg_bytes_per_solve}


class LocalShardPlan(ShardedPlan):
    """Shard ``rank`` of ``shards`` with NO transport (fmgsr_shard_plan_create_local):
    the shard's kernels and slab-edge fix-ups on this GPU, halos never
    exchanged.  Times one shard's share of a sharded solve on one GPU; the
    output is not a solution."""

    def __init__(self, cfg, B: int, shards: int, rank: int, dtype=torch.float64,
                 coarse: int = -1, use_graph: bool = True):
        N.require_cuda()
        self.key = key_from_config(cfg, B, dtype, use_graph=use_graph, coarse=coarse)
        d = _desc(self.key)
        h = C.c_void_p()
        N.check(N.lib().fmgsr_shard_plan_create_local(C.byref(d), int(shards), int(rank),
                                                      C.byref(h)), "shard_plan_create_local")
        self._h = h
        self.shards, self.rank = shards, rank
        self.rows = 2 ** self.key.m // shards


STEP_KINDS = ("loadf", "cascade_hi", "cascade_lo", "coarse_fmg", "top", "down", "coarse_v", "up")
COMM_KINDS = ("send", "recv", "allgather", "fixup")


def comm_schedule(cfg, B: int, shards: int, rank: int, dtype=torch.float64, coarse: int = -1):
    """The transport schedule of shard ``rank`` (fmgsr_shard_schedule; host
    only, no GPU needed): ``(records, cutoff, halo_rows)`` with one dict per
    send / recv / all-gather / fix-up in the order the plan issues them."""
    key = key_from_config(cfg, B, dtype, coarse=coarse)
    d = _desc(key)
    n, cut, halo = C.c_int64(), C.c_int32(), C.c_int64()
    L = N.lib()
    N.check(L.fmgsr_shard_schedule(C.byref(d), int(shards), int(rank), None, 0, C.byref(n),
                                   C.byref(cut), C.byref(halo)), "shard_schedule")
    recs = (N.CommRec * max(1, n.value))()
    N.check(L.fmgsr_shard_schedule(C.byref(d), int(shards), int(rank), recs, n.value,
                                   C.byref(n), C.byref(cut), C.byref(halo)), "shard_schedule")
    out = [{"step": r.step, "step_kind": STEP_KINDS[r.step_kind], "level": r.level,
            "array_level": r.array_level,
            "kind": COMM_KINDS[r.kind], "peer": r.peer, "tag": r.tag, "bytes": r.bytes,
            "addr": r.addr} for r in recs[:n.value]]
    return out, cut.value, halo.value
