"""The patch-slab transport schedule checked on the host, no GPU:
``fmgsr_shard_schedule`` runs a shard's plan dry (same step list, same level
ping-pong state, every device call skipped) and exports every ncclSend /
ncclRecv / ncclAllGather / fix-up it would issue.  Across all ranks of a
sharded solve:

* every step's sends k -> p pair one-to-one, IN ISSUE ORDER (NCCL p2p has no
  tags), with the receives p posts from k: same count, same bytes, same tag;
* a halo row block lands on the same virtual-global rows it left from;
* every rank issues the identical all-gather sequence (collectives must
  match) on identical replicated buffers;
* fix-ups run exactly at the slab edges that have a neighbour.

So the NCCL path cannot deadlock on a mismatched group or deliver a halo to
the wrong rows.  Reference anchor: the additive, order-independent patch
contract (_kernels_numba.py:79-91) is what makes patches
shardable; the driver schedule is cycles.py:137-222."""

from collections import defaultdict

import pytest

import paper_1207_6720_b200 as fm
from paper_1207_6720_b200.shard import comm_schedule

GEOMS = {  # name: (m0, m, P, b, n_sr, B)
    "config2": (3, 16, 64, 4, 1, 1024),
    "config4": (3, 24, 4096, 8, 1, 64),
    "odd_b_sr0": (3, 16, 64, 3, 0, 96),
    "sr2_b1": (3, 14, 64, 1, 2, 64),
}


def _cfg(m0, m, P, b, n_sr):
    return fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr,
                           smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))


@pytest.mark.parametrize("name", sorted(GEOMS))
@pytest.mark.parametrize("S", [2, 4, 8])
def test_schedule_pairs_and_collectives_match(name, S):
    m0, m, P, b, n_sr, B = GEOMS[name]
    cfg = _cfg(m0, m, P, b, n_sr)
    scheds, cuts = [], set()
    for r in range(S):
        recs, cut, halo = comm_schedule(cfg, B, S, r)
        scheds.append(recs)
        cuts.add((cut, halo))
    assert len(cuts) == 1, "every rank must agree on the cutoff and halo"
    (cut, halo), = cuts
    assert m0 < cut < m
    nsteps = {max(x["step"] for x in s) for s in scheds}
    ld, es = B, 8
    for step in range(max(nsteps) + 1):
        by = [[x for x in s if x["step"] == step] for s in scheds]
        # point to point, in issue order per ordered pair
        for k in range(S):
            for p in range(S):
                snd = [x for x in by[k] if x["kind"] == "send" and x["peer"] == p]
                rcv = [x for x in by[p] if x["kind"] == "recv" and x["peer"] == k]
                assert len(snd) == len(rcv), (step, k, p)
                if snd:
                    assert abs(k - p) == 1, "slabs talk to their two neighbours only"
                for a, z in zip(snd, rcv):
                    assert (a["tag"], a["bytes"], a["array_level"]) == \
                           (z["tag"], z["bytes"], z["array_level"]), (step, k, p)
                    L = a["array_level"]
                    if L >= 0:  # halo rows: same virtual-global rows on both sides
                        assert a["bytes"] == halo * ld * es
                        rows = 2 ** L // S
                        assert z["addr"] - a["addr"] == (k - p) * rows * ld * es
                    else:  # tau edge record: 5 values per column
                        assert a["bytes"] == 5 * ((B + 31) // 32 * 32) * es
        # collectives: identical sequence on every rank, on the same replicated buffer
        gat = [[(x["bytes"], x["addr"], x["array_level"]) for x in by[r]
                if x["kind"] == "allgather"] for r in range(S)]
        assert all(g == gat[0] for g in gat), step
        for bytes_, _, L in gat[0]:
            assert L == cut and bytes_ == (2 ** cut // S) * ld * es
        # fix-ups exactly at the interior slab edges of epilogue visits
        for r in range(S):
            fx = [x for x in by[r] if x["kind"] == "fixup"]
            if fx:
                assert {x["tag"] for x in fx} == ({0} if r > 0 else set()) | \
                                                  ({1} if r < S - 1 else set())
    # every sharded level visit exchanges something; nothing below the cutoff does
    for s in scheds:
        for x in s:
            if x["kind"] in ("send", "recv") and x["array_level"] >= 0:
                assert x["array_level"] > cut


def test_schedule_counts_config4():
    """Config 4 at 8 shards: the exchange rounds the design budgets for."""
    m0, m, P, b, n_sr, B = GEOMS["config4"]
    recs, cut, halo = comm_schedule(_cfg(m0, m, P, b, n_sr), B, 8, 3)
    rounds = {x["step"] for x in recs if x["kind"] in ("send", "recv")}
    gathers = [x for x in recs if x["kind"] == "allgather"]
    assert halo == b + 8
    # one grouped exchange round per sharded visit (+ the forcing / cascade halos)
    assert 100 <= len(rounds) <= 200
    assert len(gathers) == 2 * (m - cut) + 1  # u and f at each descent into the cutoff + f once


def test_schedule_rejects_unshardable():
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, 8), n_sr=1,
                          smoother=fm.SmootherConfig(ns=2, n_patches=4, buffer=2))
    with pytest.raises(ValueError):
        comm_schedule(cfg, 32, 2, 0)
