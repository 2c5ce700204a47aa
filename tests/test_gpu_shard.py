"""Patch-slab sharding with S virtual shards on one device: the
sharded schedule -- slab visits, halo and tau-edge-record exchanges, the
all-gather at the replication cutoff, redundant coarse levels -- must give
the unsharded solve bit for bit."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,P,b,n_sr,B,shards,coarse", [
    (12, 64, 4, 1, 64, 2, -1),
    (12, 64, 4, 1, 64, 4, 7),     # cutoff forced low: many sharded levels
    (13, 256, 8, 1, 32, 8, 6),    # config-4 style buffer, 8 shards
    (12, 32, 3, 0, 96, 4, 6),     # odd buffer, no SR, B not a power of two
    (12, 64, 1, 2, 64, 2, 6),     # b = 1 and two SR levels
    (13, 256, 8, 1, 128, 8, 6),   # two RHS columns per lane on the slabs, 8 shards
])
def test_shard_group_matches_unsharded(fm, m, P, b, n_sr, B, shards, coarse):
    from paper_1207_6720_b200.shard import ShardGroup

    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + shards))
    want = fm.fmg_solve(cfg, f, coarse=coarse)[0]
    g = ShardGroup(cfg, B, shards, coarse=coarse)
    assert g.cutoff < m  # something is sharded
    got = g.solve(f)
    torch.cuda.synchronize()
    assert torch.equal(got, want), (g.cutoff, g.halo)
    # replay of the captured graph gives the same bits
    got2 = g.solve(f)
    assert torch.equal(got2, want)


def test_shard_group_rejects_unshardable(fm):
    from paper_1207_6720_b200.shard import ShardGroup

    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, 8), n_sr=1,
                          smoother=fm.SmootherConfig(ns=2, n_patches=4, buffer=2))
    with pytest.raises(ValueError):
        ShardGroup(cfg, 32, 2)  # ns = 2 has no fused path
