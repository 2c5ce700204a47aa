"""The fused level visits and the f cascade as single ABI calls
(fmgsr_visit_{top,down,up}_*, fmgsr_f_cascade_*): each returns, bit for bit,
what the reference's operator composition returns on every column (the
oracle restates those operators: prolong_fmg / prolong_correction, the
additive patch smoother, restrict, coarse_rhs)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _patches(n, W, b):
    olo = np.arange(0, n, W, dtype=np.int64)
    ohi = olo + W
    elo = np.maximum(olo - b, 0)
    ehi = np.minimum(ohi + b, n)
    return olo, ohi, elo, ehi


def _smooth(O, u_in, f, n, W, b, uc=None):
    k = n.bit_length() - 1
    return O.smooth_patches(u_in, f, 4.0 ** k, *_patches(n, W, b), 1, uc=uc)


def _batch(n, B, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, B, generator=g, device="cuda", dtype=torch.float64)


CASES = [(1024, 64, 16, 4), (1024, 33, 64, 1), (512, 128, 8, 3), (2048, 64, 2048, 0), (256, 1, 4, 8),
         # short patches (owned width <= 8: the group kernel, kernels_group.cu): two and
         # four interleaved chains per lane, odd / zero buffers, ragged column counts
         (16384, 64, 4, 8), (16384, 96, 2, 8), (8192, 40, 8, 5), (4096, 33, 4, 1), (2048, 64, 8, 0),
         (64, 5, 2, 8), (32, 70, 4, 3)]


@pytest.mark.parametrize("n,B,W,b", CASES)
def test_visit_top_matches_composition(fm, oracle, n, B, W, b):
    from paper_1207_6720_b200 import visits

    if W < 4:
        pytest.skip("epilogue needs W >= 4")
    uH = _batch(n // 2, B, 1)
    f = _batch(n, B, 2) * 1e3
    u, uH2, fH = visits.visit_top(uH, f, W, b)
    none_u, uH3, fH3 = visits.visit_top(uH, f, W, b, store_u=False)
    assert none_u is None
    assert torch.equal(uH2, uH3) and torch.equal(fH, fH3)
    uHh, fh = uH.cpu().numpy(), f.cpu().numpy()
    for r in range(B):
        ur = _smooth(oracle, oracle.prolong_fmg(uHh[:, r]), fh[:, r], n, W, b)
        assert np.array_equal(u[:, r].cpu().numpy(), ur)
        assert np.array_equal(uH2[:, r].cpu().numpy(), oracle.restrict(ur))
        assert np.array_equal(fH[:, r].cpu().numpy(), oracle.coarse_rhs(fh[:, r], ur))


@pytest.mark.parametrize("n,B,W,b", CASES)
def test_visit_down_matches_composition(fm, oracle, n, B, W, b):
    from paper_1207_6720_b200 import visits

    if W < 4:
        pytest.skip("epilogue needs W >= 4")
    u = _batch(n, B, 3)
    f = _batch(n, B, 4) * 1e3
    for _ in range(2):  # the workspace counters return to their start state
        un, uH, fH = visits.visit_down(u, f, W, b)
    un2, none_uH, fH2 = visits.visit_down(u, f, W, b, restrict_u=False)
    assert none_uH is None and torch.equal(un2, un) and torch.equal(fH2, fH)
    uh, fh = u.cpu().numpy(), f.cpu().numpy()
    for r in range(B):
        ur = _smooth(oracle, uh[:, r], fh[:, r], n, W, b)
        assert np.array_equal(un[:, r].cpu().numpy(), ur)
        assert np.array_equal(uH[:, r].cpu().numpy(), oracle.restrict(ur))
        assert np.array_equal(fH[:, r].cpu().numpy(), oracle.coarse_rhs(fh[:, r], ur))


@pytest.mark.parametrize("n,B,W,b", CASES)
@pytest.mark.parametrize("sr", [False, True])
def test_visit_up_matches_composition(fm, oracle, n, B, W, b, sr):
    from paper_1207_6720_b200 import visits

    u = _batch(n, B, 5)
    uH = _batch(n // 2, B, 6)
    f = _batch(n, B, 7) * 1e3
    got = visits.visit_up(None if sr else u, uH, f, W, b, sr=sr)
    uh, uHh, fh = u.cpu().numpy(), uH.cpu().numpy(), f.cpu().numpy()
    for r in range(B):
        if sr:
            want = _smooth(oracle, oracle.prolong_fmg(uHh[:, r]), fh[:, r], n, W, b, uc=uHh[:, r])
        else:
            u_in = uh[:, r] + oracle.prolong_correction(uHh[:, r] - oracle.restrict(uh[:, r]))
            want = _smooth(oracle, u_in, fh[:, r], n, W, b)
        assert np.array_equal(got[:, r].cpu().numpy(), want)


@pytest.mark.parametrize("n,B,levels", [(4096, 64, 9), (1024, 3, 10), (256, 40, 1)])
def test_f_cascade_matches_repeated_restriction(fm, oracle, n, B, levels):
    from paper_1207_6720_b200 import visits

    f = _batch(n, B, 8)
    outs = visits.f_cascade(f, levels)
    assert len(outs) == levels
    fh = f.cpu().numpy()
    for r in range(B):
        x = fh[:, r]
        for j in range(levels):
            x = oracle.restrict(x)
            assert np.array_equal(outs[j][:, r].cpu().numpy(), x)


def test_visit_arguments_are_validated(fm):
    from paper_1207_6720_b200 import visits

    f = torch.zeros(64, 2, device="cuda", dtype=torch.float64)
    with pytest.raises(ValueError):
        visits.visit_down(f, f, 3, 1)       # odd owned width
    with pytest.raises(ValueError):
        visits.visit_down(f, f, 2, 1)       # epilogue needs W >= 4
    with pytest.raises(ValueError):
        visits.visit_top(f, f, 8, 1)        # u_coarse on the wrong level
    with pytest.raises(ValueError):
        visits.f_cascade(f, 7)              # more levels than the field has


@pytest.mark.parametrize("n_sr", [0, 1, 2])
def test_fmg_driver_from_fused_visits_matches_plan(fm, n_sr):
    """The reference's FMG-FAS-SR schedule (cycles.py:137-222) driven from
    Python with one fused-visit call per level visit reproduces the native
    plan's solution bit for bit (P = 4 patches, b = 2: owned width >= 4 on
    every smoothed level, so every visit is a fused one)."""
    from paper_1207_6720_b200 import visits

    m0, m, P, b, B = 3, 10, 4, 2, 64
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=12))
    want = fm.fmg_solve(cfg, f)[0]

    W = {l: max(2, 2 ** l // P) for l in range(m0, m + 1)}
    sr = {l: l > m - n_sr for l in range(m0, m + 1)}
    f_orig = {m: f}
    for j, fl in enumerate(visits.f_cascade(f, m - m0)):   # cycles.py:178-180
        f_orig[m - 1 - j] = fl
    u = {m0: fm.direct_solve(f_orig[m0])}                   # cycles.py:183
    for t in range(m0 + 1, m + 1):                          # cycles.py:187-199
        fw = {t: f_orig[t]}
        ut, u[t - 1], fw[t - 1] = visits.visit_top(u[t - 1], f_orig[t], W[t], b,
                                                   store_u=not sr[t])
        u[t] = ut
        for l in range(t - 1, m0, -1):                      # down leg, cycles.py:95-106
            u[l], ul1, fw[l - 1] = visits.visit_down(u[l], fw[l], W[l], b,
                                                     restrict_u=l - 1 > m0)
            if ul1 is not None:
                u[l - 1] = ul1
        u[m0] = fm.direct_solve(fw[m0])
        for l in range(m0 + 1, t + 1):                      # up leg, cycles.py:109-134
            u[l] = visits.visit_up(None if sr[l] else u[l], u[l - 1], fw[l], W[l], b, sr=sr[l])
    assert torch.equal(u[m], want)
