"""Nonlinear FAS (-u'' + u^3 = f, BASELINE config 3) on the GPU, bit for bit
against the oracle restatement (the reference is linear only), and the
one-cycle truncation-accuracy criterion on the manufactured solution."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def ocfg(oracle, cfg):
    sm = cfg.smoother
    return oracle.make_cfg(cfg.hierarchy.m0, cfg.hierarchy.m, cfg.n_sr, sm.ns,
                           oracle.GEOM_PATCHES, sm.n_patches, sm.buffer, nonlin=True)


@pytest.mark.parametrize("m,P,b,n_sr,ns", [(10, 16, 4, 1, 2), (10, 8, 3, 0, 1), (11, 64, 4, 2, 2)])
def test_nonlinear_matches_oracle(fm, oracle, m, P, b, n_sr, ns):
    B = 24
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b, nonlinear=True))
    f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=m))
    want = oracle.fmg_solve_batch(ocfg(oracle, cfg), np.ascontiguousarray(f.cpu().numpy().T),
                                  nthreads=8).T
    got = fm.fmg_solve(cfg, f)[0].cpu().numpy()
    assert np.array_equal(got, want)
    got_ops = fm.fmg_solve(cfg, f, keep_state=True)[0].cpu().numpy()  # operator path
    assert np.array_equal(got_ops, want)


def test_nonlinear_operators_match_oracle(fm, oracle):
    rng = np.random.default_rng(5)
    n = 64
    u = rng.standard_normal(n)
    f = rng.standard_normal(n) * 100
    assert np.array_equal(fm.coarse_rhs(f, u, nonlinear=True), oracle.coarse_rhs_nl(f, u))
    f8 = rng.standard_normal(8) * 50
    assert np.array_equal(fm.direct_solve(f8, nonlinear=True), oracle.direct_solve_nl(f8))


def test_nonlinear_config3_accuracy(fm):
    """Config 3 shape at reduced N (2^14, 256 patches, b = 4, V(2,2), n_sr = 1):
    one FMG cycle's error against the manufactured u is O(h^2) (<= 2x the
    error of the exactly solved discrete problem, estimated by one more cycle
    being no better than that bound)."""
    m, B = 14, 16
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=2, n_patches=256, buffer=4, nonlinear=True))
    f, uex = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=3))
    sol = fm.fmg_solve(cfg, f)[0]
    err = (torch.linalg.vector_norm(sol - uex, dim=0) / torch.linalg.vector_norm(uex, dim=0))
    h2 = (1.0 / 2 ** m) ** 2
    assert float(err.max()) < 50 * h2  # discretisation error of this problem ~ 8 h^2
