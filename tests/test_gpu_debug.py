"""Memory-safety and stale-read checks of the native plan, standing in for
compute-sanitizer (closed on this GPU pool):

* guard zones (FMGSR_GUARDS=1): every workspace array sits between 4 KiB
  guards, and the caller's forcing / solution between guard rows; no solve
  may change a guard byte (out-of-bounds writes);
* NaN poisoning (FMGSR_DEBUG_POISON): each solve first fills every level
  field, edge record and scratch with NaN, and after each FMG step the SR
  levels below it -- the reference's debug_sr (cycles.py:161-165, 209-212;
  test_cycles.py:168-190): a read of anything not produced earlier in the
  same solve (or of a dead SR level) would surface as NaN; the solution must
  stay bit-identical to the oracle."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [  # m, P, b, n_sr, ns, nl, B, plan options
    (11, 16, 4, 1, 1, False, 32, dict()),                 # scalar lanes, bulk-TMA ring
    (11, 16, 3, 1, 1, False, 64, dict()),                 # two-column lanes
    (11, 32, 2, 2, 1, False, 40, dict()),                 # ragged batch, two SR levels
    (11, 64, 4, 0, 1, False, 64, dict(coarse=0)),         # no on-chip levels
    (11, 64, 4, 1, 1, False, 64, dict(fused=False)),      # unfused operator kernels
    (10, 8, 2, 1, 2, True, 32, dict()),                   # V(2,2) nonlinear
    (10, 16, 3, 0, 2, False, 32, dict()),                 # V(2,2) linear
    (10, 4, 2, 1, 1, False, 1, dict()),                   # whole solve on chip
    (12, 1024, 8, 1, 1, False, 64, dict(coarse=0)),       # short patches: the group kernel on every level
    (12, 512, 5, 2, 1, False, 40, dict(coarse=5)),        # ... odd buffer, ragged batch, two SR levels
]


@pytest.mark.parametrize("m,P,b,n_sr,ns,nl,B,opts", CASES)
def test_guards_and_poison(fm, oracle, monkeypatch, m, P, b, n_sr, ns, nl, B, opts):
    monkeypatch.setenv("FMGSR_GUARDS", "1")
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b, nonlinear=nl))
    n = 2 ** m
    if nl:
        f, _ = fm.nonlinear_batch(n, fm.nonlinear_scales(B, seed=m))
    else:
        f, _ = fm.fourier_batch(n, fm.fourier_coefficients(B, seed=m + P))
    oc = oracle.make_cfg(3, m, n_sr, ns, oracle.GEOM_PATCHES, P, b, nonlin=nl)
    want = oracle.fmg_solve_batch(oc, np.ascontiguousarray(f.cpu().numpy().T), nthreads=8).T
    plan = fm.FmgPlan(fm.key_from_config(cfg, B, torch.float64, **opts))
    assert plan.check_guards() == 0
    plan.set_debug(True)
    G = 64  # guard rows around the caller's buffers
    fbuf = torch.full((n + 2 * G, B), 7.25, dtype=torch.float64, device="cuda")
    sbuf = torch.full((n + 2 * G, B), -3.5, dtype=torch.float64, device="cuda")
    fbuf[G:G + n] = f
    for _ in range(2):  # capture + replay
        plan.solve(fbuf[G:G + n], sbuf[G:G + n])
        torch.cuda.synchronize()
        assert np.array_equal(sbuf[G:G + n].cpu().numpy(), want)
    assert bool((fbuf[:G] == 7.25).all()) and bool((fbuf[G + n:] == 7.25).all())
    assert bool((sbuf[:G] == -3.5).all()) and bool((sbuf[G + n:] == -3.5).all())
    assert torch.equal(fbuf[G:G + n], f)  # the forcing is read-only
    assert plan.check_guards() == 0
    plan.set_debug(False)
    del plan



def test_guards_absent_without_env(fm, monkeypatch):
    monkeypatch.delenv("FMGSR_GUARDS", raising=False)
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, 8), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=4, buffer=2))
    plan = fm.FmgPlan(fm.key_from_config(cfg, 8, torch.float64))
    assert plan.check_guards() == -1
