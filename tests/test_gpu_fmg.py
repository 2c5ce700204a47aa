"""Whole FMG-FAS(-SR) solves on the GPU: golden vectors from the reference,
the C oracle on batches, the reference's driver invariants
(test_cycles.py), and the one-cycle O(h^2) accuracy criterion."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GEOM = {0: "halo", 1: "global", 2: "patches"}


def config_from_params(fm, params):
    m0, m, n_sr, ns, kind, P, b = (int(x) for x in params)
    if kind == 2:
        sm = fm.SmootherConfig(ns=ns, n_patches=P, buffer=b)
    elif kind == 1:
        sm = fm.SmootherConfig(ns=ns, halo_mode=fm.HaloMode.GLOBAL)
    else:
        sm = fm.SmootherConfig(ns=ns, halo_mode=fm.HaloMode(str(b)))
    return fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr, smoother=sm)


@pytest.mark.parametrize("path", ["plan_fused", "plan_fused_nocoarse", "plan_coarse_all",
                                  "plan_unfused", "operators"])
def test_fmg_matches_golden(fm, golden, path):
    for name in golden["fmg_cases"]:
        p = str(name) + "/"
        cfg = config_from_params(fm, golden[p + "params"])
        forcing = golden[p + "forcing"]
        if path == "operators":
            got, _ = fm.fmg_solve(cfg, forcing, keep_state=True)
        elif path == "plan_fused_nocoarse":
            got, _ = fm.fmg_solve(cfg, forcing, coarse=0)
        elif path == "plan_coarse_all":  # every level but the finest on chip
            got, _ = fm.fmg_solve(cfg, forcing, coarse=cfg.hierarchy.m)
        else:
            got, _ = fm.fmg_solve(cfg, forcing, fused=(path == "plan_fused"))
        assert np.array_equal(got, golden[p + "solution"]), (path, str(name))


def oracle_cfg(oracle, cfg):
    sm = cfg.smoother
    if sm.n_patches is not None:
        return oracle.make_cfg(cfg.hierarchy.m0, cfg.hierarchy.m, cfg.n_sr, sm.ns,
                               oracle.GEOM_PATCHES, sm.n_patches, sm.buffer)
    if sm.halo_mode is fm_global(sm):
        return oracle.make_cfg(cfg.hierarchy.m0, cfg.hierarchy.m, cfg.n_sr, sm.ns,
                               oracle.GEOM_GLOBAL, 1, 0)
    return oracle.make_cfg(cfg.hierarchy.m0, cfg.hierarchy.m, cfg.n_sr, sm.ns, oracle.GEOM_HALO,
                           1, sm.halo_mode.halo)


def fm_global(sm):
    from paper_1207_6720_b200.mesh import HaloMode

    return HaloMode.GLOBAL


@pytest.mark.parametrize("m,P,b,n_sr,ns", [
    (10, 4, 2, 1, 1),        # config 1 geometry
    (12, 64, 4, 1, 1),       # config 2 geometry, reduced N
    (12, 64, 4, 0, 1),
    (12, 16, 1, 1, 1),       # config 5 cells, odd buffer
    (12, 1024, 8, 1, 1),
    (12, 256, 4, 2, 1),
    (13, 4096, 8, 1, 1),     # config 4 geometry (W = 2 on every level)
    (14, 4096, 8, 1, 1),     # ... with a width-4 finest level: group kernel on every grid level
    (11, 512, 40, 1, 1),     # buffer beyond the group kernel's limit: width-2 levels unfused
    (11, 256, 33, 0, 1),     # width 8 with a 33-cell buffer (streaming kernel), no SR
    (10, 16, 4, 1, 2),       # V(2,2)
    (10, 8, 3, 0, 2),
])
def test_fmg_batch_matches_oracle(fm, oracle, m, P, b, n_sr, ns):
    B = 40
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + P + b))
    want = oracle.fmg_solve_batch(oracle_cfg(oracle, cfg), np.ascontiguousarray(f.cpu().numpy().T),
                                  nthreads=8).T
    variants = {"auto": dict(), "unfused": dict(fused=False), "no_coarse": dict(coarse=0),
                "coarse_m0": dict(coarse=4), "coarse_mid": dict(coarse=m - 3),
                "coarse_all": dict(coarse=m), "whole_on_chip": dict(coarse=m + 1)}
    for name, kw in variants.items():
        got = fm.fmg_solve(cfg, f, **kw)[0].cpu().numpy()
        assert np.array_equal(got, want), name


def test_zero_forcing_gives_zero(fm):
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 5), n_sr=1,
                          smoother=fm.SmootherConfig(halo_mode=fm.HaloMode.HALO2))
    sol, _ = fm.fmg_solve(cfg, np.zeros(32))
    assert not np.any(sol)


def test_rejects_bad_config_and_size(fm):
    with pytest.raises(ValueError):
        fm.SolverConfig(hierarchy=fm.build_hierarchy(1, 6))
    with pytest.raises(ValueError):
        fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6), n_sr=4)
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 5))
    with pytest.raises(ValueError):
        fm.fmg_solve(cfg, np.zeros(16))


@pytest.mark.parametrize("mode,ns,n_sr", [
    (("halo", 2), 1, 2), (("halo", 4), 2, 1), (("global", 0), 1, 3), (("patches", 8), 1, 2)])
def test_expand_sr_reproduces_finest_field(fm, mode, ns, n_sr):
    if mode[0] == "patches":
        sm = fm.SmootherConfig(ns=ns, n_patches=mode[1], buffer=3)
    elif mode[0] == "global":
        sm = fm.SmootherConfig(ns=ns, halo_mode=fm.HaloMode.GLOBAL)
    else:
        sm = fm.SmootherConfig(ns=ns, halo_mode=fm.HaloMode(str(mode[1])))
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6), n_sr=n_sr, smoother=sm)
    forcing = fm.manufactured_rhs(64)
    solution, diag = fm.fmg_solve(cfg, forcing, keep_state=True)
    rebuilt = fm.expand_sr(diag.state, cfg)
    assert np.array_equal(rebuilt[:, 0].cpu().numpy(), solution)
    # and the fast path (native plan) gives the same field
    fast, _ = fm.fmg_solve(cfg, forcing)
    assert np.array_equal(fast, solution)


@pytest.mark.parametrize("mode", [fm_mode for fm_mode in ("2", "4")])
def test_debug_sr_poisoning_changes_nothing(fm, mode):
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 6), n_sr=2,
                          smoother=fm.SmootherConfig(halo_mode=fm.HaloMode(mode)))
    forcing = fm.manufactured_rhs(64)
    plain, _ = fm.fmg_solve(cfg, forcing)
    poisoned, _ = fm.fmg_solve(cfg, forcing, debug_sr=True)
    assert np.all(np.isfinite(poisoned))
    assert np.array_equal(plain, poisoned)


def test_final_working_rhs_is_original(fm):
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 5), n_sr=1,
                          smoother=fm.SmootherConfig(halo_mode=fm.HaloMode.HALO2))
    forcing = fm.manufactured_rhs(32)
    _, diag = fm.fmg_solve(cfg, forcing, keep_state=True)
    st = diag.state
    assert torch.equal(st.f_work[5], st.f_orig[5])
    assert np.array_equal(st.f_orig[5][:, 0].cpu().numpy(), forcing)
    assert np.array_equal(st.f_orig[4][:, 0].cpu().numpy(), fm.restrict(forcing))


@pytest.mark.parametrize("mode", ["2", "4", "global"])
def test_cycle_contracts_algebraic_error(fm, mode):
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(2, 7),
                          smoother=fm.SmootherConfig(halo_mode=fm.HaloMode(mode)))
    _, diag = fm.fmg_solve(cfg, fm.manufactured_rhs(128), collect_diagnostics=True)
    assert len(diag.levels) == 5
    for lev in diag.levels:
        assert lev.error_after_cycle < lev.error_after_prolong
        assert lev.gamma < 0.5
        assert np.isfinite(lev.residual_after_cycle)


def test_config1_truncation_accuracy(fm):
    """BASELINE config 1: N=2^10, m0=3, 4 SR patches, b=2, V(1,1), n_sr=1:
    one FMG cycle reaches the discretisation error (<= 2x direct solve)."""
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, 10), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=4, buffer=2))
    f, uex = fm.sine_problem(1024)
    sol, _ = fm.fmg_solve(cfg, f)
    direct = fm.direct_fine_solve(f)
    e_fmg = fm.rel_l2_error(sol, uex)
    e_dir = fm.rel_l2_error(direct, uex)
    assert e_fmg <= 2.0 * e_dir


@pytest.mark.slow
def test_config2_full_size(fm, oracle):
    """BASELINE config 2 at full size: N=2^16, P=64, b=4, B=1024, n_sr=1.
    Bitwise against the oracle on 8 seeded RHS; O(h^2) criterion on all."""
    m, B = 16, 1024
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    coef = fm.fourier_coefficients(B, seed=0)
    f, uex = fm.fourier_batch(2 ** m, coef)
    sol, _ = fm.fmg_solve(cfg, f)
    cols = [0, 1, 63, 64, 255, 511, 777, 1023]
    fh = f[:, cols].cpu().numpy().T.copy()
    want = oracle.fmg_solve_batch(oracle_cfg(oracle, cfg), fh, nthreads=8).T
    assert np.array_equal(sol[:, cols].cpu().numpy(), want)
    direct = fm.direct_fine_solve(f)
    err = torch.linalg.vector_norm(sol - uex, dim=0) / torch.linalg.vector_norm(uex, dim=0)
    derr = torch.linalg.vector_norm(direct - uex, dim=0) / torch.linalg.vector_norm(uex, dim=0)
    assert bool((err <= 2.0 * derr).all())


def test_float32_variant_bound(fm):
    """fp32 variant against the fp64 result: per-RHS inf-relative gap within the
    stated bound (2e-3 at N=2^12, growing ~ N)."""
    m, B = 12, 32
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=9))
    s64 = fm.fmg_solve(cfg, f)[0]
    s32 = fm.fmg_solve(cfg, f.float())[0]
    assert s32.dtype == torch.float32
    gap = (s32.double() - s64).abs().amax(0) / s64.abs().amax(0)
    assert float(gap.max()) <= 2e-3


def test_solve_host_pipelined_matches_device_solve(fm):
    """fmgsr_plan_solve_host: chunks of RHS pipelined H2D / solve / D2H give the
    same bits as the device-resident solve of the whole batch."""
    m, B, chunks = 11, 64, 4
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=21))
    want = fm.fmg_solve(cfg, f)[0].cpu()
    plan = fm.get_plan(fm.key_from_config(cfg, B // chunks, torch.float64))
    hf = f.cpu().pin_memory()
    hs = torch.zeros_like(hf).pin_memory()
    plan.solve_host(hf, hs, chunks)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(hs, want)


def test_solve_host_streaming_consecutive_batches(fm):
    """FMGSR_HOST_INPUTS_READY: back-to-back host solves of different batches
    overlap on the copy streams and each lands its own exact solution."""
    m, B, chunks = 11, 64, 4
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    plan = fm.get_plan(fm.key_from_config(cfg, B // chunks, torch.float64))
    fs = [fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=30 + i))[0] for i in range(3)]
    wants = [fm.fmg_solve(cfg, f)[0].cpu() for f in fs]
    hfs = [f.cpu().pin_memory() for f in fs]
    hss = [torch.zeros_like(h).pin_memory() for h in hfs]
    for hf, hs in zip(hfs, hss):
        plan.solve_host(hf, hs, chunks, inputs_ready=True)
    torch.cuda.current_stream().synchronize()
    for hs, want in zip(hss, wants):
        assert torch.equal(hs, want)


@pytest.mark.parametrize("m,P,b,n_sr", [(12, 64, 4, 1), (11, 16, 1, 2), (12, 4096, 8, 1)])
def test_warp_coarse_kernel_matches_oracle(fm, oracle, monkeypatch, m, P, b, n_sr):
    """The warp-per-column coarse kernel (default for V(2,2) / nonlinear,
    FMGSR_COARSE=warp for V(1,1)) on the linear V(1,1) path, bit for bit."""
    monkeypatch.setenv("FMGSR_COARSE", "warp")
    B = 33  # a batch no other test uses: fresh plans read the environment
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + b))
    want = oracle.fmg_solve_batch(oracle_cfg(oracle, cfg), np.ascontiguousarray(f.cpu().numpy().T),
                                  nthreads=8).T
    for kw in (dict(), dict(coarse=m - 2), dict(coarse=5)):
        got = fm.fmg_solve(cfg, f, **kw)[0].cpu().numpy()
        assert np.array_equal(got, want), kw


def _ordered_functional(sol, w, W, scale):
    """CPU restatement of the functional's summation order: per patch of W
    owned cells a sequential sum of w*u, then a sequential sum over patches."""
    n, B = sol.shape
    out = []
    for r in range(B):
        tot = 0.0
        for p in range(n // W):
            acc = 0.0
            for i in range(p * W, (p + 1) * W):
                acc = acc + (float(w[i, r]) * float(sol[i, r]) if w is not None else float(sol[i, r]))
            tot = tot + acc
        out.append(tot * scale)
    return np.array(out)


@pytest.mark.parametrize("m,P,b,n_sr,ns,nl,fused", [
    (11, 64, 4, 1, 1, False, True),    # fused: the reduction rides in the final visit
    (11, 64, 4, 0, 1, False, True),    # n_sr = 0: FAS-correction final visit
    (11, 64, 4, 1, 1, False, False),   # unfused plan
    (10, 16, 3, 1, 2, False, True),    # V(2,2)
    (10, 16, 4, 1, 2, True, True),     # nonlinear
])
def test_functional_output_matches_ordered_sum(fm, m, P, b, n_sr, ns, nl, fused):
    B = 8
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b, nonlinear=nl))
    if nl:
        f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=2))
    else:
        f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=5))
    plan = fm.get_plan(fm.key_from_config(cfg, B, torch.float64, fused=fused))
    sol = plan.solve(f).cpu().numpy()
    W = cfg.smoother.geometry(2 ** m).W
    g = torch.Generator(device="cuda").manual_seed(9)
    w = torch.rand(2 ** m, B, generator=g, device="cuda", dtype=torch.float64)
    got_w = plan.solve_functional(f, w).cpu().numpy()
    got_h = plan.solve_functional(f).cpu().numpy()
    assert np.array_equal(got_w, _ordered_functional(sol, w.cpu().numpy(), W, 1.0))
    assert np.array_equal(got_h, _ordered_functional(sol, None, W, 2.0 ** -m))
    # and it is the midpoint integral of the solution
    assert np.allclose(got_h, sol.sum(0) / 2 ** m, rtol=1e-13, atol=0)
    # the plain solve still works after functional graphs were captured
    assert np.array_equal(plan.solve(f).cpu().numpy(), sol)


@pytest.mark.parametrize("m,P,b,n_sr", [(12, 64, 4, 1), (12, 64, 4, 0), (12, 16, 1, 2),
                                        (12, 1024, 8, 1), (11, 4, 3, 1)])
def test_two_column_lanes_match_oracle(fm, oracle, m, P, b, n_sr):
    """B a multiple of 64: the visit kernels run two RHS columns per lane
    (V2 lanes); bit for bit against the oracle on every column, and the
    functional output reduces the same bits."""
    B = 128
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=1, n_patches=P, buffer=b))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + 7 * b + P))
    want = oracle.fmg_solve_batch(oracle_cfg(oracle, cfg), np.ascontiguousarray(f.cpu().numpy().T),
                                  nthreads=8).T
    for kw in (dict(), dict(fused=False), dict(coarse=0)):
        got = fm.fmg_solve(cfg, f, **kw)[0].cpu().numpy()
        assert np.array_equal(got, want), kw
    plan = fm.get_plan(fm.key_from_config(cfg, B, torch.float64))
    W = cfg.smoother.geometry(2 ** m).W
    got_h = plan.solve_functional(f).cpu().numpy()
    assert np.array_equal(got_h, _ordered_functional(want, None, W, 2.0 ** -m))


def test_two_column_lanes_fp32_match_scalar_lanes(fm):
    """fp32: a batch of 64 (two columns per lane) equals the same columns
    solved as two batches of 32 (one column per lane), bit for bit."""
    m = 12
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(64, seed=17))
    f = f.float()
    whole = fm.fmg_solve(cfg, f)[0]
    halves = torch.cat([fm.fmg_solve(cfg, f[:, :32].contiguous())[0],
                        fm.fmg_solve(cfg, f[:, 32:].contiguous())[0]], dim=1)
    assert torch.equal(whole, halves)


def _random_configs(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        m = int(rng.integers(6, 13))
        P = int(2 ** rng.integers(0, m - 2))
        b = int(rng.integers(0, 10))
        ns = int(rng.integers(1, 3))
        n_sr = int(rng.integers(0, 3))
        B = int(rng.choice([1, 7, 33, 64, 96, 128, 192]))
        coarse = int(rng.choice([-1, 0, m - 1, m, m + 1]))
        nl = bool(rng.integers(0, 4) == 0)
        out.append((m, P, b, ns, n_sr, B, coarse, nl))
    return out


@pytest.mark.parametrize("m,P,b,ns,n_sr,B,coarse,nl", _random_configs(64, 2026))
def test_random_configurations_match_oracle(fm, oracle, m, P, b, ns, n_sr, B, coarse, nl):
    """Seeded random sweep over geometry (P, odd and even buffers), V(1,1) /
    V(2,2), SR depth, linear / nonlinear, batch shapes (scalar lanes, two-column
    lanes, ragged) and coarse-level placement (auto, none, on-chip cutoffs,
    whole solve on chip): every column bit for bit against the oracle."""
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                          smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b, nonlinear=nl))
    if nl:
        f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=m + b))
    else:
        f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + b))
    oc = oracle.make_cfg(3, m, n_sr, ns, oracle.GEOM_PATCHES, P, b, nonlin=nl)
    want = oracle.fmg_solve_batch(oc, np.ascontiguousarray(f.cpu().numpy().T), nthreads=8).T
    got = fm.fmg_solve(cfg, f, coarse=coarse)[0].cpu().numpy()
    assert np.array_equal(got, want)


def test_plan_probe_events_time_the_finest_visits(fm):
    """fmgsr_plan_probe_ms: CUDA events recorded inside the replayed graph
    around the finest top / up visits (what bench.py's roofline divides by);
    -1 when the whole solve runs inside the on-chip coarse kernel."""
    m, B = 13, 64
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=1, n_patches=64, buffer=4))
    f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=3))
    plan = fm.get_plan(fm.key_from_config(cfg, B, torch.float64))
    sol = plan.solve(f)
    torch.cuda.synchronize()
    t, u = plan.probe_ms()
    assert 0 < t < 1e3 and 0 < u < 1e3
    assert torch.equal(sol, plan.solve(f))  # the probe nodes change nothing
    small = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, 10), n_sr=1,
                            smoother=fm.SmootherConfig(ns=1, n_patches=4, buffer=2))
    f1, _ = fm.fourier_batch(2 ** 10, fm.fourier_coefficients(1, seed=3))
    whole = fm.get_plan(fm.key_from_config(small, 1, torch.float64))
    whole.solve(f1)
    torch.cuda.synchronize()
    if whole.info()["coarse_cutoff"] == 10:
        assert whole.probe_ms() == (-1.0, -1.0)


