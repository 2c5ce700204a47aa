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


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_split_division_is_ieee_division(fm, dtype):
    """The smoother's x / J (reciprocal of J ahead of the dependency chain +
    two Markstein corrections) is bitwise the IEEE division: random x over the
    whole exponent range (incl. zeros, subnormals, inf, nan) against J in the
    Jacobian's range 2*4^k + 3u^2, plus J at and next to powers of two."""
    from paper_1207_6720_b200 import _native as N

    g = torch.Generator(device="cuda").manual_seed(11)
    n = 1 << 24
    idt = torch.int64 if dtype == torch.float64 else torch.int32
    nbits = 64 if dtype == torch.float64 else 32
    # x: uniformly random bit patterns (every exponent, both signs)
    raw = torch.randint(-(2 ** (nbits - 1)), 2 ** (nbits - 1) - 1, (n,), generator=g, device="cuda",
                        dtype=torch.int64).to(idt)
    x = raw.view(dtype).clone()
    x[:64] = torch.tensor([0.0, -0.0, float("inf"), float("-inf"), float("nan")] * 12 + [1.0] * 4,
                          dtype=dtype, device="cuda")
    k = torch.randint(1, 21, (n,), generator=g, device="cuda").to(dtype)
    u = torch.randn(n, generator=g, device="cuda", dtype=torch.float64).to(dtype) * \
        torch.exp2(torch.randint(-30, 12, (n,), generator=g, device="cuda").to(dtype))
    J = 2 * torch.exp2(2 * k) + 3 * u * u
    J[: n // 8] = torch.exp2(torch.randint(3, 60, (n // 8,), generator=g, device="cuda").to(dtype))
    J[n // 8: n // 4] = torch.nextafter(J[: n // 8], torch.tensor(0.0, dtype=dtype, device="cuda"))
    J[n // 4: 3 * n // 8] = torch.nextafter(J[: n // 8], torch.tensor(float("inf"), dtype=dtype,
                                                                       device="cuda"))
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.call("fmgsr_div_check", dtype, x.data_ptr(), J.data_ptr(), None, n, bad.data_ptr(),
           N.stream_ptr())
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
    # moderate magnitudes, where the fast path is taken
    x2 = torch.randn(n, generator=g, device="cuda", dtype=torch.float64).to(dtype) * 1e3
    N.call("fmgsr_div_check", dtype, x2.data_ptr(), J.data_ptr(), None, n, bad.data_ptr(),
           N.stream_ptr())
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


@pytest.mark.parametrize("nonlinear", [True, False])
def test_ns2_omega_matches_oracle(fm, oracle, nonlinear):
    """V(2,2) streaming smoother with omega != 1 (the OMEGA1 = false kernels)."""
    B, m = 40, 10
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=2, n_patches=16, buffer=3, omega=0.8,
                                                     nonlinear=nonlinear))
    f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=4))
    oc = oracle.make_cfg(3, m, 1, 2, oracle.GEOM_PATCHES, 16, 3, nonlin=nonlinear, omega=0.8)
    want = oracle.fmg_solve_batch(oc, np.ascontiguousarray(f.cpu().numpy().T), nthreads=8).T
    got = fm.fmg_solve(cfg, f)[0].cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("nonlinear", [True, False])
def test_ns2_two_column_lanes_match_oracle(fm, oracle, nonlinear):
    """V(2,2) with B = 64 and long chains (W >= 256 on levels 10-12): the
    FAS-correction visits run two RHS columns per lane; every column bit for
    bit against the oracle."""
    m, P, b, B = 12, 4, 4, 64
    cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=1,
                          smoother=fm.SmootherConfig(ns=2, n_patches=P, buffer=b,
                                                     nonlinear=nonlinear))
    if nonlinear:
        f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=4))
    else:
        f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=4))
    oc = oracle.make_cfg(3, m, 1, 2, oracle.GEOM_PATCHES, P, b, nonlin=nonlinear)
    want = oracle.fmg_solve_batch(oc, np.ascontiguousarray(f.cpu().numpy().T), nthreads=8).T
    for kw in (dict(), dict(coarse=0)):
        got = fm.fmg_solve(cfg, f, **kw)[0].cpu().numpy()
        assert np.array_equal(got, want), kw


# ---- pinned to the reference's own driver (oracle/gen_golden_nl.py) ---------------------------
def _nl_golden():
    import os

    return np.load(os.path.join(os.path.dirname(__file__), "golden", "nonlinear.npz"))


def test_nonlinear_matches_reference_driver(fm):
    """Every reduced-size case of tests/golden/nonlinear.npz (the reference's
    FMG driver with the Newton-GS lane, N(u) tau and Newton coarse solve
    injected), solved as columns of one batch (column 0 the case, the rest
    scaled copies): the case column bit for bit, through the fused plan and the
    operator path."""
    g = _nl_golden()
    for name in g["cases"]:
        m0, m, n_sr, ns, _, P, b = (int(x) for x in g[f"{name}/params"])
        cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr,
                              smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b,
                                                         nonlinear=True))
        f0 = g[f"{name}/forcing"]
        F = np.stack([f0 * s for s in (1.0, 0.5, 2.0, 1.5)], axis=1)
        f = torch.as_tensor(np.ascontiguousarray(F), device="cuda")
        for kw in (dict(), dict(keep_state=True), dict(coarse=0)):
            got = fm.fmg_solve(cfg, f, **kw)[0][:, 0].cpu().numpy()
            assert np.array_equal(got, g[f"{name}/solution"]), (str(name), kw)


@pytest.mark.slow
def test_nonlinear_config3_full_size_reference_hash(fm):
    """Config 3 at its full size (N = 2^20, 256 patches, b = 4, V(2,2), one SR
    level, nonlinear): the hash-forcing column inside a 256-column batch (the
    bench's batch shape and kernels) reproduces the reference-driver SHA-256."""
    import hashlib

    g = _nl_golden()
    for name in g["hash_cases"]:
        m0, m, n_sr, ns, _, P, b, salt = (int(x) for x in g[f"{name}/params"])
        i = np.arange(2 ** m, dtype=np.uint64)
        h = (i * np.uint64(2654435761) + np.uint64(salt)) % np.uint64(1 << 32)
        f0 = float(g[f"{name}/scale"]) * (h.astype(np.float64) / float(1 << 32) - 0.5)
        cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr,
                              smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b,
                                                         nonlinear=True))
        B = 256
        fcol = torch.as_tensor(f0, device="cuda")
        f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=7))
        f[:, 5] = fcol
        sol = fm.fmg_solve(cfg, f)[0]
        got = sol[:, 5].cpu().numpy()
        assert np.array_equal(got[:64], g[f"{name}/head"])
        assert hashlib.sha256(np.ascontiguousarray(got).tobytes()).digest() == \
            bytes(g[f"{name}/sha256"])
