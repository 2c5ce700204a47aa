"""The CPU oracle (oracle/fmgsr_oracle.c) pinned against the reference:
golden vectors produced by the reference itself (oracle/gen_golden.py), the
reference's hand-worked known answers, and scipy's LAPACK for the coarsest
solve.  No GPU needed."""

import os

import numpy as np
import pytest
from scipy.linalg import solve_banded, solveh_banded


def test_stencils_match_golden(oracle, golden):
    for n in (4, 8, 64):
        p = f"stencil_n{n}/"
        u, f = golden[p + "u"], golden[p + "f"]
        assert np.array_equal(oracle.apply_operator(u), golden[p + "apply_operator"])
        assert np.array_equal(oracle.restrict(u), golden[p + "restrict"])
        assert np.array_equal(oracle.prolong_correction(u), golden[p + "prolong_correction"])
        assert np.array_equal(oracle.prolong_fmg(u), golden[p + "prolong_fmg"])
        assert np.array_equal(oracle.tau_correction(u), golden[p + "tau"])
        assert np.array_equal(oracle.coarse_rhs(f, u), golden[p + "coarse_rhs"])


def test_direct_solve_matches_golden(oracle, golden):
    for n in (4, 8, 16, 64):
        for f, u in zip(golden[f"direct_n{n}/f"], golden[f"direct_n{n}/u"]):
            assert np.array_equal(oracle.direct_solve(f), u)


@pytest.mark.parametrize("n", [4, 8, 16, 32, 256])
def test_direct_solve_is_lapack_ptsv_bitwise(oracle, n):
    """solveh_banded with a 2-row band runs LAPACK ?ptsv (dpttrf + dptts2)."""
    rng = np.random.default_rng(n)
    inv = float(4 ** (n.bit_length() - 1))
    ab = np.empty((2, n))
    ab[0, :] = -inv
    ab[0, 0] = 0.0
    ab[1, :] = 2 * inv
    ab[1, 0] = ab[1, -1] = 3 * inv
    for _ in range(50):
        f = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)
        assert np.array_equal(oracle.direct_solve(f), solveh_banded(ab, f))


def test_banded_lu_matches_reference_direct_fine_solve(oracle):
    """orc_banded_lu_solve against the reference's own direct_fine_solve
    (problem.py:61-77, scipy solve_banded -> LAPACK dgbsv), bit for bit."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "direct_fine.npz"))
    for n in (4, 8, 16, 64, 256, 1024):
        for f, u in zip(g[f"n{n}/f"], g[f"n{n}/u"]):
            assert np.array_equal(oracle.banded_lu_solve(f), u)


def test_sweeps_match_golden(oracle, golden):
    s = "sweeps/"
    u, f, uc, ih = golden[s + "u"], golden[s + "f"], golden[s + "uc"], float(golden[s + "inv_h2"])
    k = 0
    for (a, b) in golden[s + "windows"]:
        for fw in (True, False):
            assert np.array_equal(oracle.gs_sweep(u, f, ih, a, b, fw), golden[s + "gs"][k])
            assert np.array_equal(oracle.kaczmarz_sweep(u, uc, a, b, fw), golden[s + "kaczmarz"][k])
            k += 1


def _patches(n, W, b):
    os_ = np.arange(0, n, W)
    oe = os_ + W
    return os_, oe, np.maximum(0, os_ - b), np.minimum(n, oe + b)


def test_smooth_matches_golden(oracle, golden):
    s = "smooth/"
    u, f, uc = golden[s + "u"], golden[s + "f"], golden[s + "uc"]
    n = len(u)
    for case, want in zip(golden[s + "cases"], golden[s + "out"]):
        kind, mode, P, b, ns, cr = (int(x) for x in case)
        if kind == 0:
            W, bb = (n, 0) if mode == -1 else (2, mode)
        else:
            W, bb = max(2, n // P), b
        got = oracle.smooth_patches(u, f, 4.0 ** 6, *_patches(n, W, bb), ns, uc=uc if cr else None)
        assert np.array_equal(got, want), case


def test_fmg_matches_golden(oracle, golden):
    for name in golden["fmg_cases"]:
        p = str(name) + "/"
        m0, m, n_sr, ns, kind, P, b = (int(x) for x in golden[p + "params"])
        cfg = oracle.make_cfg(m0, m, n_sr, ns, kind, P, b)
        assert np.array_equal(oracle.fmg_solve(cfg, golden[p + "forcing"]),
                              golden[p + "solution"]), str(name)


def test_batch_driver_matches_single(oracle):
    rng = np.random.default_rng(4)
    cfg = oracle.make_cfg(3, 9, 1, 1, oracle.GEOM_PATCHES, 8, 3)
    rows = rng.standard_normal((6, 512))
    got = oracle.fmg_solve_batch(cfg, rows, nthreads=3)
    for r in range(6):
        assert np.array_equal(got[r], oracle.fmg_solve(cfg, rows[r]))


# ---- the reference's known answers (test_stencils.py:31-57, test_smoothers.py:24-28,82-84)
def test_known_answers(oracle):
    assert oracle.apply_operator(np.ones(4)).tolist() == [32.0, 0.0, 0.0, 32.0]
    assert oracle.restrict(np.array([1.0, 3.0, 5.0, 7.0])).tolist() == [2.0, 6.0]
    assert oracle.prolong_correction(np.array([4.0, 8.0])).tolist() == [2.0, 5.0, 7.0, 4.0]
    out = oracle.prolong_fmg(np.ones(8))
    assert out[0] == out[-1] == 0.53125 and out[1] == out[-2] == 1.109375
    assert out[2] == out[-3] == 1.078125 and np.all(out[3:-3] == 1.0)
    gs = oracle.gs_sweep(np.zeros(4), np.ones(4), 16.0, 0, 4, True)
    assert np.allclose(gs, [1 / 48, 1 / 24, 5 / 96, 11 / 288], rtol=0, atol=1e-16)
    assert oracle.kaczmarz_sweep(np.array([1.0, 3.0]), np.array([5.0]), 0, 2).tolist() == [4.0, 6.0]


def test_odd_window_kaczmarz_semantics(oracle):
    """SURVEY trap 1: an odd window start projects the pair straddling the
    frozen cell ws-1 (numba lane semantics); an odd stop leaves we-1 alone."""
    u = np.arange(8, dtype=float)
    uc = np.full(4, 10.0)
    out = oracle.kaczmarz_sweep(u, uc, 1, 5, True)
    assert not np.array_equal(out[0:4], u[0:4])  # pairs 0 and 1 projected
    assert np.array_equal(out[4:], u[4:])


def test_config1_one_cycle_truncation_accuracy(oracle):
    """One FMG cycle reaches the discretisation error (reference acceptance
    criterion 5): rel-L2 error <= 2x the direct solve's, BASELINE config 1."""
    n = 1024
    x = (np.arange(n) + 0.5) / n
    f = np.pi ** 2 * np.sin(np.pi * x)
    uex = np.sin(np.pi * x)
    cfg = oracle.make_cfg(3, 10, 1, 1, oracle.GEOM_PATCHES, 4, 2)
    sol = oracle.fmg_solve(cfg, f)
    inv = float(n * n)
    ab = np.zeros((3, n))
    ab[0, 1:] = -inv
    ab[1, :] = 2 * inv
    ab[1, 0] = ab[1, -1] = 3 * inv
    ab[2, :-1] = -inv
    direct = solve_banded((1, 1), ab, f)
    e = np.linalg.norm(sol - uex) / np.linalg.norm(uex)
    ed = np.linalg.norm(direct - uex) / np.linalg.norm(uex)
    assert e <= 2.0 * ed


def test_geometry_rule_reproduces_reference_partition(oracle):
    # W = max(2, n/P): with n/P <= 2 it is the reference's HALO_b partition
    for n in (16, 64):
        assert oracle.level_geometry(n, oracle.GEOM_PATCHES, n, 4) == (2, 4)
        assert oracle.level_geometry(n, oracle.GEOM_HALO, 1, 2) == (2, 2)
        assert oracle.level_geometry(n, oracle.GEOM_GLOBAL, 1, 0) == (n, 0)
    assert oracle.level_geometry(2 ** 16, oracle.GEOM_PATCHES, 64, 4) == (1024, 4)


# ---- nonlinear FAS restatement (config 3; the reference is linear only) -------------------
def _newton_fine(oracle, f):
    """Discrete solution of L u + u^3 = f by Newton with a banded LU (independent)."""
    n = len(f)
    inv = float(n * n)
    u = np.zeros(n)
    for _ in range(30):
        r = f - (oracle.apply_operator(u) + u ** 3)
        ab = np.zeros((3, n))
        ab[0, 1:] = -inv
        ab[1, :] = 2 * inv + 3 * u ** 2
        ab[1, 0] = 3 * inv + 3 * u[0] ** 2
        ab[1, -1] = 3 * inv + 3 * u[-1] ** 2
        ab[2, :-1] = -inv
        u = u + solve_banded((1, 1), ab, r)
    return u


@pytest.mark.parametrize("ns", [1, 2])
def test_nonlinear_one_cycle_truncation_accuracy(oracle, ns):
    """Manufactured u = s x(1-x)e^x: one FMG cycle lands within 2x of the
    discrete solution's discretisation error, at second order."""
    errs = []
    for m in (8, 10, 12):
        n = 2 ** m
        x = (np.arange(n) + 0.5) / n
        s = 1.7
        u = s * x * (1 - x) * np.exp(x)
        f = s * x * (x + 3) * np.exp(x) + u ** 3
        cfg = oracle.make_cfg(3, m, 1, ns, oracle.GEOM_PATCHES, min(256, n // 4), 4, nonlin=True)
        sol = oracle.fmg_solve(cfg, f)
        e = np.linalg.norm(sol - u) / np.linalg.norm(u)
        ed = np.linalg.norm(_newton_fine(oracle, f) - u) / np.linalg.norm(u)
        assert e <= 2.0 * ed
        errs.append(e)
    assert errs[0] / errs[1] > 10 and errs[1] / errs[2] > 10  # ~16 per two levels


def test_nonlinear_coarse_newton_solves(oracle):
    rng = np.random.default_rng(3)
    f = rng.standard_normal(8) * 50
    u = oracle.direct_solve_nl(f)
    assert np.max(np.abs(oracle.apply_nonlinear(u) - f)) < 1e-12 * np.max(np.abs(f))


def test_nonlinear_reduces_to_linear_for_tiny_fields(oracle):
    """With u ~ 1e-8 the cubic term is below rounding: the nonlinear sweep
    equals the linear one to ~1e-15 relative."""
    rng = np.random.default_rng(9)
    u = rng.standard_normal(32) * 1e-8
    f = rng.standard_normal(32) * 1e-8
    a = oracle.gs_sweep(u, f, 4.0 ** 5, 0, 32, True)
    b = oracle.gs_sweep_nl(u, f, 4.0 ** 5, 0, 32, True)
    assert np.max(np.abs(a - b)) <= 1e-14 * np.max(np.abs(a))


def test_oracle_matches_reference_at_full_config2_size():
    """The oracle restatement against the reference's own solve of one seeded
    RHS of config 2 at full size (N = 2^16, 64 patches, b = 4; fixture from
    oracle/gen_golden_full.py): SHA-256 of the solution bytes."""
    import hashlib

    from oracle import oracle as O

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "full_size.npz"))
    m0, m, n_sr, ns, _, P, b = (int(x) for x in g["c2/params"])
    sol = O.fmg_solve(O.make_cfg(m0, m, n_sr, ns, O.GEOM_PATCHES, P, b), g["c2/forcing"])
    assert hashlib.sha256(np.ascontiguousarray(sol).tobytes()).digest() == bytes(g["c2/sha256"])


def _hash_rhs(n, salt):
    i = np.arange(n, dtype=np.uint64)
    h = (i * np.uint64(2654435761) + np.uint64(salt)) % np.uint64(1 << 32)
    return h.astype(np.float64) / float(1 << 32) - 0.5


@pytest.mark.parametrize("case", ["h_c2", "h_c5_P256_b4", "h_c5_P16_b1", "h_c5_P1024_b8", "h_c4",
                                  "h_c3lin", "h_c2_sr0", "h_c2_sr2", "h_c5_P64_b1", "h_c5_P16_b8"])
def test_oracle_matches_reference_hashes_at_full_size(case):
    """The oracle against the reference's own solutions at the full BASELINE
    sizes of configs 2, 5 and 4 (N up to 2^24), for the machine-independent
    hash forcing of oracle/gen_golden_full.py: SHA-256 of the solution bytes."""
    import hashlib

    from oracle import oracle as O

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "full_size.npz"))
    m0, m, n_sr, ns, _, P, b, salt = (int(x) for x in g[f"{case}/params"])
    sol = O.fmg_solve(O.make_cfg(m0, m, n_sr, ns, O.GEOM_PATCHES, P, b), _hash_rhs(2 ** m, salt))
    assert np.array_equal(sol[:64], g[f"{case}/head"])
    assert hashlib.sha256(np.ascontiguousarray(sol).tobytes()).digest() == bytes(g[f"{case}/sha256"])


# ---- nonlinear FAS pinned to the reference's own driver (oracle/gen_golden_nl.py) -------------
_NL = os.path.join(os.path.dirname(__file__), "golden", "nonlinear.npz")


def test_oracle_nonlinear_matches_reference_driver():
    """The nonlinear restatement against the reference's OWN FMG driver, patch
    assembly and Kaczmarz pass with the pointwise Newton-GS lane, the N(u) tau
    and the Newton coarse solve injected through its lane registry and
    module-level names (backends.py:22-47, cycles.py:22-28): bit for bit at
    reduced sizes (V(1,1) .. V(3,3), SR depths 0-2, odd buffers)."""
    from oracle import oracle as O

    g = np.load(_NL)
    for name in g["cases"]:
        m0, m, n_sr, ns, _, P, b = (int(x) for x in g[f"{name}/params"])
        cfg = O.make_cfg(m0, m, n_sr, ns, O.GEOM_PATCHES, P, b, nonlin=True)
        got = O.fmg_solve(cfg, g[f"{name}/forcing"])
        assert np.array_equal(got, g[f"{name}/solution"]), str(name)


def test_oracle_nonlinear_config3_full_size_hash():
    """Config 3's full geometry (N = 2^20, 256 patches, b = 4, V(2,2), n_sr = 1),
    nonlinear, through the reference's driver: SHA-256 of the solution."""
    import hashlib

    from oracle import oracle as O

    g = np.load(_NL)
    for name in g["hash_cases"]:
        m0, m, n_sr, ns, _, P, b, salt = (int(x) for x in g[f"{name}/params"])
        f = float(g[f"{name}/scale"]) * _hash_rhs(2 ** m, salt)
        sol = O.fmg_solve(O.make_cfg(m0, m, n_sr, ns, O.GEOM_PATCHES, P, b, nonlin=True), f)
        assert np.array_equal(sol[:64], g[f"{name}/head"])
        assert hashlib.sha256(np.ascontiguousarray(sol).tobytes()).digest() == \
            bytes(g[f"{name}/sha256"])
