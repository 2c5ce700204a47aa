"""The additive patch smoother on the GPU (reference _kernels_numba.py:60-92,
smoothers.py:129-207): golden vectors, oracle parity over geometries
including odd buffers (SURVEY trap 1), batches, and patch-order invariance."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_smooth_matches_golden(fm, golden):
    s = "smooth/"
    u, f, uc = golden[s + "u"], golden[s + "f"], golden[s + "uc"]
    n = len(u)
    lane = fm.backends.active()
    for case, want in zip(golden[s + "cases"], golden[s + "out"]):
        kind, mode, P, b, ns, cr = (int(x) for x in case)
        if kind == 0:
            hm = {2: fm.HaloMode.HALO2, 4: fm.HaloMode.HALO4, -1: fm.HaloMode.GLOBAL}[mode]
            got = fm.smooth_level(u, f, fm.SmootherConfig(ns=ns, halo_mode=hm), 2,
                                  cr=fm.CrContext(uc) if cr else None)
            assert np.array_equal(got, want), case
            # the explicit-patch-array kernel agrees too
            got2 = fm.smooth_level(u, f, fm.SmootherConfig(ns=ns, halo_mode=hm), 2,
                                   cr=fm.CrContext(uc) if cr else None,
                                   patches=fm.partition(n, hm))
            assert np.array_equal(got2, want), case
        else:
            g = fm.level_geometry(n, n_patches=P, buffer=b)
            arrays = fm.mesh.patch_arrays(g.patches())
            got = lane.smooth_patches(u, f, float(4 ** 6), *arrays, ns, 1.0, bool(cr),
                                      uc if cr else None, 0.5)
            assert np.array_equal(got, want), case
            got2 = lane.smooth_uniform(u, f, g.W, g.b, ns, 1.0, uc if cr else None, 0.5)
            assert np.array_equal(got2, want), case


@pytest.mark.parametrize("ns", [1, 2, 3])
@pytest.mark.parametrize("cr", [False, True])
def test_smooth_batch_matches_oracle(fm, oracle, ns, cr):
    rng = np.random.default_rng(100 + ns + 10 * cr)
    n, B = 256, 45
    U = torch.as_tensor(rng.standard_normal((n, B)), device="cuda")
    Fd = torch.as_tensor(rng.standard_normal((n, B)), device="cuda")
    C = torch.as_tensor(rng.standard_normal((n // 2, B)), device="cuda")
    uh, fh, ch = U.cpu().numpy(), Fd.cpu().numpy(), C.cpu().numpy()
    lane = fm.backends.active()
    for P, b in ((1, 0), (2, 7), (4, 3), (8, 1), (16, 5), (32, 2), (128, 4), (128, 9)):
        g = fm.level_geometry(n, n_patches=P, buffer=b)
        arr = fm.mesh.patch_arrays(g.patches())
        got = lane.smooth_uniform(U, Fd, g.W, g.b, ns, 1.0, C if cr else None, 0.5).cpu().numpy()
        for j in range(B):
            want = oracle.smooth_patches(uh[:, j], fh[:, j], 4.0 ** 8, *arr, ns,
                                         uc=ch[:, j] if cr else None)
            assert np.array_equal(got[:, j], want), (P, b, j)


def test_patch_order_invariant(fm):
    # reference test_smoothers.py:146-159: shuffled explicit patch lists
    rng = np.random.default_rng(32)
    n = 256
    u = rng.standard_normal(n)
    f = rng.standard_normal(n)
    cfg = fm.SmootherConfig(ns=2, halo_mode=fm.HaloMode.HALO2)
    cr = fm.CrContext(fm.restrict(u))
    base = fm.smooth_level(u, f, cfg, 2, cr=cr)
    patches = fm.partition(n, fm.HaloMode.HALO2)
    for _ in range(10):
        shuffled = list(patches)
        rng.shuffle(shuffled)
        out = fm.smooth_level(u, f, cfg, 2, cr=cr, patches=shuffled)
        assert np.array_equal(out, base)


def test_global_is_alternating_gs(fm):
    rng = np.random.default_rng(33)
    u = rng.standard_normal(32)
    f = rng.standard_normal(32)
    got = fm.smooth_level(u, f, fm.SmootherConfig(ns=2, halo_mode=fm.HaloMode.GLOBAL), 2)
    want = fm.patch_gs_sweep(fm.patch_gs_sweep(u, f, (0, 32), "forward"), f, (0, 32), "backward")
    assert np.array_equal(got, want)


def test_minimum_slice_config2_geometry(fm, oracle):
    """cuda smooth_patches == reference smooth_patches per RHS, bit for
    bit, at the config-2 geometry (N=2^16, P=64, b=4) with B=1024."""
    n, B, P, b = 2 ** 16, 1024, 64, 4
    gen = torch.Generator(device="cuda").manual_seed(7)
    U = torch.randn((n, B), device="cuda", dtype=torch.float64, generator=gen)
    Fd = torch.randn((n, B), device="cuda", dtype=torch.float64, generator=gen)
    C = torch.randn((n // 2, B), device="cuda", dtype=torch.float64, generator=gen)
    g = fm.level_geometry(n, n_patches=P, buffer=b)
    arr = fm.mesh.patch_arrays(g.patches())
    lane = fm.backends.active()
    for cr in (False, True):
        got = lane.smooth_patches(U, Fd, float(4 ** 16), *arr, 1, 1.0, cr, C if cr else None, 0.5)
        got = got.cpu().numpy()
        uh, fh, ch = U.cpu().numpy(), Fd.cpu().numpy(), C.cpu().numpy()
        for j in (0, 1, 31, 32, 500, 1023):
            want = oracle.smooth_patches(uh[:, j], fh[:, j], 4.0 ** 16, *arr, 1,
                                         uc=ch[:, j] if cr else None)
            assert np.array_equal(got[:, j], want), (cr, j)
