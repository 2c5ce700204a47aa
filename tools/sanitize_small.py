"""Small solves that reach every kernel family and launch path, for
``compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck}``: the
fused visit kernel with the cross-warp edge-record protocol (scalar lanes with
the bulk-TMA mbarrier ring, two-column lanes with cp.async), the on-chip CTA
coarse kernel and the whole-solve-on-chip mode, the V(2,2) / nonlinear
streaming kernel and the warp coarse kernel, the unfused operator kernels,
virtual shards (halo copies, slab-edge fix-ups, cutoff gather), the functional
output and the host-buffer pipeline.  Every solve is checked bit for bit
against the oracle so a sanitizer run also proves the results unchanged.

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1207_6720_b200 as fm  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1207_6720_b200.shard import ShardGroup  # noqa: E402


def cfg_of(m, P, b, n_sr=1, ns=1, nl=False):
    return fm.SolverConfig(hierarchy=fm.build_hierarchy(3, m), n_sr=n_sr,
                           smoother=fm.SmootherConfig(ns=ns, n_patches=P, buffer=b, nonlinear=nl))


def want(m, P, b, f, n_sr=1, ns=1, nl=False):
    oc = O.make_cfg(3, m, n_sr, ns, O.GEOM_PATCHES, P, b, nonlin=nl)
    return O.fmg_solve_batch(oc, np.ascontiguousarray(f.cpu().numpy().T), nthreads=8).T


def check(name, got, ref):
    g = got.cpu().numpy() if torch.is_tensor(got) else got
    assert np.array_equal(g, ref), name
    print("ok", name, flush=True)


cases = [  # name, m, P, b, n_sr, ns, nl, B
    ("scalar_bulk_edges", 11, 16, 4, 1, 1, False, 32),
    ("v2_cpasync_edges", 11, 16, 3, 1, 1, False, 64),
    ("ragged_B", 10, 32, 2, 0, 1, False, 40),
    ("ns2_nonlinear", 10, 8, 2, 1, 2, True, 32),
    ("ns2_linear", 10, 16, 3, 0, 2, False, 32),
]
for name, m, P, b, n_sr, ns, nl, B in cases:
    cfg = cfg_of(m, P, b, n_sr, ns, nl)
    if nl:
        f, _ = fm.nonlinear_batch(2 ** m, fm.nonlinear_scales(B, seed=m))
    else:
        f, _ = fm.fourier_batch(2 ** m, fm.fourier_coefficients(B, seed=m + P))
    ref = want(m, P, b, f, n_sr, ns, nl)
    check(name, fm.fmg_solve(cfg, f)[0], ref)
    check(name + "/no_coarse", fm.fmg_solve(cfg, f, coarse=0)[0], ref)
    check(name + "/unfused", fm.fmg_solve(cfg, f, fused=False)[0], ref)
    if not nl and ns == 1:
        check(name + "/operators", fm.fmg_solve(cfg, f, keep_state=True)[0], ref)

# whole solve on chip (config 1: one RHS)
cfg = cfg_of(10, 4, 2)
f, _ = fm.fourier_batch(2 ** 10, fm.fourier_coefficients(1, seed=1))
check("whole_on_chip", fm.fmg_solve(cfg, f)[0], want(10, 4, 2, f))

# virtual shards
cfg = cfg_of(12, 64, 4)
f, _ = fm.fourier_batch(2 ** 12, fm.fourier_coefficients(64, seed=3))
ref = want(12, 64, 4, f)
g = ShardGroup(cfg, 64, 4, coarse=7)
check("shard_group_S4", g.solve(f), ref)
del g

# functional output and the host-buffer pipeline
plan = fm.FmgPlan(fm.key_from_config(cfg, 32, torch.float64))
fs = f[:, :32].contiguous()
J = plan.solve_functional(fs)
sol = plan.solve(fs)
torch.cuda.synchronize()
Jc = (sol.sum(0) * 2.0 ** -12).cpu().numpy()
assert np.allclose(J.cpu().numpy(), Jc, rtol=1e-12, atol=0), "functional"
print("ok functional", flush=True)
hf = f.cpu().pin_memory()
hs = torch.empty_like(hf).pin_memory()
plan.solve_host(hf, hs, 2)
torch.cuda.synchronize()
check("solve_host", hs, ref)
print("SANITIZE-SMALL DONE", flush=True)
