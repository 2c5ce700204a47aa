"""Study harness: the reference's study API on the GPU solver,
checked against fixtures the reference itself produced
(oracle/gen_study.py -> tests/golden/study_ref.json)."""

import json
import os

import numpy as np
import pytest

import paper_1207_6720_b200 as fmp
from paper_1207_6720_b200 import harness
from paper_1207_6720_b200.mesh import HaloMode

REF = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "study_ref.json")))


def _records():
    return [harness.StudyRecord(r["n"], r["n_sr"], HaloMode(r["halo"]), r["ns"], r["rel_error"],
                                r["quad_ref"], 1.0) for r in REF["study"]]


def test_memory_model_matches_reference():
    for c in REF["memory"]:
        cfg = fmp.SolverConfig(hierarchy=fmp.build_hierarchy(c["m0"], c["m"]), n_sr=c["n_sr"],
                               smoother=fmp.SmootherConfig(halo_mode=HaloMode(c["halo"])))
        r = harness.memory_report(cfg)
        assert [r.cells_stored_full, r.sr_working_set, r.total_modeled] == c["model"], c


def test_quad_ref_and_grid():
    for r in REF["study"]:
        assert harness.quad_ref(int(np.log2(r["n"]))) == r["quad_ref"]
    grid = harness.full_grid_configs()
    assert len(grid) == 24 and grid[0] == (0, HaloMode.HALO2, 1) and grid[-1] == (3, HaloMode.GLOBAL, 2)


def test_observed_order_matches_reference():
    recs = _records()
    for o in REF["order"]:
        curve = [r for r in recs if (r.halo_mode.label, r.ns, r.n_sr) == (o["halo"], o["ns"], o["n_sr"])]
        assert harness.observed_order(curve) == o["order"]
    with pytest.raises(ValueError):
        harness.observed_order(recs[:2])


def test_csv_schema_byte_for_byte(tmp_path):
    p = tmp_path / "s.csv"
    harness.emit_csv(_records()[:6], p)
    assert p.read_bytes() == REF["csv"].encode("ascii")


def test_study_argument_errors():
    with pytest.raises(ValueError):
        harness.run_study(2, 6, [(0, "2", 1)], m0=2)
    with pytest.raises(ValueError):
        harness.run_study(6, 5, [(0, "2", 1)])
    with pytest.raises(ValueError):
        harness.run_study(4, 5, [(0, "2", 1)], nmodes_div=0)


@pytest.mark.gpu
def test_full_study_on_gpu_matches_reference(fm):
    """Every (config, n) cell of run_full_study(4, 8) solved on the device has
    the reference's relative error exactly (the solutions are bit-identical)."""
    recs = harness.run_full_study(4, 8)
    assert len(recs) == len(REF["study"])
    for got, want in zip(recs, REF["study"]):
        assert (got.n, got.n_sr, got.halo_mode.label, got.ns) == \
            (want["n"], want["n_sr"], want["halo"], want["ns"])
        assert got.rel_error == want["rel_error"], want
        assert got.runtime_ms > 0


@pytest.mark.gpu
def test_seed_check_passes_on_gpu(fm):
    got = harness.seed_check()
    assert [[n, ok] for n, ok, _ in got] == REF["seed_check"]
    assert all(ok for _, ok, _ in got)
