"""TEST INFRASTRUCTURE ONLY -- study-harness fixtures from the real reference.

Runs the UNMODIFIED reference ``fmgsr`` (``/root/reference/pkg/src``, numba
lane) study harness and writes ``tests/golden/study_ref.json``:
  * ``memory``: ``harness.memory_report`` for a set of configurations,
  * ``study``: ``harness.run_full_study(4, 8)`` records (runtime dropped: it is
    a wall-clock figure), the full 24-configuration grid,
  * ``order``: ``harness.observed_order`` of each configuration's curve,
  * ``csv``: ``harness.emit_csv`` of the first records with the runtime column
    pinned to 1.0 (to compare the CSV formatting byte for byte),
  * ``seed_check``: names and verdicts of ``harness.seed_check()``.

    python oracle/gen_study.py
"""

from __future__ import annotations

import json
import os
import tempfile

from gen_golden import _import_reference

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "study_ref.json")


def main() -> None:
    fm = _import_reference()
    from fmgsr import harness
    from fmgsr.mesh import HaloMode

    mem = []
    for m0, m, n_sr, halo in [(2, 12, 0, "2"), (2, 12, 3, "4"), (3, 10, 1, "2"), (2, 8, 2, "global"),
                              (3, 16, 1, "4"), (2, 9, 2, "2"), (3, 12, 0, "global")]:
        cfg = fm.SolverConfig(hierarchy=fm.build_hierarchy(m0, m), n_sr=n_sr,
                              smoother=fm.SmootherConfig(halo_mode=HaloMode(halo)))
        r = harness.memory_report(cfg)
        mem.append({"m0": m0, "m": m, "n_sr": n_sr, "halo": halo,
                    "model": [r.cells_stored_full, r.sr_working_set, r.total_modeled]})
    recs = harness.run_full_study(4, 8)
    study = [{"n": r.n, "n_sr": r.n_sr, "halo": r.halo_mode.label, "ns": r.ns,
              "rel_error": r.rel_error, "quad_ref": r.quad_ref} for r in recs]
    order = {}
    for r in recs:
        order.setdefault((r.halo_mode.label, r.ns, r.n_sr), []).append(r)
    orders = [{"halo": k[0], "ns": k[1], "n_sr": k[2], "order": harness.observed_order(v)}
              for k, v in order.items() if len(v) >= 3]
    pinned = [harness.StudyRecord(r.n, r.n_sr, r.halo_mode, r.ns, r.rel_error, r.quad_ref, 1.0)
              for r in recs[:6]]
    path = os.path.join(tempfile.mkdtemp(), "s.csv")
    harness.emit_csv(pinned, path)
    checks = [[name, bool(ok)] for name, ok, _ in harness.seed_check()]
    with open(OUT, "w") as fh:
        json.dump({"memory": mem, "study": study, "order": orders, "csv": open(path).read(),
                   "seed_check": checks}, fh, indent=0)
    print("wrote", OUT, len(study), "study records")


if __name__ == "__main__":
    main()
