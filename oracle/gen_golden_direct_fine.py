"""TEST INFRASTRUCTURE ONLY -- fixtures of the reference's independent check
solve ``fmgsr.problem.direct_fine_solve`` (problem.py:61-77: the level
operator assembled as a 3-row band and solved by scipy ``solve_banded`` ->
LAPACK dgbsv), from the UNMODIFIED reference on seeded right-hand sides.
Writes ``tests/golden/direct_fine.npz``; the oracle restatement
(``orc_banded_lu_solve``) and the device kernel (``fmgsr_banded_lu_solve``)
are pinned to it bit for bit.

    python oracle/gen_golden_direct_fine.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gen_golden import _import_reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "direct_fine.npz")


def main():
    fm = _import_reference()
    from fmgsr import problem

    out = {}
    for n in (4, 8, 16, 64, 256, 1024):
        rng = np.random.default_rng([7, n])
        f = np.stack([rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3) for _ in range(2)]
                     + [problem.manufactured_rhs(n)])
        out[f"n{n}/f"] = f
        out[f"n{n}/u"] = np.stack([problem.direct_fine_solve(r) for r in f])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, sorted(out), fm.__name__)


if __name__ == "__main__":
    main()
