"""Grid hierarchy and patch geometry (host side).

Mirrors the reference's ``fmgsr.mesh`` (reference mesh.py:17-158): level k
has 2**k cells of width 2**-k, patches own a half-open cell range inside a
clamped extended range.  The kernels never see patch objects: every standard
partition is *uniform* (owned width W, buffer b), so a level's geometry is
the pair (W, b) and the device derives each patch's ranges from its index.

Geometries
  * ``HaloMode.HALO2`` / ``HALO4`` -- the reference partition: W = 2
    (``PATCH_WIDTH``), b = 2 or 4 (mesh.py:130-136);
  * ``HaloMode.GLOBAL`` -- one patch, W = n, b = 0 (mesh.py:122-125);
  * P patches with a b-cell buffer (BASELINE configs): W_l = max(2, n_l/P).
    Wherever n_l / P <= 2 this is exactly the reference's HALO_b partition.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import ClassVar

import numpy as np

PATCH_WIDTH = 2


class HaloMode(enum.Enum):
    """Halo policy of the standard partition (reference mesh.py:22-45)."""

    HALO2 = "2"
    HALO4 = "4"
    GLOBAL = "global"

    @property
    def halo(self) -> int | None:
        return None if self is HaloMode.GLOBAL else int(self.value)

    @property
    def label(self) -> str:
        return self.value


@dataclass(frozen=True)
class Hierarchy:
    """Levels m0..m (reference mesh.py:48-76)."""

    m0: int
    m: int

    REFINEMENT_RATIO: ClassVar[int] = 2

    def __post_init__(self) -> None:
        if self.m0 < 1:
            raise ValueError(f"coarsest exponent must be >= 1, got m0={self.m0}")
        if self.m <= self.m0:
            raise ValueError(f"need at least two levels: m={self.m} must exceed m0={self.m0}")

    @property
    def levels(self) -> range:
        return range(self.m0, self.m + 1)

    def size(self, level: int) -> int:
        return 2 ** level

    def spacing(self, level: int) -> float:
        return 2.0 ** (-level)


def build_hierarchy(m0: int, m: int) -> Hierarchy:
    return Hierarchy(m0=m0, m=m)


@dataclass(frozen=True)
class Patch:
    """Owned range inside an extended range, both half-open (mesh.py:84-99)."""

    owned: tuple[int, int]
    extended: tuple[int, int]

    def __post_init__(self) -> None:
        (os_, oe), (es, ee) = self.owned, self.extended
        if not (es <= os_ < oe <= ee):
            raise ValueError(f"owned {self.owned} not inside extended {self.extended}")


@dataclass(frozen=True)
class LevelGeometry:
    """Uniform partition of one level: owned width W, buffer b (clamped)."""

    n: int
    W: int
    b: int

    @property
    def n_patches(self) -> int:
        return self.n // self.W

    def patches(self) -> list[Patch]:
        return [Patch((s, s + self.W), (max(0, s - self.b), min(self.n, s + self.W + self.b)))
                for s in range(0, self.n, self.W)]


def level_geometry(n: int, mode: HaloMode = HaloMode.HALO2, n_patches: int | None = None,
                   buffer: int | None = None) -> LevelGeometry:
    """Geometry of a level of n cells.

    ``n_patches`` selects the P-patch rule W = max(2, n/P) with ``buffer``
    cells (default: the halo of ``mode``); otherwise the reference partition.
    """
    if n_patches is not None:
        b = buffer if buffer is not None else (mode.halo if mode.halo is not None else 0)
        return LevelGeometry(n, max(PATCH_WIDTH, n // n_patches), b)
    if mode is HaloMode.GLOBAL:
        if n < 1:
            raise ValueError(f"level size must be positive, got {n}")
        return LevelGeometry(n, n, 0)
    if n % 2 != 0:
        raise ValueError(f"patch modes need an even level size, got {n}")
    if n < 4:
        raise ValueError(f"patch modes need at least 4 cells, got {n}")
    return LevelGeometry(n, PATCH_WIDTH, mode.halo if buffer is None else buffer)


def partition(n: int, mode: HaloMode) -> list[Patch]:
    """The reference's ordered patch list (mesh.py:102-136)."""
    return level_geometry(n, mode).patches()


def patch_arrays(patches: list[Patch]) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """Four int64 arrays (owned_lo, owned_hi, ext_lo, ext_hi), mesh.py:139-147."""
    a = np.array([[p.owned[0], p.owned[1], p.extended[0], p.extended[1]] for p in patches],
                 dtype=np.int64).reshape(-1, 4)
    return tuple(np.ascontiguousarray(a[:, k]) for k in range(4))
