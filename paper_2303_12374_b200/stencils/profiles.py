"""Synthetic vertical grid and reference-state profiles (host side, tiny).

Per SURVEY.md §8d: layer thicknesses ``dz[k] ~ U(0.8, 1.2)`` drawn from a
splitmix64 stream, ``zh`` (half levels) accumulated upward from
``zh[kstart] = 0``, ``z`` at cell centres, ``dzh = z[k] - z[k-1]``,
``rhoref = exp(-z/H)``, ``rhorefh = exp(-zh/H)`` with H = 10 up to 64 levels
and stretched with deeper grids (``scale_height``).  Arrays have one entry per
GLOBAL ghost-padded level; a z-slab slices its window (no exchange needed).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..rng import SplitMix64

__all__ = ["FIELD_SEED_BASE", "FIELD_SPECS", "Profiles", "make_profiles"]

FIELD_SEED_BASE = 230312374
#: field -> (seed offset, low, high); seed = FIELD_SEED_BASE + offset
FIELD_SPECS = {
    "u": (0, -1.0, 1.0),
    "v": (1, -1.0, 1.0),
    "w": (2, -1.0, 1.0),
    "ut": (3, -1.0, 1.0),
    "vt": (4, -1.0, 1.0),
    "wt": (5, -1.0, 1.0),
    "evisc": (6, 0.01, 0.1),
    "s": (7, -1.0, 1.0),
    "st": (8, -1.0, 1.0),
    "u_next": (9, -1.0, 1.0),
    "v_next": (10, -1.0, 1.0),
    "w_next": (11, -1.0, 1.0),
}
_PROFILE_SEED_OFFSET = 100


@dataclass(frozen=True)
class Profiles:
    dz: np.ndarray
    dzi: np.ndarray
    dzhi: np.ndarray
    rhoref: np.ndarray
    rhorefh: np.ndarray

    def window(self, k_offset: int, count: int) -> "Profiles":
        sl = slice(k_offset, k_offset + count)
        return Profiles(*(a[sl].copy() for a in (self.dz, self.dzi, self.dzhi, self.rhoref, self.rhorefh)))

    def as_dtype(self, dtype) -> "Profiles":
        return Profiles(*(a.astype(dtype) for a in (self.dz, self.dzi, self.dzhi, self.rhoref, self.rhorefh)))


def make_profiles(kcells: int, kgc: int) -> Profiles:
    """Float64 profiles over ``kcells`` global levels (ghosts included)."""
    stream = SplitMix64(FIELD_SEED_BASE + _PROFILE_SEED_OFFSET)
    dz = np.array([0.8 + 0.4 * stream.next_float() for _ in range(kcells)], dtype=np.float64)
    zh = np.zeros(kcells + 1)
    for k in range(kgc, kcells):
        zh[k + 1] = zh[k] + dz[k]
    for k in range(kgc - 1, -1, -1):
        zh[k] = zh[k + 1] - dz[k]
    z = 0.5 * (zh[:-1] + zh[1:])
    dzh = np.empty(kcells)
    dzh[1:] = z[1:] - z[:-1]
    dzh[0] = dz[0]
    height = scale_height(kcells, kgc)
    return Profiles(
        dz=dz,
        dzi=1.0 / dz,
        dzhi=1.0 / dzh,
        rhoref=np.exp(-z / height),
        rhorefh=np.exp(-zh[:-1] / height),
    )


def scale_height(kcells: int, kgc: int) -> float:
    """Density scale height of the synthetic reference state.

    SURVEY §8d gives ``exp(-z/10)``; with dz ~ 1 per level that is kept for
    grids up to 64 levels, and deeper grids stretch it with the domain
    (10 per 64 levels): unstretched, ``rhoref`` at z ~ 1000 is ~1e-44, below
    fp32's normal range, so an fp32 1024-level grid would divide by flushed
    denormals and compute inf/NaN in its top ~15 % of planes (caught by the
    bench-shape parity test).  The profile stays a global function of the
    level, so z-slabs still slice it without an exchange."""
    ktot = kcells - 2 * kgc
    return 10.0 * max(1.0, ktot / 64.0)
