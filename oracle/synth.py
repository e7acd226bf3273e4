"""NumPy twin of ``klb_synth_field`` (include/klb200.h) — TEST INFRASTRUCTURE.

Value of element (i, j, k) of a ghost-padded field stream ``seed``::

    n = ((k + k_offset) * jcells + j') * icells + i'        (global logical index)
    h = mix64(seed + (n + 1) * 0x9E3779B97F4A7C15)           (draw n+1 of SplitMix64(seed))
    v = lo + (hi - lo) * ((h >> 11) * 2**-53)                (two IEEE ops, no FMA)

with (i', j') wrapped periodically into the interior (x/y ghost cells are
periodic copies).  Bit-exact with the device generator, so oracle and GPU see
identical inputs without moving multi-GB arrays over PCIe.
"""

from __future__ import annotations

import numpy as np

__all__ = ["synth_values", "synth_field"]

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def synth_values(seed: int, n: np.ndarray, lo: float, hi: float) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (n.astype(np.uint64) + np.uint64(1)) * _GOLDEN
        h = _mix64(z)
    x = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * x


def synth_field(seed: int, lo: float, hi: float, icells: int, jcells: int, kcells_local: int, igc: int, jgc: int,
                k_offset: int = 0, periodic_xy: bool = True, dtype=np.float64) -> np.ndarray:
    """(kcells_local, jcells, icells) array of the field in ``dtype``."""
    i = np.arange(icells, dtype=np.int64)
    j = np.arange(jcells, dtype=np.int64)
    if periodic_xy:
        itot, jtot = icells - 2 * igc, jcells - 2 * jgc
        i = igc + (i - igc) % itot
        j = jgc + (j - jgc) % jtot
    k = np.arange(kcells_local, dtype=np.int64) + k_offset
    n = (k[:, None, None] * jcells + j[None, :, None]) * icells + i[None, None, :]
    return synth_values(seed, n, lo, hi).astype(dtype)
