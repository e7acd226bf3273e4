"""Ghost-padded grid layout in HBM.

A field of the (itot, jtot, ktot) interior with igc/jgc/kgc ghost layers is
stored C-order ``[k][j][i]`` with a padded row pitch::

    element (i, j, k)  ->  base + lead + i + j*jj + k*kk      (elements)

* ``jj`` (row pitch) is ``icells`` rounded up to ``align`` elements (128 B);
* ``lead`` = ``align - igc`` so the first INTERIOR cell of every row
  (i = igc) sits on a 128-byte boundary — coalesced, vector-aligned rows;
* ``kk = jj * jcells`` — z-planes are contiguous, so a halo plane for the
  multi-GPU z-slab exchange is one contiguous ``kk * elem`` byte range.

Kernels receive a pointer to element (0, 0, 0) (``base + lead``) plus ``jj``,
``kk`` and the interior bounds ``istart = igc .. iend = igc + itot`` (same
for j, k), exactly like MicroHH's ``advec_u_g`` / ``diff_uvw_g``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["GridLayout", "DTYPES"]

DTYPES = {"fp32": np.float32, "fp64": np.float64}
_ELEM = {"fp32": 4, "fp64": 8}


@dataclass(frozen=True)
class GridLayout:
    itot: int
    jtot: int
    ktot: int
    precision: str = "fp32"
    igc: int = 3
    jgc: int = 3
    kgc: int = 3
    align_bytes: int = 128

    def __post_init__(self) -> None:
        if self.precision not in _ELEM:
            raise ValueError(f"precision must be fp32 or fp64, got {self.precision!r}")
        if min(self.itot, self.jtot, self.ktot) < 1:
            raise ValueError("interior extents must be >= 1")
        if self.align_bytes < 16 or self.align_bytes % 16:
            raise ValueError("align_bytes must be a multiple of 16 (TMA strides, 16-byte vector rows)")

    # -- element geometry --------------------------------------------------------
    @property
    def elem_bytes(self) -> int:
        return _ELEM[self.precision]

    @property
    def dtype(self):
        return DTYPES[self.precision]

    @property
    def element_type(self) -> str:
        return "f32" if self.precision == "fp32" else "f64"

    @property
    def align(self) -> int:
        return self.align_bytes // self.elem_bytes

    @property
    def icells(self) -> int:
        return self.itot + 2 * self.igc

    @property
    def jcells(self) -> int:
        return self.jtot + 2 * self.jgc

    @property
    def kcells(self) -> int:
        return self.ktot + 2 * self.kgc

    @property
    def jj(self) -> int:
        # +1: the TMA tensor map is built over the 16-byte-aligned base just below
        # element (0,0,0) (one element lower), so a row must hold icells + 1.
        return -(-(self.icells + 1) // self.align) * self.align

    @property
    def lead(self) -> int:
        # smallest offset putting the first interior cell (i = igc) on an
        # alignment boundary
        return -(-self.igc // self.align) * self.align - self.igc

    @property
    def kk(self) -> int:
        return self.jj * self.jcells

    @property
    def alloc_elems(self) -> int:
        """Elements to allocate: lead + kcells planes (+ one row of slack)."""
        return self.lead + self.kk * self.kcells + self.jj

    @property
    def alloc_bytes(self) -> int:
        return self.alloc_elems * self.elem_bytes

    @property
    def span_elems(self) -> int:
        """Elements from (0,0,0) to the end of the allocation (what a capture stores)."""
        return self.alloc_elems - self.lead

    # -- bounds ------------------------------------------------------------------
    @property
    def istart(self) -> int:
        return self.igc

    @property
    def iend(self) -> int:
        return self.igc + self.itot

    @property
    def jstart(self) -> int:
        return self.jgc

    @property
    def jend(self) -> int:
        return self.jgc + self.jtot

    @property
    def kstart(self) -> int:
        return self.kgc

    @property
    def kend(self) -> int:
        return self.kgc + self.ktot

    @property
    def cells(self) -> int:
        return self.itot * self.jtot * self.ktot

    def offset(self, i: int, j: int, k: int) -> int:
        """Element offset of (i, j, k) from the pointer passed to kernels."""
        return i + j * self.jj + k * self.kk

    # -- host views ----------------------------------------------------------------
    def host_view(self, flat: np.ndarray) -> np.ndarray:
        """(kcells, jcells, icells) strided view of a flat allocation-sized array."""
        if flat.size < self.alloc_elems:
            raise ValueError("array smaller than the layout")
        base = flat[self.lead:self.lead + self.kk * self.kcells]
        return base.reshape(self.kcells, self.jcells, self.jj)[:, :, : self.icells]

    def interior(self, view: np.ndarray) -> np.ndarray:
        return view[self.kstart:self.kend, self.jstart:self.jend, self.istart:self.iend]

    def slab(self, k_begin: int, k_count: int) -> "GridLayout":
        """Layout of a z-slab of ``k_count`` interior planes (same x/y layout)."""
        del k_begin
        return GridLayout(self.itot, self.jtot, k_count, self.precision, self.igc, self.jgc, self.kgc, self.align_bytes)
