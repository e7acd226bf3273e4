"""ctypes binding of oracle/_build/libstencil_ref.so — TEST INFRASTRUCTURE ONLY.

Runs the C restatement over numpy (kcells, jcells, icells) arrays (contiguous,
pitch = icells) on a thread pool of z-chunks; used as the timed CPU baseline
(bench.py) and cross-checked against the NumPy oracle (tests/test_oracle.py,
tests/test_family_oracle.py).  advec_u / diff_uvw: stencil_ref.c (fp32 and
fp64 arithmetic); the §8f family: family_ref.c (float64 arithmetic).
"""

from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

_LIB = Path(__file__).resolve().parent / "_build" / "libstencil_ref.so"
_handle = None


def available() -> bool:
    return _LIB.exists()


def _lib():
    global _handle
    if _handle is None:
        _handle = C.CDLL(str(_LIB))
    return _handle


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _chunks(kstart, kend, threads):
    n = kend - kstart
    step = max(1, -(-n // threads))
    return [(k, min(k + step, kend)) for k in range(kstart, kend, step)]


def advec_u(ut, u, v, w, rhoref, rhorefh, dzi, dxi, dyi, ghost=(3, 3, 3), threads=1, pool=None):
    """In-place ut += advection tendency over the interior (arrays of one dtype)."""
    suffix = "f32" if ut.dtype == np.float32 else "f64"
    fn = getattr(_lib(), f"advec_u_{suffix}")
    real = C.c_float if suffix == "f32" else C.c_double
    kc, jc, ic = ut.shape
    gi, gj, gk = ghost

    def run(kr):
        fn(_ptr(ut), _ptr(u), _ptr(v), _ptr(w), _ptr(rhoref), _ptr(rhorefh), _ptr(dzi), real(dxi), real(dyi),
           C.c_int(ic), C.c_ssize_t(ic * jc), gi, ic - gi, gj, jc - gj, kr[0], kr[1])

    _map(run, _chunks(gk, kc - gk, threads), threads, pool)


def diff_uvw(ut, vt, wt, e, u, v, w, dzi, dzhi, rhoref, rhorefh, dxi, dyi, ghost=(3, 3, 3), threads=1, pool=None):
    suffix = "f32" if ut.dtype == np.float32 else "f64"
    fn = getattr(_lib(), f"diff_uvw_{suffix}")
    real = C.c_float if suffix == "f32" else C.c_double
    kc, jc, ic = ut.shape
    gi, gj, gk = ghost

    def run(kr):
        fn(_ptr(ut), _ptr(vt), _ptr(wt), _ptr(e), _ptr(u), _ptr(v), _ptr(w), _ptr(dzi), _ptr(dzhi), _ptr(rhoref),
           _ptr(rhorefh), real(dxi), real(dyi), C.c_int(ic), C.c_ssize_t(ic * jc), gi, ic - gi, gj, jc - gj, kr[0],
           kr[1])

    _map(run, _chunks(gk, kc - gk, threads), threads, pool)


def _family(name, arrays, scalars, ghost, threads, pool):
    """oracle/family_ref.c kernel ``name`` (float64 arrays, in place on the
    first) over the interior, z-chunks on ``threads``."""
    if any(a.dtype != np.float64 for a in arrays):
        raise TypeError("family_ref.c computes in float64")
    fn = getattr(_lib(), f"{name}_f64")
    kc, jc, ic = arrays[0].shape
    gi, gj, gk = ghost

    def run(kr):
        fn(*(_ptr(a) for a in arrays), *(C.c_double(x) for x in scalars), C.c_int(ic), C.c_ssize_t(ic * jc), gi,
           ic - gi, gj, jc - gj, kr[0], kr[1])

    _map(run, _chunks(gk, kc - gk, threads), threads, pool)


def advec_v(vt, u, v, w, rhoref, rhorefh, dzi, dxi, dyi, ghost=(3, 3, 3), threads=1, pool=None):
    _family("advec_v", (vt, u, v, w, rhoref, rhorefh, dzi), (dxi, dyi), ghost, threads, pool)


def advec_w(wt, u, v, w, rhoref, rhorefh, dzhi, dxi, dyi, ghost=(3, 3, 3), threads=1, pool=None):
    _family("advec_w", (wt, u, v, w, rhoref, rhorefh, dzhi), (dxi, dyi), ghost, threads, pool)


def advec_s(st, s, u, v, w, rhoref, rhorefh, dzi, dxi, dyi, ghost=(3, 3, 3), threads=1, pool=None):
    _family("advec_s", (st, s, u, v, w, rhoref, rhorefh, dzi), (dxi, dyi), ghost, threads, pool)


def diff_c(st, s, evisc, dzi, dzhi, rhoref, rhorefh, dxi, dyi, tpri, ghost=(3, 3, 3), threads=1, pool=None):
    _family("diff_c", (st, s, evisc, dzi, dzhi, rhoref, rhorefh), (dxi, dyi, tpri), ghost, threads, pool)


def evisc_smag(evisc, u, v, w, dzi, dzhi, dxi, dyi, cs, ghost=(3, 3, 3), threads=1, pool=None):
    _family("evisc_smag", (evisc, u, v, w, dzi, dzhi), (dxi, dyi, cs), ghost, threads, pool)


def _map(fn, items, threads, pool):
    if threads <= 1 and pool is None:
        for it in items:
            fn(it)
        return
    if pool is not None:
        list(pool.map(fn, items))
        return
    with ThreadPoolExecutor(max_workers=threads) as tp:
        list(tp.map(fn, items))


def synth_field(seed, lo, hi, icells, jcells, kcells, igc, jgc, k_offset=0, dtype=np.float64, threads=1, pool=None):
    """C twin of oracle.synth.synth_field (bit-exact), z-chunks on ``threads``."""
    out = np.empty((kcells, jcells, icells), dtype=dtype)
    suffix = "f32" if out.dtype == np.float32 else "f64"
    fn = getattr(_lib(), f"synth_field_{suffix}")

    def run(kr):
        fn(_ptr(out), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.c_double(lo), C.c_double(hi), icells, jcells, igc, jgc,
           k_offset, kr[0], kr[1])

    _map(run, _chunks(0, kcells, threads), threads, pool)
    return out
