"""NumPy restatement of the MicroHH interior stencils — TEST INFRASTRUCTURE.

PARITY UNPINNED against upstream MicroHH: the kernels are a third-party
dependency (MicroHH, gmd-10-3145-2017, cited at /root/reference/PAPER.md:350-352;
no version pin, no vendored copy — /root/reference/pkg/.gitignore:1-2) whose
source is absent from /root/reference.  The only reference call site is the
bodiless ``grid3d`` declaration (/root/reference/pkg/src/kltune/presets.py:17-20,
54-76).  These functions restate SURVEY.md Appendix A (advec_2i5::advec_u,
diff_smag2::diff_uvw interior formulas) and are pinned by known-answer tests
(tests/test_oracle.py).

Arrays are (kcells, jcells, icells) float64 views with ``g`` ghost layers on
every axis; all arithmetic is float64 (fp32 inputs are promoted), the GPU
result is compared with ``max|gpu - ref| / max|ref|`` per output array.
"""

from __future__ import annotations

import numpy as np

__all__ = ["interp2", "interp6_ws", "interp5_ws", "advec_u", "diff_uvw"]


def interp2(a, b):
    return 0.5 * (a + b)


def interp6_ws(a, b, c, d, e, f):
    """6th-order centred interpolation to the face between c and d."""
    return (37.0 * (c + d) - 8.0 * (b + e) + (a + f)) / 60.0


def interp5_ws(a, b, c, d, e, f):
    """Odd part of the 5th-order upwind interpolation (kills constants)."""
    return (10.0 * (d - c) - 5.0 * (e - b) + (f - a)) / 60.0


def _flux(vel, a, b, c, d, e, f):
    return vel * interp6_ws(a, b, c, d, e, f) - np.abs(vel) * interp5_ws(a, b, c, d, e, f)


class _Shift:
    """X[di, dj, dk] -> X[k+dk, j+dj, i+di] over the interior box."""

    def __init__(self, shape, gi, gj, gk, ni, nj, nk):
        self.gi, self.gj, self.gk = gi, gj, gk
        self.ni, self.nj, self.nk = ni, nj, nk

    def __call__(self, arr, di=0, dj=0, dk=0):
        return arr[self.gk + dk:self.gk + dk + self.nk,
                   self.gj + dj:self.gj + dj + self.nj,
                   self.gi + di:self.gi + di + self.ni]


def _box(arr, g, n):
    gi, gj, gk = g
    ni, nj, nk = n
    return _Shift(arr.shape, gi, gj, gk, ni, nj, nk)


def advec_u(ut, u, v, w, rhoref, rhorefh, dzi, dxi, dyi, ghost=(3, 3, 3), interior=None):
    """Return ``ut`` + advection tendency (new float64 array; inputs untouched).

    SURVEY.md Appendix A.2.  ``ghost`` = (igc, jgc, kgc); ``interior`` =
    (itot, jtot, ktot), inferred from the shapes when omitted.
    """
    u, v, w = (np.asarray(x, dtype=np.float64) for x in (u, v, w))
    out = np.array(ut, dtype=np.float64, copy=True)
    gi, gj, gk = ghost
    if interior is None:
        interior = (u.shape[2] - 2 * gi, u.shape[1] - 2 * gj, u.shape[0] - 2 * gk)
    X = _box(u, ghost, interior)
    ni, nj, nk = interior
    ks = slice(gk, gk + nk)
    rho = np.asarray(rhoref, np.float64)[ks][:, None, None]
    rhoh_bot = np.asarray(rhorefh, np.float64)[ks][:, None, None]
    rhoh_top = np.asarray(rhorefh, np.float64)[gk + 1:gk + 1 + nk][:, None, None]
    dz_i = np.asarray(dzi, np.float64)[ks][:, None, None]

    def run(axis_shift):
        return [X(u, **{axis_shift: o}) for o in (-3, -2, -1, 0, 1, 2, 3)]

    ux = run("di")
    uy = run("dj")
    uz = run("dk")

    ue = interp2(ux[3], ux[4])
    uw = interp2(ux[2], ux[3])
    fx = _flux(ue, *ux[1:7]) - _flux(uw, *ux[0:6])

    vn = interp2(X(v, -1, 1, 0), X(v, 0, 1, 0))
    vs = interp2(X(v, -1, 0, 0), X(v, 0, 0, 0))
    fy = _flux(vn, *uy[1:7]) - _flux(vs, *uy[0:6])

    wtop = interp2(X(w, -1, 0, 1), X(w, 0, 0, 1))
    wbot = interp2(X(w, -1, 0, 0), X(w, 0, 0, 0))
    fz = rhoh_top * _flux(wtop, *uz[1:7]) - rhoh_bot * _flux(wbot, *uz[0:6])

    X(out)[...] += -fx * dxi - fy * dyi - fz / rho * dz_i
    return out


def diff_uvw(ut, vt, wt, evisc, u, v, w, dzi, dzhi, rhoref, rhorefh, dxi, dyi, ghost=(3, 3, 3), interior=None):
    """Return (ut, vt, wt) + Smagorinsky diffusion tendencies."""
    e, u, v, w = (np.asarray(x, dtype=np.float64) for x in (evisc, u, v, w))
    out_u = np.array(ut, dtype=np.float64, copy=True)
    out_v = np.array(vt, dtype=np.float64, copy=True)
    out_w = np.array(wt, dtype=np.float64, copy=True)
    gi, gj, gk = ghost
    if interior is None:
        interior = (u.shape[2] - 2 * gi, u.shape[1] - 2 * gj, u.shape[0] - 2 * gk)
    X = _box(u, ghost, interior)
    nk = interior[2]

    def prof(a, dk=0):
        return np.asarray(a, np.float64)[gk + dk:gk + dk + nk][:, None, None]

    rh_top, rh_bot = prof(rhorefh, 1), prof(rhorefh)
    rho, rho_m = prof(rhoref), prof(rhoref, -1)
    dz_i, dz_i_m = prof(dzi), prof(dzi, -1)
    dzh_top, dzh = prof(dzhi, 1), prof(dzhi)
    q = 0.25
    e0 = X(e)

    # ---- ut ----
    en = q * (X(e, -1, 0, 0) + e0 + X(e, -1, 1, 0) + X(e, 0, 1, 0))
    es = q * (X(e, -1, -1, 0) + X(e, 0, -1, 0) + X(e, -1, 0, 0) + e0)
    et = q * (X(e, -1, 0, 0) + e0 + X(e, -1, 0, 1) + X(e, 0, 0, 1))
    eb = q * (X(e, -1, 0, -1) + X(e, 0, 0, -1) + X(e, -1, 0, 0) + e0)
    u0 = X(u)
    X(out_u)[...] += (
        (e0 * (X(u, 1) - u0) * dxi - X(e, -1) * (u0 - X(u, -1)) * dxi) * 2.0 * dxi
        + (en * ((X(u, 0, 1) - u0) * dyi + (X(v, 0, 1) - X(v, -1, 1)) * dxi)
           - es * ((u0 - X(u, 0, -1)) * dyi + (X(v) - X(v, -1)) * dxi)) * dyi
        + (rh_top * et * ((X(u, 0, 0, 1) - u0) * dzh_top + (X(w, 0, 0, 1) - X(w, -1, 0, 1)) * dxi)
           - rh_bot * eb * ((u0 - X(u, 0, 0, -1)) * dzh + (X(w) - X(w, -1)) * dxi)) / rho * dz_i
    )

    # ---- vt ----
    ee = q * (X(e, 0, -1, 0) + e0 + X(e, 1, -1, 0) + X(e, 1, 0, 0))
    ew = q * (X(e, -1, -1, 0) + X(e, -1, 0, 0) + X(e, 0, -1, 0) + e0)
    et = q * (X(e, 0, -1, 0) + e0 + X(e, 0, -1, 1) + X(e, 0, 0, 1))
    eb = q * (X(e, 0, -1, -1) + X(e, 0, 0, -1) + X(e, 0, -1, 0) + e0)
    v0 = X(v)
    X(out_v)[...] += (
        (ee * ((X(v, 1) - v0) * dxi + (X(u, 1) - X(u, 1, -1)) * dyi)
         - ew * ((v0 - X(v, -1)) * dxi + (X(u) - X(u, 0, -1)) * dyi)) * dxi
        + (e0 * (X(v, 0, 1) - v0) * dyi - X(e, 0, -1) * (v0 - X(v, 0, -1)) * dyi) * 2.0 * dyi
        + (rh_top * et * ((X(v, 0, 0, 1) - v0) * dzh_top + (X(w, 0, 0, 1) - X(w, 0, -1, 1)) * dyi)
           - rh_bot * eb * ((v0 - X(v, 0, 0, -1)) * dzh + (X(w) - X(w, 0, -1)) * dyi)) / rho * dz_i
    )

    # ---- wt ----
    ee = q * (X(e, 0, 0, -1) + e0 + X(e, 1, 0, -1) + X(e, 1, 0, 0))
    ew = q * (X(e, -1, 0, -1) + X(e, -1, 0, 0) + X(e, 0, 0, -1) + e0)
    en = q * (X(e, 0, 0, -1) + e0 + X(e, 0, 1, -1) + X(e, 0, 1, 0))
    es = q * (X(e, 0, -1, -1) + X(e, 0, -1, 0) + X(e, 0, 0, -1) + e0)
    w0 = X(w)
    X(out_w)[...] += (
        (ee * ((X(w, 1) - w0) * dxi + (X(u, 1) - X(u, 1, 0, -1)) * dzh)
         - ew * ((w0 - X(w, -1)) * dxi + (X(u) - X(u, 0, 0, -1)) * dzh)) * dxi
        + (en * ((X(w, 0, 1) - w0) * dyi + (X(v, 0, 1) - X(v, 0, 1, -1)) * dzh)
           - es * ((w0 - X(w, 0, -1)) * dyi + (X(v) - X(v, 0, 0, -1)) * dzh)) * dyi
        + (rho * e0 * (X(w, 0, 0, 1) - w0) * dz_i - rho_m * X(e, 0, 0, -1) * (w0 - X(w, 0, 0, -1)) * dz_i_m)
        / prof(rhorefh) * 2.0 * dzh
    )
    return out_u, out_v, out_w
