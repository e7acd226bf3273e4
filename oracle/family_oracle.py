"""NumPy restatement of the rest of the MicroHH stencil family — TEST INFRASTRUCTURE.

SURVEY.md §8(f) row 2 ("remaining MicroHH stencils in the same family"):
``advec_v``, ``advec_w`` and the scalar ``advec_s`` of advec_2i5; the scalar
diffusion ``diff_c`` and the neutral Smagorinsky eddy viscosity
(``evisc_smag``: strain rate + viscosity, the step before ``diff_uvw``) of
diff_smag2.

PARITY UNPINNED against upstream MicroHH, exactly like stencil_oracle.py:
the kernels are a third-party dependency (MicroHH, gmd-10-3145-2017, cited
at /root/reference/PAPER.md:350-352) absent from /root/reference; the paper
names only advec_u / diff_uvw.  These functions are the
builder's restatement, in the notation of SURVEY.md Appendix A, with the same
builder decisions: >= 3 ghost layers on every axis, one interior formula for
every cell (no near-wall special cases), every interior k evaluated (w at the
wall level included).  They are pinned by known-answer tests
(tests/test_family_oracle.py).  Only tests/ and bench.py's CPU legs import
this module.

Staggering (Arakawa C): u at (i-1/2, j, k), v at (i, j-1/2, k), w at
(i, j, k-1/2), scalars / evisc / rhoref at centres, rhorefh at k-1/2.
``X[di, dj, dk]`` is ``X[k+dk, j+dj, i+di]``; all arithmetic float64.
"""

from __future__ import annotations

import numpy as np

from .stencil_oracle import _box, _flux, interp2

__all__ = ["advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag", "strain2", "rk3_uvw", "diff_uvw_rk3"]


def _setup(fields, ghost, interior):
    arrs = [np.asarray(f, dtype=np.float64) for f in fields]
    gi, gj, gk = ghost
    a0 = arrs[0]
    if interior is None:
        interior = (a0.shape[2] - 2 * gi, a0.shape[1] - 2 * gj, a0.shape[0] - 2 * gk)
    return arrs, _box(a0, ghost, interior), interior


def _prof(a, gk, nk, dk=0):
    return np.asarray(a, np.float64)[gk + dk:gk + dk + nk][:, None, None]


def _runs(X, a, key):
    return [X(a, **{key: o}) for o in (-3, -2, -1, 0, 1, 2, 3)]


def _advect(X, phi, vel_x, vel_y, vel_z, rh_top, rh_bot, fac):
    """-(div of the 5th-order upwind fluxes of ``phi``); face velocities are
    (west, east), (south, north), (bottom, top) pairs, ``fac`` the z metric."""
    px, py, pz = _runs(X, phi, "di"), _runs(X, phi, "dj"), _runs(X, phi, "dk")
    fx = _flux(vel_x[1], *px[1:7]) - _flux(vel_x[0], *px[0:6])
    fy = _flux(vel_y[1], *py[1:7]) - _flux(vel_y[0], *py[0:6])
    fz = rh_top * _flux(vel_z[1], *pz[1:7]) - rh_bot * _flux(vel_z[0], *pz[0:6])
    return fx, fy, fz * fac


def advec_v(vt, u, v, w, rhoref, rhorefh, dzi, dxi, dyi, ghost=(3, 3, 3), interior=None):
    """vt + advection of v at (i, j-1/2, k): x faces carry u averaged over rows
    j-1, j; y faces v averaged to the centres; z faces w averaged over rows
    j-1, j (times rhorefh); divided by rhoref[k] / dz[k]."""
    (u, v, w), X, n = _setup((u, v, w), ghost, interior)
    out = np.array(vt, dtype=np.float64, copy=True)
    gk, nk = ghost[2], n[2]
    vx = (interp2(X(u, 0, -1), X(u)), interp2(X(u, 1, -1), X(u, 1)))
    vy = (interp2(X(v, 0, -1), X(v)), interp2(X(v), X(v, 0, 1)))
    vz = (interp2(X(w, 0, -1), X(w)), interp2(X(w, 0, -1, 1), X(w, 0, 0, 1)))
    fx, fy, fz = _advect(X, v, vx, vy, vz, _prof(rhorefh, gk, nk, 1), _prof(rhorefh, gk, nk),
                         _prof(dzi, gk, nk) / _prof(rhoref, gk, nk))
    X(out)[...] += -fx * dxi - fy * dyi - fz
    return out


def advec_w(wt, u, v, w, rhoref, rhorefh, dzhi, dxi, dyi, ghost=(3, 3, 3), interior=None):
    """wt + advection of w at (i, j, k-1/2): x faces carry u averaged over
    levels k-1, k; y faces v likewise; z faces (at centres k-1, k) w averaged
    times rhoref[k-1] / rhoref[k]; divided by rhorefh[k] / dzh[k]."""
    (u, v, w), X, n = _setup((u, v, w), ghost, interior)
    out = np.array(wt, dtype=np.float64, copy=True)
    gk, nk = ghost[2], n[2]
    vx = (interp2(X(u, 0, 0, -1), X(u)), interp2(X(u, 1, 0, -1), X(u, 1)))
    vy = (interp2(X(v, 0, 0, -1), X(v)), interp2(X(v, 0, 1, -1), X(v, 0, 1)))
    vz = (interp2(X(w, 0, 0, -1), X(w)), interp2(X(w), X(w, 0, 0, 1)))
    fx, fy, fz = _advect(X, w, vx, vy, vz, _prof(rhoref, gk, nk), _prof(rhoref, gk, nk, -1),
                         _prof(dzhi, gk, nk) / _prof(rhorefh, gk, nk))
    X(out)[...] += -fx * dxi - fy * dyi - fz
    return out


def advec_s(st, s, u, v, w, rhoref, rhorefh, dzi, dxi, dyi, ghost=(3, 3, 3), interior=None):
    """st + advection of a cell-centred scalar: face velocities are the
    staggered components themselves (u[i], u[i+1], ...)."""
    (s, u, v, w), X, n = _setup((s, u, v, w), ghost, interior)
    out = np.array(st, dtype=np.float64, copy=True)
    gk, nk = ghost[2], n[2]
    fx, fy, fz = _advect(X, s, (X(u), X(u, 1)), (X(v), X(v, 0, 1)), (X(w), X(w, 0, 0, 1)),
                         _prof(rhorefh, gk, nk, 1), _prof(rhorefh, gk, nk),
                         _prof(dzi, gk, nk) / _prof(rhoref, gk, nk))
    X(out)[...] += -fx * dxi - fy * dyi - fz
    return out


def diff_c(st, s, evisc, dzi, dzhi, rhoref, rhorefh, dxi, dyi, tpri, ghost=(3, 3, 3), interior=None):
    """st + Smagorinsky diffusion of a scalar with eddy diffusivity
    evisc / Pr_t (``tpri`` = 1 / Pr_t), face diffusivities the two-point
    means of evisc; z faces weighted by rhorefh and dzh, divided by rhoref dz."""
    (s, e), X, n = _setup((s, evisc), ghost, interior)
    out = np.array(st, dtype=np.float64, copy=True)
    gk, nk = ghost[2], n[2]
    s0, e0 = X(s), X(e)
    ee, ew = 0.5 * (e0 + X(e, 1)) * tpri, 0.5 * (X(e, -1) + e0) * tpri
    en, es = 0.5 * (e0 + X(e, 0, 1)) * tpri, 0.5 * (X(e, 0, -1) + e0) * tpri
    et, eb = 0.5 * (e0 + X(e, 0, 0, 1)) * tpri, 0.5 * (X(e, 0, 0, -1) + e0) * tpri
    X(out)[...] += (
        (ee * (X(s, 1) - s0) - ew * (s0 - X(s, -1))) * dxi * dxi
        + (en * (X(s, 0, 1) - s0) - es * (s0 - X(s, 0, -1))) * dyi * dyi
        + (_prof(rhorefh, gk, nk, 1) * et * (X(s, 0, 0, 1) - s0) * _prof(dzhi, gk, nk, 1)
           - _prof(rhorefh, gk, nk) * eb * (s0 - X(s, 0, 0, -1)) * _prof(dzhi, gk, nk))
        / _prof(rhoref, gk, nk) * _prof(dzi, gk, nk)
    )
    return out


def strain2(u, v, w, dzi, dzhi, dxi, dyi, ghost=(3, 3, 3), interior=None):
    """Squared strain rate 2 S_ij S_ij at cell centres: the diagonal terms at
    the centre, each off-diagonal term the mean of its four surrounding edges."""
    (u, v, w), X, n = _setup((u, v, w), ghost, interior)
    gk, nk = ghost[2], n[2]
    dz, dzh, dzh1 = _prof(dzi, gk, nk), _prof(dzhi, gk, nk), _prof(dzhi, gk, nk, 1)
    diag = 2.0 * (((X(u, 1) - X(u)) * dxi) ** 2 + ((X(v, 0, 1) - X(v)) * dyi) ** 2
                  + ((X(w, 0, 0, 1) - X(w)) * dz) ** 2)

    def sxy(di, dj):  # edge (i-1/2+di, j-1/2+dj): du/dy + dv/dx
        return ((X(u, di, dj) - X(u, di, dj - 1)) * dyi + (X(v, di, dj) - X(v, di - 1, dj)) * dxi) ** 2

    def sxz(di, dk, dzh_):  # edge (i-1/2+di, k-1/2+dk): du/dz + dw/dx
        return ((X(u, di, 0, dk) - X(u, di, 0, dk - 1)) * dzh_ + (X(w, di, 0, dk) - X(w, di - 1, 0, dk)) * dxi) ** 2

    def syz(dj, dk, dzh_):  # edge (j-1/2+dj, k-1/2+dk): dv/dz + dw/dy
        return ((X(v, 0, dj, dk) - X(v, 0, dj, dk - 1)) * dzh_ + (X(w, 0, dj, dk) - X(w, 0, dj - 1, dk)) * dyi) ** 2

    # 2 x (1/8 of the sum over four edges): each squared (du_i/dx_j + du_j/dx_i) edge value
    # holds S_ij^2 + S_ji^2 = 2 S_ij^2 (x4), so a uniform shear alpha gives alpha^2
    off = 0.25 * (sxy(0, 0) + sxy(0, 1) + sxy(1, 0) + sxy(1, 1)
                   + sxz(0, 0, dzh) + sxz(0, 1, dzh1) + sxz(1, 0, dzh) + sxz(1, 1, dzh1)
                   + syz(0, 0, dzh) + syz(0, 1, dzh1) + syz(1, 0, dzh) + syz(1, 1, dzh1))
    return diag + off


def evisc_smag(evisc, u, v, w, dzi, dzhi, dxi, dyi, cs, ghost=(3, 3, 3), interior=None):
    """Neutral Smagorinsky eddy viscosity written over the interior of a copy
    of ``evisc``: (cs * (dx dy dz)^(1/3))^2 * sqrt(2 S_ij S_ij)."""
    out = np.array(evisc, dtype=np.float64, copy=True)
    s2 = strain2(u, v, w, dzi, dzhi, dxi, dyi, ghost, interior)
    _, X, n = _setup((u,), ghost, interior)
    gk, nk = ghost[2], n[2]
    mlen = np.cbrt(1.0 / (dxi * dyi * _prof(dzi, gk, nk)))
    X(out)[...] = (cs * mlen) ** 2 * np.sqrt(s2)
    return out


def rk3_uvw(ut, vt, wt, u, v, w, rk_a, rk_bdt, ghost=(3, 3, 3), interior=None):
    """One low-storage RK3 substep on the interior: a + rk_bdt * at and
    rk_a * at for (u, ut), (v, vt), (w, wt).  Returns (ut, vt, wt, u, v, w)."""
    arrs, X, _ = _setup((ut, vt, wt, u, v, w), ghost, interior)
    out = [np.array(a, copy=True) for a in arrs]
    for t, a in ((0, 3), (1, 4), (2, 5)):
        X(out[a])[...] += rk_bdt * X(arrs[t])
        X(out[t])[...] = rk_a * X(arrs[t])
    return tuple(out)


def diff_uvw_rk3(ut, vt, wt, evisc, u, v, w, u_next, v_next, w_next, dzi, dzhi, rhoref, rhorefh, dxi, dyi, rk_a,
                 rk_bdt, ghost=(3, 3, 3), interior=None):
    """diff_uvw followed by one RK3 substep into the next-substep buffers
    (SURVEY §8f row 1): T = t + diffusion; t <- rk_a T; next <- cur + rk_bdt T
    on the interior (ghost cells of every array keep their inputs).  Returns
    (ut, vt, wt, u_next, v_next, w_next)."""
    from .stencil_oracle import diff_uvw

    tu, tv, tw = diff_uvw(ut, vt, wt, evisc, u, v, w, dzi, dzhi, rhoref, rhorefh, dxi, dyi, ghost, interior)
    arrs, X, _ = _setup((u, v, w, ut, vt, wt, u_next, v_next, w_next), ghost, interior)
    res = []
    for t_new, t_old in ((tu, arrs[3]), (tv, arrs[4]), (tw, arrs[5])):
        out = np.array(t_old, copy=True)
        X(out)[...] = rk_a * X(t_new)
        res.append(out)
    for cur, t_new, nxt in ((arrs[0], tu, arrs[6]), (arrs[1], tv, arrs[7]), (arrs[2], tw, arrs[8])):
        out = np.array(nxt, copy=True)
        X(out)[...] = X(cur) + rk_bdt * X(t_new)
        res.append(out)
    return tuple(res)
