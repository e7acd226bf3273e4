"""Known-answer tests pinning the NumPy restatement of the rest of the MicroHH
stencil family (oracle/family_oracle.py; parity with upstream MicroHH is
unpinned, like the advec_u / diff_uvw oracle)."""

import numpy as np
import pytest

from oracle import family_oracle as fo
from paper_2303_12374_b200.stencils.profiles import make_profiles

SHAPE = (14, 13, 15)  # (kcells, jcells, icells), 3 ghost layers


def _grid(kc, j, i):
    k3, j3, i3 = np.meshgrid(np.arange(kc, dtype=float), np.arange(j, dtype=float), np.arange(i, dtype=float),
                             indexing="ij")
    return k3, j3, i3


@pytest.mark.parametrize("name", ["advec_v", "advec_w", "advec_s"])
def test_constant_field_and_velocity_give_zero_advection(name):
    prof = make_profiles(SHAPE[0], 3)
    const = np.full(SHAPE, 0.37)
    u, v, w = np.full(SHAPE, 0.7), np.full(SHAPE, -0.3), np.zeros(SHAPE)
    zero = np.zeros(SHAPE)
    if name == "advec_s":
        out = fo.advec_s(zero, const, u, v, w, prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
    elif name == "advec_v":
        out = fo.advec_v(zero, u, const, w, prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
        u, v = np.full(SHAPE, 0.7), np.full(SHAPE, 0.37)
        out = fo.advec_v(zero, u, v, w, prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
    else:
        out = fo.advec_w(zero, u, v, np.zeros(SHAPE), prof.rhoref, prof.rhorefh, prof.dzhi, 1.0, 1.0)
    assert np.max(np.abs(out)) < 1e-13


def test_advec_s_of_a_linear_profile_in_uniform_flow_is_exact():
    """5th-order upwind fluxes reproduce a linear scalar exactly: with uniform
    u and rho, the tendency is -u ds/dx."""
    kc, jc, ic = SHAPE
    _, _, i3 = _grid(kc, jc, ic)
    s = 0.25 * i3
    u, v, w = np.full(SHAPE, 0.8), np.zeros(SHAPE), np.zeros(SHAPE)
    ones = np.ones(kc)
    out = fo.advec_s(np.zeros(SHAPE), s, u, v, w, ones, ones, ones, 2.0, 1.0)
    inner = out[3:-3, 3:-3, 3:-3]
    assert np.allclose(inner, -0.8 * 0.25 * 2.0, atol=1e-13)


@pytest.mark.parametrize("upwind", [1.0, -1.0])
def test_advec_v_flux_is_upwind_biased(upwind):
    """A jump in v advected by u: the 5th-order upwind flux depends on the sign
    of the face velocity (interp5 enters with -|u|)."""
    prof = make_profiles(SHAPE[0], 3)
    v = np.where(np.arange(SHAPE[2])[None, None, :] < 7, 1.0, 0.0) * np.ones(SHAPE)
    u = np.full(SHAPE, upwind)
    out = fo.advec_v(np.zeros(SHAPE), u, v, np.zeros(SHAPE), prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
    mirrored = fo.advec_v(np.zeros(SHAPE), -u, v, np.zeros(SHAPE), prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
    assert not np.allclose(out, -mirrored)


def test_diff_c_kills_linear_profiles_and_conserves():
    kc, jc, ic = SHAPE
    k3, j3, i3 = _grid(kc, jc, ic)
    ones = np.ones(kc)
    e = np.full(SHAPE, 0.05)
    lin = 0.3 * i3 - 0.2 * j3 + 0.1 * k3
    out = fo.diff_c(np.zeros(SHAPE), lin, e, ones, ones, ones, ones, 1.0, 1.0, 3.0)
    assert np.max(np.abs(out[3:-3, 3:-3, 3:-3])) < 1e-13
    # a periodic bump in x: the x-diffusion sums to zero over a full period
    s = np.cos(2 * np.pi * (i3 - 3) / (ic - 6))
    out = fo.diff_c(np.zeros(SHAPE), s, e, ones, ones, ones, ones, 1.0, 1.0, 3.0)
    assert abs(out[3:-3, 3:-3, 3:-3].sum()) < 1e-10


def test_strain2_of_uniform_shear_and_solid_rotation():
    kc, jc, ic = SHAPE
    k3, j3, i3 = _grid(kc, jc, ic)
    prof = make_profiles(kc, 3)
    one = np.ones(kc)
    alpha = 0.6
    # simple shear u = alpha * y: 2 S_ij S_ij = alpha^2
    s2 = fo.strain2(alpha * j3, np.zeros(SHAPE), np.zeros(SHAPE), one, one, 1.0, 1.0)
    assert np.allclose(s2, alpha ** 2, atol=1e-13)
    # solid-body rotation u = -y, v = x has no strain
    s2 = fo.strain2(-(j3 - 0.5), i3 - 0.5, np.zeros(SHAPE), one, one, 1.0, 1.0)
    assert np.max(np.abs(s2)) < 1e-12
    # uniform stretching u = a x: 2 S_ij S_ij = 2 a^2
    s2 = fo.strain2(alpha * i3, np.zeros(SHAPE), np.zeros(SHAPE), prof.dzi, prof.dzhi, 1.0, 1.0)
    assert np.allclose(s2, 2 * alpha ** 2, atol=1e-13)


def test_evisc_smag_scales_with_mixing_length():
    kc, jc, ic = SHAPE
    _, j3, _ = _grid(kc, jc, ic)
    one = np.ones(kc)
    ev = fo.evisc_smag(np.zeros(SHAPE), 0.6 * j3, np.zeros(SHAPE), np.zeros(SHAPE), one * 0.5, one * 0.5, 1.0, 1.0,
                       0.1)
    # mlen = (1 * 1 * 2)^(1/3), |S| = 0.6
    assert np.allclose(ev[3:-3, 3:-3, 3:-3], (0.1 * 2 ** (1 / 3)) ** 2 * 0.6, atol=1e-14)
    assert np.all(ev[:3] == 0)
