"""Known-answer tests pinning the NumPy stencil oracle (parity with upstream
MicroHH is unpinned — see oracle/__init__.py) and the synthetic-field twin."""

import numpy as np
import pytest

from oracle import stencil_oracle as so
from oracle.synth import synth_field, synth_values
from paper_2303_12374_b200.rng import SplitMix64
from paper_2303_12374_b200.stencils.profiles import make_profiles


def test_interp6_exact_for_cell_averages_of_quintics_and_interp5_kills_constants():
    """interp6_ws is the finite-volume face reconstruction: exact for cell
    averages of polynomials up to degree 5; interp5_ws vanishes on constants."""
    edges = np.arange(-3.0, 3.5, 1.0)  # 6 cells around the face at x = 0
    rng = np.random.default_rng(0)
    for _ in range(20):
        coef = rng.normal(size=6)
        prim = np.polynomial.polynomial.polyint(coef)
        avg = np.diff(np.polynomial.polynomial.polyval(edges, prim))
        face = np.polynomial.polynomial.polyval(0.0, coef)
        assert abs(so.interp6_ws(*avg) - face) < 1e-12 * (1 + np.abs(avg).max())
        assert so.interp5_ws(*np.full(6, avg[0])) == 0.0


def _fields(shape, seed=1):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, shape) for _ in range(3)]


def test_constant_velocity_constant_u_gives_zero_advection():
    shape = (14, 12, 13)
    u = np.full(shape, 0.7)
    v = np.full(shape, -0.3)
    w = np.zeros(shape)
    prof = make_profiles(shape[0], 3)
    ut = np.zeros(shape)
    out = so.advec_u(ut, u, v, w, prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
    assert np.max(np.abs(out)) < 1e-13


def test_constant_fields_give_zero_diffusion():
    shape = (9, 10, 11)
    e = np.full(shape, 0.05)
    u, v, w = (np.full(shape, c) for c in (0.3, -0.2, 0.1))
    prof = make_profiles(shape[0], 3)
    z = np.zeros(shape)
    for out in so.diff_uvw(z, z, z, e, u, v, w, prof.dzi, prof.dzhi, prof.rhoref, prof.rhorefh, 1.0, 1.0):
        assert np.max(np.abs(out)) < 1e-15


def test_periodic_shift_equivariance_in_x():
    """Shifting all fields periodically in x shifts the tendency (interior)."""
    g, n = 3, (16, 10, 8)
    shape = (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g)
    fields = {}
    for name, seed in (("u", 1), ("v", 2), ("w", 3), ("e", 4)):
        core = np.random.default_rng(seed).uniform(-1, 1, (shape[0], shape[1], n[0]))
        fields[name] = core
    def pad(core):
        return np.concatenate([core[:, :, -g:], core, core[:, :, :g]], axis=2)
    prof = make_profiles(shape[0], g)
    base = so.advec_u(np.zeros(shape), pad(fields["u"]), pad(fields["v"]), pad(fields["w"]), prof.rhoref,
                      prof.rhorefh, prof.dzi, 1.0, 1.0)
    shifted = so.advec_u(np.zeros(shape), *(pad(np.roll(fields[k], 5, axis=2)) for k in "uvw"), prof.rhoref,
                         prof.rhorefh, prof.dzi, 1.0, 1.0)
    inner = (slice(g, -g), slice(g, -g), slice(g, -g))
    assert np.allclose(np.roll(base[inner], 5, axis=2), shifted[inner], atol=1e-13)


def test_advection_of_linear_profile_matches_analytic():
    """u = a + b*x with constant v = w = 0 and uniform grid: ut = -d(uu)/dx = -2 u b (exact for quadratics)."""
    g, n = 3, (12, 8, 6)
    shape = (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g)
    x = np.arange(shape[2]) - 0.5  # u at i-1/2
    u = np.broadcast_to(0.3 + 0.05 * x, shape).copy()
    z = np.zeros(shape)
    prof = make_profiles(shape[0], g)
    out = so.advec_u(z, u, z, z, prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)
    inner = out[g:-g, g:-g, g:-g]
    expect = -2 * u[g:-g, g:-g, g:-g] * 0.05
    assert np.allclose(inner, expect, atol=1e-12)


def test_synth_twin_is_splitmix_stream():
    seed = 230312374
    stream = SplitMix64(seed)
    ref = [(stream.next_u64() >> 11) * 2.0 ** -53 for _ in range(50)]
    got = synth_values(seed, np.arange(50), 0.0, 1.0)
    assert np.array_equal(got, np.array(ref))


def test_synth_periodic_ghosts():
    f = synth_field(5, -1, 1, 10 + 6, 7 + 6, 4, 3, 3)
    assert np.array_equal(f[:, :, :3], f[:, :, 10:13]) and np.array_equal(f[:, :3, :], f[:, 7:10, :])
    part = synth_field(5, -1, 1, 16, 13, 2, 3, 3, k_offset=2)
    assert np.array_equal(part, f[2:4])


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
def test_c_restatement_matches_numpy_oracle(kernel):
    from oracle import cref
    from oracle.synth import synth_field
    from paper_2303_12374_b200.stencils.problem import KERNEL_FIELDS
    from paper_2303_12374_b200.stencils.profiles import FIELD_SEED_BASE, FIELD_SPECS

    if not cref.available():
        pytest.skip("oracle/_build/libstencil_ref.so not built (make -C oracle)")
    g, n = 3, (20, 14, 9)
    shape = (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g)
    f = {}
    for name in KERNEL_FIELDS[kernel]:
        s, lo, hi = FIELD_SPECS[name]
        f[name] = synth_field(FIELD_SEED_BASE + s, lo, hi, shape[2], shape[1], shape[0], g, g)
    prof = make_profiles(shape[0], g)
    if kernel == "advec_u":
        ref = {"ut": so.advec_u(f["ut"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0)}
        got = {"ut": f["ut"].copy()}
        cref.advec_u(got["ut"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh, prof.dzi, 1.0, 1.0, threads=3)
    else:
        r = so.diff_uvw(f["ut"], f["vt"], f["wt"], f["evisc"], f["u"], f["v"], f["w"], prof.dzi, prof.dzhi,
                        prof.rhoref, prof.rhorefh, 1.0, 1.0)
        ref = dict(zip(("ut", "vt", "wt"), r))
        got = {k: f[k].copy() for k in ("ut", "vt", "wt")}
        cref.diff_uvw(got["ut"], got["vt"], got["wt"], f["evisc"], f["u"], f["v"], f["w"], prof.dzi, prof.dzhi,
                      prof.rhoref, prof.rhorefh, 1.0, 1.0, threads=2)
    for name in ref:
        assert np.max(np.abs(got[name] - ref[name])) <= 1e-12 * np.max(np.abs(ref[name]))


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw", "diff_uvw_rk3", "evisc_smag"])
def test_oracle_window_equals_whole_grid(kernel):
    """The bounded-window oracle the large-shape GPU parity tests use
    (tests/test_gpu_bench_parity.py) equals the whole-grid oracle, for a grid
    and for a z-slab of it (global plane offset)."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from stencil_helpers import oracle_outputs, oracle_window
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(20, 12, 16, "fp32")
    full, _ = oracle_outputs(kernel, lay)
    win = oracle_window(kernel, lay, 5, 11)
    for name, arr in win.items():
        assert np.array_equal(arr, lay.interior(full[name])[2:8])
    slab = GridLayout(20, 12, 8, "fp32")  # global interior planes 4..12 = padded offset 4
    win = oracle_window(kernel, slab, 3, 11, k_offset=4, kcells_global=lay.kcells)
    for name, arr in win.items():
        assert np.array_equal(arr, lay.interior(full[name])[4:12])


@pytest.mark.parametrize("kernel,precision", [("advec_u", "fp32"), ("diff_uvw", "fp64"), ("diff_uvw", "fp32"),
                                              ("diff_uvw_rk3", "fp64"), ("advec_v", "fp32"), ("advec_w", "fp64"),
                                              ("advec_s", "fp32"), ("diff_c", "fp64"), ("evisc_smag", "fp32"),
                                              ("evisc_smag", "fp64"), ("rk3_uvw", "fp32")])
def test_cref_chunks_cover_the_grid_like_the_numpy_oracle(kernel, precision):
    """The full-volume GPU parity check (stencil_helpers.full_volume_error)
    streams the C restatement over z-chunks with their inputs regenerated per
    chunk; stitched together they must equal the NumPy oracle of the whole
    grid, and a z-slab (k_offset) must equal the same planes of the grid."""
    from oracle import cref

    if not cref.available():
        pytest.skip("oracle/_build not built")
    from stencil_helpers import cref_chunks, oracle_outputs

    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(20, 14, 11, precision)
    ref, _ = oracle_outputs(kernel, lay)
    covered = 0
    for kb, ke, out in cref_chunks(kernel, lay, chunk=4, threads=2):
        covered += ke - kb
        for n, r in out.items():
            want = lay.interior(ref[n])[kb - lay.kstart:ke - lay.kstart]
            assert np.allclose(r, want, rtol=0, atol=1e-12 * np.max(np.abs(want))), (n, kb)
    assert covered == lay.ktot
    # a slab of planes 4..8 of the same grid (its own 3 ghost planes read the neighbours' planes)
    slab = GridLayout(20, 14, 4, precision)
    for kb, ke, out in cref_chunks(kernel, slab, k_offset=4, kcells_global=lay.kcells, chunk=3, threads=1):
        for n, r in out.items():
            lo = kb - slab.kstart + 4
            want = lay.interior(ref[n])[lo:lo + ke - kb]
            assert np.allclose(r, want, rtol=0, atol=1e-12 * np.max(np.abs(want))), (n, kb)
