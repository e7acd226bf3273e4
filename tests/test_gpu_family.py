"""GPU parity of the rest of the MicroHH stencil family (SURVEY §8f row 2:
advec_v, advec_w, advec_s, diff_c, evisc_smag) against the NumPy restatement
(oracle/family_oracle.py), through the same NVRTC / C-ABI launch path as the
hot-path kernels.  Bar: max|gpu - ref| / max|ref| <= 1e-5 (fp32), 1e-12 (fp64)."""

import numpy as np
import pytest

from stencil_helpers import TOL, oracle_outputs, rel_error, run_config

pytestmark = pytest.mark.gpu

FAMILY = ["advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag"]


@pytest.fixture(scope="module")
def compiler(gpu_ctx):
    from paper_2303_12374_b200.cuda import NvrtcCompiler

    return NvrtcCompiler(gpu_ctx)


def _space(kernel, precision):
    from paper_2303_12374_b200.stencils.definitions import definition_for

    return definition_for(kernel, precision).space


@pytest.mark.parametrize("kernel", FAMILY)
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_family_default_and_sampled_configs_match_oracle(gpu_ctx, compiler, kernel, precision):
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(45, 23, 19, precision)
    ref, _ = oracle_outputs(kernel, lay)
    space = _space(kernel, precision)
    cfgs = [space.default_config()[0]] + space.sample_random(5 if precision == "fp32" else 6, 4)
    for cfg in cfgs:
        got = run_config(gpu_ctx, compiler, kernel, lay, cfg)
        for name in ref:
            err = rel_error(got[name], ref[name], lay)
            assert err <= TOL[precision], (cfg, name, err)


@pytest.mark.parametrize("kernel", FAMILY)
def test_family_k_subrange_launch(gpu_ctx, compiler, kernel):
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(32, 24, 20, "fp64")
    kr = (lay.kstart + 4, lay.kstart + 13)
    ref, _ = oracle_outputs(kernel, lay, k_range=kr)
    cfg = dict(_space(kernel, "fp64").default_config()[0], block_x=32, block_y=4, tile_z=2, contiguous_z=True)
    got = run_config(gpu_ctx, compiler, kernel, lay, cfg, k_range=kr)
    for name in ref:
        diff = np.max(np.abs(got[name].astype(np.float64) - ref[name]))
        assert diff <= 1e-12 * np.max(np.abs(ref[name])), (name, diff)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_rk3_fused_diffusion_matches_oracle(gpu_ctx, compiler, precision):
    """diff_uvw_rk3: the diffusion tendency with the RK3
    substep fused into its store, in every staging family (DIRECT, ZMARCH,
    TMA incl. packed column tiles), against the oracle diff_uvw + RK3."""
    from paper_2303_12374_b200.stencils.definitions import FAMILY_PINS, family_space
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(45, 23, 19, precision)
    ref, _ = oracle_outputs("diff_uvw_rk3", lay)
    space = _space("diff_uvw_rk3", precision)
    cfgs = [space.default_config()[0]]
    for fam in FAMILY_PINS:
        cfgs += family_space("diff_uvw_rk3", fam, precision).sample_random(13, 2)
    base = space.default_config()[0]
    cfgs.append(dict(base, staging="TMA", contiguous_x=True, block_x=16, block_y=4, tile_x=4, tile_y=2, depth=1,
                     zchunk=8, unravel="XYZ"))
    for cfg in cfgs:
        assert space.is_valid(cfg), cfg
        got = run_config(gpu_ctx, compiler, "diff_uvw_rk3", lay, cfg)
        for name in ref:
            err = rel_error(got[name], ref[name], lay)
            assert err <= TOL[precision], (cfg["staging"], name, err)


def test_rk3_pass_matches_oracle(gpu_ctx, compiler):
    from paper_2303_12374_b200.stencils.layout import GridLayout

    for precision in ("fp32", "fp64"):
        lay = GridLayout(45, 23, 19, precision)
        ref, _ = oracle_outputs("rk3_uvw", lay)
        base = _space("rk3_uvw", precision).default_config()[0]
        # default (scalar), then the vector path: consecutive column tiles of
        # 2 / 4 cells, the last chunk of every row crossing iend (45 columns)
        cfgs = [base,
                dict(base, contiguous_x=True, tile_x=2, block_x=16, block_y=2, tile_y=2, tile_z=2),
                dict(base, contiguous_x=True, tile_x=4, block_x=16, block_y=4, block_z=2, unroll_x=True),
                dict(base, contiguous_x=True, tile_x=4, block_x=32, contiguous_z=True, tile_z=4, unravel="ZYX")]
        for cfg in cfgs:
            got = run_config(gpu_ctx, compiler, "rk3_uvw", lay, cfg)
            for name in ref:
                assert rel_error(got[name], ref[name], lay) <= TOL[precision], (cfg, name)


@pytest.mark.parametrize("kernel", ["advec_v", "advec_w", "advec_s"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_family_tma_advection_matches_oracle(gpu_ctx, compiler, kernel, precision):
    """TMA-staged flux-form advection of the family (advec_family_tma.cuh):
    sampled TMA configurations plus fixed column-tile shapes on ragged grids
    (partial thread tiles and blocks), against the oracle."""
    from paper_2303_12374_b200.stencils.definitions import family_space
    from paper_2303_12374_b200.stencils.layout import GridLayout

    space = _space(kernel, precision)
    base = space.default_config()[0]
    cfgs = family_space(kernel, "TMA", precision).sample_random(17, 3)
    cfgs += [dict(base, staging="TMA", contiguous_x=True, block_x=32, block_y=4, tile_x=2, tile_y=2, depth=2,
                  zchunk=16, unravel="XYZ"),
             dict(base, staging="TMA", contiguous_x=True, block_x=16, block_y=2, tile_x=4, tile_y=3, depth=1,
                  zchunk=8)]
    for grid in ((45, 23, 19), (130, 37, 41)):
        lay = GridLayout(*grid, precision)
        ref, _ = oracle_outputs(kernel, lay)
        for cfg in cfgs:
            assert space.is_valid(cfg), cfg
            got = run_config(gpu_ctx, compiler, kernel, lay, cfg)
            for name in ref:
                err = rel_error(got[name], ref[name], lay)
                assert err <= TOL[precision], (grid, cfg, name, err)


@pytest.mark.parametrize("kernel", ["advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag"])
def test_family_tma_misaligned_fields_use_scalar_path(gpu_ctx, compiler, kernel):
    """Pointers shifted off the 16-byte grid: the uniform scalar-access branch
    of the family TMA kernel gives the oracle result too."""
    from paper_2303_12374_b200.capture import scalar_env_from_args
    from paper_2303_12374_b200.cuda import DeviceArray, DeviceBuffer
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    precision = "fp32"
    lay = GridLayout(70, 29, 23, precision)
    ref, _ = oracle_outputs(kernel, lay)
    cfg = dict(_space(kernel, precision).default_config()[0], staging="TMA", contiguous_x=True, block_x=16,
               block_y=4, tile_x=4, tile_y=2, depth=2, zchunk=8)
    prob = StencilProblem(kernel, lay, gpu_ctx)
    shifted = {}
    try:
        args = []
        for a in prob.args():
            if isinstance(a, DeviceBuffer) and a.element_count == lay.span_elems:
                arr = DeviceArray(lay.alloc_bytes + 64)
                dst = arr.ptr + lay.elem_bytes
                check(lib().klb_memcpy_dtod(dst, a.ptr - lay.lead * lay.elem_bytes, lay.alloc_bytes, None))
                shifted[a.position] = arr
                a = DeviceBuffer(a.position, a.role, a.element_type, dst + lay.lead * lay.elem_bytes,
                                 a.element_count, owner=arr)
            args.append(a)
        gpu_ctx.synchronize()
        d = prob.definition
        env = scalar_env_from_args(args)
        problem = d.derive_problem_size(env)
        exe = compiler.compile(d.render_compile_request(cfg, problem, env), gpu_ctx.ident)
        exe.load()
        exe.launch(d.derive_geometry(cfg, problem, env), args, timed=True)
        name = prob.outputs()[0]
        flat = np.frombuffer(shifted[0].download(lay.alloc_bytes, offset_bytes=lay.elem_bytes), dtype=lay.dtype)
        assert rel_error(lay.host_view(flat), ref[name], lay) <= TOL[precision]
    finally:
        for arr in shifted.values():
            arr.free()
        prob.close()


def test_rk3_vector_config_on_misaligned_fields_takes_the_scalar_path(gpu_ctx, compiler):
    """rk3_uvw's vector path needs every row start vector-aligned; with the
    fields shifted one element off the 16-byte grid the same column-tile
    configuration must take the scalar loop and still match the oracle."""
    from paper_2303_12374_b200.capture import scalar_env_from_args
    from paper_2303_12374_b200.cuda import DeviceArray, DeviceBuffer
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    precision = "fp32"
    lay = GridLayout(45, 23, 19, precision)
    ref, _ = oracle_outputs("rk3_uvw", lay)
    cfg = dict(_space("rk3_uvw", precision).default_config()[0], contiguous_x=True, tile_x=4, block_x=16, block_y=4)
    prob = StencilProblem("rk3_uvw", lay, gpu_ctx)
    shifted, names = {}, {}
    try:
        args = []
        for a in prob.args():
            if isinstance(a, DeviceBuffer) and a.element_count == lay.span_elems:
                arr = DeviceArray(lay.alloc_bytes + 64)
                dst = arr.ptr + lay.elem_bytes
                check(lib().klb_memcpy_dtod(dst, a.ptr - lay.lead * lay.elem_bytes, lay.alloc_bytes, None))
                shifted[a.position] = arr
                a = DeviceBuffer(a.position, a.role, a.element_type, dst + lay.lead * lay.elem_bytes,
                                 a.element_count, owner=arr)
            args.append(a)
        gpu_ctx.synchronize()
        d = prob.definition
        env = scalar_env_from_args(args)
        problem = d.derive_problem_size(env)
        exe = compiler.compile(d.render_compile_request(cfg, problem, env), gpu_ctx.ident)
        exe.load()
        exe.launch(d.derive_geometry(cfg, problem, env), args, timed=True)
        order = ("ut", "vt", "wt", "u", "v", "w")  # ARG_LAYOUT["rk3_uvw"] buffer order
        assert sorted(shifted) == list(range(6))
        for pos, name in enumerate(order):
            flat = np.frombuffer(shifted[pos].download(lay.alloc_bytes, offset_bytes=lay.elem_bytes), dtype=lay.dtype)
            assert rel_error(lay.host_view(flat), ref[name], lay) <= TOL[precision], name
    finally:
        for arr in shifted.values():
            arr.free()
        prob.close()


@pytest.mark.parametrize("kernel", ["diff_c", "evisc_smag"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_family_tma_plane_march_matches_oracle(gpu_ctx, compiler, kernel, precision):
    """TMA z-march over 1-halo planes (kl_plane_tma.cuh) for diff_c and
    evisc_smag: sampled TMA configurations plus fixed tiles, ragged grids."""
    from paper_2303_12374_b200.stencils.definitions import family_space
    from paper_2303_12374_b200.stencils.layout import GridLayout

    space = _space(kernel, precision)
    base = space.default_config()[0]
    cfgs = family_space(kernel, "TMA", precision).sample_random(19, 3)
    cfgs += [dict(base, staging="TMA", block_x=32, block_y=4, tile_x=1, tile_y=2, depth=2, zchunk=16),
             dict(base, staging="TMA", contiguous_x=True, block_x=16, block_y=2, tile_x=4, tile_y=3, depth=1,
                  zchunk=8, unravel="XYZ"),
             dict(base, staging="TMA", contiguous_x=True, block_x=32, block_y=2, tile_x=4, tile_y=4, depth=2,
                  zchunk=16, unravel="XYZ"),
             dict(base, staging="TMA", contiguous_x=True, block_x=64, block_y=1, tile_x=2, tile_y=1, depth=3,
                  zchunk=32, unravel="XYZ")]
    for grid in ((45, 23, 19), (130, 37, 41)):
        lay = GridLayout(*grid, precision)
        ref, _ = oracle_outputs(kernel, lay)
        for cfg in cfgs:
            assert space.is_valid(cfg), cfg
            got = run_config(gpu_ctx, compiler, kernel, lay, cfg)
            for name in ref:
                err = rel_error(got[name], ref[name], lay)
                assert err <= TOL[precision], (grid, cfg, name, err)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_evisc_tma_shared_x_edges_match_oracle(gpu_ctx, compiler, precision):
    """evisc_smag TMA with ``xshare``: 31 output columns per warp, lane 31 a
    helper whose west-face edges are its neighbours' east-face edges (warp
    shuffles) — block widths 32..128 on ragged grids (partial warps and
    blocks along x), a k sub-range, and the scalar store path."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    space = _space("evisc_smag", precision)
    base = space.default_config()[0]
    cases = [dict(block_x=32, block_y=4, tile_y=2, depth=2, zchunk=16),
             dict(block_x=64, block_y=2, tile_y=4, depth=1, zchunk=8, unravel="XYZ"),
             dict(block_x=128, block_y=2, tile_y=4, depth=2, zchunk=32, unravel="XYZ")]
    for grid, k_range in (((45, 23, 19), None), ((130, 37, 41), None), ((200, 30, 24), (6, 21))):
        lay = GridLayout(*grid, precision)
        ref, _ = oracle_outputs("evisc_smag", lay, k_range=k_range)
        for case in cases:
            cfg = dict(base, staging="TMA", tile_x=1, xshare=1, **case)
            assert space.is_valid(cfg), case
            got = run_config(gpu_ctx, compiler, "evisc_smag", lay, cfg, k_range=k_range)
            err = rel_error(got["evisc"], ref["evisc"], lay)
            assert err <= TOL[precision], (grid, case, err)
