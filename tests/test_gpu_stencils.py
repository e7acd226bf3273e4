"""GPU parity: NVRTC-compiled stencils vs the NumPy oracle (tests/stencil_helpers.py).

Bar (BASELINE.json north_star): max|gpu - ref| / max|ref| <= 1e-5 (fp32),
<= 1e-12 (fp64) per output array, ref computed in float64 from the same inputs.
"""

import numpy as np
import pytest

from stencil_helpers import TOL, host_fields, oracle_outputs, rel_error, run_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def compiler(gpu_ctx):
    from paper_2303_12374_b200.cuda import NvrtcCompiler

    return NvrtcCompiler(gpu_ctx)


def _default(kernel, precision):
    from paper_2303_12374_b200.stencils.definitions import definition_for

    return definition_for(kernel, precision).space.default_config()[0]


def test_device_synth_is_bit_exact(gpu_ctx):
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    for precision in ("fp32", "fp64"):
        lay = GridLayout(37, 29, 11, precision)
        prob = StencilProblem("diff_uvw", lay, gpu_ctx)
        try:
            want = host_fields(lay, prob.fields)
            for name in prob.fields:
                got = prob.download(name)
                assert np.array_equal(got, want[name]), (precision, name)
        finally:
            prob.close()


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_default_config_matches_oracle(gpu_ctx, compiler, kernel, precision):
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(64, 64, 64, precision) if kernel == "diff_uvw" else GridLayout(48, 40, 24, precision)
    got = run_config(gpu_ctx, compiler, kernel, lay, _default(kernel, precision))
    ref, _ = oracle_outputs(kernel, lay)
    for name in ref:
        err = rel_error(got[name], ref[name], lay)
        assert err <= TOL[precision], (name, err)


def _sample_configs(kernel, precision, n, seed):
    """n configurations per staging family (DIRECT / ZMARCH / TMA)."""
    from paper_2303_12374_b200.stencils.definitions import FAMILY_PINS, definition_for, family_space

    space = definition_for(kernel, precision).space
    cfgs = []
    for fam in FAMILY_PINS:
        for c in family_space(kernel, fam, precision).sample_random(seed, n):
            assert space.is_valid(c)
            cfgs.append(c)
    return cfgs


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_sampled_configs_match_oracle(gpu_ctx, compiler, kernel, precision):
    """Random Table-2 + B200 configurations on a ragged grid (extents not multiples of any tile)."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(45, 23, 19, precision)
    ref, _ = oracle_outputs(kernel, lay)
    for cfg in _sample_configs(kernel, precision, 3, seed=7 if precision == "fp32" else 11):
        got = run_config(gpu_ctx, compiler, kernel, lay, cfg)
        for name in ref:
            err = rel_error(got[name], ref[name], lay)
            assert err <= TOL[precision], (cfg, name, err)


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
def test_k_subrange_launch(gpu_ctx, compiler, kernel):
    """Launching a k sub-range (the multi-GPU interior/boundary split) only touches those planes."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(32, 24, 20, "fp64")
    kr = (lay.kstart + 4, lay.kstart + 13)
    ref, _ = oracle_outputs(kernel, lay, k_range=kr)
    for cfg in (_default(kernel, "fp64"), dict(_default(kernel, "fp64"), staging="ZMARCH", zchunk=8, block_x=32, block_y=4),
                dict(_default(kernel, "fp64"), staging="TMA", zchunk=8, block_x=32, block_y=4, depth=2)):
        got = run_config(gpu_ctx, compiler, kernel, lay, cfg, k_range=kr)
        for name in ref:
            diff = np.max(np.abs(got[name].astype(np.float64) - ref[name]))
            assert diff <= 1e-12 * np.max(np.abs(ref[name])), (cfg["staging"], name, diff)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_tma_configs_rejected_by_an_earlier_tuner_run(gpu_ctx, compiler, precision):
    """Regression: advec_u TMA configurations the replay verifier once flagged."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    base = _default("advec_u", precision)
    cases = [dict(block_x=32, block_y=1, tile_y=1, depth=1, zchunk=8, min_blocks=2),
             dict(block_x=32, block_y=4, tile_y=1, depth=3, zchunk=64, min_blocks=2),
             dict(block_x=64, block_y=2, tile_y=1, depth=3, zchunk=8, min_blocks=3),
             dict(block_x=32, block_y=2, tile_y=2, depth=2, zchunk=32, min_blocks=5)]
    lay = GridLayout(96, 40, 70, precision)
    ref, _ = oracle_outputs("advec_u", lay)
    for case in cases:
        cfg = dict(base, staging="TMA", **case)
        got = run_config(gpu_ctx, compiler, "advec_u", lay, cfg)
        err = rel_error(got["ut"], ref["ut"], lay)
        assert err <= TOL[precision], (case, err)


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
def test_tma_repeated_launches_are_stable(gpu_ctx, compiler, kernel):
    """Intermittent-race guard: the same TMA configuration, launched repeatedly on
    a grid with many z-chunks, must reproduce the oracle every time (an earlier
    advec_u TMA build read the w plane of a chunk's first steps before its
    mbarrier completed — caught by the tuner's replay verification)."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    lay = GridLayout(256, 64, 96, "fp32")
    ref, _ = oracle_outputs(kernel, lay)
    cfg = dict(_default(kernel, "fp32"), staging="TMA", block_x=128, block_y=1, tile_y=1, depth=2, zchunk=8)
    for _ in range(4):
        got = run_config(gpu_ctx, compiler, kernel, lay, cfg)
        for name in ref:
            assert rel_error(got[name], ref[name], lay) <= TOL["fp32"], name


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_advec_tma_column_tiles_match_oracle(gpu_ctx, compiler, precision):
    """advec_u TMA with tile_x consecutive columns per thread (vectorised
    shared-memory reads / ut stores), on grids whose x extent leaves partial
    thread tiles and partial blocks."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    from paper_2303_12374_b200.stencils.definitions import definition_for

    space = definition_for("advec_u", precision).space
    base = _default("advec_u", precision)
    cases = [dict(block_x=32, block_y=4, tile_x=2, tile_y=2, depth=2, zchunk=16),
             dict(block_x=16, block_y=8, tile_x=4, tile_y=1, depth=1, zchunk=8),
             dict(block_x=16, block_y=2, tile_x=4, tile_y=3, depth=3, zchunk=64),
             dict(block_x=64, block_y=1, tile_x=2, tile_y=4, depth=1, zchunk=32)]
    for grid in ((45, 23, 19), (130, 37, 41)):
        lay = GridLayout(*grid, precision)
        ref, _ = oracle_outputs("advec_u", lay)
        for case in cases:
            cfg = dict(base, staging="TMA", contiguous_x=True, **case)
            assert space.is_valid(cfg), case
            got = run_config(gpu_ctx, compiler, "advec_u", lay, cfg)
            err = rel_error(got["ut"], ref["ut"], lay)
            assert err <= TOL[precision], (grid, case, err)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_advec_tma_balanced_row_runs_match_oracle(gpu_ctx, compiler, precision):
    """advec_u TMA with ``ysplit`` > 0: the y extent cut into near-equal row
    runs (grid sized to whole waves, definitions.YSPLIT_VALUES) — runs shorter
    than the block's rows, strips past a run's end idle — on ragged grids and
    on a k sub-range (the planes outside it untouched)."""
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.stencils.layout import GridLayout

    space = definition_for("advec_u", precision).space
    base = _default("advec_u", precision)
    cases = [dict(block_x=32, block_y=4, tile_x=2, tile_y=2, depth=2, zchunk=16, ysplit=1),
             dict(block_x=16, block_y=4, tile_x=4, tile_y=2, depth=2, zchunk=8, ysplit=2),
             dict(block_x=32, block_y=8, tile_x=4, tile_y=1, depth=1, zchunk=32, ysplit=2)]
    for grid, k_range in (((45, 23, 19), None), ((130, 37, 41), None), ((96, 61, 30), (5, 27))):
        lay = GridLayout(*grid, precision)
        ref, _ = oracle_outputs("advec_u", lay, k_range=k_range)
        for case in cases:
            cfg = dict(base, staging="TMA", contiguous_x=True, **case)
            assert space.is_valid(cfg), case
            got = run_config(gpu_ctx, compiler, "advec_u", lay, cfg, k_range=k_range)
            err = rel_error(got["ut"], ref["ut"], lay)
            assert err <= TOL[precision], (grid, case, err)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_diff_tma_column_tiles_match_oracle(gpu_ctx, compiler, precision):
    """diff_uvw TMA with tile_x consecutive columns per thread (x-face reuse,
    vectorised shared-memory reads and tendency stores), on grids whose x/y
    extents leave partial thread tiles and partial blocks."""
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.stencils.layout import GridLayout

    space = definition_for("diff_uvw", precision).space
    base = _default("diff_uvw", precision)
    cases = [dict(block_x=32, block_y=4, tile_x=2, tile_y=2, depth=2, zchunk=16, contiguous_x=True),
             dict(block_x=16, block_y=8, tile_x=4, tile_y=1, depth=1, zchunk=8, contiguous_x=True),
             dict(block_x=16, block_y=2, tile_x=4, tile_y=4, depth=3, zchunk=64, contiguous_x=True),
             dict(block_x=64, block_y=2, tile_x=1, tile_y=4, depth=1, zchunk=32, unravel="XYZ"),
             dict(block_x=128, block_y=2, tile_x=1, tile_y=4, depth=1, zchunk=64, unravel="XYZ")]
    for grid in ((45, 23, 19), (130, 37, 41)):
        lay = GridLayout(*grid, precision)
        ref, _ = oracle_outputs("diff_uvw", lay)
        for case in cases:
            cfg = dict(base, staging="TMA", **case)
            assert space.is_valid(cfg), case
            got = run_config(gpu_ctx, compiler, "diff_uvw", lay, cfg)
            for name in ref:
                err = rel_error(got[name], ref[name], lay)
                assert err <= TOL[precision], (grid, case, name, err)


_MISALIGNED_CFG = {
    "advec_u": dict(staging="TMA", contiguous_x=True, block_x=32, block_y=4, tile_x=2, tile_y=2, depth=2, zchunk=8),
    "diff_uvw": dict(staging="TMA", contiguous_x=True, block_x=16, block_y=4, tile_x=4, tile_y=2, depth=2, zchunk=8),
}


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_tma_misaligned_fields_use_scalar_path(gpu_ctx, compiler, kernel, precision):
    """Fields whose interior rows are NOT 16-byte aligned (pointers shifted by
    one element, as a replayed capture or a foreign allocation may be): the
    kernel's uniform fallback to scalar shared-memory access must give the
    same result as the aligned, vectorised path."""
    from paper_2303_12374_b200.capture import scalar_env_from_args
    from paper_2303_12374_b200.cuda import DeviceArray, DeviceBuffer
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(70, 29, 23, precision)
    ref, _ = oracle_outputs(kernel, lay)
    cfg = dict(_default(kernel, precision), **_MISALIGNED_CFG[kernel])
    prob = StencilProblem(kernel, lay, gpu_ctx)
    shifted = {}
    try:
        args = []
        for a in prob.args():
            if isinstance(a, DeviceBuffer) and a.element_count == lay.span_elems:
                arr = DeviceArray(lay.alloc_bytes + 64)
                dst = arr.ptr + lay.elem_bytes  # one element off the 16-byte grid
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
        assert args[0].ptr % 16 != (prob.field_ptr("ut") % 16)
        for pos, name in enumerate(prob.outputs()):
            flat = np.frombuffer(shifted[pos].download(lay.alloc_bytes, offset_bytes=lay.elem_bytes), dtype=lay.dtype)
            err = rel_error(lay.host_view(flat), ref[name], lay)
            assert err <= TOL[precision], (name, err)
    finally:
        for arr in shifted.values():
            arr.free()
        prob.close()
