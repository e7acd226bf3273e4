"""Stencil definitions on the reference API; NVRTC compiles sampled
configurations of every kernel/precision for sm_100a (no GPU needed)."""

import pytest

from paper_2303_12374_b200.backend import DeviceIdent
from paper_2303_12374_b200.capture import scalar_env_from_args, ScalarArg
from paper_2303_12374_b200.stencils.definitions import ARG_LAYOUT, FAMILY_PINS, KERNELS, PRECISIONS, definition_for
from paper_2303_12374_b200.stencils.layout import GridLayout

B200 = DeviceIdent("NVIDIA B200", "Blackwell", {"compute_capability": "10.0"})


def scalars(kernel, lay):
    nb = len(ARG_LAYOUT[kernel]["buffers"])
    vals = dict(dxi=1.0, dyi=1.0, jj=lay.jj, kk=lay.kk, istart=lay.istart, jstart=lay.jstart, kstart=lay.kstart,
                iend=lay.iend, jend=lay.jend, kend=lay.kend)
    out = []
    vals.update(tpri=3.0, cs=0.23)
    for i, n in enumerate(ARG_LAYOUT[kernel]["scalars"]):
        out.append(ScalarArg(nb + i, "f32" if n in ("dxi", "dyi", "tpri", "cs") else "i32", vals[n]))
    return out


def test_layout_alignment():
    for prec, align in (("fp32", 32), ("fp64", 16)):
        lay = GridLayout(1024, 1024, 128, prec)
        assert lay.jj % align == 0 and (lay.lead + lay.istart) % align == 0
        assert lay.jj >= lay.icells and lay.kk == lay.jj * lay.jcells


@pytest.mark.parametrize("kernel", KERNELS)
def test_default_config_is_the_paper_default(kernel):
    d = definition_for(kernel, "fp32")
    cfg, ok = d.space.default_config()
    assert ok and cfg["block_x"] == 256 and cfg["staging"] == "DIRECT" and cfg["zchunk"] == 1
    lay = GridLayout(256, 256, 256, "fp32")
    env = scalar_env_from_args(scalars(kernel, lay))
    problem = d.derive_problem_size(env)
    assert problem == (256, 256, 256)
    geom = d.derive_geometry(cfg, problem, env)
    assert geom.block == (256, 1, 1) and geom.grid == (256 * 256, 1, 1) and geom.shared_mem_bytes == 0


def test_precision_is_in_the_kernel_key():
    keys = {definition_for(k, p).kernel_key() for k in KERNELS for p in PRECISIONS}
    assert len(keys) == 4


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("precision", list(PRECISIONS))
def test_nvrtc_compiles_sampled_configs(kernel, precision):
    from paper_2303_12374_b200.cuda._abi import library_path
    from paper_2303_12374_b200.cuda.compiler import NvrtcCompiler

    if not library_path().exists():
        pytest.skip("libklb200.so not built")
    d = definition_for(kernel, precision)
    lay = GridLayout(40, 24, 16, precision)
    env = scalar_env_from_args(scalars(kernel, lay))
    problem = d.derive_problem_size(env)
    comp = NvrtcCompiler()
    cfgs = d.space.sample_random(3, 3) + [c for c in d.space.sample_random(4, 300) if c["staging"] == "ZMARCH"][:2]
    for staging, bx in (("ZMARCH", 16), ("TMA", 16), ("TMA", 64)):
        cfg = d.space.default_config()[0]
        cfg.update(FAMILY_PINS[staging], tile_x=1, contiguous_x=False, contiguous_y=False, block_x=bx, block_y=4,
                   zchunk=16, depth=1 if staging == "TMA" else 0)
        assert d.space.is_valid(cfg), cfg
        cfgs.append(cfg)
    futures = comp.compile_many([d.render_compile_request(c, problem, env) for c in cfgs], B200)
    for fut in futures:
        img = fut.result()
        assert img.lowered_name == f"{kernel}_{precision}" and len(img.cubin) > 1000


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("precision", list(PRECISIONS))
def test_tma_shared_memory_fits_the_optin_limit(kernel, precision):
    """Every TMA point of the (precision-specific) space launches within the
    B200 opt-in shared-memory limit, and the restriction admits large tiles
    (the ring is bounded by bytes, not by a fixed cell count)."""
    from paper_2303_12374_b200.stencils.definitions import SMEM_OPTIN_BYTES, family_space

    d = definition_for(kernel, precision)
    lay = GridLayout(512, 512, 512, precision)
    env = scalar_env_from_args(scalars(kernel, lay))
    problem = d.derive_problem_size(env)
    cfgs = family_space(kernel, "TMA", precision).sample_random(5, 400)
    assert cfgs
    biggest = 0
    for c in cfgs:
        assert d.space.is_valid(c)
        smem = d.derive_geometry(c, problem, env).shared_mem_bytes
        assert 0 < smem <= SMEM_OPTIN_BYTES, c
        biggest = max(biggest, smem)
    assert biggest > 96 * 1024
    assert any(c["tile_x"] > 1 for c in cfgs)


def test_space_fingerprints_differ_by_precision_only_where_limits_do():
    keys = {(k, p): definition_for(k, p).space.fingerprint() for k in KERNELS for p in PRECISIONS}
    assert keys["diff_uvw", "fp32"] != keys["diff_uvw", "fp64"]
    assert keys["advec_u", "fp32"] != keys["advec_u", "fp64"]


@pytest.mark.parametrize("kernel", KERNELS)
def test_nvrtc_compiles_column_tiles(kernel):
    """TMA column tiles (tile_x consecutive columns; the fp32 advec_u ones use
    packed FFMA2/FADD2 arithmetic) compile for sm_100a in both precisions."""
    from paper_2303_12374_b200.cuda._abi import library_path
    from paper_2303_12374_b200.cuda.compiler import NvrtcCompiler

    if not library_path().exists():
        pytest.skip("libklb200.so not built")
    comp = NvrtcCompiler()
    for precision in PRECISIONS:
        d = definition_for(kernel, precision)
        lay = GridLayout(64, 24, 16, precision)
        env = scalar_env_from_args(scalars(kernel, lay))
        problem = d.derive_problem_size(env)
        reqs = []
        for tx, bx in ((2, 32), (4, 16)):
            cfg = d.space.default_config()[0]
            cfg.update(FAMILY_PINS["TMA"], tile_x=tx, contiguous_x=True, contiguous_y=False, block_x=bx, block_y=4,
                       tile_y=2, zchunk=16, depth=1)
            assert d.space.is_valid(cfg), cfg
            reqs.append(d.render_compile_request(cfg, problem, env))
        for fut in comp.compile_many(reqs, B200):
            assert len(fut.result().cubin) > 1000


@pytest.mark.parametrize("kernel", ["advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag"])
def test_family_kernels_compile_and_key_by_precision(kernel):
    """The §8f family: Table-2 DIRECT space, precision in the kernel key,
    NVRTC compiles sampled configurations for sm_100a."""
    from paper_2303_12374_b200.cuda._abi import library_path
    from paper_2303_12374_b200.cuda.compiler import NvrtcCompiler

    keys = {definition_for(kernel, p).kernel_key() for p in PRECISIONS}
    assert len(keys) == 2
    if not library_path().exists():
        pytest.skip("libklb200.so not built")
    comp = NvrtcCompiler()
    reqs = []
    for precision in PRECISIONS:
        d = definition_for(kernel, precision)
        assert d.space.default_config()[0]["staging"] == "DIRECT"
        lay = GridLayout(40, 24, 16, precision)
        env = scalar_env_from_args(scalars(kernel, lay))
        problem = d.derive_problem_size(env)
        assert problem == (40, 24, 16)
        for cfg in [d.space.default_config()[0]] + d.space.sample_random(2, 2):
            reqs.append(d.render_compile_request(cfg, problem, env))
    for fut in comp.compile_many(reqs, B200):
        assert fut.result().lowered_name.startswith(kernel)


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw", "diff_uvw_rk3", "advec_v", "advec_w", "advec_s", "diff_c",
                                    "evisc_smag", "rk3_uvw"])
def test_capture_metadata_with_embedded_source_fits_the_format_cap(kernel):
    """A capture embeds the definition with its source; the .klcap metadata
    block is capped at 64 KiB (reference capture.py:37), so the assembled
    NVRTC sources are comment-stripped."""
    from paper_2303_12374_b200.capture import ScalarArg, metadata_block

    for precision in PRECISIONS:
        d = definition_for(kernel, precision)
        descs = [(i, "input", "f32", 1, 4, 0) for i in range(14)]
        blob = metadata_block(d, (1024, 1024, 1024), [ScalarArg(20, "i32", 1)] * 12, descs, "app", "t")
        assert len(blob) < 60 * 1024, len(blob)


def test_advec_u_ysplit_sizes_the_grid_to_whole_waves():
    """advec_u's ``ysplit`` knob (TMA only): the grid holds ~ysplit blocks per
    SM of the B200 (148), never fewer row runs than ceil(jtot / rows per
    block) (the kernel traps otherwise), and 0 keeps the natural tiling."""
    from paper_2303_12374_b200.stencils.definitions import B200_SMS, definition_for
    from paper_2303_12374_b200.stencils.layout import GridLayout

    d = definition_for("advec_u", "fp32")
    lay = GridLayout(256, 256, 256, "fp32")
    env = {"arg9": lay.jj, "arg10": lay.kk}
    base = dict(d.space.default_config()[0], staging="TMA", block_x=32, block_y=8, tile_x=4, tile_y=1,
                contiguous_x=True, zchunk=64, depth=2)
    grids = {}
    for ys in (0, 1, 2):
        cfg = dict(base, ysplit=ys)
        assert d.space.is_valid(cfg), ys
        grids[ys] = d.derive_geometry(cfg, (256, 256, 256), env).grid[0]
        req = d.render_compile_request(cfg, (256, 256, 256), env)
        assert f"-D KL_YBAL={ys}" in req.defines
    nbxz = 2 * 4
    assert grids[0] == nbxz * 32                      # 256 rows / 8 per block
    assert grids[1] == nbxz * 32                      # 148 / 8 = 18 runs < 32 needed: natural count kept
    assert grids[2] == nbxz * (2 * B200_SMS // nbxz) == 296  # 37 runs of <= 7 rows, 2 blocks per SM
    assert not d.space.is_valid(dict(d.space.default_config()[0], ysplit=1))  # DIRECT: pinned to 0


def test_advec_u_ysplit_never_makes_empty_row_runs():
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.stencils.layout import GridLayout

    d = definition_for("advec_u", "fp32")
    lay = GridLayout(45, 23, 19, "fp32")
    env = {"arg9": lay.jj, "arg10": lay.kk}
    cfg = dict(d.space.default_config()[0], staging="TMA", block_x=32, block_y=4, tile_x=2, tile_y=2,
               contiguous_x=True, zchunk=8, depth=2, ysplit=2)
    g = d.derive_geometry(cfg, (45, 23, 19), env).grid[0]
    assert g == 1 * 3 * 23  # nbx * nbz * min(jtot, 296 / 3): one row per run, none empty


def test_evisc_xshare_grid_counts_31_columns_per_warp():
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.stencils.layout import GridLayout

    d = definition_for("evisc_smag", "fp32")
    lay = GridLayout(512, 512, 512, "fp32")
    env = {"arg9": lay.jj, "arg10": lay.kk}
    cfg = dict(d.space.default_config()[0], staging="TMA", block_x=128, block_y=2, tile_x=1, tile_y=4, zchunk=64,
               depth=2)
    g0 = d.derive_geometry(dict(cfg, xshare=0), (512, 512, 512), env).grid[0]
    g1 = d.derive_geometry(dict(cfg, xshare=1), (512, 512, 512), env).grid[0]
    assert g0 == 4 * 64 * 8 and g1 == 5 * 64 * 8  # ceil(512 / 124) = 5 blocks along x
    assert "-D KL_XSHARE=1" in d.render_compile_request(dict(cfg, xshare=1), (512, 512, 512), env).defines
    assert not d.space.is_valid(dict(cfg, xshare=1, tile_x=2, contiguous_x=True))


@pytest.mark.parametrize("fused,base", [("diff_uvw_peer", "diff_uvw"), ("advec_u_peer", "advec_u"),
                                        ("diff_uvw_rk3", "diff_uvw")])
@pytest.mark.parametrize("precision", PRECISIONS)
def test_fused_variants_share_their_base_kernel_space_and_launch(fused, base, precision):
    """A fused variant selects from its base kernel's wisdom (slab.SlabDriver,
    build()): same space fingerprint, and for the same configuration and
    problem the same grid, block, shared memory and tunable defines."""
    from paper_2303_12374_b200.stencils.layout import GridLayout

    fd, bd = definition_for(fused, precision), definition_for(base, precision)
    assert fd.space.fingerprint() == bd.space.fingerprint()
    lay = GridLayout(256, 192, 128, precision)
    vals = dict(dxi=1.0, dyi=1.0, rk_a=0.5, rk_bdt=0.01, jj=lay.jj, kk=lay.kk, istart=lay.istart,
                jstart=lay.jstart, kstart=lay.kstart, iend=lay.iend, jend=lay.jend, kend=lay.kend,
                peer_klo=lay.kstart, peer_khi=lay.kend, peer_shift_lo=5, peer_shift_hi=-5)

    def env(k):
        nb = len(ARG_LAYOUT[k]["buffers"])
        return {f"arg{nb + i}": vals[n] for i, n in enumerate(ARG_LAYOUT[k]["scalars"])}

    extra = {"ysplit": 2} if "ysplit" in bd.space.param_names else {}
    cands = [dict(bd.space.default_config()[0], staging="TMA", zchunk=z, depth=1, block_x=32, block_y=4,
                  tile_x=tx, tile_y=2, contiguous_x=True, **extra) for tx, z in ((4, 64), (2, 32))]
    cfg = next(c for c in cands if bd.space.is_valid(c))
    pf, pb = fd.derive_problem_size(env(fused)), bd.derive_problem_size(env(base))
    assert pf == pb
    gf, gb = fd.derive_geometry(cfg, pf, env(fused)), bd.derive_geometry(cfg, pb, env(base))
    assert (gf.grid, gf.block, gf.shared_mem_bytes) == (gb.grid, gb.block, gb.shared_mem_bytes)
    df = set(fd.render_compile_request(cfg, pf, env(fused)).defines)
    db = set(bd.render_compile_request(cfg, pb, env(base)).defines)
    assert df == db
