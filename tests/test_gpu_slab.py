"""Multi-GPU z-slab path on ONE GPU: virtual ranks exchange halos with D2D
copies (CopyExchanger, the same plan klb_halo_exchange_z runs over NCCL) and
launch their interior/boundary sub-ranges through WisdomKernel; the result
must equal the undecomposed grid's (same compiled configuration everywhere, so
to the last bits)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _poison_ghosts(driver):
    """NaN-fill the ghost planes the exchange is responsible for."""
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.halo import HALO_REACH

    lay = driver.layout
    plane = lay.kk * lay.elem_bytes
    for name, (down, up) in HALO_REACH[driver.kernel].items():
        base = driver.problem.field_ptr(name)
        if driver.below >= 0 and up:
            check(lib().klb_memset_d8(base + (lay.kstart - up) * plane, 0xFF, up * plane, None))
        if driver.above >= 0 and down:
            check(lib().klb_memset_d8(base + lay.kend * plane, 0xFF, down * plane, None))
    driver.ctx.synchronize()


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
@pytest.mark.parametrize("staging", ["DIRECT", "TMA"])
def test_virtual_ranks_match_single_grid(gpu_ctx, tmp_path, kernel, staging):
    from paper_2303_12374_b200.cuda import NvrtcCompiler
    from paper_2303_12374_b200.halo import HALO_REACH, CopyExchanger
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.wisdom import WisdomFile, WisdomRecord

    grid, nranks, precision = (64, 48, 30), 3, "fp64"
    d = definition_for(kernel, precision)
    cfg = d.space.default_config()[0]
    if staging == "TMA":
        cfg.update(staging="TMA", zchunk=8, block_x=32, block_y=4, depth=2)
    assert d.space.is_valid(cfg)
    # pin the configuration for every problem size via wisdom (selection -> same_device_nearest)
    WisdomFile(d.kernel_key(), records=[WisdomRecord(gpu_ctx.ident, (1, 1, 1), cfg, 1.0)]).save(
        tmp_path / f"{d.kernel_key()}.wisdom")
    comp = NvrtcCompiler(gpu_ctx)

    whole = SlabDriver(kernel, precision, grid, gpu_ctx, compiler=comp, wisdom_dir=tmp_path)
    whole.step()
    gpu_ctx.synchronize()
    ref = {n: whole.problem.download(n).copy() for n in whole.problem.outputs()}
    whole.close()

    ranks = [SlabDriver(kernel, precision, grid, gpu_ctx, rank=r, nranks=nranks, compiler=comp, wisdom_dir=tmp_path)
             for r in range(nranks)]
    for drv in ranks:
        _poison_ghosts(drv)
    ex = CopyExchanger([{n: drv.problem.field_ptr(n) for n in HALO_REACH[kernel]} for drv in ranks])
    lay = ranks[0].layout
    ex.exchange_all(ranks[0].compute, HALO_REACH[kernel], lay.elem_bytes, lay.kk,
                    [(drv.layout.kstart, drv.layout.kend) for drv in ranks])
    gpu_ctx.synchronize()
    for drv in ranks:
        assert set(drv.ranges) <= {"interior", "lower", "upper"}
        if staging == "TMA":
            # resolve() pre-compiles every sub-range and switches step() to
            # bound launches (one C-ABI call each)
            drv.resolve()
            assert set(drv._bound) == set(drv.ranges)
        drv.step()
    gpu_ctx.synchronize()
    g = lay.kgc
    for drv in ranks:
        off, count = drv.slab.offset, drv.slab.count
        for name in ref:
            got = drv.problem.download(name)[g:g + count]
            want = ref[name][g + off:g + off + count]
            # same configuration everywhere -> identical per-cell arithmetic; allow last-bit
            # differences where a carried face is evaluated in the prologue instead of the
            # loop body (FMA contraction may differ between the two)
            err = np.max(np.abs(got - want)) / np.max(np.abs(want))
            assert err <= 1e-13, (drv.rank, name, err)
        assert drv.wisdom.reports and all(r.configuration == cfg for r in drv.wisdom.reports)
        drv.close()


@pytest.mark.parametrize("kernel,precision", [("diff_uvw", "fp32"), ("diff_uvw", "fp64"), ("advec_u", "fp32"),
                                              ("advec_u", "fp64")])
def test_fused_peer_halo_virtual_ranks_match_single_grid(gpu_ctx, tmp_path, kernel, precision):
    """halo="fused": every virtual rank launches diff_uvw_peer / advec_u_peer
    ONCE over its whole slab; the planes outside the slab come from the neighbours' fields
    (LocalPeers: other allocations on this device), so the ghost planes are
    poisoned and never exchanged — and the tendencies equal the undecomposed
    grid's, for equal slabs (30 planes: 10/10/10) and unequal ones (31:
    11/10/10, so a neighbour's allocation has another plane count)."""
    from paper_2303_12374_b200.cuda import NvrtcCompiler
    from paper_2303_12374_b200.halo import LocalPeers
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.wisdom import WisdomFile, WisdomRecord

    from paper_2303_12374_b200.stencils.problem import PEER_KERNELS

    comp = NvrtcCompiler(gpu_ctx)
    d = definition_for(kernel, precision)
    cfg = dict(d.space.default_config()[0], staging="TMA", zchunk=8, block_x=32, block_y=4, depth=2)
    if kernel == "advec_u":  # column pairs: the packed fp32 main loop
        cfg.update(tile_x=2, contiguous_x=True, block_x=16)
    assert d.space.is_valid(cfg), cfg
    WisdomFile(d.kernel_key(), records=[WisdomRecord(gpu_ctx.ident, (1, 1, 1), cfg, 1.0)]).save(
        tmp_path / f"{d.kernel_key()}.wisdom")
    fields = PEER_KERNELS[f"{kernel}_peer"]
    for grid in ((64, 48, 30), (48, 40, 31)):
        whole = SlabDriver(kernel, precision, grid, gpu_ctx, compiler=comp, wisdom_dir=tmp_path)
        whole.step()
        gpu_ctx.synchronize()
        ref = {n: whole.problem.download(n).copy() for n in whole.problem.outputs()}
        whole.close()
        nranks = 3
        drivers = []
        peers = LocalPeers([])
        for r in range(nranks):
            drv = SlabDriver(kernel, precision, grid, gpu_ctx, rank=r, nranks=nranks, compiler=comp,
                             wisdom_dir=tmp_path, halo="fused", exchanger=peers.for_rank(r))
            drivers.append(drv)
        peers.ranks = [({n: drv.problem.field_ptr(n) for n in fields}, drv.layout.kstart, drv.layout.kend)
                       for drv in drivers]
        for drv in drivers:
            _poison_ghosts(drv)
        for drv in drivers:
            drv.resolve()
            assert set(drv.ranges) == {"slab"} and set(drv._bound) == {"slab"}
            assert drv.step() == 1
        gpu_ctx.synchronize()
        g = drivers[0].layout.kgc
        for drv in drivers:
            off, count = drv.slab.offset, drv.slab.count
            for name in ref:
                got = drv.problem.download(name)[g:g + count]
                want = ref[name][g + off:g + off + count]
                err = np.max(np.abs(got - want)) / np.max(np.abs(want))
                assert err <= 1e-13 if precision == "fp64" else err <= 1e-6, (grid, drv.rank, name, err)
            rep = drv.wisdom.reports[0]
            assert rep.configuration == cfg and rep.problem == (grid[0], grid[1], count)
        for drv in drivers:
            drv.close()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_rk3_time_loop_fused_halo_virtual_ranks_match_oracle(gpu_ctx, tmp_path, precision):
    """Four substeps of the low-storage RK3 time loop (SlabDriver.rk3_substep:
    diff_uvw_rk3 into the alternate buffers + periodic x/y ghost fill) on one
    undecomposed grid and on 3 virtual ranks whose launches read the
    neighbours' CURRENT buffers (diff_uvw_rk3_peer; u/v/w and u_next/v_next/
    w_next alternate, so the peer arguments alternate too) — every rank's
    tendencies and velocities equal the oracle's time loop."""
    from paper_2303_12374_b200.cuda import NvrtcCompiler
    from paper_2303_12374_b200.halo import LocalPeers
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.wisdom import WisdomFile, WisdomRecord
    from stencil_helpers import oracle_rk3_loop

    comp = NvrtcCompiler(gpu_ctx)
    d = definition_for("diff_uvw_rk3", precision)
    cfg = dict(d.space.default_config()[0], staging="TMA", zchunk=8, block_x=32, block_y=4, depth=2)
    WisdomFile(d.kernel_key(), records=[WisdomRecord(gpu_ctx.ident, (1, 1, 1), cfg, 1.0)]).save(
        tmp_path / f"{d.kernel_key()}.wisdom")
    grid, nsub, dt = (48, 40, 31), 4, 0.05
    lay = GridLayout(*grid, precision)
    want_t, want_u = oracle_rk3_loop(lay, nsub, dt)
    tol = 1e-5 if precision == "fp32" else 1e-12
    g = lay.kgc
    cur = ("u", "v", "w") if nsub % 2 == 0 else ("u_next", "v_next", "w_next")

    def check(drv, off, count, what):
        for name, ref in list(want_t.items()) + [(c, want_u[n]) for c, n in zip(cur, ("u", "v", "w"))]:
            got = drv.problem.download(name)[g:g + count, g:-g, g:g + grid[0]].astype(np.float64)
            r = ref[g + off:g + off + count, g:-g, g:g + grid[0]]
            err = np.max(np.abs(got - r)) / np.max(np.abs(ref[g:-g, g:-g, g:g + grid[0]]))
            assert err <= tol, (what, name, err)

    whole = SlabDriver("diff_uvw_rk3", precision, grid, gpu_ctx, compiler=comp, wisdom_dir=tmp_path)
    for s in range(nsub):
        assert whole.rk3_substep(s, dt) == 2
    gpu_ctx.synchronize()
    check(whole, 0, grid[2], "whole grid")
    whole.close()

    nranks = 3
    peers = LocalPeers([])
    drivers = [SlabDriver("diff_uvw_rk3", precision, grid, gpu_ctx, rank=r, nranks=nranks, compiler=comp,
                          wisdom_dir=tmp_path, halo="fused", exchanger=peers.for_rank(r)) for r in range(nranks)]
    peers.ranks = [({n: drv.problem.field_ptr(n) for n in drv.problem.fields}, drv.layout.kstart, drv.layout.kend)
                   for drv in drivers]
    for drv in drivers:
        _poison_ghosts(drv)
    for s in range(nsub):  # one stream: rank r's substep s after every rank's substep s-1
        for drv in drivers:
            drv.rk3_substep(s, dt)
    gpu_ctx.synchronize()
    for drv in drivers:
        check(drv, drv.slab.offset, drv.slab.count, f"rank {drv.rank}")
        assert all(r.configuration == cfg for r in drv.wisdom.reports)
        drv.close()


def test_nccl_single_rank_exchange_is_a_noop(gpu_ctx):
    """The NCCL path end to end on one GPU: unique id, comm init, grouped
    send/recv call with no neighbours (the only topology one GPU allows)."""
    from paper_2303_12374_b200.cuda._abi import lib
    from paper_2303_12374_b200.halo import NcclExchanger
    from paper_2303_12374_b200.slab import SlabDriver

    import ctypes

    ver = ctypes.c_int()
    if lib().klb_nccl_version(ctypes.byref(ver)) != 0:
        pytest.skip("libnccl.so.2 not loadable on this host")
    ex = NcclExchanger(0, 1, NcclExchanger.unique_id())
    drv = SlabDriver("diff_uvw", "fp32", (64, 32, 16), gpu_ctx, rank=0, nranks=1, exchanger=ex)
    drv.step()
    gpu_ctx.synchronize()
    drv.close()
    ex.close()
    assert ver.value >= 22700


@pytest.mark.parametrize("kernel,copy_streams,align", [("advec_u", 1, 128), ("diff_uvw", 1, 128), ("diff_uvw", 2, 128),
                                                      ("advec_u", 3, 128), ("diff_uvw", 1, 16), ("advec_u", 2, 16)])
def test_host_streamed_step_matches_device_step(gpu_ctx, tmp_path, kernel, copy_streams, align):
    """SlabDriver.step_host (fields in pinned host memory, chunked H2D |
    launch | D2H on overlapped streams, one or several copy streams per
    direction) returns the same tendencies as step() on device-resident
    fields, and leaves the host inputs untouched."""
    from paper_2303_12374_b200.cuda import HostPinned, NvrtcCompiler
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.wisdom import WisdomFile, WisdomRecord

    grid, precision = (64, 40, 37), "fp64"
    d = definition_for(kernel, precision)
    cfg = d.space.default_config()[0]
    cfg.update(staging="TMA", zchunk=8, block_x=32, block_y=4, depth=2)
    WisdomFile(d.kernel_key(), records=[WisdomRecord(gpu_ctx.ident, (1, 1, 1), cfg, 1.0)]).save(
        tmp_path / f"{d.kernel_key()}.wisdom")
    drv = SlabDriver(kernel, precision, grid, gpu_ctx, compiler=NvrtcCompiler(gpu_ctx), wisdom_dir=tmp_path,
                     align_bytes=align)
    prob, lay = drv.problem, drv.layout
    assert lay.align_bytes == align
    nbytes = lay.alloc_bytes
    host = {}
    for n in prob.fields:
        host[n] = HostPinned(nbytes)
        check(lib().klb_memcpy_dtoh(host[n].ptr, prob.fields[n].ptr, nbytes, None))
    gpu_ctx.synchronize()
    before = {n: host[n].array(lay.dtype).copy() for n in host}
    drv.step()
    gpu_ctx.synchronize()
    ref = {n: prob.download(n).copy() for n in prob.outputs()}
    # scramble the device copies: step_host must bring everything it reads from the host
    for n, arr in prob.fields.items():
        check(lib().klb_memset_d8(arr.ptr, 0xFF, nbytes, None))
    gpu_ctx.synchronize()
    launches = drv.step_host({n: b.ptr for n, b in host.items()}, chunks=5, copy_streams=copy_streams)
    drv.compute.synchronize()
    assert launches == 5
    h2d, d2h = drv.stream_bytes
    plane = lay.kk * lay.elem_bytes
    assert d2h == len(ref) * lay.ktot * plane
    for n in prob.fields:
        got = host[n].array(lay.dtype)
        if n in ref:
            have, want = lay.interior(lay.host_view(got)), lay.interior(ref[n])
            err = np.max(np.abs(have - want)) / np.max(np.abs(want))
            assert err <= 1e-13, (n, err)
        else:
            assert np.array_equal(got, before[n]), n
    for b in host.values():
        b.free()
    drv.close()
