"""Oracle parity of the kernels the benchmark times, at the shapes it times them.

Every launch goes through the application path the bench uses —
``WisdomKernel`` over the committed ``wisdom/`` (select -> NVRTC -> load ->
launch) — and is compared with the float64 oracle (``oracle/``, SURVEY
Appendix A; parity UNPINNED against upstream MicroHH) on
the same synthetic inputs, over EVERY interior cell of the benchmarked grid
against the C restatement (``full_volume_error``: float64 arithmetic, inputs
regenerated per 32-plane z-chunk by the C synth twin, so host memory stays
bounded at 1024^3; the fused RK3 kernel as cref's diff_uvw + the RK3
epilogue).

Bar (BASELINE.json north_star): max|gpu - ref| / max|ref| <= 1e-5 (fp32),
<= 1e-12 (fp64) per output array.

Cases = BASELINE configs 1-4 (+ the north-star 512^3 fp32 pair, the fused
RK3 kernel and its unfused rk3_uvw baseline, and the §8f family kernels at
the 512^3 shape the bench's ``family`` rows time; config 5's runtime
selection at shapes without a record of their own), and config 4's N = 2/4/8
z-slab ranks: the 1024^2 x {511, 254,
126}-plane interior sub-ranges and single-plane boundary sub-ranges, each
selected from wisdom for its own shape, exactly as ``bench.py --gpus N``
launches them on every rank.
"""

from __future__ import annotations

import json
import os
from pathlib import Path

import pytest

from stencil_helpers import TOL, full_volume_error, window_error

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
WISDOM = ROOT / "wisdom"
RESULTS = os.environ.get("KL_PARITY_LOG")  # optional JSON-lines record of every case

CASES = [
    # (tag, kernel, precision, grid, match kind the committed wisdom must give)
    ("config 1", "diff_uvw", "fp64", (64, 64, 64), "exact"),
    ("config 2", "advec_u", "fp32", (256, 256, 256), "exact"),
    ("config 3", "advec_u", "fp64", (512, 512, 512), "exact"),
    ("config 3", "diff_uvw", "fp64", (512, 512, 512), "exact"),
    ("config 4", "diff_uvw", "fp32", (1024, 1024, 1024), "exact"),
    ("north_star", "advec_u", "fp32", (512, 512, 512), "exact"),
    ("north_star", "diff_uvw", "fp32", (512, 512, 512), "exact"),
    ("§8f fusion", "diff_uvw_rk3", "fp32", (512, 512, 512), "exact"),
    ("§8f fusion", "diff_uvw_rk3", "fp64", (512, 512, 512), "exact"),
    ("§8f fusion", "rk3_uvw", "fp32", (512, 512, 512), "exact"),
    ("§8f fusion", "rk3_uvw", "fp64", (512, 512, 512), "exact"),
] + [("§8f family", k, p, (512, 512, 512), "exact")
     for k in ("advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag") for p in ("fp32", "fp64")] + [
    # config 5: shapes with no record of their own, where runtime selection
    # picks the nearest tuned problem's configuration (portability.QUERIES)
    ("config 5", "advec_u", "fp32", (192, 192, 192), "same_device_nearest"),
    ("config 5", "diff_uvw", "fp64", (384, 384, 384), "same_device_nearest"),
    ("config 5", "diff_uvw", "fp32", (768, 768, 768), "same_device_nearest"),
    ("config 5", "advec_u", "fp64", (320, 200, 150), "same_device_nearest"),
]


#: restated in C by oracle/cref (stencil_ref.c, family_ref.c; + the RK3 epilogue)
FULL_VOLUME = ("advec_u", "diff_uvw", "diff_uvw_rk3", "rk3_uvw", "advec_v", "advec_w", "advec_s", "diff_c",
               "evisc_smag")


def _windows(lay, n=8):
    if lay.ktot <= 64:
        return [(lay.kstart, lay.kend)]
    mid = lay.kstart + lay.ktot // 2
    return [(lay.kstart, lay.kstart + n), (mid - n // 2, mid + n // 2), (lay.kend - n, lay.kend)]


def _record(entry: dict) -> None:
    print(json.dumps(entry))
    if RESULTS:
        with open(RESULTS, "a", encoding="utf-8") as fh:
            fh.write(json.dumps(entry) + "\n")


@pytest.fixture(scope="module")
def compiler(gpu_ctx):
    from paper_2303_12374_b200.cuda import NvrtcCompiler

    return NvrtcCompiler(gpu_ctx)


@pytest.mark.parametrize("tag,kernel,precision,grid,kind", CASES,
                         ids=[f"{k}_{p}_{g[0]}x{g[1]}x{g[2]}" for _, k, p, g, _ in CASES])
def test_wisdom_selected_kernel_matches_oracle(gpu_ctx, compiler, tag, kernel, precision, grid, kind):
    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(*grid, precision)
    prob = StencilProblem(kernel, lay, gpu_ctx)
    try:
        wk = WisdomKernel(prob.definition, compiler, wisdom_dir=WISDOM, capture_policy=CapturePolicy())
        report = wk.launch(gpu_ctx.ident, prob.args())
        gpu_ctx.synchronize()
        if kernel in FULL_VOLUME:
            errors = {"all planes": full_volume_error(prob, kernel)}
            checked = f"every interior cell ({lay.cells})"
        else:
            errors = {f"{kb}:{ke}": window_error(prob, kernel, kb, ke) for kb, ke in _windows(lay)}
            checked = "planes " + ", ".join(errors)
    finally:
        prob.close()
    worst = max(e for w in errors.values() for e in w.values())
    _record({"case": tag, "kernel": kernel, "precision": precision, "grid": list(grid),
             "match_kind": report.match_kind, "config": report.configuration, "worst_rel_err": worst,
             "tolerance": TOL[precision], "checked": checked, "errors": errors})
    assert report.match_kind == kind, report.match_kind
    assert worst <= TOL[precision], errors


@pytest.mark.parametrize("align", [16])
def test_bench_row_pitch_matches_oracle(gpu_ctx, compiler, align):
    """Config 4 on the layout the bench runs it on (``bench.py --row-align``,
    default 16: rows packed at 16-byte pitch, so the host-streamed step moves
    no padding): the whole 1024^3 grid through the committed wisdom, every
    interior cell against the oracle."""
    from paper_2303_12374_b200.slab import SlabDriver

    drv = SlabDriver("diff_uvw", "fp32", (1024, 1024, 1024), gpu_ctx, compiler=compiler, wisdom_dir=WISDOM,
                     align_bytes=align)
    try:
        assert drv.layout.jj == 1032 and drv.layout.align_bytes == align
        chosen = drv.resolve()
        drv.step()
        gpu_ctx.synchronize()
        errors = {"all planes": full_volume_error(drv.problem, "diff_uvw")}
    finally:
        drv.close()
    worst = max(errors["all planes"].values())
    _record({"case": f"config 4, {align}-byte row pitch", "selection":
             {n: {"match_kind": k, "config": c} for n, (c, k) in chosen.items()}, "worst_rel_err": worst,
             "checked": "every interior cell (1073741824)", "errors": errors})
    assert all(k == "exact" for _, k in chosen.values())
    assert worst <= TOL["fp32"], errors


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_slab_rank_subranges_match_oracle(gpu_ctx, compiler, nranks):
    """Config 4 at N ranks: rank 1's slab (interior sub-range + its boundary
    planes, each wisdom-selected for its own shape) as SlabDriver launches
    them, checked over every cell of the slab.  The slab's ghost planes hold the neighbours' planes (the device
    generator indexes by global plane — what the halo exchange maintains), so
    the result must equal the whole-grid oracle on the rank's planes."""
    from paper_2303_12374_b200.slab import SlabDriver

    drv = SlabDriver("diff_uvw", "fp32", (1024, 1024, 1024), gpu_ctx, rank=1, nranks=nranks, exchanger=None,
                     compiler=compiler, wisdom_dir=WISDOM)
    try:
        chosen = drv.resolve()
        drv.step()
        gpu_ctx.synchronize()
        lay = drv.layout
        shapes = {name: ke - kb for name, (kb, ke) in drv.ranges.items()}
        errors = {"all planes": full_volume_error(drv.problem, "diff_uvw")}
    finally:
        drv.close()
    worst = max(e for w in errors.values() for e in w.values())
    _record({"case": f"config 4 slab rank 1 of {nranks}", "subrange_planes": shapes,
             "selection": {n: {"match_kind": k, "config": c} for n, (c, k) in chosen.items()},
             "worst_rel_err": worst, "checked": f"every interior cell of the slab ({lay.cells})", "errors": errors})
    interior = {2: 511, 4: 254, 8: 126}[nranks]
    assert shapes["interior"] == interior and shapes.get("lower", shapes.get("upper")) == 1
    assert worst <= TOL["fp32"], errors


@pytest.mark.parametrize("nranks", [2, 8])
def test_fused_halo_slab_matches_oracle(gpu_ctx, compiler, nranks):
    """Config 4 at N ranks with the fused halo (``--halo fused``): rank 1's
    ONE slab launch of diff_uvw_peer, selected from the committed diff_uvw
    wisdom for the slab's shape, reads the planes outside its slab from its
    neighbours' fields (virtual ranks on this device: separate allocations
    generated at their own global planes), its own ghost planes poisoned —
    checked over every cell of the slab."""
    from paper_2303_12374_b200.halo import LocalPeers
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.problem import PEER_KERNELS

    grid = (1024, 1024, 1024)
    ranks = [r for r in (0, 1, 2) if r < nranks]
    peers = LocalPeers([])
    drivers = {}
    try:
        for r in ranks:
            fused = r == 1
            drivers[r] = SlabDriver("diff_uvw", "fp32", grid, gpu_ctx, rank=r, nranks=nranks, compiler=compiler,
                                    wisdom_dir=WISDOM, halo="fused" if fused else "exchange",
                                    exchanger=peers.for_rank(r) if fused else None)
        fields = PEER_KERNELS["diff_uvw_peer"]
        peers.ranks = [({n: drivers[r].problem.field_ptr(n) for n in fields}, drivers[r].layout.kstart,
                        drivers[r].layout.kend) if r in drivers else ({}, 0, 0) for r in range(max(ranks) + 1)]
        drv = drivers[1]
        lay = drv.layout
        plane = lay.kk * lay.elem_bytes
        from paper_2303_12374_b200.cuda._abi import check, lib

        for n in fields:  # the fused launch must never read its own ghost planes
            base = drv.problem.field_ptr(n)
            check(lib().klb_memset_d8(base + (lay.kstart - lay.kgc) * plane, 0xFF, lay.kgc * plane, None))
            if drv.above >= 0:
                check(lib().klb_memset_d8(base + lay.kend * plane, 0xFF, lay.kgc * plane, None))
        gpu_ctx.synchronize()
        chosen = drv.resolve()
        assert drv.step() == 1
        gpu_ctx.synchronize()
        errors = {"all planes": full_volume_error(drv.problem, "diff_uvw")}
    finally:
        for d in drivers.values():
            d.close()
    worst = max(errors["all planes"].values())
    _record({"case": f"config 4 fused-halo slab rank 1 of {nranks}", "selection":
             {n: {"match_kind": k, "config": c} for n, (c, k) in chosen.items()}, "worst_rel_err": worst,
             "checked": f"every interior cell of the slab ({lay.cells})", "errors": errors})
    assert chosen["slab"][1] == "exact"
    assert worst <= TOL["fp32"], errors
