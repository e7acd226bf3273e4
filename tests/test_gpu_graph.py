"""CUDA-graph replay of bound launches (klb_stream_*_capture / klb_graph_*).

``WisdomKernel.graph`` captures ``repeat`` launches of the wisdom-selected
configuration on a stream; replaying the graph must leave exactly the bytes
the same launches leave when enqueued one by one (the kernel parameters — TMA
descriptors included — are copied into the graph at capture), and one
captured application must match the oracle.
"""

from pathlib import Path

import numpy as np
import pytest

from stencil_helpers import TOL, oracle_outputs, rel_error

pytestmark = pytest.mark.gpu

WISDOM = Path(__file__).resolve().parent.parent / "wisdom"


@pytest.mark.parametrize("kernel,precision,grid", [("diff_uvw", "fp64", (64, 64, 64)),
                                                   ("advec_u", "fp32", (96, 40, 70)),
                                                   ("diff_uvw_rk3", "fp32", (72, 40, 33))])
def test_graph_replay_matches_eager_launches(gpu_ctx, kernel, precision, grid):
    from paper_2303_12374_b200.cuda import NvrtcCompiler, Stream
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(*grid, precision)
    prob = StencilProblem(kernel, lay, gpu_ctx)
    stream = Stream.create()
    try:
        wk = WisdomKernel(prob.definition, NvrtcCompiler(gpu_ctx), wisdom_dir=WISDOM)
        n = 4
        run = wk.bind(gpu_ctx.ident, prob.args(), stream=stream)
        for _ in range(n):
            run()
        stream.synchronize()
        eager = {name: prob.download(name).copy() for name in prob.outputs()}

        prob.regenerate()
        before = {name: prob.download(name).copy() for name in prob.outputs()}
        g = wk.graph(gpu_ctx.ident, prob.args(), stream, repeat=n)
        stream.synchronize()
        for name in before:  # capturing records the launches, it does not run them
            assert np.array_equal(prob.download(name), before[name]), name
        g.launch(stream)
        stream.synchronize()
        for name in eager:
            assert np.array_equal(prob.download(name), eager[name]), name
        g.close()

        prob.regenerate()
        one = wk.graph(gpu_ctx.ident, prob.args(), stream, repeat=1)
        one.launch(stream)
        stream.synchronize()
        ref, _ = oracle_outputs(kernel, lay)
        for name in ref:
            assert rel_error(prob.download(name), ref[name], lay) <= TOL[precision], name
        one.close()
    finally:
        prob.close()
        stream.close()


def test_failed_capture_leaves_the_stream_usable(gpu_ctx):
    from paper_2303_12374_b200.cuda import Graph, NvrtcCompiler, Stream
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(40, 24, 12, "fp64")
    prob = StencilProblem("advec_u", lay, gpu_ctx)
    stream = Stream.create()
    try:
        wk = WisdomKernel(prob.definition, NvrtcCompiler(gpu_ctx), wisdom_dir=WISDOM)
        run = wk.bind(gpu_ctx.ident, prob.args(), stream=stream)
        with pytest.raises(RuntimeError, match="abandon"):
            with Graph.capture(stream):
                run()
                raise RuntimeError("abandon the capture")
        with pytest.raises(ValueError):
            Graph.capture(Stream()).__enter__()  # the legacy default stream cannot be captured
        prob.regenerate()
        run()  # the stream left capture mode: eager launches work again
        stream.synchronize()
        ref, _ = oracle_outputs("advec_u", lay)
        assert rel_error(prob.download("ut"), ref["ut"], lay) <= TOL["fp64"]
    finally:
        prob.close()
        stream.close()


def test_chained_step_graph_matches_the_oracle_chain(gpu_ctx):
    """A time-step fragment as one graph: evisc_smag (u, v, w -> evisc) then the
    fused diff_uvw + RK3 substep reading that evisc and the same u, v, w
    (StencilProblem.share_fields).  Graph replay == eager launches bit for bit,
    and both match the oracle chain (evisc_smag -> diff_uvw_rk3 on its output)."""
    from oracle import family_oracle
    from paper_2303_12374_b200.cuda import Graph, NvrtcCompiler, Stream
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import CS, RK_A, RK_BDT, StencilProblem
    from paper_2303_12374_b200.stencils.profiles import make_profiles
    from stencil_helpers import host_fields

    lay = GridLayout(70, 38, 29, "fp64")
    pe = StencilProblem("evisc_smag", lay, gpu_ctx)
    pd = StencilProblem("diff_uvw_rk3", lay, gpu_ctx)
    stream = Stream.create()
    try:
        pd.share_fields(pe, ("evisc", "u", "v", "w"))
        comp = NvrtcCompiler(gpu_ctx)
        run_e = WisdomKernel(pe.definition, comp, wisdom_dir=WISDOM).bind(gpu_ctx.ident, pe.args(), stream=stream)
        run_d = WisdomKernel(pd.definition, comp, wisdom_dir=WISDOM).bind(gpu_ctx.ident, pd.args(), stream=stream)
        outs = ("evisc", "ut", "vt", "wt", "u_next", "v_next", "w_next")

        def fetch():
            return {n: (pe if n == "evisc" else pd).download(n).copy() for n in outs}

        run_e()
        run_d()
        stream.synchronize()
        eager = fetch()

        pe.regenerate()
        pd.regenerate()
        with Graph.capture(stream) as g:
            run_e()
            run_d()
        g.launch(stream)
        stream.synchronize()
        got = fetch()
        for n in outs:
            assert np.array_equal(got[n], eager[n]), n
        g.close()

        f = host_fields(lay, ("evisc", "u", "v", "w", "ut", "vt", "wt", "u_next", "v_next", "w_next"))
        prof = make_profiles(lay.kcells, lay.kgc).as_dtype(lay.dtype)
        gh = (lay.igc, lay.jgc, lay.kgc)
        evisc = family_oracle.evisc_smag(f["evisc"], f["u"], f["v"], f["w"], prof.dzi, prof.dzhi, 1.0, 1.0, CS,
                                         ghost=gh)
        ref = dict(zip(("ut", "vt", "wt", "u_next", "v_next", "w_next"),
                       family_oracle.diff_uvw_rk3(f["ut"], f["vt"], f["wt"], evisc, f["u"], f["v"], f["w"],
                                                  f["u_next"], f["v_next"], f["w_next"], prof.dzi, prof.dzhi,
                                                  prof.rhoref, prof.rhorefh, 1.0, 1.0, RK_A, RK_BDT, ghost=gh)))
        ref["evisc"] = evisc
        for n in outs:
            assert rel_error(got[n], ref[n], lay) <= TOL["fp64"], n
    finally:
        pd.close()
        pe.close()
        stream.close()


@pytest.mark.parametrize("kernel,precision,grid", [("diff_uvw", "fp64", (64, 64, 64)),
                                                   ("advec_u", "fp32", (96, 40, 70)),
                                                   ("diff_uvw", "fp32", (130, 70, 50))])
def test_pdl_launches_are_ordered(gpu_ctx, kernel, precision, grid):
    """Programmatic dependent launch (klb_launch_ex KLB_LAUNCH_PDL): each
    application of a read-modify-write stencil may start launching while the
    previous one drains, but its griddepcontrol.wait must hold every global
    access until that one completed — 12 chained applications, eager and as a
    captured graph, leave exactly the bytes of 12 ordinary launches."""
    from paper_2303_12374_b200.cuda import NvrtcCompiler, Stream
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(*grid, precision)
    prob = StencilProblem(kernel, lay, gpu_ctx)
    stream = Stream.create()
    n = 12
    try:
        wk = WisdomKernel(prob.definition, NvrtcCompiler(gpu_ctx), wisdom_dir=WISDOM)
        plain = wk.bind(gpu_ctx.ident, prob.args(), stream=stream)
        for _ in range(n):
            plain()
        stream.synchronize()
        want = {name: prob.download(name).copy() for name in prob.outputs()}

        prob.regenerate()
        pdl = wk.bind(gpu_ctx.ident, prob.args(), stream=stream, pdl=True)
        for _ in range(n):
            pdl()
        stream.synchronize()
        for name in want:
            assert np.array_equal(prob.download(name), want[name]), name

        prob.regenerate()
        g = wk.graph(gpu_ctx.ident, prob.args(), stream, repeat=n, pdl=True)
        g.launch(stream)
        stream.synchronize()
        for name in want:
            assert np.array_equal(prob.download(name), want[name]), name
        g.close()
    finally:
        prob.close()
        stream.close()


def test_chained_step_graph_with_pdl(gpu_ctx):
    """evisc_smag -> diff_uvw_rk3 (the second reads the first's evisc) with
    programmatic dependent launch inside one graph: bit-identical to the
    plain chain."""
    from paper_2303_12374_b200.cuda import Graph, NvrtcCompiler, Stream
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(128, 96, 64, "fp32")
    pe = StencilProblem("evisc_smag", lay, gpu_ctx)
    pd = StencilProblem("diff_uvw_rk3", lay, gpu_ctx)
    stream = Stream.create()
    try:
        pd.share_fields(pe, ("evisc", "u", "v", "w"))
        comp = NvrtcCompiler(gpu_ctx)
        we = WisdomKernel(pe.definition, comp, wisdom_dir=WISDOM)
        wd = WisdomKernel(pd.definition, comp, wisdom_dir=WISDOM)
        outs = ("evisc", "ut", "vt", "wt", "u_next", "v_next", "w_next")

        def fetch():
            return {n: (pe if n == "evisc" else pd).download(n).copy() for n in outs}

        def chain(pdl, steps=3):
            run_e = we.bind(gpu_ctx.ident, pe.args(), stream=stream, pdl=pdl)
            run_d = wd.bind(gpu_ctx.ident, pd.args(), stream=stream, pdl=pdl)
            with Graph.capture(stream) as g:
                for _ in range(steps):
                    run_e()
                    run_d()
            pe.regenerate()
            pd.regenerate()
            g.launch(stream)
            stream.synchronize()
            g.close()
            return fetch()

        plain, fast = chain(False), chain(True)
        for n in outs:
            assert np.array_equal(fast[n], plain[n]), n
    finally:
        pd.close()
        pe.close()
        stream.close()
