"""Shared GPU-test helpers: run a stencil configuration and compare with the oracle."""

from __future__ import annotations

import numpy as np

from oracle import family_oracle, stencil_oracle
from oracle.synth import synth_field
from paper_2303_12374_b200.stencils.layout import GridLayout
from paper_2303_12374_b200.stencils.problem import CS, KERNEL_FIELDS, RK_A, RK_BDT, TPRI, StencilProblem
from paper_2303_12374_b200.stencils.profiles import FIELD_SEED_BASE, FIELD_SPECS, make_profiles

TOL = {"fp32": 1e-5, "fp64": 1e-12}


def host_fields(layout: GridLayout, names, k_offset=0):
    out = {}
    for n in names:
        off, lo, hi = FIELD_SPECS[n]
        out[n] = synth_field(FIELD_SEED_BASE + off, lo, hi, layout.icells, layout.jcells, layout.kcells, layout.igc,
                             layout.jgc, k_offset=k_offset, dtype=layout.dtype)
    return out


def oracle_outputs(kernel: str, layout: GridLayout, dxi=1.0, dyi=1.0, k_range=None):
    """Oracle result for the full interior (or local planes ``k_range``)."""
    f = host_fields(layout, KERNEL_FIELDS[kernel])
    prof = make_profiles(layout.kcells, layout.kgc).as_dtype(layout.dtype)
    res = _oracle_compute(kernel, f, prof, layout, dxi, dyi)
    if k_range is not None:
        kb, ke = k_range
        for name, arr in res.items():
            orig = f[name].astype(np.float64)
            arr[:kb] = orig[:kb]
            arr[ke:] = orig[ke:]
    return res, f


def oracle_window(kernel: str, layout: GridLayout, kb: int, ke: int, k_offset: int = 0,
                  kcells_global: int | None = None, dxi=1.0, dyi=1.0):
    """Oracle outputs on local planes ``[kb, ke)`` of a grid ``layout`` whose
    local plane 0 is global ghost-padded plane ``k_offset`` (a z-slab; 0 for
    a whole grid) — only planes ``kb - kgc .. ke + kgc`` are generated, so the
    check is bounded however large the grid.  Returns ``{output: (ke-kb,
    jtot, itot) float64}`` (interior i/j)."""
    g = layout.kgc
    sub = GridLayout(layout.itot, layout.jtot, ke - kb, layout.precision, layout.igc, layout.jgc, g)
    f = host_fields(sub, KERNEL_FIELDS[kernel], k_offset=k_offset + kb - g)
    kcg = kcells_global if kcells_global is not None else layout.kcells
    prof = make_profiles(kcg, g).window(k_offset + kb - g, sub.kcells).as_dtype(layout.dtype)
    res = _oracle_compute(kernel, f, prof, sub, dxi, dyi)
    return {n: sub.interior(a) for n, a in res.items()}


def cyclic_xy(a: np.ndarray, layout: GridLayout) -> np.ndarray:
    """MicroHH boundary_cyclic on the interior planes of a (kcells, jcells,
    icells) array: x/y ghost cells take the interior cell they wrap onto
    (the oracle of ``klb_cyclic_xy``)."""
    gi, gj, gk = layout.igc, layout.jgc, layout.kgc
    ii = gi + (np.arange(a.shape[2]) - gi) % layout.itot
    jj = gj + (np.arange(a.shape[1]) - gj) % layout.jtot
    out = np.array(a, copy=True)
    out[gk:a.shape[0] - gk] = a[gk:a.shape[0] - gk][:, jj][:, :, ii]
    return out


def oracle_rk3_loop(layout: GridLayout, nsub: int, dt: float, dxi=1.0, dyi=1.0):
    """``nsub`` substeps of the low-storage RK3 time loop SlabDriver.rk3_substep
    runs (diff_uvw_rk3 into the alternate buffers, then the periodic x/y ghost
    fill), over the whole grid.  Returns (tendencies, current u/v/w) by name
    ({"ut", "vt", "wt"}, {"u", "v", "w"}), float64."""
    from paper_2303_12374_b200.slab import SlabDriver

    f = {n: a.astype(np.float64) for n, a in host_fields(layout, KERNEL_FIELDS["diff_uvw_rk3"]).items()}
    prof = make_profiles(layout.kcells, layout.kgc).as_dtype(layout.dtype)
    g = (layout.igc, layout.jgc, layout.kgc)
    cur = [f["u"], f["v"], f["w"]]
    nxt = [f["u_next"], f["v_next"], f["w_next"]]
    t = [f["ut"], f["vt"], f["wt"]]
    for s in range(nsub):
        rk_a, rk_bdt = SlabDriver.RK3_A[(s % 3 + 1) % 3], SlabDriver.RK3_B[s % 3] * dt
        out = family_oracle.diff_uvw_rk3(*t, f["evisc"], *cur, *nxt, prof.dzi, prof.dzhi, prof.rhoref, prof.rhorefh,
                                         dxi, dyi, rk_a, rk_bdt, ghost=g)
        t = list(out[:3])
        nxt, cur = cur, [cyclic_xy(a, layout) for a in out[3:]]
    return dict(zip(("ut", "vt", "wt"), t)), dict(zip(("u", "v", "w"), cur))


def download_planes(prob: StencilProblem, name: str, kb: int, ke: int) -> np.ndarray:
    """Interior i/j of local planes ``[kb, ke)`` of a device field, (ke-kb, jtot, itot)."""
    lay = prob.layout
    e = lay.elem_bytes
    raw = prob.fields[name].download((ke - kb) * lay.kk * e, (lay.lead + kb * lay.kk) * e)
    arr = np.frombuffer(raw, dtype=lay.dtype).reshape(ke - kb, lay.jcells, lay.jj)
    return arr[:, lay.jstart:lay.jend, lay.istart:lay.iend]


def window_error(prob: StencilProblem, kernel: str, kb: int, ke: int) -> dict:
    """max|gpu - ref| / max|ref| per output over local planes [kb, ke)."""
    ref = oracle_window(kernel, prob.layout, kb, ke, prob.k_offset, prob.kcells_global, prob.dxi, prob.dyi)
    out = {}
    for name, r in ref.items():
        got = download_planes(prob, name, kb, ke).astype(np.float64)
        # a NaN/inf anywhere (output or reference) is an unbounded error
        err = float(np.max(np.abs(got - r)) / np.max(np.abs(r)))
        out[name] = err if np.isfinite(err) else float("inf")
    return out


def cref_chunks(kernel: str, layout: GridLayout, k_offset: int = 0, kcells_global: int | None = None,
                dxi: float = 1.0, dyi: float = 1.0, chunk: int = 32, threads: int | None = None,
                rk_a: float = RK_A, rk_bdt: float = RK_BDT, tpri: float = TPRI, cs: float = CS):
    """Yield ``(kb, ke, {output: (ke-kb, jtot, itot) float64})`` over every
    interior plane of ``layout`` (local plane 0 = global plane ``k_offset``):
    the C restatement (oracle/cref, float64 arithmetic on inputs of the
    layout's precision) on z-chunks of ``chunk`` planes, each chunk's inputs
    (+ ghost reach) generated by the C synth twin — host memory stays bounded
    at any grid size.  advec_u / diff_uvw (stencil_ref.c), the §8f family
    advec_v/w/s, diff_c, evisc_smag (family_ref.c), and diff_uvw_rk3 /
    rk3_uvw (cref's diff_uvw + the RK3 epilogue of family_oracle, elementwise
    in float64)."""
    import os

    from oracle import cref

    g = layout.kgc
    threads = threads or os.cpu_count() or 1
    base = make_profiles(kcells_global if kcells_global is not None else layout.kcells, g)
    for kb in range(layout.kstart, layout.kend, chunk):
        ke = min(kb + chunk, layout.kend)
        sub = GridLayout(layout.itot, layout.jtot, ke - kb, layout.precision, layout.igc, layout.jgc, g)
        k0 = k_offset + kb - g
        f = {}
        for n in KERNEL_FIELDS[kernel]:
            off, lo, hi = FIELD_SPECS[n]
            a = cref.synth_field(FIELD_SEED_BASE + off, lo, hi, sub.icells, sub.jcells, sub.kcells, sub.igc, sub.jgc,
                                 k_offset=k0, dtype=layout.dtype, threads=threads)
            f[n] = a.astype(np.float64)
        prof = base.window(k0, sub.kcells).as_dtype(layout.dtype)
        pf = {k: np.ascontiguousarray(getattr(prof, k), dtype=np.float64) for k in ("rhoref", "rhorefh", "dzi", "dzhi")}
        gh = (sub.igc, sub.jgc, g)
        if kernel == "advec_u":
            cref.advec_u(f["ut"], f["u"], f["v"], f["w"], pf["rhoref"], pf["rhorefh"], pf["dzi"], dxi, dyi, ghost=gh,
                         threads=threads)
            outs = ("ut",)
        elif kernel in ("diff_uvw", "diff_uvw_rk3"):
            cref.diff_uvw(f["ut"], f["vt"], f["wt"], f["evisc"], f["u"], f["v"], f["w"], pf["dzi"], pf["dzhi"],
                          pf["rhoref"], pf["rhorefh"], dxi, dyi, ghost=gh, threads=threads)
            outs = ("ut", "vt", "wt")
            if kernel == "diff_uvw_rk3":
                for c, t in (("u", "ut"), ("v", "vt"), ("w", "wt")):
                    f[c + "_next"] = f[c] + rk_bdt * f[t]  # interior cells only are compared
                    f[t] = rk_a * f[t]
                outs += ("u_next", "v_next", "w_next")
        elif kernel == "advec_v":
            cref.advec_v(f["vt"], f["u"], f["v"], f["w"], pf["rhoref"], pf["rhorefh"], pf["dzi"], dxi, dyi, ghost=gh,
                         threads=threads)
            outs = ("vt",)
        elif kernel == "advec_w":
            cref.advec_w(f["wt"], f["u"], f["v"], f["w"], pf["rhoref"], pf["rhorefh"], pf["dzhi"], dxi, dyi,
                         ghost=gh, threads=threads)
            outs = ("wt",)
        elif kernel == "advec_s":
            cref.advec_s(f["st"], f["s"], f["u"], f["v"], f["w"], pf["rhoref"], pf["rhorefh"], pf["dzi"], dxi, dyi,
                         ghost=gh, threads=threads)
            outs = ("st",)
        elif kernel == "diff_c":
            cref.diff_c(f["st"], f["s"], f["evisc"], pf["dzi"], pf["dzhi"], pf["rhoref"], pf["rhorefh"], dxi, dyi,
                        tpri, ghost=gh, threads=threads)
            outs = ("st",)
        elif kernel == "evisc_smag":
            cref.evisc_smag(f["evisc"], f["u"], f["v"], f["w"], pf["dzi"], pf["dzhi"], dxi, dyi, cs, ghost=gh,
                            threads=threads)
            outs = ("evisc",)
        elif kernel == "rk3_uvw":
            for c, t in (("u", "ut"), ("v", "vt"), ("w", "wt")):
                f[c] = f[c] + rk_bdt * f[t]
                f[t] = rk_a * f[t]
            outs = ("ut", "vt", "wt", "u", "v", "w")
        else:
            raise ValueError(f"no C restatement of {kernel}")
        yield kb, ke, {n: sub.interior(f[n]) for n in outs}


def full_volume_error(prob: StencilProblem, kernel: str, chunk: int = 32) -> dict:
    """max|gpu - ref| / max|ref| per output over EVERY interior cell of the
    device problem (all its local planes), reference = ``cref_chunks``."""
    diff, scale = {}, {}
    for kb, ke, ref in cref_chunks(kernel, prob.layout, prob.k_offset, prob.kcells_global, prob.dxi, prob.dyi,
                                   chunk, rk_a=prob.rk_a, rk_bdt=prob.rk_bdt, tpri=prob.tpri, cs=prob.cs):
        for n, r in ref.items():
            got = download_planes(prob, n, kb, ke).astype(np.float64)
            d = float(np.max(np.abs(got - r)))
            diff[n] = max(diff.get(n, 0.0), d if np.isfinite(d) else float("inf"))
            scale[n] = max(scale.get(n, 0.0), float(np.max(np.abs(r))))
    return {n: diff[n] / scale[n] for n in diff}


def _oracle_compute(kernel, f, prof, layout, dxi, dyi):
    g = (layout.igc, layout.jgc, layout.kgc)
    if kernel == "advec_u":
        res = {"ut": stencil_oracle.advec_u(f["ut"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh, prof.dzi, dxi,
                                             dyi, ghost=g)}
    elif kernel == "advec_v":
        res = {"vt": family_oracle.advec_v(f["vt"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh, prof.dzi, dxi,
                                           dyi, ghost=g)}
    elif kernel == "advec_w":
        res = {"wt": family_oracle.advec_w(f["wt"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh, prof.dzhi,
                                           dxi, dyi, ghost=g)}
    elif kernel == "advec_s":
        res = {"st": family_oracle.advec_s(f["st"], f["s"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh,
                                           prof.dzi, dxi, dyi, ghost=g)}
    elif kernel == "diff_c":
        res = {"st": family_oracle.diff_c(f["st"], f["s"], f["evisc"], prof.dzi, prof.dzhi, prof.rhoref,
                                          prof.rhorefh, dxi, dyi, TPRI, ghost=g)}
    elif kernel == "rk3_uvw":
        res = dict(zip(("ut", "vt", "wt", "u", "v", "w"),
                       family_oracle.rk3_uvw(f["ut"], f["vt"], f["wt"], f["u"], f["v"], f["w"], RK_A, RK_BDT, ghost=g)))
    elif kernel == "diff_uvw_rk3":
        res = dict(zip(("ut", "vt", "wt", "u_next", "v_next", "w_next"),
                       family_oracle.diff_uvw_rk3(f["ut"], f["vt"], f["wt"], f["evisc"], f["u"], f["v"], f["w"],
                                                  f["u_next"], f["v_next"], f["w_next"], prof.dzi, prof.dzhi,
                                                  prof.rhoref, prof.rhorefh, dxi, dyi, RK_A, RK_BDT, ghost=g)))
    elif kernel == "evisc_smag":
        res = {"evisc": family_oracle.evisc_smag(f["evisc"], f["u"], f["v"], f["w"], prof.dzi, prof.dzhi, dxi, dyi,
                                                 CS, ghost=g)}
    else:
        ut, vt, wt = stencil_oracle.diff_uvw(f["ut"], f["vt"], f["wt"], f["evisc"], f["u"], f["v"], f["w"], prof.dzi,
                                             prof.dzhi, prof.rhoref, prof.rhorefh, dxi, dyi, ghost=g)
        res = {"ut": ut, "vt": vt, "wt": wt}
    return res


def rel_error(got: np.ndarray, ref: np.ndarray, layout: GridLayout) -> float:
    gi = layout.interior(got).astype(np.float64)
    ri = layout.interior(ref)
    scale = np.max(np.abs(ri))
    err = float(np.max(np.abs(gi - ri)) / scale)
    return err if np.isfinite(err) else float("inf")


def run_config(ctx, compiler, kernel, layout, config, k_range=None):
    prob = StencilProblem(kernel, layout, ctx)
    try:
        d = prob.definition
        args = prob.args(k_range)
        from paper_2303_12374_b200.capture import scalar_env_from_args

        env = scalar_env_from_args(args)
        problem = d.derive_problem_size(env)
        exe = compiler.compile(d.render_compile_request(config, problem, env), ctx.ident)
        exe.load()
        exe.launch(d.derive_geometry(config, problem, env), args, timed=True)
        return {n: prob.download(n).copy() for n in prob.outputs()}
    finally:
        prob.close()
