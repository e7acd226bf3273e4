"""``SlabDriver`` — one rank's share of a z-slab decomposed stencil application.

Wires the pieces of ``halo.py`` to the runtime launch path:

* fields of the rank's slab live in HBM (``StencilProblem`` with the global
  plane offset, so the synthetic data are those of the undecomposed grid);
* every sub-range (interior / lower / upper, ``SlabRank.subranges``) is
  launched through ``WisdomKernel.launch`` — the application-facing API —
  so each gets its own wisdom selection and compiled instance;
* ``step()`` issues: halo exchange on the comm stream (peer-memory pulls over
  CUDA IPC, NCCL send/recv, or D2D copies for virtual ranks), the interior
  launch on the compute stream concurrently, then the boundary launches
  after the exchange event;
* ``halo="fused"`` (diff_uvw, advec_u): no exchange and no sub-ranges — ONE launch of
  ``diff_uvw_peer`` over the whole slab, whose TMA staging reads the planes
  just outside the slab straight from the neighbours' fields through
  peer-mapped pointers (``IpcExchanger.peer_fields``; ``LocalPeers`` for
  virtual ranks), between two cross-rank fences (the neighbours' inputs are
  final / they are done reading ours).

All launches are asynchronous; callers time steps with CUDA events on
``compute`` (the comm stream is joined back into it every step).
"""

from __future__ import annotations

from pathlib import Path

from .capture import CapturePolicy
from .cuda.device import DeviceContext, Event, Stream
from .dispatch import WisdomKernel
from .halo import HALO_REACH, SlabDecomposition, SlabRank
from .stencils.definitions import definition_for
from .stencils.layout import GridLayout
from .stencils.problem import PEER_KERNELS, StencilProblem
from .stencils.profiles import make_profiles

__all__ = ["SlabDriver", "FUSED_HALO"]

#: kernels with a fused-halo variant (the planes outside the slab read from
#: the neighbours' fields inside the TMA staging) -> that variant
FUSED_HALO = {"diff_uvw": "diff_uvw_peer", "advec_u": "advec_u_peer", "diff_uvw_rk3": "diff_uvw_rk3_peer"}


class SlabDriver:
    def __init__(self, kernel: str, precision: str, grid: tuple[int, int, int], ctx: DeviceContext, *,
                 rank: int = 0, nranks: int = 1, exchanger=None, compiler=None,
                 wisdom_dir: str | Path | None = None, ghost: int = 3, halo: str = "exchange",
                 align_bytes: int = 128) -> None:
        from .cuda.compiler import NvrtcCompiler

        if halo not in ("exchange", "fused"):
            raise ValueError(f"halo must be 'exchange' or 'fused', not {halo!r}")
        if halo == "fused" and kernel not in FUSED_HALO:
            raise ValueError(f"the fused halo exists for {tuple(FUSED_HALO)}")
        self.fused = halo == "fused"
        if self.fused and nranks > 1 and exchanger is None:
            raise ValueError("the fused halo needs an exchanger that maps the neighbours' fields")
        self.kernel, self.precision, self.grid = kernel, precision, tuple(grid)
        self.ctx = ctx
        self.rank, self.nranks = rank, nranks
        self.exchanger = exchanger
        # ``align_bytes``: the row-pitch quantum of the fields (stencils/layout.py);
        # 16 packs rows densely (less padding to stream in step_host)
        self.global_layout = GridLayout(*grid, precision, ghost, ghost, ghost, align_bytes)
        self.decomposition = SlabDecomposition(grid[2], nranks)
        self.slab = SlabRank(self.decomposition, rank, ghost, kernel)
        self.layout = GridLayout(grid[0], grid[1], self.slab.count, precision, ghost, ghost, ghost, align_bytes)
        profiles = make_profiles(self.global_layout.kcells, ghost)
        self.compute = ctx.stream
        self.comm = Stream.create() if exchanger is not None and not self.fused else None
        self.problem = StencilProblem(FUSED_HALO[kernel] if self.fused else kernel, self.layout, ctx,
                                      k_offset=self.slab.offset, kcells_global=self.global_layout.kcells,
                                      profiles=profiles, stream=self.compute)
        self.compiler = compiler or NvrtcCompiler(ctx)
        # the fused kernel selects from its base kernel's wisdom (same space and problem sizes)
        base_key = definition_for(kernel, precision).kernel_key() if self.fused else None
        self.wisdom = WisdomKernel(self.problem.definition, self.compiler, wisdom_dir=wisdom_dir or ".",
                                   capture_policy=CapturePolicy(), wisdom_key=base_key)
        self.ranges = {"slab": (self.layout.kstart, self.layout.kend)} if self.fused else self.slab.subranges()
        self._peers_attached = not (self.fused and exchanger is not None and nranks > 1)
        self._rk3_cache: dict = {}  # (parity, stage, dt) -> launch arguments (rk3_substep)
        self._rk3_peers: dict = {}  # parity -> the neighbours' current fields
        self.args = {name: self.problem.args(rng) for name, rng in self.ranges.items()}
        self.below, self.above = self.decomposition.neighbours(rank)
        self._ev_start = Event()
        self._ev_halo = Event()
        self.kernel_events: list[tuple[Event, Event]] = []
        self.reports = {}
        self._stream_state = None
        self._bound: dict = {}
        self._h2d = self._d2h = None
        self.stream_bytes = (0, 0)  # (h2d, d2h) bytes of the last step_host

    # -- setup -------------------------------------------------------------------------
    def attach_peers(self) -> None:
        """Fused halo: map the neighbours' evisc/u/v/w and point the slab
        launch's peer arguments at them (collective over the ranks when the
        exchanger maps IPC memory; done once, on first use)."""
        if self._peers_attached:
            return
        lay = self.layout
        names = PEER_KERNELS[self.problem.kernel]
        got = self.exchanger.peer_fields({n: self.problem.field_ptr(n) for n in names}, lay.kstart, lay.kend)
        sides = {}
        for side, (ptrs, ks, ke) in got.items():
            # the neighbour's allocation differs from ours only in its plane count
            count = lay.span_elems + ((ke - ks) - (lay.kend - lay.kstart)) * lay.kk
            sides[side] = (ptrs, count, ke if side == "below" else ks)
        self.problem.set_peers(below=sides.get("below"), above=sides.get("above"))
        self.args = {name: self.problem.args(rng) for name, rng in self.ranges.items()}
        self._peers_attached = True

    def resolve(self) -> dict:
        """Select + compile every sub-range before timing; returns name -> (config, match_kind)."""
        self.attach_peers()
        out = {}
        for name, args in self.args.items():
            report = self.wisdom.launch(self.ctx.ident, args, stream=self.compute)
            self.reports[name] = report
            out[name] = (report.configuration, report.match_kind)
        self.compute.synchronize()
        self.problem.regenerate(self.problem.outputs())
        # bound launches for the steady state (one C-ABI call per sub-range)
        self._bound = {name: self.wisdom.bind(self.ctx.ident, args, stream=self.compute)
                       for name, args in self.args.items()}
        return out

    @property
    def local_cells(self) -> int:
        return self.layout.cells

    def cells_in(self, name: str) -> int:
        kb, ke = self.ranges[name]
        return self.layout.itot * self.layout.jtot * (ke - kb)

    # -- one application step -------------------------------------------------------------
    def exchange(self, after: Event | None = None) -> None:
        """Halo exchange on the comm stream, ordered after ``after`` (default:
        the work enqueued on the compute stream so far)."""
        if self.exchanger is None:
            return
        if after is None:
            after = self._ev_start.record(self.compute)
        self.comm.wait(after)
        lay = self.layout
        # fields with the same reach share one NCCL group (diff_uvw: all four)
        groups: dict[tuple[int, int], list[int]] = {}
        for field, reach in HALO_REACH[self.kernel].items():
            groups.setdefault(reach, []).append(self.problem.field_ptr(field))
        for (down, up), ptrs in groups.items():
            self.exchanger.exchange(self.comm, ptrs, lay.elem_bytes, lay.kk, lay.kstart, lay.kend, down, up,
                                    self.below, self.above)
        self._ev_halo.record(self.comm)

    def step(self, time_kernel: tuple[Event, Event] | None = None) -> int:
        """Enqueue one step; returns the number of kernels launched."""
        ident = self.ctx.ident
        bound = self._bound

        def run(name):
            if name in bound:
                bound[name]()
            else:
                self.wisdom.launch(ident, self.args[name], stream=self.compute)

        if self.fused:
            self.attach_peers()
            ex = self.exchanger
            if ex is not None:
                ex.fence_ready(self.compute, self.below, self.above)
            if time_kernel is not None:
                time_kernel[0].record(self.compute)
            run("slab")
            if time_kernel is not None:
                time_kernel[1].record(self.compute)
            if ex is not None:
                ex.fence_done(self.compute, self.below, self.above)
            return 1
        self.exchange()
        launched = 0

        if "interior" in self.args:
            if time_kernel is not None:
                time_kernel[0].record(self.compute)
            run("interior")
            if time_kernel is not None:
                time_kernel[1].record(self.compute)
            launched += 1
        if self.exchanger is not None:
            self.compute.wait(self._ev_halo)
        for name in ("lower", "upper"):
            if name in self.args:
                run(name)
                launched += 1
        return launched

    # -- RK3 time loop (diff_uvw_rk3) ----------------------------------------------------
    #: MicroHH's low-storage RK3 (Williamson) coefficients
    RK3_A = (0.0, -5.0 / 9.0, -153.0 / 128.0)
    RK3_B = (1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0)

    def rk3_substep(self, s: int, dt: float) -> int:
        """Substep ``s`` (0, 1, 2, ... — three per time step) of a low-storage
        RK3 time loop over the slab with diff_uvw_rk3: the tendencies T = t +
        diffusion give t <- A[(s+1)%3] T and next <- cur + B[s%3] dt T, where
        cur / next are (u, v, w) / (u_next, v_next, w_next) on even substeps
        and swapped on odd ones (the buffers alternate); then the x/y ghost
        cells of next are refilled periodically (``klb_cyclic_xy``).  With
        ``halo="fused"`` the launch reads the neighbours' current fields
        through their peer mappings — no exchange; the fences order it after
        the neighbours' previous substep and before their next one.  Returns
        the number of kernel launches (2: the stencil and the ghost fill)."""
        from .cuda._abi import check, lib

        if self.kernel != "diff_uvw_rk3" or (self.nranks > 1 and not self.fused):
            raise ValueError("rk3_substep runs diff_uvw_rk3 (with halo='fused' when the grid is decomposed)")
        parity = s % 2
        args = self._rk3_args(parity, s % 3, dt)
        if self.exchanger is not None and self.nranks > 1:
            self.exchanger.fence_ready(self.compute, self.below, self.above)
        self.wisdom.launch(self.ctx.ident, args, stream=self.compute)
        lay = self.layout
        for name in (("u_next", "v_next", "w_next") if parity == 0 else ("u", "v", "w")):
            check(lib().klb_cyclic_xy(self.problem.field_ptr(name), lay.elem_bytes, 0, lay.icells, lay.jcells,
                                      lay.jj, lay.kk, lay.igc, lay.jgc, lay.kstart, lay.kend, self.compute.handle))
        if self.exchanger is not None and self.nranks > 1:
            self.exchanger.fence_done(self.compute, self.below, self.above)
        return 2

    def _rk3_args(self, parity: int, sub: int, dt: float) -> list:
        """Launch arguments of substep parity / RK stage (memoised): the
        current/next buffers swapped on odd substeps, the neighbours' current
        fields as the peer arguments, the stage's coefficients."""
        key = (parity, sub, dt)
        cache = self._rk3_cache
        if key in cache:
            return cache[key]
        from .capture import ScalarArg
        from .cuda.device import DeviceBuffer
        from .stencils.definitions import ARG_LAYOUT

        prob = self.problem
        if self.fused and self.exchanger is not None and self.nranks > 1:
            peers = self._rk3_peers
            if not peers:  # collective, same order on every rank: both buffer sets of the neighbours
                lay = self.layout
                for par, names in ((0, ("u", "v", "w")), (1, ("u_next", "v_next", "w_next"))):
                    ptrs = {"evisc": prob.field_ptr("evisc")}
                    ptrs.update({f: prob.field_ptr(n) for f, n in zip(("u", "v", "w"), names)})
                    got = self.exchanger.peer_fields(ptrs, lay.kstart, lay.kend)
                    peers[par] = {side: (p, lay.span_elems + ((ke - ks) - (lay.kend - lay.kstart)) * lay.kk,
                                         ke if side == "below" else ks) for side, (p, ks, ke) in got.items()}
            prob.set_peers(below=peers[parity].get("below"), above=peers[parity].get("above"))
        args = prob.args(self.ranges["slab"] if self.fused else None)
        layout = ARG_LAYOUT[prob.kernel]
        pos = {name: i for i, (name, _) in enumerate(layout["buffers"])}
        if parity:
            for a, b in (("u", "u_next"), ("v", "v_next"), ("w", "w_next")):
                ia, ib = pos[a], pos[b]
                da, db = args[ia], args[ib]
                args[ia] = DeviceBuffer(ia, da.role, da.element_type, db.ptr, db.element_count, owner=db.owner)
                args[ib] = DeviceBuffer(ib, db.role, db.element_type, da.ptr, da.element_count, owner=da.owner)
        nb = len(layout["buffers"])
        for name, value in (("rk_a", self.RK3_A[(sub + 1) % 3]), ("rk_bdt", self.RK3_B[sub] * dt)):
            i = nb + layout["scalars"].index(name)
            args[i] = ScalarArg(i, args[i].dtype, value)
        cache[key] = args
        return args

    def step_host(self, host: dict[str, int], chunks: int = 16, copy_streams: int = 1) -> int:
        """One step streamed from/to pinned host memory (``stream.py``).

        ``host`` maps every field to a pinned host buffer laid out exactly like
        the device allocation (``layout.alloc_bytes``); inputs and RMW outputs
        are read from it, the tendencies written back.  Enqueued on the
        compute, h2d, d2h (and comm) streams and joined back into ``compute``;
        returns the number of kernels launched.  ``copy_streams`` > 1 spreads
        the chunks' uploads (and downloads) round-robin over that many
        streams per direction, so several copy engines share the link."""
        from .cuda._abi import check, lib
        from .stream import stream_plan

        if self.fused:
            raise ValueError("step_host streams the exchange variant (halo='exchange')")
        lay = self.layout
        if self._stream_state is None or self._stream_state[0] != (chunks, copy_streams):
            fields = tuple(self.problem.fields)
            plan = stream_plan(self.kernel, fields, self.problem.outputs(), self.ranges, lay.kcells, lay.kstart,
                               lay.kend, self.below, self.above, chunks)
            args = {st.name: self.problem.args(st.k_range) for st in plan}
            events = [(Event(), Event()) for _ in plan]
            if self._h2d is None or len(self._h2d) != copy_streams:
                for st in (self._h2d or []) + (self._d2h or []):
                    st.close()
                self._h2d = [Stream.create() for _ in range(copy_streams)]
                self._d2h = [Stream.create() for _ in range(copy_streams)]
                self._ev_join = [Event() for _ in range(copy_streams)]
            self._stream_state = ((chunks, copy_streams), plan, args, events)
        _, plan, args, events = self._stream_state
        ns = len(self._h2d)
        plane = lay.kk * lay.elem_bytes
        lead = lay.lead * lay.elem_bytes
        dev = {n: a.ptr for n, a in self.problem.fields.items()}
        ident = self.ctx.ident

        start = self._ev_start.record(self.compute)
        for st in self._h2d + self._d2h:
            st.wait(start)
        n_boundary = sum(1 for st in plan if st.after_halo)
        for i, st in enumerate(plan):
            up = self._h2d[i % ns]
            for c in st.uploads:
                off = lead + c.p0 * plane
                check(lib().klb_memcpy_htod(dev[c.field] + off, host[c.field] + off, (c.p1 - c.p0) * plane,
                                            up.handle))
            events[i][0].record(up)
            if self.exchanger is not None and i + 1 == max(n_boundary, 1):
                self.exchange(after=events[i][0])
        order = [i for i, st in enumerate(plan) if not st.after_halo] + [i for i, st in enumerate(plan) if st.after_halo]
        waited_halo = False
        for i in order:
            st = plan[i]
            self.compute.wait(events[i][0])
            if st.after_halo and self.exchanger is not None and not waited_halo:
                self.compute.wait(self._ev_halo)
                waited_halo = True
            self.wisdom.launch(ident, args[st.name], stream=self.compute)
            events[i][1].record(self.compute)
            down = self._d2h[i % ns]
            down.wait(events[i][1])
            for c in st.downloads:
                off = lead + c.p0 * plane
                check(lib().klb_memcpy_dtoh(host[c.field] + off, dev[c.field] + off, (c.p1 - c.p0) * plane,
                                            down.handle))
        if self.exchanger is not None and not waited_halo:
            self.compute.wait(self._ev_halo)
        for ev, down in zip(self._ev_join, self._d2h):
            self.compute.wait(ev.record(down))
        self.stream_bytes = (sum((c.p1 - c.p0) * plane for st in plan for c in st.uploads),
                             sum((c.p1 - c.p0) * plane for st in plan for c in st.downloads))
        return len(plan)

    def close(self) -> None:
        """Collective when the exchanger maps peer memory (IPC): every rank
        unmaps its neighbours' fields before any rank frees its own."""
        detach = getattr(self.exchanger, "detach", None)
        if callable(detach):
            detach([self.problem.field_ptr(n) for n in self.problem.fields])
        self.problem.close()
        if self.comm is not None:
            self.comm.close()
        for s in (self._h2d or []) + (self._d2h or []):
            s.close()
