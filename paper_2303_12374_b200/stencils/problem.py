"""Device-resident stencil problems: fields in HBM + the launch argument list.

``StencilProblem(kernel, layout, ctx)`` allocates every field the kernel
touches in the ghost-padded pitched layout (``layout.GridLayout``), fills them
on the device with the deterministic generator (``klb_synth_field``; the
oracle twin is ``oracle/synth.py``), uploads the 1-D profiles, and builds the
MicroHH-ordered argument list of ``DeviceBuffer`` / ``ScalarArg`` the
``WisdomKernel`` / ``CudaExecutable`` launch API takes (positions from
``definitions.ARG_LAYOUT``).

For z-slab decomposition (``k_offset``/``kcells_global``) a rank's local
fields hold global planes ``[k_offset, k_offset + layout.kcells)``; the
generator indexes by global plane, so a slab's ghost planes initially equal
its neighbours' interior planes, and the halo exchange keeps them so.
"""

from __future__ import annotations

import numpy as np

from ..capture import ScalarArg
from ..cuda._abi import check, lib
from ..cuda.device import DeviceArray, DeviceBuffer, DeviceContext, Stream
from .definitions import ARG_LAYOUT, definition_for
from .layout import GridLayout
from .profiles import FIELD_SEED_BASE, FIELD_SPECS, Profiles, make_profiles

__all__ = ["StencilProblem", "KERNEL_FIELDS", "BYTES_PER_CELL_WORDS", "PEER_KERNELS"]

KERNEL_FIELDS = {
    "advec_u": ("ut", "u", "v", "w"),
    "diff_uvw": ("ut", "vt", "wt", "evisc", "u", "v", "w"),
    "advec_v": ("vt", "u", "v", "w"),
    "advec_w": ("wt", "u", "v", "w"),
    "advec_s": ("st", "s", "u", "v", "w"),
    "diff_c": ("st", "s", "evisc"),
    "evisc_smag": ("evisc", "u", "v", "w"),
    "diff_uvw_rk3": ("ut", "vt", "wt", "evisc", "u", "v", "w", "u_next", "v_next", "w_next"),
    "diff_uvw_peer": ("ut", "vt", "wt", "evisc", "u", "v", "w"),
    "advec_u_peer": ("ut", "u", "v", "w"),
    "diff_uvw_rk3_peer": ("ut", "vt", "wt", "evisc", "u", "v", "w", "u_next", "v_next", "w_next"),
    "rk3_uvw": ("ut", "vt", "wt", "u", "v", "w"),
}
#: algorithmic HBM words per interior cell: advec_u reads u,v,w,ut
#: and writes ut; diff_uvw reads evisc,u,v,w,ut,vt,wt and writes ut,vt,wt;
#: advec_v/w as advec_u; advec_s reads s,u,v,w,st and writes st; diff_c reads
#: s,evisc,st and writes st; evisc_smag reads u,v,w and writes evisc.
BYTES_PER_CELL_WORDS = {"advec_u": 5, "diff_uvw": 10, "advec_v": 5, "advec_w": 5, "advec_s": 6, "diff_c": 4,
                        "evisc_smag": 4,
                        # diff_uvw + RK3 epilogue: reads evisc,u,v,w,ut,vt,wt, writes ut,vt,wt,u',v',w'
                        "diff_uvw_rk3": 13,
                        # diff_uvw with its z-halo read from the neighbours' fields: same words per cell
                        "diff_uvw_peer": 10, "advec_u_peer": 5, "diff_uvw_rk3_peer": 13,
                        # the separate RK3 pass: read + write u,v,w,ut,vt,wt
                        "rk3_uvw": 12}
#: MicroHH defaults of the model constants the family kernels take
TPRI = 3.0  # 1 / Pr_t (Pr_t = 1/3)
CS = 0.23   # Smagorinsky constant
#: RK3 substep used by diff_uvw_rk3 / rk3_uvw: MicroHH's second substep of the
#: Williamson low-storage scheme (cA = -5/9, cB = 15/16) with dt = 0.01
RK_A = -5.0 / 9.0
RK_BDT = 15.0 / 16.0 * 0.01
_PROFILE_FIELDS = ("rhoref", "rhorefh", "dzi", "dzhi")
#: the fused-halo kernels' neighbour-field arguments -> the local field they mirror
_PEER_FIELDS = {f"{f}_{side}": f for side in ("lo", "hi") for f in ("evisc", "u", "v", "w")}
#: fields each fused-halo kernel reads from its neighbours (its halo'd inputs)
PEER_KERNELS = {"diff_uvw_peer": ("evisc", "u", "v", "w"), "advec_u_peer": ("u", "w"),
                "diff_uvw_rk3_peer": ("evisc", "u", "v", "w")}
#: peer_klo / peer_khi of a side without a neighbour: a plane no launch reaches
_NO_PEER = 1 << 30


class StencilProblem:
    def __init__(self, kernel: str, layout: GridLayout, ctx: DeviceContext, *, k_offset: int = 0,
                 kcells_global: int | None = None, profiles: Profiles | None = None,
                 dxi: float = 1.0, dyi: float = 1.0, tpri: float = TPRI, cs: float = CS,
                 rk_a: float = RK_A, rk_bdt: float = RK_BDT, stream: Stream | None = None) -> None:
        if kernel not in ARG_LAYOUT:
            raise ValueError(f"unknown kernel {kernel!r}")
        self.kernel = kernel
        self.layout = layout
        self.ctx = ctx
        self.k_offset = k_offset
        self.kcells_global = kcells_global if kcells_global is not None else layout.kcells
        self.definition = definition_for(kernel, layout.precision)
        self.dxi, self.dyi = dxi, dyi
        self.tpri, self.cs = tpri, cs
        self.rk_a, self.rk_bdt = rk_a, rk_bdt
        self.stream = stream or ctx.stream
        glob = profiles if profiles is not None else make_profiles(self.kcells_global, layout.kgc)
        self.profiles = glob.window(k_offset, layout.kcells).as_dtype(layout.dtype)
        self.fields: dict[str, DeviceArray] = {}
        self._borrowed: set[str] = set()  # fields aliased from another problem (share_fields)
        # diff_uvw_peer: neighbour fields (name -> (pointer, element count)) and
        # (peer_klo, peer_khi, peer_shift_lo, peer_shift_hi); default: none
        self.peers: dict[str, tuple[int, int]] = {}
        self.peer_bounds = (-_NO_PEER, _NO_PEER, 0, 0)
        for name in KERNEL_FIELDS[kernel]:
            arr = DeviceArray(layout.alloc_bytes)
            arr.zero(self.stream)
            self.fields[name] = arr
        self.regenerate()
        self.profile_arrays: dict[str, DeviceArray] = {}
        for name in _PROFILE_FIELDS:
            data = np.ascontiguousarray(getattr(self.profiles, name))
            arr = DeviceArray(data.nbytes)
            arr.upload(data, stream=self.stream)
            self.profile_arrays[name] = arr
        self._args = self._build_args()

    # -- data ----------------------------------------------------------------------
    def regenerate(self, names=None) -> None:
        """(Re)fill fields with the deterministic synthetic values."""
        lay = self.layout
        for name in names or self.fields:
            seed_off, lo, hi = FIELD_SPECS[name]
            check(lib().klb_synth_field(
                self.fields[name].ptr, lay.elem_bytes, lay.lead, lay.icells, lay.jcells, lay.kcells, lay.jj, lay.kk,
                lay.igc, lay.jgc, self.k_offset, self.kcells_global, FIELD_SEED_BASE + seed_off, lo, hi, 1,
                self.stream.handle))
        self.stream.synchronize()

    def field_ptr(self, name: str) -> int:
        """Device pointer of element (0, 0, 0) — what kernels receive."""
        return self.fields[name].ptr + self.layout.lead * self.layout.elem_bytes

    def download(self, name: str) -> np.ndarray:
        """(kcells, jcells, icells) host view of a field."""
        flat = self.fields[name].download_array(self.layout.dtype)
        return self.layout.host_view(flat)

    def outputs(self) -> tuple[str, ...]:
        return tuple(n for n, role in ARG_LAYOUT[self.kernel]["buffers"] if role == "output")

    # -- launch arguments --------------------------------------------------------------
    def _build_args(self) -> list:
        lay = self.layout
        elem = lay.element_type
        args: list = []
        pos = 0
        for name, role in ARG_LAYOUT[self.kernel]["buffers"]:
            if name in self.fields:
                args.append(DeviceBuffer(pos, role, elem, self.field_ptr(name), lay.span_elems, owner=self.fields[name]))
            elif name in _PEER_FIELDS:  # no neighbour on that side: the local field, never reached
                local = _PEER_FIELDS[name]
                ptr, count = self.peers.get(name, (self.field_ptr(local), lay.span_elems))
                args.append(DeviceBuffer(pos, role, elem, ptr, count, owner=self.fields[local]))
            else:
                arr = self.profile_arrays[name]
                args.append(DeviceBuffer(pos, role, elem, arr.ptr, arr.nbytes // lay.elem_bytes, owner=arr))
            pos += 1
        scalars = {
            "dxi": (elem, self.dxi), "dyi": (elem, self.dyi), "jj": ("i32", lay.jj), "kk": ("i32", lay.kk),
            "istart": ("i32", lay.istart), "jstart": ("i32", lay.jstart), "kstart": ("i32", lay.kstart),
            "iend": ("i32", lay.iend), "jend": ("i32", lay.jend), "kend": ("i32", lay.kend),
            "tpri": (elem, self.tpri), "cs": (elem, self.cs), "rk_a": (elem, self.rk_a),
            "rk_bdt": (elem, self.rk_bdt),
            "peer_klo": ("i32", self.peer_bounds[0]), "peer_khi": ("i32", self.peer_bounds[1]),
            "peer_shift_lo": ("i32", self.peer_bounds[2]), "peer_shift_hi": ("i32", self.peer_bounds[3]),
        }
        for name in ARG_LAYOUT[self.kernel]["scalars"]:
            dtype, value = scalars[name]
            args.append(ScalarArg(pos, dtype, value))
            pos += 1
        return args

    def args(self, k_range: tuple[int, int] | None = None) -> list:
        """Launch args, optionally restricted to local planes ``[kb, ke)``."""
        if k_range is None:
            return list(self._args)
        kb, ke = k_range
        pos_ks = len(ARG_LAYOUT[self.kernel]["buffers"]) + ARG_LAYOUT[self.kernel]["scalars"].index("kstart")
        pos_ke = len(ARG_LAYOUT[self.kernel]["buffers"]) + ARG_LAYOUT[self.kernel]["scalars"].index("kend")
        out = list(self._args)
        out[pos_ks] = ScalarArg(pos_ks, "i32", kb)
        out[pos_ke] = ScalarArg(pos_ke, "i32", ke)
        return out

    def set_peers(self, below=None, above=None) -> None:
        """diff_uvw_peer / advec_u_peer: read the planes outside this slab
        from the neighbours' fields.  ``below`` / ``above`` = ``(pointers,
        element count, plane)``: the neighbour's field pointers of element
        (0,0,0) by name (``PEER_KERNELS[kernel]``; device memory this context can address — a CUDA
        IPC mapping or another allocation of this device), the element count
        from there (its ``layout.span_elems``) and its local ``kend`` (below)
        / ``kstart`` (above), so that local plane ``kstart - 1`` maps to
        ``kend_below - 1`` and ``kend`` to ``kstart_above``."""
        if self.kernel not in PEER_KERNELS:
            raise ValueError(f"set_peers applies to the fused-halo kernels {tuple(PEER_KERNELS)}")
        lay = self.layout
        peers: dict[str, tuple[int, int]] = {}
        klo, khi, shlo, shhi = -_NO_PEER, _NO_PEER, 0, 0
        for side, info in (("lo", below), ("hi", above)):
            if info is None:
                continue
            ptrs, count, plane = info
            for f in PEER_KERNELS[self.kernel]:
                if (ptrs[f] - self.field_ptr(f)) % 16:
                    raise ValueError(f"peer {f}_{side} has another 16-byte phase than the local field")
                peers[f"{f}_{side}"] = (int(ptrs[f]), int(count))
            if side == "lo":
                klo, shlo = lay.kstart, int(plane) - lay.kstart
            else:
                khi, shhi = lay.kend, int(plane) - lay.kend
        self.peers, self.peer_bounds = peers, (klo, khi, shlo, shhi)
        self._args = self._build_args()

    def share_fields(self, other: "StencilProblem", names) -> None:
        """Use ``other``'s device buffers for ``names`` — kernels chained in one
        time step (evisc_smag's evisc feeding diff_uvw, the tendencies the
        advection and diffusion kernels accumulate into) read and write the
        same fields instead of copies.  The borrowed buffers stay owned by
        ``other``; ``regenerate`` refills them like this problem's own."""
        if other.layout != self.layout:
            raise ValueError("shared fields need identical layouts")
        for name in names:
            if name not in self.fields or name not in other.fields:
                raise KeyError(f"{name!r} is not a field of both {self.kernel} and {other.kernel}")
            if name not in self._borrowed:
                self.fields[name].free()
            self.fields[name] = other.fields[name]
            self._borrowed.add(name)
        self._args = self._build_args()

    def scalar_env(self) -> dict[str, int]:
        from ..capture import scalar_env_from_args

        return scalar_env_from_args(self._args)

    @property
    def algorithmic_bytes(self) -> int:
        return BYTES_PER_CELL_WORDS[self.kernel] * self.layout.elem_bytes * self.layout.cells

    def close(self) -> None:
        own = [a for n, a in self.fields.items() if n not in self._borrowed]
        for arr in own + list(self.profile_arrays.values()):
            arr.free()
        self.fields.clear()
        self.profile_arrays.clear()
