"""Multi-GPU z-slab decomposition with halo exchange.

The global (itot, jtot, ktot) grid is cut into contiguous z-slabs, one per
rank; each rank holds its slab plus ``kgc`` ghost planes on both sides in the
same pitched layout as a single-GPU grid.  One application step:

    comm stream    : exchange halo planes of the INPUT fields with rank r+-1
    compute stream : stencil over interior planes [kstart+h_lo, kend-h_hi)
                     (reads no ghost plane -> overlaps the exchange)
                     wait(exchange) ; stencil over the boundary planes

The exchange only writes ghost planes and only reads interior input planes,
while the interior launch only reads interior input planes and writes the
(output) tendency fields, so the overlap is race-free by construction.  Each
sub-range is its own problem size, so ``WisdomKernel`` selects a separate
configuration for it (the paper's per-problem selection).

Exchange plan (``halo_plan``) — every rank passes the same per-field reach:
  ``down`` = planes a rank reads ABOVE its slab (stencil reach towards +k),
  ``up``   = planes it reads BELOW its slab (reach towards -k);
  send [kstart, kstart+down) -> below   | recv [kstart-up, kstart) <- below
  send [kend-up, kend)       -> above   | recv [kend, kend+down)   <- above
This is the protocol ``klb_halo_exchange_z`` (NCCL send/recv) and
``klb_halo_pull_z`` (peer memory over CUDA IPC, ``IpcExchanger``: the
receiver-side half of the plan, copy engines reading the neighbour's planes
over NVLink) implement in C; the ``CopyExchanger`` (several virtual ranks on
one GPU, D2D copies) implements the same plan in Python, and so does the
CPU-test transport over gloo (tests/test_halo.py).

Reach per kernel (from the stencil definitions):
  advec_u : u (down 3, up 3), w (down 1, up 0), v none
  diff_uvw: evisc, u, v, w (down 1, up 1)
  (the §8f family in HALO_REACH below, from oracle/family_oracle.py)
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

__all__ = [
    "HALO_REACH", "SlabDecomposition", "halo_plan", "NcclExchanger", "IpcExchanger", "CopyExchanger", "LocalPeers",
    "SlabRank",
]

#: kernel -> {field: (down, up)}
HALO_REACH = {
    "advec_u": {"u": (3, 3), "w": (1, 0)},
    "diff_uvw": {"evisc": (1, 1), "u": (1, 1), "v": (1, 1), "w": (1, 1)},
    "advec_v": {"v": (3, 3), "w": (1, 0)},
    "advec_w": {"w": (3, 3), "u": (0, 1), "v": (0, 1)},
    "advec_s": {"s": (3, 3), "w": (1, 0)},
    "diff_c": {"s": (1, 1), "evisc": (1, 1)},
    "evisc_smag": {"u": (1, 1), "v": (1, 1), "w": (1, 0)},
    "diff_uvw_rk3": {"evisc": (1, 1), "u": (1, 1), "v": (1, 1), "w": (1, 1)},
    "diff_uvw_peer": {"evisc": (1, 1), "u": (1, 1), "v": (1, 1), "w": (1, 1)},
    "advec_u_peer": {"u": (3, 3), "w": (1, 0)},
    "diff_uvw_rk3_peer": {"evisc": (1, 1), "u": (1, 1), "v": (1, 1), "w": (1, 1)},
    "rk3_uvw": {},
}


def kernel_reach(kernel: str) -> tuple[int, int]:
    """(max down, max up) over the kernel's exchanged fields."""
    reach = HALO_REACH[kernel].values()
    return max((d for d, _ in reach), default=0), max((u for _, u in reach), default=0)


@dataclass(frozen=True)
class SlabDecomposition:
    """Split ``ktot`` interior planes over ``nranks`` (sizes differ by <= 1)."""

    ktot: int
    nranks: int

    def __post_init__(self) -> None:
        if self.nranks < 1 or self.ktot < self.nranks:
            raise ValueError("need 1 <= nranks <= ktot")

    def planes(self, rank: int) -> tuple[int, int]:
        """(global interior offset, plane count) of ``rank``'s slab."""
        base, extra = divmod(self.ktot, self.nranks)
        count = base + (1 if rank < extra else 0)
        offset = rank * base + min(rank, extra)
        return offset, count

    def neighbours(self, rank: int) -> tuple[int, int]:
        below = rank - 1 if rank > 0 else -1
        above = rank + 1 if rank < self.nranks - 1 else -1
        return below, above


def halo_plan(kstart: int, kend: int, down: int, up: int, below: int, above: int):
    """List of (op, peer, first_plane, nplanes) for one field, in issue order."""
    ops = []
    if below >= 0:
        if down:
            ops.append(("send", below, kstart, down))
        if up:
            ops.append(("recv", below, kstart - up, up))
    if above >= 0:
        if up:
            ops.append(("send", above, kend - up, up))
        if down:
            ops.append(("recv", above, kend, down))
    return ops


class NcclExchanger:
    """Halo exchange over NCCL point-to-point (one communicator per job)."""

    def __init__(self, rank: int, nranks: int, unique_id: bytes) -> None:
        from .cuda._abi import check, lib

        self.rank, self.nranks = rank, nranks
        comm = C.c_void_p()
        uid = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        check(lib().klb_nccl_comm_init(C.byref(comm), nranks, uid, rank))
        self.comm = comm.value

    @staticmethod
    def unique_id() -> bytes:
        from .cuda._abi import check, lib

        buf = (C.c_ubyte * 128)()
        check(lib().klb_nccl_unique_id(buf))
        return bytes(buf)

    def exchange(self, stream, ptrs, elem_bytes: int, kk: int, kstart: int, kend: int, down: int, up: int,
                 below: int, above: int) -> None:
        from .cuda._abi import check, lib

        arr = (C.c_uint64 * len(ptrs))(*ptrs)
        check(lib().klb_halo_exchange_z(self.comm, stream.handle, len(ptrs), arr, elem_bytes, kk, kstart, kend, down,
                                        up, below, above))

    def close(self) -> None:
        from .cuda._abi import lib

        if self.comm:
            lib().klb_nccl_comm_destroy(self.comm)
            self.comm = None


class IpcExchanger:
    """Halo exchange over peer memory (CUDA IPC), receiver-pulled.

    Each rank maps its neighbours' field allocations once
    (``klb_ipc_mem_handle`` / ``klb_ipc_mem_open``: over NVLink between GPUs,
    or another process's allocation on the same GPU) and pulls the planes it
    needs into its own ghost planes with copy-engine copies
    (``klb_halo_pull_z``) on the comm stream, overlapped with the interior
    launch.  Ordering across processes uses interprocess events, made
    race-free by two host barriers of the ``ProcessGroup`` per exchange::

        comm: record ready      (my input planes are final for this step)
        ---- barrier A ----     (every rank's ready is enqueued)
        comm: wait ready(below, above); pull their planes; record pulled
        ---- barrier B ----     (every rank's pulled is enqueued)
        comm: wait pulled(below, above)

    The last wait orders everything after the exchange on this rank — the
    boundary launches and any later write of the inputs by the application —
    after the neighbours have finished reading this rank's planes (no
    write-after-read race in a time loop).  The barriers only order host
    enqueues; the GPU never waits on the host.  Same ``exchange`` signature as
    ``NcclExchanger``; the plan is ``halo_plan``'s receiver side."""

    def __init__(self, group) -> None:
        from .cuda._abi import check, lib

        self.group = group
        self.rank, self.nranks = group.rank, group.nranks
        self._events = []
        handles = []
        for _ in range(2):  # ready, pulled
            ev = C.c_void_p()
            h = (C.c_ubyte * 64)()
            check(lib().klb_ipc_event_create(C.byref(ev), h))
            self._events.append(ev.value)
            handles.append(bytes(h))
        self.ready, self.pulled = self._events
        peers = group.allgather(b"".join(handles))
        self._peer_events: dict[int, tuple[int, int]] = {}
        for r in (self.rank - 1, self.rank + 1):
            if 0 <= r < self.nranks:
                evs = []
                for i in range(2):
                    ev = C.c_void_p()
                    h = (C.c_ubyte * 64).from_buffer_copy(peers[r][64 * i:64 * (i + 1)])
                    check(lib().klb_ipc_event_open(h, C.byref(ev)))
                    evs.append(ev.value)
                self._peer_events[r] = tuple(evs)
        self._maps: dict[tuple, dict] = {}  # (local pointer tuple, kstart, kend) -> peer mappings
        self._opened: dict[tuple, list[int]] = {}  # same key -> the mapped bases to close

    @staticmethod
    def probe(group) -> tuple[bool, str]:
        """Collective: can every rank map its neighbours' device memory and
        open their interprocess events?  Each rank exports a small buffer and
        an event, opens its neighbours', copies one value from each, and the
        outcome is agreed over the group (every rank returns the same
        ``(ok, reason)``), so a job falls back to another transport as a whole."""
        import struct

        from .cuda._abi import KlbError, check, lib
        from .cuda.device import DeviceArray

        buf = DeviceArray(256)
        mark = struct.pack("<Q", 0x6B6C62000000 + group.rank)
        ev = C.c_void_p()
        opened, peer_events, why = [], [], ""
        try:
            check(lib().klb_memcpy_htod(buf.ptr, mark, 8, None))
            check(lib().klb_device_synchronize())
            h, off, eh = (C.c_ubyte * 64)(), C.c_uint64(), (C.c_ubyte * 64)()
            check(lib().klb_ipc_mem_handle(buf.ptr, h, C.byref(off)))
            check(lib().klb_ipc_event_create(C.byref(ev), eh))
            blob = bytes(h) + struct.pack("<Q", off.value) + bytes(eh)
        except KlbError as err:
            blob, why = b"\0" * 136, f"rank {group.rank}: export failed: {err}"
        peers = group.allgather(blob)
        ok = not why
        for r in (group.rank - 1, group.rank + 1):
            if not ok or not 0 <= r < group.nranks:
                continue
            try:
                base = C.c_uint64()
                check(lib().klb_ipc_mem_open((C.c_ubyte * 64).from_buffer_copy(peers[r][:64]), C.byref(base)))
                opened.append(base.value)
                off_r, = struct.unpack_from("<Q", peers[r], 64)
                got = C.create_string_buffer(8)
                check(lib().klb_memcpy_dtoh(got, base.value + off_r, 8, None))
                check(lib().klb_device_synchronize())
                if got.raw != struct.pack("<Q", 0x6B6C62000000 + r):
                    raise KlbError(-1, "peer value mismatch")
                pe = C.c_void_p()
                check(lib().klb_ipc_event_open((C.c_ubyte * 64).from_buffer_copy(peers[r][72:136]), C.byref(pe)))
                peer_events.append(pe.value)
            except KlbError as err:
                ok, why = False, f"rank {group.rank}: peer {r}: {err}"
        verdict = group.allgather(struct.pack("<?", ok) + why.encode()[:200].ljust(200, b"\0"))
        group.barrier()  # every peer finished reading before anything is unmapped / freed
        for base in opened:
            lib().klb_ipc_mem_close(base)
        for pe in peer_events:
            lib().klb_event_destroy(pe)
        if ev.value:
            lib().klb_event_destroy(ev.value)
        group.barrier()
        buf.free()
        bad = [v[1:].rstrip(b"\0").decode(errors="replace") for v in verdict if not v[0]]
        return (not bad), "; ".join(bad)

    def _attach(self, ptrs, kstart: int, kend: int) -> dict:
        """Collective on first use of a field set: map the neighbours' fields."""
        import struct

        from .cuda._abi import check, lib

        key = (tuple(ptrs), kstart, kend)
        entry = self._maps.get(key)
        if entry is not None:
            return entry
        blob = struct.pack("<ii", kstart, kend)
        for p in ptrs:
            h = (C.c_ubyte * 64)()
            off = C.c_uint64()
            check(lib().klb_ipc_mem_handle(p, h, C.byref(off)))
            blob += bytes(h) + struct.pack("<Q", off.value)
        allb = self.group.allgather(blob)
        entry = {}
        for side, r in (("below", self.rank - 1), ("above", self.rank + 1)):
            if not 0 <= r < self.nranks:
                continue
            ks, ke = struct.unpack_from("<ii", allb[r], 0)
            mapped = []
            for i in range(len(ptrs)):
                at = 8 + 72 * i
                h = (C.c_ubyte * 64).from_buffer_copy(allb[r][at:at + 64])
                off, = struct.unpack_from("<Q", allb[r], at + 64)
                base = C.c_uint64()
                check(lib().klb_ipc_mem_open(h, C.byref(base)))
                self._opened.setdefault(key, []).append(base.value)
                mapped.append(base.value + off)
            entry[side] = (mapped, ks, ke)
        self._maps[key] = entry
        return entry

    def peer_fields(self, fields: dict[str, int], kstart: int, kend: int) -> dict:
        """Collective: the neighbours' pointers of ``fields`` (name -> local
        pointer) mapped into this process, ``{"below"|"above": (name ->
        pointer, their kstart, their kend)}`` — what the fused-halo kernel
        (diff_uvw_peer) reads the planes outside the slab from."""
        names = list(fields)
        entry = self._attach([fields[n] for n in names], kstart, kend)
        return {side: (dict(zip(names, mapped)), ks, ke) for side, (mapped, ks, ke) in entry.items()}

    def fence_ready(self, stream, below: int, above: int) -> None:
        """Order ``stream`` after the neighbours' work that produced their
        input planes (each rank records, a host barrier, each waits)."""
        from .cuda._abi import check, lib

        check(lib().klb_event_record(self.ready, stream.handle))
        self.group.barrier()
        for r in (below, above):
            if r >= 0:
                check(lib().klb_stream_wait_event(stream.handle, self._peer_events[r][0]))

    def fence_done(self, stream, below: int, above: int) -> None:
        """Order ``stream``'s later work after the neighbours have finished
        reading this rank's planes (no write-after-read race in a time loop)."""
        from .cuda._abi import check, lib

        check(lib().klb_event_record(self.pulled, stream.handle))
        self.group.barrier()
        for r in (below, above):
            if r >= 0:
                check(lib().klb_stream_wait_event(stream.handle, self._peer_events[r][1]))

    def exchange(self, stream, ptrs, elem_bytes: int, kk: int, kstart: int, kend: int, down: int, up: int,
                 below: int, above: int) -> None:
        from .cuda._abi import check, lib

        entry = self._attach(ptrs, kstart, kend)
        n = len(ptrs)
        self.fence_ready(stream, below, above)
        arr = (C.c_uint64 * n)(*ptrs)
        lo = (C.c_uint64 * n)(*entry["below"][0]) if below >= 0 else None
        hi = (C.c_uint64 * n)(*entry["above"][0]) if above >= 0 else None
        below_kend = entry["below"][2] if below >= 0 else 0
        above_kstart = entry["above"][1] if above >= 0 else 0
        check(lib().klb_halo_pull_z(stream.handle, n, arr, lo, hi, elem_bytes, kk, kstart, kend, down, up,
                                    below_kend, above_kstart))
        self.fence_done(stream, below, above)

    def detach(self, ptrs=None) -> None:
        """Collective: unmap the neighbours' allocations mapped for field sets
        of the local pointers ``ptrs`` (all when None) — before the fields are
        freed.  Mappings of other field sets (another driver sharing this
        exchanger, e.g. a fused-halo slab launch holding peer pointers) stay."""
        from .cuda._abi import lib

        lib().klb_device_synchronize()
        self.group.barrier()  # nobody still copies from a mapping being closed
        mine = None if ptrs is None else set(ptrs)
        for key in list(self._maps):
            if mine is None or set(key[0]) <= mine:
                for base in self._opened.pop(key, []):
                    lib().klb_ipc_mem_close(base)
                del self._maps[key]
        self.group.barrier()  # every peer has unmapped before anyone frees

    def close(self) -> None:
        from .cuda._abi import lib

        if self._events:
            self.detach()
            for a, b in self._peer_events.values():
                lib().klb_event_destroy(a)
                lib().klb_event_destroy(b)
            for ev in self._events:
                lib().klb_event_destroy(ev)
            self._events, self._peer_events = [], {}


class LocalPeers:
    """Virtual ranks on ONE device for the fused-halo kernel: rank ``r``'s
    neighbours' fields are plain allocations of the same context, and every
    rank's launches go to one stream, so the fences are no-ops.  ``ranks[r]``
    = (field name -> pointer of element (0,0,0), kstart, kend) over all the
    rank's fields; ``for_rank(r)`` is the per-rank view ``SlabDriver(halo=
    "fused")`` takes as its exchanger.  As with ``IpcExchanger.peer_fields``
    (which pairs the ranks' pointer lists position by position) a request
    {key: my pointer} returns, per key, the neighbour's pointer of the SAME
    field as mine — so {"u": my u_next} yields the neighbour's u_next."""

    def __init__(self, ranks: list[tuple[dict[str, int], int, int]]) -> None:
        self.ranks = ranks

    def for_rank(self, r: int) -> "LocalPeers._View":
        return LocalPeers._View(self, r)

    class _View:
        def __init__(self, owner: "LocalPeers", rank: int) -> None:
            self.owner, self.rank = owner, rank

        def peer_fields(self, fields: dict[str, int], kstart: int, kend: int) -> dict:
            mine = {p: n for n, p in self.owner.ranks[self.rank][0].items()}
            out = {}
            for side, r in (("below", self.rank - 1), ("above", self.rank + 1)):
                if 0 <= r < len(self.owner.ranks):
                    ptrs, ks, ke = self.owner.ranks[r]
                    out[side] = ({k: ptrs[mine[p]] for k, p in fields.items()}, ks, ke)
            return out

        def fence_ready(self, stream, below: int, above: int) -> None:
            pass

        def fence_done(self, stream, below: int, above: int) -> None:
            pass


class CopyExchanger:
    """Virtual ranks on ONE device: the halo plan executed as D2D copies.

    ``ranks[r]`` maps field name -> device pointer of local element (0,0,0).
    Used to test the decomposition on a single GPU (gpurun gives one).
    """

    def __init__(self, ranks: list[dict[str, int]]) -> None:
        self.ranks = ranks

    def exchange_all(self, stream, fields: dict[str, tuple[int, int]], elem_bytes: int, kk: int,
                     bounds: list[tuple[int, int]]) -> None:
        from .cuda._abi import check, lib

        plane = kk * elem_bytes
        n = len(self.ranks)
        for r in range(n):
            kstart, kend = bounds[r]
            below, above = (r - 1 if r > 0 else -1), (r + 1 if r < n - 1 else -1)
            for name, (down, up) in fields.items():
                for op, peer, first, count in halo_plan(kstart, kend, down, up, below, above):
                    if op != "recv":
                        continue
                    # the peer sends the matching planes of its own slab
                    pk0, pk1 = bounds[peer]
                    src_first = pk1 - count if peer < r else pk0
                    check(lib().klb_memcpy_dtod(self.ranks[r][name] + first * plane,
                                                self.ranks[peer][name] + src_first * plane, count * plane,
                                                stream.handle))


@dataclass
class SlabRank:
    """Per-rank view of a decomposition: local offsets and sub-ranges."""

    decomposition: SlabDecomposition
    rank: int
    kgc: int
    kernel: str

    @property
    def offset(self) -> int:
        return self.decomposition.planes(self.rank)[0]

    @property
    def count(self) -> int:
        return self.decomposition.planes(self.rank)[1]

    @property
    def kstart(self) -> int:
        return self.kgc

    @property
    def kend(self) -> int:
        return self.kgc + self.count

    def subranges(self) -> dict[str, tuple[int, int]]:
        """interior / lower / upper local plane ranges (empty ones omitted).

        Ranks at the global bottom/top read physical ghost planes that need no
        exchange, so their outer boundary folds into the interior range.
        """
        below, above = self.decomposition.neighbours(self.rank)
        down, up = kernel_reach(self.kernel)
        lo = self.kstart + (up if below >= 0 else 0)
        hi = self.kend - (down if above >= 0 else 0)
        lo, hi = min(lo, self.kend), max(hi, self.kstart)
        if hi <= lo:  # slab thinner than the reach: everything waits for the halo
            return {"lower": (self.kstart, self.kend)}
        out = {"interior": (lo, hi)}
        if lo > self.kstart:
            out["lower"] = (self.kstart, lo)
        if hi < self.kend:
            out["upper"] = (hi, self.kend)
        return out
