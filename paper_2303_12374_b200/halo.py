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
This is the protocol ``klb_halo_exchange_z`` (NCCL) implements in C; the
``CopyExchanger`` (several virtual ranks on one GPU, D2D copies) and the
``HostExchanger`` (NumPy arrays over torch.distributed/gloo, CPU tests)
implement the same plan in Python.

Reach per kernel (from the stencil definitions):
  advec_u : u (down 3, up 3), w (down 1, up 0), v none
  diff_uvw: evisc, u, v, w (down 1, up 1)
  (the §8f family in HALO_REACH below, from oracle/family_oracle.py)
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

__all__ = [
    "HALO_REACH", "SlabDecomposition", "halo_plan", "NcclExchanger", "CopyExchanger", "HostExchanger",
    "StagedExchanger", "SlabRank",
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


class HostExchanger:
    """The halo plan over torch.distributed (gloo) on NumPy (kcells, jcells, icells) arrays."""

    def __init__(self, rank: int, nranks: int) -> None:
        self.rank, self.nranks = rank, nranks

    def exchange(self, arrays, kstart: int, kend: int, down: int, up: int, below: int, above: int) -> None:
        import numpy as np
        import torch
        import torch.distributed as dist

        reqs, sinks = [], []
        for arr in arrays:
            for op, peer, first, count in halo_plan(kstart, kend, down, up, below, above):
                if op == "send":
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr[first:first + count])), peer))
                else:
                    buf = torch.empty(arr[first:first + count].shape, dtype=torch.from_numpy(arr[:1]).dtype)
                    reqs.append(dist.irecv(buf, peer))
                    sinks.append((arr, first, count, buf))
        for req in reqs:
            req.wait()
        for arr, first, count, buf in sinks:
            arr[first:first + count] = buf.numpy()


class StagedExchanger:
    """The same exchange as ``NcclExchanger`` with the planes relayed through
    pinned host memory over torch.distributed (any backend; gloo here).

    Not a performance transport: it serialises on the host.  It exists so the
    whole multi-rank path (decomposition, sub-range launches, exchange
    ordering, max-over-ranks timing, bench output at N > 1) can run as several
    processes on ONE GPU — NCCL refuses two ranks on one device — which is
    what ``tests/test_gpu_multiproc.py`` does (selected in ``bench.py`` by
    ``KL_HALO_TRANSPORT=staged``).  Same signature as ``NcclExchanger.exchange``.
    """

    def __init__(self, rank: int, nranks: int) -> None:
        self.rank, self.nranks = rank, nranks

    def exchange(self, stream, ptrs, elem_bytes: int, kk: int, kstart: int, kend: int, down: int, up: int,
                 below: int, above: int) -> None:
        import numpy as np
        import torch
        import torch.distributed as dist

        from .cuda._abi import check, lib

        plane = kk * elem_bytes
        stream.synchronize()  # the planes to send are final (the comm stream waited on compute)
        reqs, sinks = [], []
        for ptr in ptrs:
            for op, peer, first, count in halo_plan(kstart, kend, down, up, below, above):
                buf = np.empty(count * plane, dtype=np.uint8)
                if op == "send":
                    check(lib().klb_memcpy_dtoh(buf.ctypes.data, ptr + first * plane, count * plane, stream.handle))
                    stream.synchronize()
                    reqs.append(dist.isend(torch.from_numpy(buf), peer))
                else:
                    t = torch.from_numpy(buf)
                    reqs.append(dist.irecv(t, peer))
                    sinks.append((ptr + first * plane, buf))
        for req in reqs:
            req.wait()
        for dst, buf in sinks:
            check(lib().klb_memcpy_htod(dst, buf.ctypes.data, buf.nbytes, stream.handle))
        stream.synchronize()

    def close(self) -> None:
        pass


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
