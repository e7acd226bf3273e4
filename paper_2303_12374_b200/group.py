"""``ProcessGroup`` — single-node rank rendezvous over the C ABI (no torch).

The multi-rank driver (``bench.py --gpus N``, ``SlabDriver`` with the IPC or
NCCL halo transport) needs a barrier, a max/sum over ranks and a way to hand
NCCL ids and CUDA-IPC handles around.  ``klb_group_*`` (include/klb200.h)
implements them on one POSIX shared-memory segment with process-shared
atomics: microsecond barriers, no sockets, no torch.distributed, and a
timeout instead of a hang when a peer dies.

The segment name must be identical on every rank and unique per job:
``group_name()`` derives it from the launcher — the parent process id (the
torchrun agent, or ``bench.py``'s own spawner) plus ``MASTER_PORT`` — or
takes ``KLB_GROUP`` when set.  No reference counterpart.
"""

from __future__ import annotations

import ctypes as C
import os
import struct

__all__ = ["ProcessGroup", "group_name", "SLOT_BYTES"]

SLOT_BYTES = 4096


def group_name(environ=None) -> str:
    env = os.environ if environ is None else environ
    if env.get("KLB_GROUP"):
        name = env["KLB_GROUP"]
    else:
        name = f"klb_{os.getppid()}_{env.get('MASTER_PORT', '0')}_{env.get('TORCHELASTIC_RUN_ID', '')}"
    name = "".join(c if c.isalnum() or c in "_-." else "_" for c in name.lstrip("/"))
    return "/" + name[:100]


class ProcessGroup:
    """``rank`` of ``nranks`` processes of one job on this node."""

    def __init__(self, rank: int, nranks: int, name: str | None = None, timeout: float = 300.0) -> None:
        from .cuda._abi import check, lib

        self.rank, self.nranks = rank, nranks
        self.name = name or group_name()
        h = C.c_void_p()
        check(lib().klb_group_open(self.name.encode(), rank, nranks, float(timeout), C.byref(h)))
        self.handle = h.value

    def barrier(self) -> None:
        from .cuda._abi import check, lib

        check(lib().klb_group_barrier(self.handle))

    def allgather(self, payload: bytes) -> list[bytes]:
        """Every rank's ``payload`` (all the same length, <= 4096 bytes)."""
        from .cuda._abi import check, lib

        n = len(payload)
        out = C.create_string_buffer(max(n * self.nranks, 1))
        check(lib().klb_group_allgather(self.handle, payload, n, out))
        raw = out.raw
        return [raw[r * n:(r + 1) * n] for r in range(self.nranks)]

    def allgather_obj(self, values: tuple[float, ...]) -> list[tuple[float, ...]]:
        fmt = f"<{len(values)}d"
        return [struct.unpack(fmt, b) for b in self.allgather(struct.pack(fmt, *values))]

    def max(self, value: float) -> float:
        return max(v[0] for v in self.allgather_obj((float(value),)))

    def sum(self, value: float) -> float:
        return float(sum(v[0] for v in self.allgather_obj((float(value),))))

    def broadcast(self, payload: bytes | None, root: int = 0, size: int | None = None) -> bytes:
        """``root``'s payload on every rank (others pass None and the size)."""
        n = len(payload) if payload is not None else int(size)
        mine = payload if self.rank == root else b"\0" * n
        return self.allgather(mine)[root]

    def close(self) -> None:
        from .cuda._abi import lib

        if self.handle:
            lib().klb_group_close(self.handle)
            self.handle = None

    def __enter__(self) -> "ProcessGroup":
        return self

    def __exit__(self, *exc) -> None:
        self.close()
