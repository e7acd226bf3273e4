"""Device context, memory and streams over the C ABI.

``DeviceContext.ident`` is the ``DeviceIdent`` wisdom records are keyed by
(reference backend.py:47-66): ``name`` is the driver's device name (e.g.
"NVIDIA B200"), ``architecture`` the family derived from the compute
capability ("Blackwell" for 10.x/12.x), ``attributes`` the measured
properties (SM count, L2, HBM size, clocks...).

``DeviceBuffer`` is the launch-argument form of a device allocation: it
carries the reference ``BufferArg`` fields (position, role, element_type) plus
a device pointer, and converts itself to a ``BufferArg`` (one synchronous D2H
copy) when a capture is taken before the launch.
"""

from __future__ import annotations

import ctypes as C
import threading
from collections.abc import Iterator
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np

from ..backend import DeviceIdent
from ..capture import ADDRESS_ALIGN, ELEMENT_SIZES, BufferArg
from ._abi import DeviceInfo, check, lib

__all__ = [
    "architecture_name", "DeviceContext", "open_device", "DeviceArray", "DeviceBuffer", "Stream", "Event",
    "HostPinned",
]

_FAMILIES = [
    ((12, 0), "Blackwell"), ((10, 0), "Blackwell"), ((9, 0), "Hopper"), ((8, 9), "Ada"), ((8, 0), "Ampere"),
    ((7, 5), "Turing"), ((7, 0), "Volta"), ((6, 0), "Pascal"),
]
_NP_TO_ELEM = {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64", np.dtype(np.int32): "i32",
               np.dtype(np.int64): "i64", np.dtype(np.uint8): "u8"}


def architecture_name(major: int, minor: int) -> str:
    for (ma, mi), family in _FAMILIES:
        if (major, minor) >= (ma, mi):
            return family
    return f"sm_{major}{minor}"


class Stream:
    """A non-blocking CUDA stream (``handle`` None = legacy default stream)."""

    def __init__(self, handle=None, owned: bool = False) -> None:
        self.handle = handle
        self._owned = owned

    @classmethod
    def create(cls, priority: int = 0) -> "Stream":
        h = C.c_void_p()
        check(lib().klb_stream_create(C.byref(h), priority))
        return cls(h.value, owned=True)

    def synchronize(self) -> None:
        check(lib().klb_stream_synchronize(self.handle))

    def wait(self, event: "Event") -> None:
        check(lib().klb_stream_wait_event(self.handle, event.handle))

    def close(self) -> None:
        if self._owned and self.handle:
            check(lib().klb_stream_destroy(self.handle))
            self.handle, self._owned = None, False


class Graph:
    """An executable CUDA graph: the launches enqueued on a stream between
    ``capture`` entry and exit, replayed by one ``launch`` (klb_graph_*).
    Kernel parameters are copied in at capture time; the buffers they point
    to must stay allocated while the graph is used."""

    def __init__(self) -> None:
        self.handle = None

    @classmethod
    @contextmanager
    def capture(cls, stream: Stream) -> Iterator["Graph"]:
        if stream is None or not stream.handle:
            raise ValueError("graph capture needs a created (non-default) stream")
        g = cls()
        check(lib().klb_stream_begin_capture(stream.handle))
        h = C.c_void_p()
        try:
            yield g
        except BaseException:
            if lib().klb_stream_end_capture(stream.handle, C.byref(h)) == 0 and h.value:
                lib().klb_graph_destroy(h.value)
            raise
        check(lib().klb_stream_end_capture(stream.handle, C.byref(h)))
        g.handle = h.value

    def launch(self, stream: Stream) -> None:
        if self.handle is None:
            raise ValueError("graph was not captured (or is closed)")
        check(lib().klb_graph_launch(self.handle, stream.handle))

    def close(self) -> None:
        if self.handle:
            check(lib().klb_graph_destroy(self.handle))
            self.handle = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass


class Event:
    def __init__(self) -> None:
        h = C.c_void_p()
        check(lib().klb_event_create(C.byref(h)))
        self.handle = h.value

    def record(self, stream: Stream | None = None) -> "Event":
        check(lib().klb_event_record(self.handle, stream.handle if stream else None))
        return self

    def synchronize(self) -> None:
        check(lib().klb_event_synchronize(self.handle))

    def elapsed_ms(self, later: "Event") -> float:
        out = C.c_float()
        check(lib().klb_event_elapsed_ms(self.handle, later.handle, C.byref(out)))
        return float(out.value)

    def __del__(self) -> None:
        try:
            if self.handle:
                lib().klb_event_destroy(self.handle)
        except Exception:
            pass


class DeviceArray:
    """Owning device allocation."""

    def __init__(self, nbytes: int) -> None:
        ptr = C.c_uint64()
        check(lib().klb_mem_alloc(max(int(nbytes), 1), C.byref(ptr)))
        self.ptr = int(ptr.value)
        self.nbytes = int(nbytes)

    def zero(self, stream: Stream | None = None) -> "DeviceArray":
        check(lib().klb_memset_d8(self.ptr, 0, self.nbytes, stream.handle if stream else None))
        return self

    def upload(self, data, offset_bytes: int = 0, stream: Stream | None = None) -> None:
        buf = np.ascontiguousarray(data) if not isinstance(data, (bytes, bytearray, memoryview)) else data
        view = memoryview(buf).cast("B")
        if offset_bytes + view.nbytes > self.nbytes:
            raise ValueError("upload past the end of the allocation")
        host = (C.c_char * view.nbytes).from_buffer_copy(view) if view.readonly else (C.c_char * view.nbytes).from_buffer(view)
        check(lib().klb_memcpy_htod(self.ptr + offset_bytes, host, view.nbytes, stream.handle if stream else None))
        if stream is None or stream.handle is None:
            check(lib().klb_device_synchronize())
        else:
            stream.synchronize()

    def download(self, nbytes: int | None = None, offset_bytes: int = 0, stream: Stream | None = None) -> bytes:
        n = self.nbytes - offset_bytes if nbytes is None else int(nbytes)
        out = C.create_string_buffer(max(n, 1))
        check(lib().klb_memcpy_dtoh(out, self.ptr + offset_bytes, n, stream.handle if stream else None))
        if stream is None or stream.handle is None:
            check(lib().klb_device_synchronize())
        else:
            stream.synchronize()
        return out.raw[:n]

    def download_array(self, dtype, offset_bytes: int = 0, count: int | None = None) -> np.ndarray:
        dt = np.dtype(dtype)
        n = (self.nbytes - offset_bytes) // dt.itemsize if count is None else count
        return np.frombuffer(self.download(n * dt.itemsize, offset_bytes), dtype=dt).copy()

    def copy_from(self, other: "DeviceArray", nbytes: int | None = None, stream: Stream | None = None) -> None:
        n = min(self.nbytes, other.nbytes) if nbytes is None else nbytes
        check(lib().klb_memcpy_dtod(self.ptr, other.ptr, n, stream.handle if stream else None))

    def free(self) -> None:
        if self.ptr:
            check(lib().klb_mem_free(self.ptr))
            self.ptr = 0

    def __del__(self) -> None:
        try:
            if getattr(self, "ptr", 0):
                lib().klb_mem_free(self.ptr)
        except Exception:
            pass


class HostPinned:
    """Page-locked host buffer (for the end-to-end H2D/D2H path)."""

    def __init__(self, nbytes: int) -> None:
        p = C.c_void_p()
        check(lib().klb_host_alloc(max(int(nbytes), 1), C.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)

    def array(self, dtype, count: int | None = None) -> np.ndarray:
        dt = np.dtype(dtype)
        n = self.nbytes // dt.itemsize if count is None else count
        raw = (C.c_char * (n * dt.itemsize)).from_address(self.ptr)
        return np.frombuffer(raw, dtype=dt, count=n)

    def free(self) -> None:
        if self.ptr:
            check(lib().klb_host_free(self.ptr))
            self.ptr = None

    def __del__(self) -> None:
        try:
            if getattr(self, "ptr", None):
                lib().klb_host_free(self.ptr)
        except Exception:
            pass


@dataclass(frozen=True)
class DeviceBuffer:
    """Launch argument referring to device memory (the B200 form of BufferArg).

    ``ptr`` points at the first element the kernel sees; ``element_count``
    elements from there form the capture payload.
    """

    position: int
    role: str
    element_type: str
    ptr: int
    element_count: int
    owner: object = field(default=None, compare=False, repr=False)

    def __post_init__(self) -> None:
        if self.role not in ("input", "output"):
            raise ValueError(f"buffer role must be input/output, got '{self.role}'")
        if self.element_type not in ELEMENT_SIZES:
            raise ValueError(f"unknown element type '{self.element_type}'")

    @property
    def nbytes(self) -> int:
        return self.element_count * ELEMENT_SIZES[self.element_type]

    def to_buffer_arg(self) -> BufferArg:
        out = C.create_string_buffer(max(self.nbytes, 1))
        check(lib().klb_memcpy_dtoh(out, self.ptr, self.nbytes, None))
        check(lib().klb_device_synchronize())
        return BufferArg(self.position, self.role, self.element_type, out.raw[: self.nbytes],
                         address_mod=self.ptr % ADDRESS_ALIGN)


class DeviceContext:
    """One GPU: primary context, identity, a default stream and an L2-flush buffer."""

    _lock = threading.Lock()
    _open: dict[int, "DeviceContext"] = {}

    def __init__(self, ordinal: int) -> None:
        info = DeviceInfo()
        check(lib().klb_init(ordinal, C.byref(info)))
        self.ordinal = ordinal
        self.info = info
        self.name = info.name.decode()
        self.compute_capability = (info.cc_major, info.cc_minor)
        self.sm_count = info.sm_count
        self.l2_bytes = info.l2_bytes
        self.max_smem_optin = info.max_smem_per_block_optin
        self.max_threads_per_sm = info.max_threads_per_sm
        self.ident = DeviceIdent(
            name=self.name,
            architecture=architecture_name(info.cc_major, info.cc_minor),
            attributes={
                "compute_capability": f"{info.cc_major}.{info.cc_minor}",
                "sm_count": info.sm_count,
                "l2_bytes": info.l2_bytes,
                "total_mem_bytes": int(info.total_mem_bytes),
                "max_smem_per_block_optin": info.max_smem_per_block_optin,
                "max_threads_per_sm": info.max_threads_per_sm,
                "regs_per_sm": info.regs_per_sm,
                "clock_khz": info.clock_khz,
                "mem_clock_khz": info.mem_clock_khz,
                "mem_bus_width_bits": info.mem_bus_width_bits,
            },
        )
        self.stream = Stream.create()
        self._flush: DeviceArray | None = None

    @property
    def arch_flag(self) -> str:
        major, minor = self.compute_capability
        suffix = "a" if major >= 9 else ""
        return f"sm_{major}{minor}{suffix}"

    def flush_buffer(self) -> DeviceArray:
        """A buffer of 2x L2 whose rewrite evicts every line between timed reps."""
        if self._flush is None:
            self._flush = DeviceArray(max(2 * self.l2_bytes, 64 << 20))
        return self._flush

    def make_current(self) -> None:
        check(lib().klb_set_device(self.ordinal))

    def synchronize(self) -> None:
        check(lib().klb_device_synchronize())

    def mem_info(self) -> tuple[int, int]:
        free, total = C.c_size_t(), C.c_size_t()
        check(lib().klb_mem_get_info(C.byref(free), C.byref(total)))
        return int(free.value), int(total.value)


def open_device(ordinal: int = 0) -> DeviceContext:
    """Process-wide singleton context per device ordinal."""
    with DeviceContext._lock:
        ctx = DeviceContext._open.get(ordinal)
        if ctx is None:
            ctx = DeviceContext._open[ordinal] = DeviceContext(ordinal)
        return ctx
