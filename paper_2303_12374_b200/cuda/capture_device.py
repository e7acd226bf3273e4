"""Device-side capture: a ``.klcap`` written straight
from device memory, byte-identical to the host writers
(reference capture.py:4-16 layout; ``capture.serialize_capture``).

The reference writer needs every payload in host memory twice (the buffer and
the serialized file, capture.py:259-275) and CRCs it there; a 1024^3 fp32
diff_uvw launch is ~30 GB.  Here:

* each device buffer's CRC-32 is computed where it lives
  (``klb_crc32_device``: per-chunk CRC registers on the GPU, chained with the
  zero-append operator — equal to ``zlib.crc32`` of the bytes), so the
  metadata, which precedes the payloads in the file, is known before any
  payload byte crosses PCIe;
* payloads then stream through two pinned staging buffers: the D2H copy of
  chunk i+1 runs while chunk i is written to the file.

Host memory in use is two chunks, whatever the grid size.  ``read_capture``
(host zlib) verifies every CRC on the way back, which is the parity check of
the device CRC (tests/test_gpu_capture_tune.py).
"""

from __future__ import annotations

import ctypes as C
import os
import tempfile
import zlib
from pathlib import Path
from typing import Sequence

from ..capture import ADDRESS_ALIGN, BufferArg, ScalarArg, header_block, metadata_block, scalar_env_from_args, _round_up
from ..kerneldef import KernelDefinition
from ._abi import check, lib
from .device import DeviceBuffer, Event, HostPinned, Stream

__all__ = ["device_crc32", "write_capture_device"]


def device_crc32(ptr: int, nbytes: int, stream: Stream | None = None) -> int:
    """zlib-compatible CRC-32 of ``nbytes`` of device memory at ``ptr``."""
    out = C.c_uint32()
    check(lib().klb_crc32_device(int(ptr), int(nbytes), stream.handle if stream is not None else None,
                                 C.byref(out)))
    return out.value


def write_capture_device(definition: KernelDefinition, args: Sequence[object], path: str | Path, *,
                         application: str = "", timestamp: str = "", chunk: int = 64 << 20,
                         stream: Stream | None = None) -> Path:
    scalars = [a for a in args if isinstance(a, ScalarArg)]
    buffers = [a for a in args if isinstance(a, (DeviceBuffer, BufferArg))]
    problem = definition.derive_problem_size(scalar_env_from_args(args))
    descs = []
    for b in buffers:
        if isinstance(b, DeviceBuffer):
            descs.append((b.position, b.role, b.element_type, b.element_count, b.nbytes,
                          device_crc32(b.ptr, b.nbytes, stream), b.ptr % ADDRESS_ALIGN))
        else:
            descs.append((b.position, b.role, b.element_type, b.element_count, len(b.data),
                          zlib.crc32(b.data) & 0xFFFFFFFF, b.address_mod))
    target = Path(path)
    meta = metadata_block(definition, problem, scalars, descs, application, timestamp, target=target)
    target.parent.mkdir(parents=True, exist_ok=True)
    fd, scratch = tempfile.mkstemp(prefix=target.name + ".", suffix=".tmp", dir=str(target.parent))
    staging = [HostPinned(chunk), HostPinned(chunk)]
    events = [Event(), Event()]
    handle = stream.handle if stream is not None else None
    try:
        with os.fdopen(fd, "wb") as out:
            out.write(header_block(meta))
            cursor = 0
            for b in buffers:
                gap = _round_up(cursor) - cursor
                if gap:
                    out.write(b"\0" * gap)
                if isinstance(b, BufferArg):
                    out.write(b.data)
                    cursor += gap + len(b.data)
                    continue
                pending = None  # (staging index, size) of the chunk in flight
                n = b.nbytes
                for i, lo in enumerate(range(0, n, chunk)):
                    k = i % 2
                    size = min(chunk, n - lo)
                    check(lib().klb_memcpy_dtoh(staging[k].ptr, b.ptr + lo, size, handle))
                    events[k].record(stream)
                    if pending is not None:
                        pk, psize = pending
                        events[pk].synchronize()
                        out.write((C.c_char * psize).from_address(staging[pk].ptr))
                    pending = (k, size)
                if pending is not None:
                    pk, psize = pending
                    events[pk].synchronize()
                    out.write((C.c_char * psize).from_address(staging[pk].ptr))
                cursor += gap + n
        os.replace(scratch, target)
    except BaseException:
        try:
            os.unlink(scratch)
        except OSError:
            pass
        raise
    finally:
        for h in staging:
            h.free()
    return target
