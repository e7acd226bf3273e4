"""Streaming capture I/O and replay placement, CPU side.

* ``CaptureFile.read_into`` streams one payload through caller buffers with a
  running CRC (what ``CudaReplayExecutor.from_file`` uploads from) and
  rejects corruption / truncation like ``read_capture`` (reference
  capture.py:306-340);
* a kernel source too large for the 64 KiB metadata block (reference
  capture.py:37, 261-263) goes to a ``source_file`` sidecar instead of
  failing the capture;
* ``address_mod128`` survives the round trip and is ignored by equality (the
  reference reader ignores unknown keys);
* ``WisdomKernel`` caches binaries per compile-time scalar values (pitches).
"""

import json
import zlib

import pytest

from paper_2303_12374_b200.capture import (BufferArg, CaptureFile, CaptureFormatError, ScalarArg, capture_from_args,
                                           read_capture, read_capture_info, serialize_capture, source_sidecar,
                                           write_capture, write_capture_stream)
from paper_2303_12374_b200.kerneldef import KernelBuilder
from paper_2303_12374_b200.presets import stencil3d_definition


def _cap(nbytes=300_000, address_mod=None, definition=None):
    d = definition or stencil3d_definition()
    payload = bytes((i * 131 + 7) & 0xFF for i in range(nbytes))
    args = [BufferArg(0, "output", "f32", payload, address_mod=address_mod), BufferArg(1, "input", "u8", payload[:777]),
            ScalarArg(2, "i32", 16), ScalarArg(3, "i32", 8), ScalarArg(4, "i32", 4)]
    return capture_from_args(d, args, application="t", timestamp="2026-01-01T00:00:00Z"), payload


class _Sink:
    def __init__(self, views):
        self.views, self.out, self.ready_calls = views, {}, []

    def __call__(self, slot, offset, size):
        self.out[offset] = bytes(memoryview(self.views[slot])[:size])

    def ready(self, slot):
        self.ready_calls.append(slot)

    def data(self):
        return b"".join(self.out[k] for k in sorted(self.out))


@pytest.mark.parametrize("chunk", [4096, 65536, 1 << 20])
def test_read_into_streams_every_payload(tmp_path, chunk):
    cap, payload = _cap()
    path = tmp_path / "a.klcap"
    write_capture_stream(cap, path, chunk=8192)
    cf = CaptureFile.open(path)
    assert cf.problem == (16, 8, 4) and cf.definition.name == cap.definition.name
    assert cf.scalar_env() == cap.scalar_env()
    for index, want in enumerate((payload, payload[:777])):
        views = [bytearray(chunk), bytearray(chunk)]
        sink = _Sink(views)
        cf.read_into(index, views, sink)
        assert sink.data() == want
        # alternating slots, each awaited before reuse
        assert sink.ready_calls == [i % 2 for i in range(len(sink.out))]


def test_read_into_rejects_corruption_and_truncation(tmp_path):
    cap, _ = _cap()
    path = tmp_path / "a.klcap"
    write_capture(cap, path)
    raw = bytearray(path.read_bytes())
    raw[-100] ^= 0x10  # the file ends with buffer 1's payload
    path.write_bytes(bytes(raw))
    views = [bytearray(4096), bytearray(4096)]
    cf = CaptureFile.open(path)
    cf.read_into(0, views, _Sink(views))  # buffer 0 intact
    with pytest.raises(CaptureFormatError, match="checksum"):
        cf.read_into(1, views, _Sink(views))
    path.write_bytes(bytes(raw[:-500]))
    with pytest.raises(CaptureFormatError, match="truncated"):
        CaptureFile.open(path).read_into(1, views, _Sink(views))


def test_address_mod_round_trip_and_reference_layout(tmp_path):
    cap, _ = _cap(address_mod=52)
    path = tmp_path / "a.klcap"
    write_capture(cap, path)
    info = read_capture_info(path)
    assert info["buffers"][0]["address_mod128"] == 52 and "address_mod128" not in info["buffers"][1]
    back = read_capture(path)
    assert back.buffers[0].address_mod == 52 and back == cap
    # a capture without device provenance is byte-identical to the plain layout
    plain, _ = _cap()
    assert b"address_mod128" not in serialize_capture(plain)


def test_oversized_source_goes_to_sidecar(tmp_path):
    from paper_2303_12374_b200.kerneldef import KernelDefinition

    base = stencil3d_definition()
    src = base.resolve_source() + ("// " + "x" * 100 + "\n") * 900  # ~92 KiB: over the 64 KiB metadata cap
    obj = base.to_json_obj(embed_source=True)
    obj["source_text"] = src
    d = KernelDefinition.from_json_obj(obj)
    cap, payload = _cap(definition=d)
    for writer in (write_capture, write_capture_stream):
        path = tmp_path / f"{writer.__name__}.klcap"
        writer(cap, path)
        side = source_sidecar(path)
        assert side.read_text() == src
        info = read_capture_info(path)
        assert info["definition"]["source_file"] == side.name and "source_text" not in info["definition"]
        back = read_capture(path)
        assert back.definition.resolve_source() == src
        assert back.buffers[0].data == payload
        assert CaptureFile.open(path).definition.resolve_source() == src


def test_wisdom_kernel_caches_per_compile_time_scalars(tmp_path):
    """Two launches with one problem size but different baked-in scalars
    (the stencils' KL_JJ/KL_KK pitch) compile twice; the reference's key
    (device, problem) alone would reuse the first binary."""
    from paper_2303_12374_b200.backend import DeviceIdent, MockCompiler
    from paper_2303_12374_b200.dispatch import WisdomKernel

    b = KernelBuilder("pitched", source_text="__global__ void pitched() {}")
    blk = b.tune("block", (32, 64), 32)
    d = b.problem_size("arg0").block(blk).grid("ceil_div(problem_x, block)").define("PITCH", "arg1").build()
    assert d.compile_time_args() == ("arg1",)
    comp = MockCompiler()
    wk = WisdomKernel(d, comp, wisdom_dir=tmp_path)
    dev = DeviceIdent("dev", "arch")
    r1 = wk.launch(dev, [ScalarArg(0, "i32", 100), ScalarArg(1, "i32", 128)])
    r2 = wk.launch(dev, [ScalarArg(0, "i32", 100), ScalarArg(1, "i32", 128)])
    r3 = wk.launch(dev, [ScalarArg(0, "i32", 100), ScalarArg(1, "i32", 256)])
    assert (r1.cache_hit, r2.cache_hit, r3.cache_hit) == (False, True, False)
    assert stencil3d_definition().compile_time_args() == ()
