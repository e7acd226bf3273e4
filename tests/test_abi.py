"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "klb200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(klb_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_ctypes_table():
    from paper_2303_12374_b200.cuda._abi import EXPORTS

    assert set(declared()) == set(EXPORTS)


def test_library_exports_all_symbols():
    from paper_2303_12374_b200.cuda._abi import lib, library_path

    if not library_path().exists():
        pytest.skip("libklb200.so not built (run __graft_entry__.build())")
    handle = lib()
    for name in declared():
        assert hasattr(handle, name), name
    assert handle.klb_abi_version() == 1


def test_no_driver_is_a_clean_error():
    from paper_2303_12374_b200.cuda._abi import KlbError, check, lib, library_path

    if not library_path().exists():
        pytest.skip("libklb200.so not built")
    n = ctypes.c_int(-1)
    rc = lib().klb_device_count(ctypes.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a GPU is visible here")
    with pytest.raises(KlbError):
        check(rc if rc else lib().klb_init(0, None))


def test_nvrtc_compiles_sm100a_without_gpu():
    """NVRTC needs no device: the runtime compile path is checkable on CPU."""
    from paper_2303_12374_b200.cuda._abi import library_path

    if not library_path().exists():
        pytest.skip("libklb200.so not built")
    from paper_2303_12374_b200.backend import CompileError, DeviceIdent
    from paper_2303_12374_b200.cuda.compiler import NvrtcCompiler
    from paper_2303_12374_b200.kerneldef import CompileRequest

    comp = NvrtcCompiler()
    dev = DeviceIdent("NVIDIA B200", "Blackwell", {"compute_capability": "10.0"})
    src = "template<int N> __global__ void k(float* x) { x[threadIdx.x] *= N; }"
    img = comp.compile_image(CompileRequest(src, "k<4>", (), ("-std=c++17",)), dev)
    assert img.lowered_name == "_Z1kILi4EEvPf" and img.cubin[:4] == b"\x7fELF"
    with pytest.raises(CompileError) as err:
        comp.compile_image(CompileRequest("__global__ void k() { syntax error }", "k", (), ()), dev)
    assert "error" in err.value.diagnostics


def test_graph_capture_without_a_device_fails_cleanly():
    """CUDA-graph capture refuses the legacy default stream before any driver
    call, and the C ABI reports a clean error (not a crash) without a GPU."""
    from paper_2303_12374_b200.cuda import Graph, Stream
    from paper_2303_12374_b200.cuda._abi import KlbError, check, lib, library_path

    with pytest.raises(ValueError):
        with Graph.capture(Stream()):
            pass
    if not library_path().exists():
        pytest.skip("libklb200.so not built")
    n = ctypes.c_int(-1)
    if lib().klb_device_count(ctypes.byref(n)) == 0 and n.value > 0:
        pytest.skip("a GPU is visible here")
    g = ctypes.c_void_p()
    with pytest.raises(KlbError):
        check(lib().klb_stream_end_capture(None, ctypes.byref(g)))
    assert g.value is None
