"""ctypes binding of ``libklb200.so`` (declared in include/klb200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2303_12374_b200/csrc``).  There is no fallback: if the
library is missing or the CUDA driver is unusable every entry point raises
``KlbError`` — the B200 path never silently degrades to CPU code.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

__all__ = ["KlbError", "lib", "library_path", "DeviceInfo", "FuncAttrs", "check", "EXPORTS"]

_PKG_DIR = Path(__file__).resolve().parent.parent
_LIB_NAME = "libklb200.so"


class KlbError(RuntimeError):
    def __init__(self, code: int, message: str) -> None:
        super().__init__(f"[klb {code}] {message}")
        self.code = code


class DeviceInfo(C.Structure):
    _fields_ = [
        ("name", C.c_char * 256),
        ("ordinal", C.c_int),
        ("cc_major", C.c_int),
        ("cc_minor", C.c_int),
        ("sm_count", C.c_int),
        ("l2_bytes", C.c_int),
        ("max_smem_per_block_optin", C.c_int),
        ("max_smem_per_sm", C.c_int),
        ("max_threads_per_sm", C.c_int),
        ("max_threads_per_block", C.c_int),
        ("regs_per_sm", C.c_int),
        ("warp_size", C.c_int),
        ("clock_khz", C.c_int),
        ("mem_clock_khz", C.c_int),
        ("mem_bus_width_bits", C.c_int),
        ("pci_bus_id", C.c_int),
        ("driver_version", C.c_int),
        ("total_mem_bytes", C.c_size_t),
        ("uuid", C.c_ubyte * 16),
    ]


class FuncAttrs(C.Structure):
    _fields_ = [
        ("num_regs", C.c_int),
        ("local_bytes", C.c_int),
        ("static_smem_bytes", C.c_int),
        ("max_threads_per_block", C.c_int),
        ("max_dynamic_smem_bytes", C.c_int),
        ("ptx_version", C.c_int),
        ("binary_version", C.c_int),
    ]


_u = C.c_uint
_i = C.c_int
_ll = C.c_longlong
_sz = C.c_size_t
_u64 = C.c_uint64
_vp = C.c_void_p
_pvp = C.POINTER(C.c_void_p)
_u3 = C.POINTER(C.c_uint)
_d = C.c_double

# name -> argtypes (all return int unless listed in _RESTYPE)
EXPORTS: dict[str, list] = {
    "klb_abi_version": [],
    "klb_last_error": [],
    "klb_device_count": [C.POINTER(_i)],
    "klb_init": [_i, C.POINTER(DeviceInfo)],
    "klb_set_device": [_i],
    "klb_device_synchronize": [],
    "klb_nvrtc_version": [C.POINTER(_i), C.POINTER(_i)],
    "klb_compile": [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), _i, _pvp, C.POINTER(_sz),
                    C.POINTER(_vp), C.POINTER(_vp)],
    "klb_free": [_vp],
    "klb_module_load": [_vp, _pvp],
    "klb_module_unload": [_vp],
    "klb_module_function": [_vp, C.c_char_p, _pvp],
    "klb_function_attributes": [_vp, C.POINTER(FuncAttrs)],
    "klb_function_set_max_dynamic_smem": [_vp, _i],
    "klb_occupancy_blocks_per_sm": [_vp, _i, _i, C.POINTER(_i)],
    "klb_launch": [_vp, _u3, _u3, _u, _vp, _pvp],
    "klb_launch_ex": [_vp, _u3, _u3, _u, _vp, _pvp, _u],
    "klb_time_launches": [_vp, _u3, _u3, _u, _vp, _pvp, _i, _i, _u64, _sz, C.POINTER(C.c_float)],
    "klb_mem_alloc": [_sz, C.POINTER(_u64)],
    "klb_mem_free": [_u64],
    "klb_mem_get_info": [C.POINTER(_sz), C.POINTER(_sz)],
    "klb_host_alloc": [_sz, _pvp],
    "klb_host_free": [_vp],
    "klb_memcpy_htod": [_u64, _vp, _sz, _vp],
    "klb_memcpy_dtoh": [_vp, _u64, _sz, _vp],
    "klb_memcpy_dtod": [_u64, _u64, _sz, _vp],
    "klb_memset_d8": [_u64, C.c_ubyte, _sz, _vp],
    "klb_stream_create": [_pvp, _i],
    "klb_stream_destroy": [_vp],
    "klb_stream_synchronize": [_vp],
    "klb_stream_wait_event": [_vp, _vp],
    "klb_event_create": [_pvp],
    "klb_event_destroy": [_vp],
    "klb_event_record": [_vp, _vp],
    "klb_event_synchronize": [_vp],
    "klb_event_elapsed_ms": [_vp, _vp, C.POINTER(C.c_float)],
    "klb_stream_begin_capture": [_vp],
    "klb_stream_end_capture": [_vp, _pvp],
    "klb_graph_launch": [_vp, _vp],
    "klb_graph_destroy": [_vp],
    "klb_module_global": [_vp, C.c_char_p, C.POINTER(_u64), C.POINTER(_sz)],
    "klb_tensor_map_encode_3d": [_vp, _i, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(C.c_uint)],
    "klb_synth_field": [_u64, _i, _ll, _i, _i, _i, _i, _ll, _i, _i, _i, _i, _u64, _d, _d, _i, _vp],
    "klb_compare_fields": [_u64, _u64, _i, _ll, _i, _i, _i, _i, _i, _i, _i, _ll, C.POINTER(_d), C.POINTER(_d), _vp],
    "klb_cyclic_xy": [_u64, _i, _ll, _i, _i, _i, _ll, _i, _i, _i, _i, _vp],
    "klb_crc32_device": [_u64, C.c_size_t, _vp, C.POINTER(C.c_uint32)],
    "klb_nccl_version": [C.POINTER(_i)],
    "klb_nccl_unique_id": [C.POINTER(C.c_ubyte)],
    "klb_nccl_comm_init": [_pvp, _i, C.POINTER(C.c_ubyte), _i],
    "klb_nccl_comm_destroy": [_vp],
    "klb_halo_exchange_z": [_vp, _vp, _i, C.POINTER(_u64), _i, _ll, _i, _i, _i, _i, _i, _i],
    "klb_group_open": [C.c_char_p, _i, _i, _d, _pvp],
    "klb_group_barrier": [_vp],
    "klb_group_allgather": [_vp, _vp, _sz, _vp],
    "klb_group_close": [_vp],
    "klb_ipc_mem_handle": [_u64, C.POINTER(C.c_ubyte), C.POINTER(_u64)],
    "klb_ipc_mem_open": [C.POINTER(C.c_ubyte), C.POINTER(_u64)],
    "klb_ipc_mem_close": [_u64],
    "klb_ipc_event_create": [_pvp, C.POINTER(C.c_ubyte)],
    "klb_ipc_event_open": [C.POINTER(C.c_ubyte), _pvp],
    "klb_halo_pull_z": [_vp, _i, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), _i, _ll, _i, _i, _i, _i, _i,
                        _i],
}
_RESTYPE = {"klb_last_error": C.c_char_p, "klb_free": None}

_lock = threading.Lock()
_handle: C.CDLL | None = None


def library_path() -> Path:
    override = os.environ.get("KLB200_LIBRARY")
    return Path(override) if override else _PKG_DIR / _LIB_NAME


def lib() -> C.CDLL:
    """The loaded library (loads once; raises if it was never built)."""
    global _handle
    if _handle is not None:
        return _handle
    with _lock:
        if _handle is None:
            path = library_path()
            if not path.exists():
                raise KlbError(-1, f"{path} not found — run __graft_entry__.build() to compile the CUDA backend")
            handle = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
            for name, argtypes in EXPORTS.items():
                fn = getattr(handle, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPE.get(name, C.c_int)
            _handle = handle
    return _handle


def check(rc: int) -> None:
    if rc != 0:
        message = lib().klb_last_error()
        raise KlbError(rc, message.decode("utf-8", "replace") if message else "unknown error")
