"""B200 backend behind the reference plugin boundary (backend.py:212-277).

``NvrtcCompiler`` / ``CudaExecutable`` implement ``CompilerInterface`` /
``ExecutableHandle``; ``CudaReplayExecutor`` implements ``Executor``; all of
them reach the GPU only through the C ABI in ``libklb200.so``
(include/klb200.h).
"""

from ._abi import KlbError, library_path
from .compiler import CompiledImage, CudaExecutable, NvrtcCompiler
from .device import DeviceArray, DeviceBuffer, DeviceContext, Event, Graph, HostPinned, Stream, open_device

__all__ = [
    "KlbError", "library_path", "CompiledImage", "CudaExecutable", "NvrtcCompiler", "DeviceArray", "DeviceBuffer",
    "DeviceContext", "Event", "Graph", "HostPinned", "Stream", "open_device", "CudaReplayExecutor",
]


def __getattr__(name):
    if name == "CudaReplayExecutor":
        from .executor import CudaReplayExecutor

        return CudaReplayExecutor
    raise AttributeError(name)
