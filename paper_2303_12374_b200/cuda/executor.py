"""``CudaReplayExecutor`` — the B200 ``Executor`` (reference backend.py:212-223).

Replays one captured launch (a ``.klcap`` Capture) or a live device-resident
``StencilProblem`` across configurations, on the GPU, in isolation:

  measure(config):
    1. render the compile request, NVRTC-compile (CUBIN cache; ``prefetch``
       compiles upcoming configurations on a thread pool)  -> compile_failed
    2. load the module, derive the launch geometry, check it against the
       device limits (threads, opt-in shared memory)           -> launch_failed
    3. verify: restore the pristine output buffers, launch once, compare every
       output with the default configuration's result on the device
       (max|a-b| / max|b| <= 1e-5 fp32, 1e-12 fp64)             -> invalid_config
    4. time: ``warmup`` launches, then ``repetitions`` launches, each preceded
       by an L2 flush (a 2x-L2 memset outside the event window) and bracketed
       by CUDA events on the replay stream; objective = median seconds.

Unlike the reference ``SubprocessExecutor`` (which launches with no buffers,
backend.py:462 — SURVEY Appendix B.4), the captured buffers ARE replayed.
``reentrant = False``: measurements are exclusive.  A sticky CUDA error
(illegal address etc.) poisons the context; the executor then reports
``launch_failed`` for everything and records ``broken`` in ``describe()``.
"""

from __future__ import annotations

import ctypes as C
import statistics
import time
from typing import Sequence

from ..backend import (
    STATUS_COMPILE_FAILED,
    STATUS_INVALID_CONFIG,
    STATUS_LAUNCH_FAILED,
    STATUS_OK,
    CompileError,
    Executor,
    LaunchError,
    Measurement,
)
from ..capture import ADDRESS_ALIGN, ELEMENT_SIZES, Capture, CaptureFile, scalar_env_from_args
from ..expr import EvalError
from ..kerneldef import DefinitionError, KernelDefinition
from ..space import Configuration
from ._abi import KlbError
from .compiler import CudaExecutable, NvrtcCompiler
from .device import DeviceArray, DeviceBuffer, DeviceContext

__all__ = ["CudaReplayExecutor", "TOLERANCE"]

TOLERANCE = {"f32": 1e-5, "f64": 1e-12}
_STICKY = {700, 701, 702, 709, 710, 714, 715, 716, 717, 718, 719, 720}


class CudaReplayExecutor(Executor):
    reentrant = False

    def __init__(self, capture: Capture | CaptureFile | None, ctx: DeviceContext, *,
                 definition: KernelDefinition | None = None,
                 args: Sequence[object] | None = None, problem=None, compiler: NvrtcCompiler | None = None,
                 warmup: int = 3, repetitions: int = 7, flush_l2: bool = True, verify: bool = True,
                 output_layout=None, chunk: int = 64 << 20) -> None:
        """Either ``capture`` (a loaded ``Capture``, or a ``CaptureFile`` whose
        payloads are streamed from disk to the device in ``chunk``-byte
        pieces — see ``from_file``) or ``definition`` + device ``args``
        (+ ``problem``) of an already resident launch."""
        self.ctx = ctx
        self.compiler = compiler or NvrtcCompiler(ctx)
        self.warmup = warmup
        self.repetitions = repetitions
        self.flush_l2 = flush_l2
        self.verify = verify
        self.output_layout = output_layout
        self.broken: str | None = None
        self._owned: list[DeviceArray] = []
        if isinstance(capture, CaptureFile):
            self.definition = capture.definition
            self.problem = tuple(capture.problem)
            self.args = self._upload_file(capture, chunk)
        elif capture is not None:
            self.definition = capture.definition
            self.problem = tuple(capture.problem)
            self.args = self._upload_capture(capture)
        else:
            if definition is None or args is None:
                raise ValueError("need a capture or definition + args")
            self.definition = definition
            self.args = list(args)
            self.problem = tuple(problem) if problem is not None else definition.derive_problem_size(
                scalar_env_from_args(self.args))
        self.scalar_env = scalar_env_from_args(self.args)
        self.outputs = [a for a in self.args if isinstance(a, DeviceBuffer) and a.role == "output"]
        self._pristine = []
        self._expected = []
        for buf in self.outputs:
            keep = DeviceArray(buf.nbytes)
            self._copy(keep.ptr, buf.ptr, buf.nbytes)
            self._pristine.append(keep)
        self._futures: dict[tuple, object] = {}
        self.default_config, _ = self.definition.space.default_config()
        if verify:
            self._compute_expected()

    # -- setup ---------------------------------------------------------------------------
    def _copy(self, dst: int, src: int, nbytes: int) -> None:
        from ._abi import check, lib

        check(lib().klb_memcpy_dtod(dst, src, nbytes, self.ctx.stream.handle))

    @classmethod
    def from_file(cls, path, ctx: DeviceContext, **kwargs) -> "CudaReplayExecutor":
        """Replay a ``.klcap`` without loading it into host memory: each
        payload is read in chunks into two pinned staging buffers, CRC-checked
        on the way, and uploaded asynchronously (the read of chunk i+1
        overlaps the H2D copy of chunk i).  Host memory: two chunks."""
        return cls(CaptureFile.open(path), ctx, **kwargs)

    def _placed(self, nbytes: int, address_mod: int | None) -> tuple[DeviceArray, int]:
        """A device allocation and the address inside it that reproduces the
        captured argument's alignment (``address_mod`` = original address mod
        ``ADDRESS_ALIGN``): the application's fields put every interior row
        on a 128-byte boundary, which the TMA kernels' vector path needs, so
        the replay must not time the misaligned fallback instead."""
        if address_mod is None:
            arr = DeviceArray(nbytes)
            return arr, arr.ptr
        arr = DeviceArray(nbytes + ADDRESS_ALIGN)
        return arr, arr.ptr + (address_mod - arr.ptr) % ADDRESS_ALIGN

    def _upload_capture(self, cap: Capture) -> list:
        from ._abi import check, lib

        args: list = list(cap.scalars)
        for b in cap.buffers:
            arr, ptr = self._placed(len(b.data), b.address_mod)
            if b.data:
                check(lib().klb_memcpy_htod(ptr, b.data, len(b.data), self.ctx.stream.handle))
                self.ctx.stream.synchronize()
            self._owned.append(arr)
            args.append(DeviceBuffer(b.position, b.role, b.element_type, ptr, b.element_count, owner=arr))
        return args

    def _upload_file(self, capfile: CaptureFile, chunk: int) -> list:
        from ._abi import check, lib
        from .device import Event, HostPinned

        stream = self.ctx.stream
        args: list = list(capfile.scalars)
        entries = capfile.buffers
        longest = max((e["byte_length"] for e in entries), default=0)
        chunk = max(ELEMENT_SIZES["f64"], min(chunk, longest))
        staging = [HostPinned(chunk), HostPinned(chunk)]
        events = [Event(), Event()]
        pending = [False, False]
        self.host_staging_bytes = 2 * chunk
        try:
            views = [(C.c_char * chunk).from_address(h.ptr) for h in staging]
            for index, e in enumerate(entries):
                arr, ptr = self._placed(e["byte_length"], e.get("address_mod128"))
                self._owned.append(arr)

                def consume(slot, offset, size, ptr=ptr):
                    check(lib().klb_memcpy_htod(ptr + offset, staging[slot].ptr, size, stream.handle))
                    events[slot].record(stream)
                    pending[slot] = True

                def ready(slot):
                    if pending[slot]:
                        events[slot].synchronize()
                        pending[slot] = False

                consume.ready = ready
                capfile.read_into(index, views, consume)
                count = e["byte_length"] // ELEMENT_SIZES[e["element_type"]]
                args.append(DeviceBuffer(e["position"], e["role"], e["element_type"], ptr, count, owner=arr))
            stream.synchronize()
        finally:
            stream.synchronize()
            for h in staging:
                h.free()
        return args

    def restore_outputs(self) -> None:
        for buf, keep in zip(self.outputs, self._pristine):
            self._copy(buf.ptr, keep.ptr, buf.nbytes)

    def _compute_expected(self) -> None:
        exe = self._build(self.default_config)
        geom = self.definition.derive_geometry(self.default_config, self.problem, self.scalar_env)
        self.restore_outputs()
        exe.launch(geom, self.args, timed=True)
        self._expected = []
        for buf in self.outputs:
            ref = DeviceArray(buf.nbytes)
            self._copy(ref.ptr, buf.ptr, buf.nbytes)
            self._expected.append(ref)
        self.ctx.stream.synchronize()
        self.restore_outputs()
        exe.close()

    # -- compilation -------------------------------------------------------------------
    def _key(self, config: Configuration) -> tuple:
        return tuple(sorted(config.items()))

    def prefetch(self, configs: Sequence[Configuration]) -> None:
        """Start NVRTC compiles of ``configs`` in the background."""
        for cfg in configs:
            key = self._key(cfg)
            if key in self._futures:
                continue
            try:
                req = self.definition.render_compile_request(cfg, self.problem, self.scalar_env)
            except EvalError:
                continue
            self._futures[key] = self.compiler.submit(req, self.ctx.ident)

    def _build(self, config: Configuration) -> CudaExecutable:
        req = self.definition.render_compile_request(config, self.problem, self.scalar_env)
        fut = self._futures.pop(self._key(config), None)
        image = fut.result() if fut is not None else self.compiler.compile_image(req, self.ctx.ident)
        exe = CudaExecutable(req, image, self.ctx)
        exe.load()
        return exe

    # -- verification ------------------------------------------------------------------
    def _compare(self, got: DeviceBuffer, ref: DeviceArray) -> tuple[float, float]:
        import ctypes as C

        from ._abi import check, lib

        lay = self.output_layout
        width = ELEMENT_SIZES[got.element_type]
        diff, mag = C.c_double(), C.c_double()
        if lay is not None:
            check(lib().klb_compare_fields(got.ptr, ref.ptr, width, 0, lay.istart, lay.iend, lay.jstart, lay.jend,
                                           lay.kstart, lay.kend, lay.jj, lay.kk, C.byref(diff), C.byref(mag),
                                           self.ctx.stream.handle))
        else:  # flat comparison over the whole buffer
            n = got.element_count
            check(lib().klb_compare_fields(got.ptr, ref.ptr, width, 0, 0, n, 0, 1, 0, 1, n, n, C.byref(diff),
                                           C.byref(mag), self.ctx.stream.handle))
        return diff.value, mag.value

    def verify_current(self) -> float:
        """Largest relative deviation of the current outputs from the expected ones."""
        worst = 0.0
        for buf, ref in zip(self.outputs, self._expected):
            diff, mag = self._compare(buf, ref)
            worst = max(worst, diff / mag if mag > 0 else diff)
        return worst

    # -- Executor --------------------------------------------------------------------------
    def measure(self, config: Configuration) -> Measurement:
        if self.broken:
            return Measurement(STATUS_LAUNCH_FAILED)
        stages: dict[str, float] = {}
        t0 = time.perf_counter()
        try:
            req = self.definition.render_compile_request(config, self.problem, self.scalar_env)
            fut = self._futures.pop(self._key(config), None)
            image = fut.result() if fut is not None else self.compiler.compile_image(req, self.ctx.ident)
            stages["compile"] = image.compile_seconds
        except (CompileError, EvalError):
            return Measurement(STATUS_COMPILE_FAILED, stage_timings=stages)
        stages["compile_wait"] = time.perf_counter() - t0
        exe = None
        try:
            t0 = time.perf_counter()
            exe = CudaExecutable(req, image, self.ctx)
            exe.load()
            stages["module_load"] = time.perf_counter() - t0
            geom = self.definition.derive_geometry(config, self.problem, self.scalar_env)
            if geom.threads_per_block > 1024 or geom.shared_mem_bytes > self.ctx.max_smem_optin:
                return Measurement(STATUS_LAUNCH_FAILED, stage_timings=stages)
            if self.verify:
                self.restore_outputs()
                exe.launch(geom, self.args, timed=True)
                err = self.verify_current()
                stages["verify_error"] = err
                tol = TOLERANCE.get(self.outputs[0].element_type, 1e-5) if self.outputs else 0.0
                if not err <= tol:
                    return Measurement(STATUS_INVALID_CONFIG, stage_timings=stages)
            flush = self.ctx.flush_buffer() if self.flush_l2 else None
            samples = exe.time_launches(geom, self.args, self.warmup, self.repetitions, flush=flush)
            if self.verify:
                self.restore_outputs()
        except (LaunchError, KlbError, EvalError, DefinitionError) as err:
            code = getattr(err, "code", None)
            text = str(err)
            if code in _STICKY or any(f"[klb {c}]" in text for c in _STICKY):
                self.broken = text
            return Measurement(STATUS_LAUNCH_FAILED, stage_timings=stages)
        finally:
            # every exit (invalid geometry, failed verification, launch error)
            # unloads the module; a poisoned context cannot unload, so skip it
            if exe is not None and not self.broken:
                try:
                    exe.close()
                except (KlbError, LaunchError):
                    pass
        objective = statistics.median(samples)
        stages["launch"] = objective
        stages["launch_min"] = min(samples)
        return Measurement(STATUS_OK, objective=objective, stage_timings=stages)

    def describe(self) -> dict:
        info = {
            "backend": "cuda",
            "device": self.ctx.ident.to_json_obj(),
            "space_fingerprint": self.definition.space.fingerprint(),
            "warmup": self.warmup,
            "repetitions": self.repetitions,
            "flush_l2": self.flush_l2,
            "verify": self.verify,
            "problem": list(self.problem),
            "precision": "fp64" if self.outputs and self.outputs[0].element_type == "f64" else "fp32",
        }
        if self.broken:
            info["broken"] = self.broken
        return info

    def close(self) -> None:
        for arr in self._owned + self._pristine + self._expected:
            arr.free()
        self._owned, self._pristine, self._expected = [], [], []
