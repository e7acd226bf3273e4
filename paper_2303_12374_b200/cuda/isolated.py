"""``IsolatedReplayExecutor`` — ``CudaReplayExecutor`` in a worker process.

The reference tuner records failures and never aborts (tuner.py:215-243), but
on a GPU a bad variant can leave a *sticky* error (illegal address, trap)
that poisons the CUDA context: every later launch in that process fails, so
an in-process executor can only report ``launch_failed`` for the rest of the
session (SURVEY.md §7 "Sticky CUDA errors from bad variants need process
isolation").  This executor keeps the replay executor in a spawned worker
process that owns its own context; when a measurement leaves the worker
broken — or hangs past ``timeout`` — the worker is discarded and the next
measurement starts a fresh one, so the session continues with a clean
context.  Within a healthy worker, compiles, uploaded buffers and the
expected outputs persist across measurements as in-process.

The worker rebuilds the problem from a ``spec``:
  ``{"capture": path}``                          a .klcap (reference layout), or
  ``{"kernel": k, "precision": p, "grid": [nx, ny, nz]}``   a live synthetic problem.
"""

from __future__ import annotations

import multiprocessing as mp
from typing import Any

from ..backend import STATUS_LAUNCH_FAILED, Executor, Measurement
from ..space import Configuration

__all__ = ["IsolatedReplayExecutor"]


def _worker(conn, spec: dict, kwargs: dict) -> None:
    from .device import open_device
    from .executor import CudaReplayExecutor

    ctx = open_device(int(spec.get("device", 0)))
    prob = None
    if "capture" in spec:
        ex = CudaReplayExecutor.from_file(spec["capture"], ctx, **kwargs)
    else:
        from ..stencils.layout import GridLayout
        from ..stencils.problem import StencilProblem

        lay = GridLayout(*spec["grid"], spec["precision"])
        prob = StencilProblem(spec["kernel"], lay, ctx)
        ex = CudaReplayExecutor(None, ctx, definition=prob.definition, args=prob.args(), output_layout=lay, **kwargs)
    conn.send(("ready", ex.describe()))
    while True:
        msg = conn.recv()
        if msg is None:
            break
        m = ex.measure(msg)
        conn.send(("result", (m.status, m.objective, dict(m.stage_timings), ex.broken)))
        if ex.broken:  # the context is poisoned: leave, the parent starts a fresh worker
            break
    conn.close()


class IsolatedReplayExecutor(Executor):
    reentrant = False

    def __init__(self, spec: dict, *, timeout: float = 120.0, **executor_kwargs: Any) -> None:
        self.spec = dict(spec)
        self.timeout = timeout
        self.kwargs = executor_kwargs
        self.restarts = 0
        self._proc = None
        self._conn = None
        self._describe: dict = {}
        self._start()

    def _start(self) -> None:
        ctx = mp.get_context("spawn")
        parent, child = ctx.Pipe()
        proc = ctx.Process(target=_worker, args=(child, self.spec, self.kwargs), daemon=True)
        proc.start()
        child.close()
        if not parent.poll(self.timeout * 5):
            proc.kill()
            raise RuntimeError("isolated replay worker did not start")
        kind, payload = parent.recv()
        self._proc, self._conn, self._describe = proc, parent, payload
        self.problem = tuple(payload.get("problem", ()))

    def _stop(self) -> None:
        if self._proc is not None:
            try:
                self._conn.send(None)
            except (OSError, EOFError, BrokenPipeError):
                pass
            self._proc.join(timeout=5)
            if self._proc.is_alive():
                self._proc.kill()
                self._proc.join()
        self._proc = self._conn = None

    def measure(self, config: Configuration) -> Measurement:
        if self._proc is None or not self._proc.is_alive():
            self._stop()
            self._start()
            self.restarts += 1
        try:
            self._conn.send(dict(config))
            if not self._conn.poll(self.timeout):
                raise TimeoutError
            _, (status, objective, stages, broken) = self._conn.recv()
        except (TimeoutError, EOFError, OSError, BrokenPipeError):
            # hung or died: discard the worker, report the configuration failed
            if self._proc is not None:
                self._proc.kill()
                self._proc.join()
            self._proc = self._conn = None
            return Measurement(STATUS_LAUNCH_FAILED, stage_timings={"isolated_restart": 1.0})
        if broken:
            self._proc.join(timeout=5)
            self._proc = self._conn = None
        return Measurement(status, objective=objective, stage_timings=stages)

    def describe(self) -> dict:
        out = dict(self._describe, isolated=True, restarts=self.restarts)
        out.pop("broken", None)
        return out

    def close(self) -> None:
        self._stop()
