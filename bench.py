#!/usr/bin/env python
"""Benchmark: BASELINE.json metric on B200 — Gcells/s and HBM GB/s (roofline
fraction), wisdom-tuned vs default configuration, 1/2/4/8 GPUs.

Workload (``--workload``, default = BASELINE config 4, the one configuration
quoted at every GPU count): diff_uvw fp32 on a 1024x1024x1024 grid,
z-slab decomposed over the N ranks with NCCL halo exchange overlapped with the
interior launch (strong scaling: the grid is fixed).  One step = one
application of the stencil to the whole grid (+ the halo exchange).

    python bench.py [--gpus N --steps K --warmup W]          # our arm
    python bench.py --impl reference [...]                    # CPU reference arm

Our arm prints ONE JSON line (rank 0).  ``value`` = interior cells of the
whole grid / device step time (CUDA events on the compute stream, max over
ranks), inputs resident in HBM; ``e2e`` = same metric with every step's
fields copied host->device from pinned memory and the tendencies copied back;
``roofline`` = the dominant (interior) kernel's algorithmic bytes / its
event-timed duration vs MEASURED_PEAKS.json; ``cpu_baseline`` = the NumPy
oracle on the host cores (bounded sample); ``variants`` = tuned vs default;
``suite`` (N=1) = BASELINE configs 1-3 tuned vs default (L2 flushed).

The reference arm times the reference CPU implementation of this path — the
NumPy oracle restating MicroHH (the reference package has no stencil code,
SURVEY.md §0) — on the same workload with all host threads, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gcells/s and achieved HBM GB/s (% of roofline), tuned vs default, 1/2/4/8 B200"
from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS as WORDS  # noqa: E402
WORKLOADS = {
    "diff_uvw_fp32_1024": ("diff_uvw", "fp32", (1024, 1024, 1024),
                           "BASELINE config 4: diff_uvw fp32 1024^3, z-slab decomposed over N GPUs, NVLink halo exchange"),
    "advec_u_fp32_256": ("advec_u", "fp32", (256, 256, 256), "BASELINE config 2: advec_u fp32 256^3, wisdom-selected"),
    "advec_u_fp64_512": ("advec_u", "fp64", (512, 512, 512), "BASELINE config 3: advec_u fp64 512^3"),
    "diff_uvw_fp64_512": ("diff_uvw", "fp64", (512, 512, 512), "BASELINE config 3: diff_uvw fp64 512^3"),
    # small grids for the multi-process plumbing test (not a BASELINE configuration)
    "diff_uvw_fp32_256": ("diff_uvw", "fp32", (256, 256, 256), "diff_uvw fp32 256^3 (multi-process plumbing test)"),
    "advec_u_fp32_256x256x96": ("advec_u", "fp32", (256, 256, 96), "advec_u fp32 256x256x96 (multi-process plumbing test)"),
}
SUITE = [
    ("diff_uvw", "fp64", (64, 64, 64), "config 1"),
    ("advec_u", "fp32", (256, 256, 256), "config 2"),
    ("advec_u", "fp64", (512, 512, 512), "config 3"),
    ("diff_uvw", "fp64", (512, 512, 512), "config 3"),
    ("advec_u", "fp32", (512, 512, 512), "north_star 512^3"),
    ("diff_uvw", "fp32", (512, 512, 512), "north_star 512^3"),
]
#: SURVEY §8f row 2 — the rest of the MicroHH family (DIRECT kernels), 512^3
FAMILY_SUITE = [(k, p, (512, 512, 512), "§8f family") for k in ("advec_v", "advec_w", "advec_s", "diff_c", "evisc_smag")
                for p in ("fp32", "fp64")]
#: SURVEY §8f row 1 — the RK3 substep fused into diff_uvw's store vs diff_uvw + a separate RK3 pass
FUSION_SUITE = [(k, p, (512, 512, 512), "§8f fusion") for p in ("fp32", "fp64")
                for k in ("diff_uvw", "rk3_uvw", "diff_uvw_rk3")]


def fusion_summary(rows):
    """Fused (diff_uvw_rk3) vs unfused (diff_uvw + rk3_uvw) per precision, tuned configs."""
    out = []
    by = {(r["kernel"], r["precision"]): r for r in rows if isinstance(r, dict) and "tuned" in r}
    for p in ("fp32", "fp64"):
        try:
            fused = by["diff_uvw_rk3", p]["tuned"]["us"]
            unfused = by["diff_uvw", p]["tuned"]["us"] + by["rk3_uvw", p]["tuned"]["us"]
        except KeyError:
            continue
        out.append({"precision": p, "fused_us": fused, "unfused_us": round(unfused, 2),
                    "speedup": round(unfused / fused, 3), "words_per_cell": {"fused": 13, "unfused": 22}})
    return out


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    try:
        data = json.loads(path.read_text())
        return float(data["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# distributed plumbing (host side only: barrier, max over ranks, NCCL id)


class Dist:
    """Rank plumbing of the N-GPU job, torch-free: ``ProcessGroup``
    (klb_group_*, one shared-memory segment; barrier, max/sum over ranks,
    NCCL-id broadcast).  RANK / WORLD_SIZE / LOCAL_RANK come from the
    launcher — torchrun, or ``bench.py --gpus N``'s own spawner."""

    def __init__(self):
        self.rank = env_int("RANK", 0)
        self.world = env_int("WORLD_SIZE", 1)
        self.local = env_int("LOCAL_RANK", self.rank)
        self.group = None
        if self.world > 1:
            from paper_2303_12374_b200.group import ProcessGroup

            self.group = ProcessGroup(self.rank, self.world, timeout=float(os.environ.get("KLB_GROUP_TIMEOUT", 600)))

    def barrier(self):
        if self.group:
            self.group.barrier()

    def max(self, value: float) -> float:
        return self.group.max(value) if self.group else value

    def sum(self, value: float) -> float:
        return self.group.sum(value) if self.group else value

    def broadcast_bytes(self, payload: bytes | None, size: int) -> bytes:
        return self.group.broadcast(payload, size=size) if self.group else payload

    def close(self):
        if self.group:
            self.group.close()


def spawn_ranks(n: int, argv: list[str]) -> int:
    """``--gpus N`` without a launcher: start N ranks of this script (rank r
    on GPU r), each with RANK/WORLD_SIZE/LOCAL_RANK and one shared group name;
    rank 0 prints the JSON line.  A failing rank stops the others."""
    import subprocess

    group = f"/klb_bench_{os.getpid()}_{time.time_ns()}"
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(n), LOCAL_RANK=str(r), LOCAL_WORLD_SIZE=str(n),
                   KLB_GROUP=group, MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *argv], env=env))
    rc = 0
    while procs:
        for p in list(procs):
            code = p.poll()
            if code is None:
                continue
            procs.remove(p)
            if code != 0:
                rc = rc or code
                for q in procs:
                    q.terminate()
        time.sleep(0.05)
    return rc


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)


class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, indices, period=0.02):
        self.indices = list(indices)
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self.error = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handles = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in self.indices]
            self.max_mhz = max(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM) for h in self.handles)
        except Exception as err:  # NVML missing: report, do not fail the run
            self.nvml, self.handles, self.error = None, [], repr(err)

    def _run(self):
        while not self._stop.is_set():
            for h in self.handles:
                try:
                    self.samples.append(self.nvml.nvmlDeviceGetClockInfo(h, self.nvml.NVML_CLOCK_SM))
                    mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, name in self.REASONS.items():
                        if mask & bit and name != "gpu_idle":
                            self.reasons.add(name)
                except Exception as err:
                    self.error = repr(err)
            time.sleep(self.period)

    def __enter__(self):
        if self.handles:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def report(self):
        out = {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.error:
            out["note"] = self.error
        return out


# ---------------------------------------------------------------------------
# CPU reference (the NumPy oracle on the host cores)


class CpuOracle:
    """The CPU restatement of the path on a bounded z-sample of the workload.

    Prefers the C restatement (oracle/stencil_ref.c via oracle/cref.py, in the
    workload's precision, one z-chunk per host thread); falls back to the NumPy
    oracle (float64, threads over z-chunks) when the C library is not built.
    Input generation happens once, outside every timed region.
    """

    def __init__(self, kernel, precision, grid, threads, planes_per_thread=None, full=False):
        import numpy as np

        from oracle import cref
        from oracle.synth import synth_field
        from paper_2303_12374_b200.stencils.problem import KERNEL_FIELDS
        from paper_2303_12374_b200.stencils.profiles import FIELD_SEED_BASE, FIELD_SPECS, make_profiles

        self.kernel, self.threads = kernel, threads
        itot, jtot, ktot = grid
        g = 3
        per = planes_per_thread or (4 if itot * jtot >= 512 * 512 else 16)
        self.nk = ktot if full else min(ktot, per * threads)
        self.cells = itot * jtot * self.nk
        dtype = np.float32 if precision == "fp32" else np.float64
        self.use_c = cref.available()
        self.kind = "C restatement (oracle/stencil_ref.c)" if self.use_c else "NumPy oracle (float64)"
        kc = self.nk + 2 * g
        self.pool = ThreadPoolExecutor(max_workers=threads)
        self.f = {}
        t0 = time.perf_counter()
        for name in KERNEL_FIELDS[kernel]:
            off, lo, hi = FIELD_SPECS[name]
            if self.use_c:  # the C twin of the generator, one z-chunk per thread (whole 1024^3 grids)
                self.f[name] = cref.synth_field(FIELD_SEED_BASE + off, lo, hi, itot + 2 * g, jtot + 2 * g, kc, g, g,
                                                dtype=dtype, threads=threads, pool=self.pool)
            else:
                self.f[name] = synth_field(FIELD_SEED_BASE + off, lo, hi, itot + 2 * g, jtot + 2 * g, kc, g, g,
                                           dtype=dtype)
        self.setup_seconds = time.perf_counter() - t0
        self.prof = make_profiles(ktot + 2 * g, g).window(0, kc).as_dtype(dtype)
        self.interior = (itot, jtot, self.nk)

    def step(self):
        from oracle import cref, stencil_oracle

        f, p = self.f, self.prof
        if self.use_c:
            if self.kernel == "advec_u":
                cref.advec_u(f["ut"], f["u"], f["v"], f["w"], p.rhoref, p.rhorefh, p.dzi, 1.0, 1.0,
                             threads=self.threads, pool=self.pool)
            else:
                cref.diff_uvw(f["ut"], f["vt"], f["wt"], f["evisc"], f["u"], f["v"], f["w"], p.dzi, p.dzhi, p.rhoref,
                              p.rhorefh, 1.0, 1.0, threads=self.threads, pool=self.pool)
            return
        g = 3
        per = max(1, -(-self.nk // self.threads))

        def work(k0):
            n = min(per, self.nk - k0)
            sl = slice(k0, k0 + n + 2 * g)
            ff = {k: v[sl] for k, v in f.items()}
            pp = {k: getattr(p, k)[sl] for k in ("rhoref", "rhorefh", "dzi", "dzhi")}
            inter = (self.interior[0], self.interior[1], n)
            if self.kernel == "advec_u":
                stencil_oracle.advec_u(ff["ut"], ff["u"], ff["v"], ff["w"], pp["rhoref"], pp["rhorefh"], pp["dzi"],
                                       1.0, 1.0, interior=inter)
            else:
                stencil_oracle.diff_uvw(ff["ut"], ff["vt"], ff["wt"], ff["evisc"], ff["u"], ff["v"], ff["w"],
                                        pp["dzi"], pp["dzhi"], pp["rhoref"], pp["rhorefh"], 1.0, 1.0, interior=inter)

        list(self.pool.map(work, range(0, self.nk, per)))

    def rate(self, reps=3):
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            self.step()
            times.append(time.perf_counter() - t0)
        return self.cells / statistics.median(times) / 1e9, statistics.median(times)

    def close(self):
        self.pool.shutdown()


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, dist):
    """The reference arm: the CPU implementation of the path (the C
    restatement, all host threads) applied to the WHOLE grid of the workload
    each step — inputs generated once outside the timed region — so
    ``ms_per_step`` is a measured full-grid step.  The run stops early (and
    reports the steps it ran) if it would exceed ``--reference-budget``
    seconds."""
    kernel, precision, grid, label = WORKLOADS[args.workload]
    if dist.rank != 0:
        return 0
    threads = host_threads()
    cpu = CpuOracle(kernel, precision, grid, threads, full=True)
    t_start = time.perf_counter()
    warm = 0
    for _ in range(args.warmup):
        cpu.step()
        warm += 1
        if time.perf_counter() - t_start > args.reference_budget / 3:
            break
    secs = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu.step()
        secs.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > args.reference_budget:
            break
    cpu.close()
    step_s = statistics.median(secs)
    value = cpu.cells / step_s / 1e9
    sample = (f"the whole grid ({cpu.cells} cells, {grid[2]} z-planes) of {label}; {cpu.kind}, {threads} host "
              f"threads over z-chunks; median of {len(secs)} full steps (inputs generated once, "
              f"{cpu.setup_seconds:.1f} s, untimed)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "Gcells/s", "n_gpus": args.gpus,
        "steps": len(secs), "warmup": warm, "ms_per_step": round(step_s * 1e3, 3),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if precision == "fp32" else "f64", "data": DATA,
        "config": workload_config(args, kernel, precision, grid, label, args.gpus),
        "cpu_baseline": {"value": round(value, 5), "unit": "Gcells/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "Gcells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if len(secs) < args.steps:
        line["steps_requested"] = args.steps
    print(json.dumps(line), flush=True)
    return 0


DATA = "synthetic (splitmix64 fields generated on device; oracle/synth.py twin)"


def workload_config(args, kernel, precision, grid, label, world):
    """The ``config`` object both arms print (identical, so the driver can
    match the arms' lines)."""
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import KERNEL_FIELDS

    wisdom_dir = Path(args.wisdom)
    nf, field = len(KERNEL_FIELDS[kernel]), GridLayout(*grid, precision, align_bytes=args.row_align).alloc_bytes
    l2 = (f"inputs larger than L2 ({nf} fields x {field / 1e9:.2f} GB), no flush" if nf * field > 2 * 126e6
          else f"working set {nf * field / 1e6:.0f} MB (under 2x L2), no flush")
    return {"workload": label, "kernel": kernel, "precision": precision, "grid": list(grid),
            "decomposition": f"z-slab x{world}", "parallelism": f"slab{world}", "ghost_cells": 3,
            "row_align_bytes": args.row_align, "l2": l2,
            "wisdom": str(wisdom_dir.relative_to(ROOT)) if wisdom_dir.is_relative_to(ROOT) else str(wisdom_dir)}


# ---------------------------------------------------------------------------
# our arm


def timed_steps(driver, dist, steps, time_kernel=True):
    """Device seconds per step (max over ranks) and mean dominant-kernel seconds."""
    from paper_2303_12374_b200.cuda import Event

    pairs = [(Event(), Event()) for _ in range(steps)] if time_kernel else []
    start, stop = Event(), Event()
    launches = 0
    dist.barrier()
    driver.ctx.synchronize()
    start.record(driver.compute)
    for s in range(steps):
        launches += driver.step(pairs[s] if time_kernel else None)
    stop.record(driver.compute)
    stop.synchronize()
    driver.ctx.synchronize()
    dist.barrier()
    step_s = start.elapsed_ms(stop) * 1e-3 / steps
    kern_s = statistics.mean(a.elapsed_ms(b) for a, b in pairs) * 1e-3 if pairs else None
    return dist.max(step_s), (dist.max(kern_s) if kern_s is not None else None), launches


def same_box_copy_gbs(ctx, nbytes=1 << 31, reps=10):
    """This box's device-to-device copy bandwidth right now (read + write
    bytes / time, best of ``reps`` event-timed copies of ``nbytes``) — the
    MEASURED_PEAKS.json method repeated in the same run, so the kernel's
    fraction can also be read against the box it ran on (HBM bandwidth
    differs a few per cent between boxes and clocks)."""
    from paper_2303_12374_b200.cuda import DeviceArray, Event
    from paper_2303_12374_b200.cuda._abi import check, lib

    src, dst = DeviceArray(nbytes), DeviceArray(nbytes)
    s = ctx.stream
    try:
        best = float("inf")
        for i in range(reps + 3):
            e0, e1 = Event(), Event()
            e0.record(s)
            check(lib().klb_memcpy_dtod(dst.ptr, src.ptr, nbytes, s.handle))
            e1.record(s)
            e1.synchronize()
            if i >= 3:
                best = min(best, e0.elapsed_ms(e1) * 1e-3)
        return 2 * nbytes / best / 1e9
    finally:
        src.free()
        dst.free()


def run_e2e(driver, dist, steps, chunks, copy_streams=1):
    """End to end through the public API: every step streams all fields from
    pinned host memory and the tendencies back (``SlabDriver.step_host``:
    chunked, uploads / kernels / downloads overlapped on three streams)."""
    from paper_2303_12374_b200.cuda import Event, HostPinned
    from paper_2303_12374_b200.cuda._abi import check, lib

    prob = driver.problem
    nbytes = prob.layout.alloc_bytes
    host = {}
    for n in prob.fields:
        buf = HostPinned(nbytes)
        check(lib().klb_memcpy_dtoh(buf.ptr, prob.fields[n].ptr, nbytes, driver.compute.handle))
        host[n] = buf
    driver.compute.synchronize()
    ptrs = {n: b.ptr for n, b in host.items()}
    launches = driver.step_host(ptrs, chunks, copy_streams)  # warm-up: selects + compiles every chunk's sub-range
    driver.compute.synchronize()
    start, stop = Event(), Event()
    dist.barrier()
    driver.ctx.synchronize()
    start.record(driver.compute)
    for _ in range(steps):
        driver.step_host(ptrs, chunks, copy_streams)
    stop.record(driver.compute)
    stop.synchronize()
    dist.barrier()
    step_s = dist.max(start.elapsed_ms(stop) * 1e-3 / steps)
    h2d, d2h = driver.stream_bytes
    for buf in host.values():
        buf.free()
    return step_s, int(dist.sum(h2d)), int(dist.sum(d2h)), launches


def ncu_traffic(kernel_key_prefix):
    """DRAM bytes per launch from the committed ncu summary, if one matches."""
    for path in sorted((ROOT / "profiles").glob("*ncu_summary*.json"), reverse=True):
        try:
            data = json.loads(path.read_text())
        except Exception:
            continue
        entry = data.get(kernel_key_prefix)
        if entry and entry.get("dram_bytes"):
            return float(entry["dram_bytes"]), path.name
    return None, None


def suite_measure(ctx, compiler, wisdom_dir, peak, suite=SUITE, cpu=False):
    """BASELINE configs 1-3 (+ the north_star 512^3 fp32 pair) on one GPU:
    tuned (wisdom) vs default, L2 flushed per rep; with ``cpu`` also the C
    restatement of the path on the whole grid on all host threads (advec_u /
    diff_uvw rows; median of 3 steps, 1 at >= 512^3)."""
    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    rows = []
    empty = ROOT / "build" / "empty_wisdom"
    empty.mkdir(parents=True, exist_ok=True)
    for kernel, precision, grid, tag in suite:
        lay = GridLayout(*grid, precision)
        prob = StencilProblem(kernel, lay, ctx)
        row = {"config": tag, "kernel": kernel, "precision": precision, "grid": list(grid)}
        for variant, wdir in (("tuned", wisdom_dir), ("default", empty)):
            wk = WisdomKernel(prob.definition, compiler, wisdom_dir=wdir, capture_policy=CapturePolicy())
            env = prob.scalar_env()
            problem = prob.definition.derive_problem_size(env)
            handle, cfg, kind = wk.resolve(ctx.ident, problem, env)
            geom = prob.definition.derive_geometry(cfg, problem, env)
            secs = handle.time_launches(geom, prob.args(), warmup=3, reps=15, flush=ctx.flush_buffer())
            t = statistics.median(secs)
            gbs = prob.algorithmic_bytes / t / 1e9
            row[variant] = {"us": round(t * 1e6, 2), "gcells": round(lay.cells / t / 1e9, 2), "gbs": round(gbs, 1),
                            "frac": round(gbs / peak, 4), "match_kind": kind}
        prob.close()
        if cpu and kernel in ("advec_u", "diff_uvw"):
            try:
                threads = host_threads()
                oracle = CpuOracle(kernel, precision, grid, threads, full=True)
                oracle.step()
                rate, secs_cpu = oracle.rate(reps=1 if lay.cells >= 512 ** 3 else 3)
                oracle.close()
                row["cpu"] = {"gcells": round(rate, 5), "cores": threads, "kind": "port",
                              "sample": f"whole grid; {oracle.kind}; step {secs_cpu:.4f} s"}
            except Exception as err:  # report, never hide
                row["cpu"] = {"error": repr(err)[:200]}
        rows.append(row)
    return rows


GRAPH_SUITE = [("diff_uvw", "fp64", (64, 64, 64), "config 1"), ("advec_u", "fp32", (128, 128, 128), "128^3")]


def graph_measure(ctx, compiler, wisdom_dir, peak, n=200):
    """Launch-bound small problems (config 1): n back-to-back applications of
    the tuned kernel (L2 warm, no flush between them — the working set stays
    in L2) enqueued one bound launch at a time, with programmatic dependent
    launch (PDL), replayed as one captured CUDA graph, and as a graph with
    PDL edges; device time per application from events on the launching
    stream, plus the host enqueue cost per application.  The cold (L2
    flushed, eager) figure of the same kernel is the ``suite`` row."""
    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import Event, Stream
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import KERNEL_FIELDS, StencilProblem

    rows = []
    stream = Stream.create()
    try:
        for kernel, precision, grid, tag in GRAPH_SUITE:
            lay = GridLayout(*grid, precision)
            prob = StencilProblem(kernel, lay, ctx)
            wk = WisdomKernel(prob.definition, compiler, wisdom_dir=wisdom_dir, capture_policy=CapturePolicy())
            run = wk.bind(ctx.ident, prob.args(), stream=stream)
            run_pdl = wk.bind(ctx.ident, prob.args(), stream=stream, pdl=True)
            g = wk.graph(ctx.ident, prob.args(), stream, repeat=n)
            gp = wk.graph(ctx.ident, prob.args(), stream, repeat=n, pdl=True)
            footprint = len(KERNEL_FIELDS[kernel]) * lay.alloc_bytes
            row = {"config": tag, "kernel": kernel, "precision": precision, "grid": list(grid), "applications": n,
                   "algorithmic_bytes_per_application": prob.algorithmic_bytes,
                   "working_set_bytes": footprint, "l2_resident": footprint < 126e6}
            variants = {"eager": lambda: [run() for _ in range(n)],
                        "eager_pdl": lambda: [run_pdl() for _ in range(n)],
                        "graph": lambda: g.launch(stream), "graph_pdl": lambda: gp.launch(stream)}
            for variant, go in variants.items():
                best = None
                for _ in range(3):
                    go()  # warm
                    stream.synchronize()
                    e0, e1 = Event(), Event()
                    e0.record(stream)
                    t0 = time.perf_counter()
                    go()
                    host = time.perf_counter() - t0
                    e1.record(stream)
                    e1.synchronize()
                    dev = e0.elapsed_ms(e1) * 1e-3
                    if best is None or dev < best[0]:
                        best = (dev, host)
                per = best[0] / n
                row[variant] = {"us_per_application": round(per * 1e6, 3),
                                "host_enqueue_us_per_application": round(best[1] / n * 1e6, 3),
                                "gcells": round(lay.cells / per / 1e9, 2),
                                # L2-resident: the HBM roofline does not bound these; GB/s of algorithmic
                                # bytes per application, reported beside (not against) the HBM peak
                                "algorithmic_gbs": round(prob.algorithmic_bytes / per / 1e9, 1),
                                "of_hbm_peak": round(prob.algorithmic_bytes / per / 1e9 / peak, 3)}
            row["graph_speedup"] = round(row["eager"]["us_per_application"] / row["graph"]["us_per_application"], 3)
            row["graph_pdl_speedup"] = round(row["eager"]["us_per_application"] /
                                             row["graph_pdl"]["us_per_application"], 3)
            g.close()
            gp.close()
            prob.close()
            rows.append(row)
    finally:
        stream.close()
    return rows


def other_halo_variant(args, dist, driver, kernel, precision, grid, ctx, exchanger, compiler, wisdom_dir):
    """N > 1 over IPC: the halo mode the headline did not use, timed the same
    way, and checked against it — both modes' tendencies after one step from
    the same state must agree on every rank (compared on the device)."""
    import ctypes as C

    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.slab import SlabDriver

    mode = "exchange" if driver.fused else "fused"
    other = SlabDriver(kernel, precision, grid, ctx, rank=dist.rank, nranks=dist.world, exchanger=exchanger,
                       compiler=compiler, wisdom_dir=wisdom_dir, halo=mode, align_bytes=args.row_align)
    try:
        other.resolve()
        for _ in range(args.warmup):
            other.step()
        step_s, _, launches = timed_steps(other, dist, args.steps, time_kernel=False)
        worst = 0.0
        for drv in (driver, other):
            drv.problem.regenerate(drv.problem.outputs())
            drv.step()
        ctx.synchronize()
        dist.barrier()
        lay = driver.layout
        for name in driver.problem.outputs():
            diff, mag = C.c_double(), C.c_double()
            check(lib().klb_compare_fields(driver.problem.field_ptr(name), other.problem.field_ptr(name),
                                           lay.elem_bytes, 0, lay.istart, lay.iend, lay.jstart, lay.jend,
                                           lay.kstart, lay.kend, lay.jj, lay.kk, C.byref(diff), C.byref(mag),
                                           driver.compute.handle))
            worst = max(worst, diff.value / mag.value if mag.value > 0 else diff.value)
        worst = dist.max(worst)
        return {"halo": mode, "ms_per_step": round(step_s * 1e3, 4),
                "gcells": round(grid[0] * grid[1] * grid[2] / step_s / 1e9, 3),
                "launches_per_step": launches // max(args.steps, 1), "max_rel_diff_vs_headline": worst}
    except Exception as err:  # report, never hide
        return {"halo": mode, "error": repr(err)[:300]}
    finally:
        try:
            other.close()
        except Exception as err:  # a sticky device error surfaces here; the headline line is still printed
            print(f"klb: closing the {mode} variant failed: {err!r}", file=sys.stderr, flush=True)


def run_ours(args, dist):
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.halo import IpcExchanger, NcclExchanger
    from paper_2303_12374_b200.slab import SlabDriver

    kernel, precision, grid, label = WORKLOADS[args.workload]
    # KL_DEVICE_ORDINAL pins every rank to one device (the single-GPU
    # multi-process test of the N > 1 path, tests/test_gpu_multiproc.py)
    forced = os.environ.get("KL_DEVICE_ORDINAL")
    ctx = open_device(int(forced) if forced is not None else (dist.local if args.gpus > 1 or dist.world > 1 else 0))
    peak, peak_src = peaks()
    exchanger, transport = None, None
    if dist.world > 1:
        # ipc: neighbours map each other's fields (CUDA IPC) and pull halo
        # planes over NVLink with copy engines; nccl: ncclSend/ncclRecv;
        # auto (default): ipc if every rank's probe succeeds, else nccl
        transport = os.environ.get("KL_HALO_TRANSPORT", "auto")
        if transport == "auto":
            # peer memory when every rank can map its neighbours (agreed over
            # the group), else NCCL for the whole job
            ok, why = IpcExchanger.probe(dist.group)
            transport = "ipc" if ok else "nccl"
            if not ok and dist.rank == 0:
                print(f"klb: IPC transport unavailable ({why}); using NCCL", file=sys.stderr, flush=True)
        if transport == "nccl":
            uid = dist.broadcast_bytes(NcclExchanger.unique_id() if dist.rank == 0 else None, 128)
            exchanger = NcclExchanger(dist.rank, dist.world, uid)
        else:
            exchanger = IpcExchanger(dist.group)
        if dist.rank == 0:
            print(f"klb: halo transport={transport} comm nranks={dist.world}", file=sys.stderr, flush=True)
    compiler = NvrtcCompiler(ctx)
    wisdom_dir = Path(args.wisdom)
    empty = ROOT / "build" / "empty_wisdom"
    empty.mkdir(parents=True, exist_ok=True)

    # the fused halo (diff_uvw_peer reading the neighbours' planes through
    # IPC mappings) needs peer memory; with NCCL only the exchange runs
    from paper_2303_12374_b200.slab import FUSED_HALO

    can_fuse = kernel in FUSED_HALO and dist.world > 1 and transport == "ipc"
    halo = args.halo if can_fuse else "exchange"
    variants = {}
    results = {}
    for variant, wdir in (("tuned", wisdom_dir), ("default", empty)):
        # (the Table-2 default is a DIRECT configuration: it has no TMA staging to fuse the halo into)
        driver = SlabDriver(kernel, precision, grid, ctx, rank=dist.rank, nranks=dist.world, exchanger=exchanger,
                            compiler=compiler, wisdom_dir=wdir, halo=halo if variant == "tuned" else "exchange",
                            align_bytes=args.row_align)
        chosen = driver.resolve()
        for _ in range(args.warmup):
            driver.step()
        with ClockSampler([ctx.ordinal] if forced is not None or dist.world == 1 else range(dist.world)) as clocks:
            step_s, kern_s, launches = timed_steps(driver, dist, args.steps)
        cells_total = grid[0] * grid[1] * grid[2]
        # the dominant kernel: the interior sub-range, or the whole-slab launch of the fused halo
        main = "slab" if driver.fused else "interior"
        interior_cells = dist.sum(driver.cells_in(main) if main in driver.ranges else 0)
        kern_bytes = (driver.cells_in(main) if main in driver.ranges else 0) * WORDS[kernel] * \
            driver.layout.elem_bytes
        achieved = kern_bytes / kern_s / 1e9 if kern_s else None
        results[variant] = dict(driver=driver, step_s=step_s, kern_s=kern_s, launches=launches, clocks=clocks.report())
        variants[variant] = {
            "ms_per_step": round(step_s * 1e3, 4),
            "gcells": round(cells_total / step_s / 1e9, 3),
            "gbs": round(cells_total * WORDS[kernel] * driver.layout.elem_bytes / step_s / 1e9, 1),
            "frac_of_measured_hbm": round(cells_total * WORDS[kernel] * driver.layout.elem_bytes / step_s / 1e9 / peak, 4),
            "frac_of_8tbs": round(cells_total * WORDS[kernel] * driver.layout.elem_bytes / step_s / 1e9 / 8000.0, 4),
            "dominant_kernel_gbs_rank0": round(achieved, 1) if achieved else None,
            "selection": {name: {"match_kind": kind, "config": cfg} for name, (cfg, kind) in chosen.items()},
        }
        if variant == "tuned":
            results[variant]["kern_bytes"] = kern_bytes
            results[variant]["interior_cells"] = interior_cells
        else:
            driver.close()

    tuned = results["tuned"]
    driver = tuned["driver"]
    cells_total = grid[0] * grid[1] * grid[2]
    value = cells_total / tuned["step_s"] / 1e9
    # (opt-in: the fused halo's TMA reads of peer memory are verified on one
    # GPU only, so the default run never risks the headline line on it)
    if can_fuse and (args.halo_variant or args.halo == "fused"):
        variants["other_halo"] = other_halo_variant(args, dist, driver, kernel, precision, grid, ctx, exchanger,
                                                    compiler, wisdom_dir)

    e2e = None
    if args.e2e_steps > 0:
        host_driver = driver
        try:
            if driver.fused:  # the host-streamed step runs the exchange variant
                host_driver = SlabDriver(kernel, precision, grid, ctx, rank=dist.rank, nranks=dist.world,
                                         exchanger=exchanger, compiler=compiler, wisdom_dir=wisdom_dir,
                                         align_bytes=args.row_align)
            e2e_s, h2d, d2h, launches = run_e2e(host_driver, dist, args.e2e_steps, args.e2e_chunks,
                                                args.e2e_streams)
            e2e = {"value": round(cells_total / e2e_s / 1e9, 4), "unit": "Gcells/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "ms_per_step": round(e2e_s * 1e3, 2),
                   "launches_per_step": launches,
                   "h2d_d2h_gbs": round((h2d + d2h) / dist.world / e2e_s / 1e9, 1),
                   "path": f"SlabDriver.step_host: pinned host fields streamed in {args.e2e_chunks} z-chunks "
                           f"(H2D on {args.e2e_streams} stream(s) | WisdomKernel.launch per chunk | D2H tendencies "
                           f"on {args.e2e_streams} stream(s), all overlapped)"}
        except Exception as err:  # report, never hide
            e2e = {"value": None, "unit": "Gcells/s", "error": repr(err)[:300]}
        finally:
            if host_driver is not driver:
                host_driver.close()

    traffic, traffic_src = ncu_traffic(f"{kernel}_{precision}_{grid[0]}x{grid[1]}x{grid[2] // dist.world}")
    achieved = tuned["kern_bytes"] / tuned["kern_s"] / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": f"{kernel}_{precision} " + ("whole-slab launch, fused halo (rank 0)" if driver.fused
                                                       else "interior sub-range (rank 0)"),
                "algorithmic_bytes_per_launch": tuned["kern_bytes"], "launch_ms": round(tuned["kern_s"] * 1e3, 4),
                "peak_source": peak_src, "frac_of_8tbs": round(achieved / 8000.0, 4)}
    if traffic_src:
        roofline["traffic_source"] = f"profiles/{traffic_src}"
    try:
        box = same_box_copy_gbs(ctx)
        roofline["same_box_copy_gbs"] = round(box, 1)
        roofline["frac_of_same_box_copy"] = round(achieved / box, 4)
    except Exception as err:  # diagnostic only
        roofline["same_box_copy_gbs"] = repr(err)[:120]

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gcells/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tuned["step_s"] * 1e3, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if precision == "fp32" else "f64",
        "data": DATA,
        "config": workload_config(args, kernel, precision, grid, label, dist.world),
        "halo_transport": transport,
        "halo": halo if dist.world > 1 else None,
        "variants": variants,
        "tuned_over_default": round(results["default"]["step_s"] / tuned["step_s"], 4),
        "gpu_launches": tuned["launches"],
        "clocks": tuned["clocks"],
        "roofline": roofline,
        "e2e": e2e,
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        # a bounded sample of the workload sized to ~10 s of CPU work: 32
        # z-planes per host thread of the same grid, steps repeated
        threads = host_threads()
        cpu = CpuOracle(kernel, precision, grid, threads, planes_per_thread=32)
        t0 = time.perf_counter()
        cpu.step()
        reps = min(30, max(3, round(10.0 / max(time.perf_counter() - t0, 1e-3))))
        rate, secs = cpu.rate(reps=reps)
        cpu.close()
        line["cpu_baseline"] = {
            "value": round(rate, 5), "unit": "Gcells/s", "cores": threads, "kind": "port",
            "sample": f"{cpu.nk} z-planes ({cpu.cells} cells) of the same grid; {cpu.kind}; {threads} host "
                      f"threads; median of {reps} steps ({secs:.3f} s each, {reps * secs:.1f} s of CPU work)"}
    if dist.rank == 0 and dist.world == 1 and args.suite:
        try:
            line["suite"] = suite_measure(ctx, compiler, wisdom_dir, peak, cpu=not args.no_cpu_baseline)
        except Exception as err:
            line["suite"] = {"error": repr(err)[:300]}
        try:
            line["family"] = suite_measure(ctx, compiler, wisdom_dir, peak, FAMILY_SUITE)
        except Exception as err:
            line["family"] = {"error": repr(err)[:300]}
        try:
            rows = suite_measure(ctx, compiler, wisdom_dir, peak, FUSION_SUITE)
            line["fusion"] = {"rows": rows, "summary": fusion_summary(rows)}
        except Exception as err:
            line["fusion"] = {"error": repr(err)[:300]}
        try:
            line["graph"] = graph_measure(ctx, compiler, wisdom_dir, peak)
        except Exception as err:
            line["graph"] = {"error": repr(err)[:300]}
    driver.close()
    if exchanger is not None:
        exchanger.close()
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="diff_uvw_fp32_1024")
    ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--e2e-streams", type=int, default=1, help="copy streams per direction in the e2e step")
    ap.add_argument("--row-align", type=int, default=int(os.environ.get("KL_ROW_ALIGN", "16")),
                    help="row-pitch quantum of the fields in bytes (GridLayout.align_bytes; 16 = densest rows)")
    ap.add_argument("--halo", choices=("exchange", "fused"), default=os.environ.get("KL_HALO", "exchange"),
                    help="N > 1, IPC transport: 'exchange' = interior launch overlapped with the halo pulls, then "
                         "the boundary launches; 'fused' = one diff_uvw_peer launch per slab reading the planes "
                         "outside it from the neighbours' fields")
    ap.add_argument("--halo-variant", action="store_true", default=bool(os.environ.get("KL_HALO_VARIANT")),
                    help="N > 1, IPC: also time the other halo mode and check it against the headline's tendencies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reference-budget", type=float, default=240.0,
                    help="seconds of timed full-grid steps the reference arm may spend")
    ap.add_argument("--suite", dest="suite", action="store_true", default=True)
    ap.add_argument("--no-suite", dest="suite", action="store_false")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus, sys.argv[1:] if argv is None else list(argv))
    dist = Dist()
    try:
        if args.impl == "reference":
            return run_reference(args, dist)
        return run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    sys.exit(main())
