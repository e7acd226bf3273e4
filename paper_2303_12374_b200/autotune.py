"""On-GPU tuning of live (device-resident) stencil problems -> wisdom files.

``kltune tune cap.klcap --backend cuda`` tunes a captured launch; for the
large grids of the benchmark (a 1024^3 fp32 diff_uvw capture is ~30 GB) this
module tunes the same launch without the disk round trip: the fields are
generated on the device (bit-identical to what a capture of the synthetic
application would hold) and ``CudaReplayExecutor`` replays them.  The result
is appended to ``<wisdom_dir>/<kernel_key>.wisdom`` with the reference's
keep-best semantics (wisdom.py:151-178), exactly like the CLI path.

    python -m paper_2303_12374_b200.autotune --kernel diff_uvw --precision fp32 \\
        --grid 1024,1024,1024 --strategy random --budget-evals 120 --wisdom wisdom/
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

from .backend import STATUS_OK
from .tuner import Budget, load_checkpoint, save_session, tune
from .wisdom import append_result, load_or_create, wisdom_path

__all__ = ["tune_problem", "main", "FOCUSED_TMA"]

#: The focused TMA sub-space the wisdom sessions enumerate exhaustively: XYZ
#: launch order (y-neighbour blocks run together, so their shared halo rows
#: are L2 hits — measured 20% faster than the other orders on diff_uvw
#: 1024^3), no register cap, zchunk 32..128, prefetch depth 1..2, every block
#: shape and thread tile of at least 32 columns.
FOCUSED_TMA = ('unravel == "XYZ" && min_blocks == 1 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && '
               'depth <= 2 && block_x * tile_x >= 32')


def tune_problem(kernel: str, precision: str, grid: tuple[int, int, int], ctx, *, strategy: str = "random",
                 budget: Budget | None = None, seed: int = 0, wisdom_dir: str | Path | None = "wisdom",
                 session_dir: str | Path | None = None, k_range: tuple[int, int] | None = None,
                 repetitions: int = 7, warmup: int = 3, restrict: str | None = None, family: str | None = None,
                 isolate: bool = False, checkpoint: bool = False, resume: bool = False, log=print):
    """One tuning session of ``kernel`` at ``grid`` on the B200 (writes the
    session into ``session_dir`` and the result into ``wisdom_dir``).
    ``checkpoint`` streams the session file while measuring; ``resume``
    continues that file if an earlier run of the same session left one
    (tuner.SessionCheckpoint / load_checkpoint)."""
    from .cuda.executor import CudaReplayExecutor
    from .stencils.layout import GridLayout
    from .stencils.problem import StencilProblem

    layout = GridLayout(*grid, precision)
    if isolate:
        # measurements in a worker process that is replaced after a sticky CUDA error (cuda/isolated.py)
        from .cuda.isolated import IsolatedReplayExecutor
        from .stencils.definitions import definition_for

        if k_range is not None:
            raise ValueError("isolated tuning of k sub-ranges is not supported")
        prob = None
        executor = IsolatedReplayExecutor({"kernel": kernel, "precision": precision, "grid": list(grid),
                                           "device": ctx.ordinal}, repetitions=repetitions, warmup=warmup,
                                          flush_l2=True, verify=True)
        definition = definition_for(kernel, precision)
    else:
        prob = StencilProblem(kernel, layout, ctx)
        args = prob.args(k_range)
        executor = CudaReplayExecutor(None, ctx, definition=prob.definition, args=args, repetitions=repetitions,
                                      warmup=warmup, flush_l2=True, verify=True, output_layout=layout)
        definition = prob.definition
    t0 = time.time()
    count = [0]

    def progress(rec):
        count[0] += 1
        m = rec.measurement
        if m.status == STATUS_OK and (count[0] % 10 == 0 or count[0] < 4):
            log(f"  [{count[0]}] {m.objective * 1e6:9.1f} us  {_short(rec.config)}")

    default_cfg = definition.space.default_config()[0]
    default_m = executor.measure(default_cfg)
    space = definition.space
    if family:
        from .stencils.definitions import family_space

        space = family_space(kernel, family, precision)
    if restrict:
        # explore a sub-space (e.g. 'staging == "ZMARCH"'); every point is valid in the
        # full space, so the session still feeds the kernel's real wisdom file
        from .space import ConfigSpace

        space = ConfigSpace(space.params, list(space.restrictions) + [restrict])
    session_path = None
    if session_dir is not None:
        Path(session_dir).mkdir(parents=True, exist_ok=True)
        tag = (f".{family.lower()}" if family else "") + (".restricted" if restrict else "")
        stem = f"{kernel}_{precision}_{'x'.join(map(str, executor.problem))}.{strategy}{tag}.seed{seed}"
        session_path = Path(session_dir) / f"{stem}.klsession"
    prior = None
    if resume and session_path is not None and session_path.exists():
        prior = load_checkpoint(session_path)
        log(f"  resuming {session_path.name}: {len(prior.evaluations)} evaluations recorded")
    session = tune(space, executor, strategy=strategy, budget=budget or Budget(max_evaluations=50),
                   seed=seed, device=ctx.ident, kernel_key=definition.kernel_key(),
                   problem=executor.problem, on_evaluation=progress, resume=prior,
                   checkpoint=session_path if (checkpoint or prior is not None) else None)
    cells = executor.problem[0] * executor.problem[1] * executor.problem[2]
    from .stencils.problem import BYTES_PER_CELL_WORDS

    words = BYTES_PER_CELL_WORDS[kernel]
    summary = {
        "kernel": kernel, "precision": precision, "grid": list(grid), "problem": list(executor.problem),
        "evaluations": len(session.evaluations), "ok": len(session.ok_evaluations()),
        "seconds": round(time.time() - t0, 1),
        "default_us": default_m.objective * 1e6 if default_m.status == STATUS_OK else None,
        "best_us": session.best_objective * 1e6 if session.best_objective else None,
        "best_config": session.best_config,
        "restrict": restrict,
        "family": family,
    }
    for tag in ("default", "best"):
        us = summary[f"{tag}_us"]
        if us:
            summary[f"{tag}_gcells"] = cells / (us * 1e-6) / 1e9
            summary[f"{tag}_gbs"] = cells * words * layout.elem_bytes / (us * 1e-6) / 1e9
    if session_path is not None:
        save_session(session, session_path)
    if wisdom_dir is not None and session.best is not None:
        wfile = load_or_create(wisdom_dir, session.kernel_key)
        append_result(wfile, session)
        wfile.save(wisdom_path(wisdom_dir, session.kernel_key))
    executor.close()
    if prob is not None:
        prob.close()
    return session, summary


def _short(cfg: dict) -> str:
    keys = ("staging", "block_x", "block_y", "block_z", "tile_x", "tile_y", "tile_z", "zchunk", "unravel", "min_blocks")
    return " ".join(f"{k}={cfg[k]}" for k in keys if k in cfg)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2303_12374_b200.autotune")
    from .stencils.definitions import ALL_KERNELS

    ap.add_argument("--kernel", choices=ALL_KERNELS, required=True)
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    ap.add_argument("--grid", default="256,256,256")
    ap.add_argument("--strategy", choices=("random", "surrogate", "exhaustive"), default="random")
    ap.add_argument("--budget-evals", type=int, default=60)
    ap.add_argument("--budget-seconds", type=float, default=900.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--wisdom", default="wisdom")
    ap.add_argument("--sessions", default=None)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--restrict", default=None, help="extra restriction expression to explore a sub-space")
    ap.add_argument("--focused", action="store_true", help="restrict to FOCUSED_TMA (with --family TMA)")
    ap.add_argument("--isolate", action="store_true",
                    help="measure in a worker process replaced after a sticky CUDA error (cuda/isolated.py)")
    ap.add_argument("--family", choices=("DIRECT", "ZMARCH", "TMA"), default=None,
                    help="tune one staging family (its fixed knobs narrowed; see definitions.family_space)")
    ap.add_argument("--checkpoint", action="store_true", help="stream the session file while measuring")
    ap.add_argument("--resume", action="store_true",
                    help="continue the session file an interrupted run of the same session left in --sessions")
    a = ap.parse_args(argv)
    from .cuda import open_device

    ctx = open_device(a.device)
    grid = tuple(int(x) for x in a.grid.split(","))
    restrict = FOCUSED_TMA if a.focused else a.restrict
    _, summary = tune_problem(a.kernel, a.precision, grid, ctx, strategy=a.strategy,
                              budget=Budget(a.budget_evals, a.budget_seconds), seed=a.seed, wisdom_dir=a.wisdom,
                              session_dir=a.sessions, restrict=restrict, family=a.family, isolate=a.isolate,
                              checkpoint=a.checkpoint, resume=a.resume)
    line = json.dumps(summary, sort_keys=True)
    print(line)
    if a.json_out:
        with open(a.json_out, "a") as fh:
            fh.write(line + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
