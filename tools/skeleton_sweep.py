"""Data-movement floor across configurations: the best distinct configurations
of a tuning session, each timed as compiled and as its KL_SKEL=1 skeleton
(TMA rings, barriers and output stores only — advec_u_tma.cuh,
evisc_smag_tma.cuh), L2 flushed.  Shows whether any tiling moves the bytes
faster than the wisdom record does (the floor the arithmetic sits on).  GPU only.

    python tools/skeleton_sweep.py --session profiles/sessions_r02/advec_u_fp32_256x256x256...klsession --top 30
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--session", required=True)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--json-out")
    ap.add_argument("--levels", default="1", help="KL_SKEL levels to time (advec_u: 2 = u boxes without halo, "
                                                  "3 = v/w boxes too)")
    a = ap.parse_args(argv)
    levels = [int(x) for x in a.levels.split(",")]

    from paper_2303_12374_b200.cuda import open_device
    from paper_2303_12374_b200.cuda.compiler import CudaExecutable
    from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
    from paper_2303_12374_b200.kerneldef import CompileRequest
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS, StencilProblem
    from paper_2303_12374_b200.tuner import load_session

    sess = load_session(a.session)
    kernel, precision = sess.kernel_key.split("-")[0].rsplit("_", 1)
    grid = tuple(sess.problem)
    ok = sorted((e for e in sess.evaluations if e.measurement.status == "ok"), key=lambda e: e.measurement.objective)
    seen, picks = set(), []
    for e in ok:
        sig = json.dumps(e.config, sort_keys=True)
        if sig not in seen:
            seen.add(sig)
            picks.append(e)
        if len(picks) >= a.top:
            break
    ctx = open_device(0)
    lay = GridLayout(*grid, precision)
    prob = StencilProblem(kernel, lay, ctx)
    d = prob.definition
    args = prob.args()
    ex = CudaReplayExecutor(None, ctx, definition=d, args=args, output_layout=lay, verify=False)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    nbytes = BYTES_PER_CELL_WORDS[kernel] * lay.elem_bytes * lay.cells
    out = open(a.json_out, "a") if a.json_out else None
    default = d.space.default_config()[0]
    for e in picks:
        cfg = dict(default, **e.config)  # sessions of an older space lack the later knobs (their defaults)
        rec = {"kernel": kernel, "precision": precision, "grid": list(grid), "config": cfg,
               "session_us": round(e.measurement.objective * 1e6, 2)}
        variants = [("full", ())] + [("skeleton" if lv == 1 else f"skeleton{lv}", (f"-D KL_SKEL={lv}",))
                                     for lv in levels]
        for tag, extra in variants:
            req = d.render_compile_request(cfg, ex.problem, ex.scalar_env)
            req = CompileRequest(req.source, req.entry, req.defines + extra, req.flags)
            geom = d.derive_geometry(cfg, ex.problem, ex.scalar_env)
            exe = CudaExecutable(req, ex.compiler.compile_image(req, ctx.ident), ctx)
            exe.load()
            secs = exe.time_launches(geom, args, 3, a.reps, flush=ctx.flush_buffer())
            exe.close()
            t = statistics.median(secs)
            rec[tag] = {"us": round(t * 1e6, 2), "frac": round(nbytes / t / 1e9 / peak, 4)}
        print(json.dumps(rec, sort_keys=True), flush=True)
        if out:
            out.write(json.dumps(rec, sort_keys=True) + "\n")
            out.flush()
    ex.close()
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
