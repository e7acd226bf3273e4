"""Probe the balanced y split (KL_YBAL, n row runs) of a TMA kernel: compile the given
configurations with -D KL_YBAL=1, launch nbx*n*nbz blocks, verify against
the default configuration's output and time (L2 flushed).  GPU only.

    python tools/ysplit_probe.py --kernel advec_u --precision fp32 --grid 256,256,256 \
        --case '{"block_y":8,"tile_y":1,"zchunk":128,"depth":4,"ysplit":37}' --case '{}'

A case may carry extra compile-time switches, e.g. '{"defines": {"KL_SKEL": 1}}'
(advec_u_tma.cuh's data-movement skeleton; its verify_err is meaningless).
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
    ap.add_argument("--kernel", default="advec_u")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="256,256,256")
    ap.add_argument("--case", action="append", required=True,
                    help='JSON overrides of the wisdom config plus "ysplit" (0 = natural tiling)')
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--json-out")
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.cuda import open_device
    from paper_2303_12374_b200.cuda.compiler import CudaExecutable
    from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
    from paper_2303_12374_b200.kerneldef import CompileRequest, LaunchGeometry
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS, StencilProblem
    from paper_2303_12374_b200.wisdom import load_or_create, select

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    d = prob.definition
    args = prob.args()
    ex = CudaReplayExecutor(None, ctx, definition=d, args=args, output_layout=lay, verify=True)
    default = d.space.default_config()[0]
    base = dict(select(load_or_create(ROOT / "wisdom", d.kernel_key()), ctx.ident, ex.problem, default).config)
    out = open(a.json_out, "a") if a.json_out else None
    bytes_ = BYTES_PER_CELL_WORDS[a.kernel] * lay.elem_bytes * lay.cells
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6458.7
    for text in a.case:
        over = json.loads(text)
        n = int(over.pop("ysplit", 0))
        extra = {str(k): int(v) for k, v in over.pop("defines", {}).items()}  # e.g. {"KL_SKEL": 1}
        cfg = dict(base, **over)
        if True:
            req = d.render_compile_request(cfg, ex.problem, ex.scalar_env)
            if n:
                req = CompileRequest(req.source, req.entry,
                                     tuple(x for x in req.defines if not x.startswith("-D KL_YBAL=")) +
                                     ("-D KL_YBAL=1",), req.flags)
            if extra:
                names = {f"-D {k}=" for k in extra}
                req = CompileRequest(req.source, req.entry,
                                     tuple(x for x in req.defines if not any(x.startswith(p) for p in names)) +
                                     tuple(f"-D {k}={v}" for k, v in extra.items()), req.flags)
            geom = d.derive_geometry(cfg, ex.problem, ex.scalar_env)
            if n:
                txy = cfg["block_x"] * cfg["tile_x"]
                nbx = -(-grid[0] // txy)
                nbz = -(-grid[2] // (cfg["block_z"] * cfg["tile_z"] * cfg["zchunk"]))
                if -(-grid[1] // n) > cfg["block_y"] * cfg["tile_y"]:
                    print(f"skip ysplit {n}: rows per block exceed the tile", flush=True)
                    continue
                geom = LaunchGeometry(block=geom.block, grid=(nbx * n * nbz, 1, 1),
                                      shared_mem_bytes=geom.shared_mem_bytes)
            try:
                exe = CudaExecutable(req, ex.compiler.compile_image(req, ctx.ident), ctx)
                exe.load()
                ex.restore_outputs()
                exe.launch(geom, args, timed=True)
                err = ex.verify_current()
                secs = exe.time_launches(geom, args, 3, a.reps, flush=ctx.flush_buffer())
                exe.close()
            except Exception as e:  # report and go on
                print(f"{json.dumps(cfg, sort_keys=True)} ysplit={n}: {e!r}", flush=True)
                continue
            t = statistics.median(secs)
            rec = {"defines": extra, "kernel": a.kernel, "precision": a.precision, "grid": list(grid), "config": cfg, "ysplit": n,
                   "blocks": geom.grid[0], "smem": geom.shared_mem_bytes, "us": t * 1e6, "min_us": min(secs) * 1e6,
                   "frac": bytes_ / t / 1e9 / peak, "verify_err": err}
            print(json.dumps(rec, sort_keys=True), flush=True)
            if out:
                out.write(json.dumps(rec, sort_keys=True) + "\n")
                out.flush()
    ex.close()
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
