"""Compile-time variants of a wisdom record, timed head to head on one box.

Each ``--variant`` is a comma-separated list of NAME=VALUE defines added to the
record's compile request (the empty string = the record as shipped); the
variants are timed interleaved for ``--rounds`` rounds (L2 flushed before
every launch, klb_time_launches) and checked bit-for-bit against the first
variant's outputs unless ``--no-check``.  GPU only.

    python tools/variant_probe.py --kernel advec_u --grid 256,256,256 \
        --variant "" --variant KL_L2HINT=1 --variant KL_L2HINT=9
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
    ap.add_argument("--variant", action="append", default=[])
    ap.add_argument("--config", action="append", default=[],
                    help="JSON config merged over the wisdom record (repeatable: each is a variant)")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--json-out")
    a = ap.parse_args(argv)

    import numpy as np

    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.cuda.compiler import CudaExecutable
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.kerneldef import CompileRequest
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS, StencilProblem

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    d = prob.definition
    env = prob.scalar_env()
    problem = d.derive_problem_size(env)
    comp = NvrtcCompiler(ctx)
    wk = WisdomKernel(d, comp, wisdom_dir=ROOT / "wisdom", capture_policy=CapturePolicy())
    _, record, kind = wk.resolve(ctx.ident, problem, env)
    configs = [dict(record, **json.loads(c)) for c in a.config] or [record]
    variants, exes, geoms = [], [], []
    for config in configs:
        base = d.render_compile_request(config, problem, env)
        for v in a.variant or [""]:
            extra = tuple(f"-D {x.strip()}" for x in v.split(",") if x.strip())
            req = CompileRequest(base.source, base.entry, base.defines + extra, base.flags)
            exe = CudaExecutable(req, comp.compile_image(req, ctx.ident), ctx)
            exe.load()
            exes.append(exe)
            geoms.append(d.derive_geometry(config, problem, env))
            variants.append((v, config))
    args = prob.args()
    outs = []
    if not a.no_check:
        for exe, geom in zip(exes, geoms):
            prob.regenerate()
            exe.launch(geom, args, timed=True)
            outs.append({n: prob.download(n).copy() for n in prob.outputs()})
        prob.regenerate()
    flush = ctx.flush_buffer()
    times = [[] for _ in exes]
    for _ in range(a.rounds):
        for i, exe in enumerate(exes):
            times[i].append(statistics.median(exe.time_launches(geoms[i], args, 3, a.reps, flush=flush)))
    nbytes = BYTES_PER_CELL_WORDS[a.kernel] * lay.elem_bytes * lay.cells
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    out = open(a.json_out, "a") if a.json_out else None
    for i, (v, config) in enumerate(variants):
        t = statistics.median(times[i])
        rec = {"kernel": a.kernel, "precision": a.precision, "grid": list(grid), "variant": v, "config": config,
               "blocks": geoms[i].grid[0], "match_kind": kind, "us": round(t * 1e6, 2), "us_rounds": [round(x * 1e6, 2) for x in times[i]],
               "frac": round(nbytes / t / 1e9 / peak, 4)}
        if outs:
            rec["bit_identical_to_first"] = all(np.array_equal(outs[i][n], outs[0][n]) for n in outs[0])
        print(json.dumps(rec, sort_keys=True), flush=True)
        if out:
            out.write(json.dumps(rec, sort_keys=True) + "\n")
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
