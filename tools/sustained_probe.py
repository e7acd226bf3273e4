"""Sustained-load head-to-head of wisdom candidates, the way the bench runs them.

The tuning objective is an isolated, L2-flushed launch; the bench's headline
is ``--steps`` back-to-back launches of the 1024^3 kernel under the board's
power cap (SM clocks settle at 1.6-1.8 GHz within milliseconds).  This tool
times the current record and a session's best configurations as batches of
``--batch`` back-to-back launches (after ``--warmup`` launches, CUDA events
around the batch; inputs far larger than L2), interleaved for ``--rounds``
rounds, and reports ms per launch — the figure the bench's ``value`` is made
of.  GPU only.

    python tools/sustained_probe.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 \
        --sessions gpurun_out/r04q/sessions/diff_uvw_fp32_1024x1024x1024*.klsession --top 6
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
    ap.add_argument("--kernel", default="diff_uvw")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="1024,1024,1024")
    ap.add_argument("--sessions", nargs="*", default=[])
    ap.add_argument("--top", type=int, default=6)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--batch", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--json-out")
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import Event, NvrtcCompiler, open_device
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS, StencilProblem
    from paper_2303_12374_b200.tuner import load_session

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    d = prob.definition
    env = prob.scalar_env()
    problem = d.derive_problem_size(env)
    comp = NvrtcCompiler(ctx)
    wk = WisdomKernel(d, comp, wisdom_dir=ROOT / "wisdom", capture_policy=CapturePolicy())
    _, record, _ = wk.resolve(ctx.ident, problem, env)
    default = d.space.default_config()[0]
    cands = [("current", dict(record))]
    seen = {json.dumps(record, sort_keys=True)}
    for path in a.sessions:
        sess = load_session(path)
        ok = sorted((e for e in sess.evaluations if e.measurement.status == "ok"), key=lambda e: e.measurement.objective)
        n = 0
        for e in ok:
            cfg = dict(default, **e.config)
            key = json.dumps(cfg, sort_keys=True)
            if key in seen:
                continue
            seen.add(key)
            cands.append((Path(path).name, cfg))
            n += 1
            if n >= a.top:
                break
    runs = []
    args = prob.args()
    for src, cfg in cands:
        exe = comp.compile(d.render_compile_request(cfg, problem, env), ctx.ident)
        exe.load()
        runs.append((src, cfg, exe.bound(d.derive_geometry(cfg, problem, env), args, stream=ctx.stream), []))
    s = ctx.stream
    for _ in range(a.rounds):
        for _, _, run, times in runs:
            for _ in range(a.warmup):
                run()
            e0, e1 = Event(), Event()
            e0.record(s)
            for _ in range(a.batch):
                run()
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_ms(e1) / a.batch)
    nbytes = BYTES_PER_CELL_WORDS[a.kernel] * lay.elem_bytes * lay.cells
    out = open(a.json_out, "a") if a.json_out else None
    for src, cfg, _, times in sorted(runs, key=lambda r: statistics.median(r[3])):
        ms = statistics.median(times)
        rec = {"kernel": a.kernel, "precision": a.precision, "grid": list(grid), "source": src, "config": cfg,
               "ms_per_launch": round(ms, 4), "ms_rounds": [round(t, 4) for t in times],
               "gcells": round(lay.cells / ms / 1e6, 2), "gbs": round(nbytes / ms / 1e6, 1)}
        print(json.dumps(rec, sort_keys=True), flush=True)
        if out:
            out.write(json.dumps(rec, sort_keys=True) + "\n")
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
