"""Host-side cost of a cached ``WisdomKernel.launch`` (the paper's launch
overhead: 294 ms first launch, ~3 us later launches of the
C++ library) on the B200 path: first launch (select + NVRTC compile + module
load) and the per-call wall time of cached launches, enqueue only (no sync),
against the bare ``klb_launch`` C-ABI call of the same packed parameters.

    python tools/dispatch_overhead.py [--kernel diff_uvw --precision fp64 --grid 64,64,64 --launches 2000]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="diff_uvw")
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--grid", default="64,64,64")
    ap.add_argument("--launches", type=int, default=2000)
    ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
    ap.add_argument("--json-out", default=None)
    a = ap.parse_args(argv)

    from paper_2303_12374_b200 import CapturePolicy, WisdomKernel
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    ctx = open_device(0)
    lay = GridLayout(*(int(x) for x in a.grid.split(",")), a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    args = prob.args()
    out = {"kernel": a.kernel, "precision": a.precision, "grid": [lay.itot, lay.jtot, lay.ktot]}
    for tag, wdir in (("tuned", a.wisdom), ("default", tempfile.mkdtemp())):
        wk = WisdomKernel(prob.definition, NvrtcCompiler(ctx), wisdom_dir=wdir, capture_policy=CapturePolicy())
        t0 = time.perf_counter()
        first = wk.launch(ctx.ident, args)
        ctx.synchronize()
        first_s = time.perf_counter() - t0
        for _ in range(50):
            wk.launch(ctx.ident, args)
        ctx.synchronize()
        per = []
        for _ in range(a.launches):
            t0 = time.perf_counter()
            wk.launch(ctx.ident, args)
            per.append(time.perf_counter() - t0)
        ctx.synchronize()
        # the bare C-ABI launch of the same cached packed parameters
        handle, cfg, _ = wk.resolve(ctx.ident, prob.definition.derive_problem_size(prob.scalar_env()),
                                    prob.scalar_env())
        geom = prob.definition.derive_geometry(cfg, prob.definition.derive_problem_size(prob.scalar_env()),
                                               prob.scalar_env())
        grid, block, smem = handle._prepare(geom)
        params, _keep, _ = handle._params(args, None)
        bare = []
        for _ in range(a.launches):
            t0 = time.perf_counter()
            check(lib().klb_launch(handle.function, grid, block, smem, ctx.stream.handle, params))
            bare.append(time.perf_counter() - t0)
        ctx.synchronize()
        bound_call = wk.bind(ctx.ident, args)
        bnd = []
        for _ in range(a.launches):
            t0 = time.perf_counter()
            bound_call()
            bnd.append(time.perf_counter() - t0)
        ctx.synchronize()
        rep = wk.overhead_report()
        out[tag] = {
            "staging": cfg["staging"], "match_kind": first.match_kind,
            "first_launch_ms": round(first_s * 1e3, 2),
            "first_stages_ms": {k: round(v * 1e3, 3) for k, v in first.stage_timings.items()},
            "cached_launch_us_median": round(statistics.median(per) * 1e6, 2),
            "cached_launch_us_p90": round(sorted(per)[int(0.9 * len(per))] * 1e6, 2),
            "bare_klb_launch_us_median": round(statistics.median(bare) * 1e6, 2),
            "bound_launch_us_median": round(statistics.median(bnd) * 1e6, 2),
            "overhead_report_subsequent_us": {k: round(v * 1e6, 2) for k, v in rep.subsequent.items()},
        }
    prob.close()
    line = json.dumps(out)
    print(line)
    if a.json_out:
        Path(a.json_out).write_text(line + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
