"""Row-pitch alignment of the HBM layout, head to head on one box.

GridLayout(align_bytes=128) pads every row to a 128-byte multiple (interior
rows start on a 128-byte boundary, 288-element fp32 rows at 256^3);
align_bytes=16 keeps rows 16-byte aligned (264 elements), so a row's right
ghost cells and the next row's left ghost cells share DRAM bursts.  For each
workload the wisdom-selected configuration runs on both layouts (interleaved
rounds, L2 flushed before every launch, klb_time_launches), and the interior
tendencies of the two layouts must be bit-identical.  GPU only.

    python tools/layout_probe.py --work advec_u:fp32:256 --work diff_uvw:fp32:1024
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

DEFAULT_WORK = ["advec_u:fp32:256", "diff_uvw:fp64:64", "advec_u:fp32:512", "diff_uvw:fp32:512",
                "advec_u:fp64:512", "diff_uvw:fp64:512", "evisc_smag:fp32:512", "diff_uvw:fp32:1024"]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--work", action="append", default=[])
    ap.add_argument("--aligns", default="128,16")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--json-out")
    a = ap.parse_args(argv)

    import numpy as np

    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS, StencilProblem

    ctx = open_device(0)
    comp = NvrtcCompiler(ctx)
    flush = ctx.flush_buffer()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    aligns = [int(x) for x in a.aligns.split(",")]
    out = open(a.json_out, "a") if a.json_out else None
    for work in a.work or DEFAULT_WORK:
        kernel, precision, n = work.split(":")
        grid = (int(n),) * 3
        runs = []
        for al in aligns:
            lay = GridLayout(*grid, precision, align_bytes=al)
            prob = StencilProblem(kernel, lay, ctx)
            d = prob.definition
            wk = WisdomKernel(d, comp, wisdom_dir=ROOT / "wisdom", capture_policy=CapturePolicy())
            env = prob.scalar_env()
            problem = d.derive_problem_size(env)
            handle, config, kind = wk.resolve(ctx.ident, problem, env)
            geom = d.derive_geometry(config, problem, env)
            handle.launch(geom, prob.args(), timed=True)
            outs = {nm: lay.interior(prob.download(nm)).copy() for nm in prob.outputs()}
            prob.regenerate()
            runs.append(dict(align=al, lay=lay, prob=prob, handle=handle, geom=geom, config=config, kind=kind,
                             outs=outs, times=[]))
        same = all(np.array_equal(runs[0]["outs"][nm], r["outs"][nm]) for r in runs[1:] for nm in runs[0]["outs"])
        for _ in range(a.rounds):
            for r in runs:
                r["times"].append(statistics.median(r["handle"].time_launches(r["geom"], r["prob"].args(), 3, a.reps,
                                                                              flush=flush)))
        nbytes = BYTES_PER_CELL_WORDS[kernel] * runs[0]["lay"].elem_bytes * runs[0]["lay"].cells
        rec = {"kernel": kernel, "precision": precision, "grid": list(grid), "config": runs[0]["config"],
               "match_kind": runs[0]["kind"], "bit_identical": same}
        for r in runs:
            t = statistics.median(r["times"])
            rec[f"align{r['align']}"] = {"jj": r["lay"].jj, "us": round(t * 1e6, 2),
                                          "us_rounds": [round(x * 1e6, 2) for x in r["times"]],
                                          "frac": round(nbytes / t / 1e9 / peak, 4)}
            r["prob"].close()
        print(json.dumps(rec, sort_keys=True), flush=True)
        if out:
            out.write(json.dumps(rec, sort_keys=True) + "\n")
            out.flush()
    return 0


if __name__ == "__main__":
    sys.exit(main())
