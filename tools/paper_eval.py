"""The paper's evaluation (§5: capture table, tuning histograms, the
cross-scenario matrix) repeated on one B200 for its eight scenarios —
advec_u / diff_uvw × 256³ / 512³ × float / double.

Per scenario:
  * capture: the first launch of the application kernel under a capture
    policy, streamed from HBM into a ``.klcap`` on local disk (time, bytes)
    — the paper's Table "Time and size required to capture kernel";
  * tuning distribution: a random session over the paper's own space (the
    DIRECT family = Table 2) of ``--random`` configurations, each as a
    fraction of the scenario's optimum; the optimum is the committed wisdom
    record (TMA staging) measured in the same process, so the B200 staging
    families show up as the gap between the best Table-2 point and 1.0;
    markers: the Table-2 default and "configuration C" (the advec_u 256³
    float optimum, the paper's reference point);
  * matrix: every scenario's optimum measured in every scenario of the same
    kernel where it is a valid point of that scenario's space (fraction of
    that scenario's optimum; n/a otherwise), and the PPM per row.
Writes one JSON document.  GPU only.

    python tools/paper_eval.py --random 150 --out paper_eval.json
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

SCENARIOS = [(k, n, p) for k in ("advec_u", "diff_uvw") for n in (256, 512) for p in ("fp32", "fp64")]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--random", type=int, default=150)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.backend import STATUS_OK
    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.report import ppm
    from paper_2303_12374_b200.stencils.definitions import family_space
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem
    from paper_2303_12374_b200.tuner import Budget, tune

    ctx = open_device(0)
    comp = NvrtcCompiler(ctx)
    out = {"device": ctx.ident.name, "scenarios": {}}
    execs, optima, tag = {}, {}, {}
    for kernel, n, prec in SCENARIOS:
        name = f"{kernel}-{n}^3-{'float' if prec == 'fp32' else 'double'}"
        tag[(kernel, n, prec)] = name
        lay = GridLayout(n, n, n, prec)
        prob = StencilProblem(kernel, lay, ctx)
        d = prob.definition
        # capture of the application's first launch, streamed from HBM
        with tempfile.TemporaryDirectory() as tmp:
            wk = WisdomKernel(d, comp, wisdom_dir=ROOT / "wisdom",
                              capture_policy=CapturePolicy(names=frozenset({d.name}), directory=tmp))
            ctx.synchronize()
            t0 = time.perf_counter()
            rep = wk.launch(ctx.ident, prob.args())
            ctx.synchronize()
            cap_s = time.perf_counter() - t0
            caps = list(Path(tmp).glob("*.klcap"))
            cap_bytes = sum(p.stat().st_size for p in caps) + sum(p.stat().st_size for p in Path(tmp).glob("*.cu"))
        prob.regenerate()
        ex = CudaReplayExecutor(None, ctx, definition=d, args=prob.args(), repetitions=a.reps, warmup=3,
                                flush_l2=True, verify=True, output_layout=lay)
        opt = ex.measure(rep.configuration)
        default = ex.measure(d.space.default_config()[0])
        sess = tune(family_space(kernel, "DIRECT", prec), ex, strategy="random",
                    budget=Budget(max_evaluations=a.random), seed=2303, device=ctx.ident,
                    kernel_key=d.kernel_key(), problem=ex.problem)
        ok = [e.measurement.objective for e in sess.evaluations if e.measurement.status == STATUS_OK]
        execs[(kernel, n, prec)] = (ex, prob, d)
        optima[(kernel, n, prec)] = (rep.configuration, opt.objective)
        fr = sorted(opt.objective / t for t in ok)
        out["scenarios"][name] = {
            "capture_seconds": round(cap_s, 3), "capture_bytes": cap_bytes,
            "optimum": {"config": rep.configuration, "match_kind": rep.match_kind,
                        "us": round(opt.objective * 1e6, 2)},
            "default_fraction": round(opt.objective / default.objective, 4),
            "table2_random": {"evaluated": len(sess.evaluations), "ok": len(ok),
                              "best_fraction": round(fr[-1], 4) if fr else None,
                              "median_fraction": round(statistics.median(fr), 4) if fr else None,
                              "fractions": [round(x, 4) for x in fr]},
        }
        print(name, out["scenarios"][name]["optimum"]["us"], out["scenarios"][name]["table2_random"]["best_fraction"],
              file=sys.stderr, flush=True)
    # configuration C (the paper's reference point) in every scenario of its kernel
    c_cfg = optima[("advec_u", 256, "fp32")][0]
    matrix = {}
    for src in SCENARIOS:
        row = {}
        for dst in SCENARIOS:
            if src[0] != dst[0]:
                continue
            ex, _, d = execs[dst]
            cfg = optima[src][0]
            if not d.space.is_valid(cfg):
                row[tag[dst]] = None
                continue
            m = ex.measure(cfg)
            row[tag[dst]] = round(optima[dst][1] / m.objective, 4) if m.status == STATUS_OK else None
        res = ppm(list(row.values()))  # (0 when a scenario's space does not hold the configuration)
        matrix[tag[src]] = {"fractions": row, "ppm": round(res.ppm, 4), "worst": round(res.worst, 4)}
    out["matrix"] = matrix
    for key in SCENARIOS:
        if key[0] == "advec_u":
            ex, _, d = execs[key]
            m = ex.measure(c_cfg) if d.space.is_valid(c_cfg) else None
            out["scenarios"][tag[key]]["configuration_C_fraction"] = (
                round(optima[key][1] / m.objective, 4) if m is not None and m.status == STATUS_OK else None)
    for ex, prob, _ in execs.values():
        ex.close()
        prob.close()
    Path(a.out).write_text(json.dumps(out, indent=1, sort_keys=True))
    return 0


if __name__ == "__main__":
    sys.exit(main())
