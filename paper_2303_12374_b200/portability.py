"""BASELINE config 5: wisdom portability sweep on B200.

Tune each kernel/precision at the anchor shapes (128^3 … 1024^3), then for
intermediate query shapes (192^3, 384^3, 768^3) compare
  * the configuration the runtime selection cascade picks from the anchors'
    wisdom (``select`` -> same_device_nearest, the paper's §4.5 heuristic), and
  * the Table-2 default,
against the per-shape tuned optimum, as ``report.fraction_of_optimum``
(optimum time / config time; 1.0 = optimal).

    python -m paper_2303_12374_b200.portability --out profiles/r01_portability.json
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

from .backend import STATUS_OK
from .report import fraction_of_optimum, ppm
from .tuner import Budget
from .wisdom import WisdomFile, select, wisdom_path

__all__ = ["sweep", "main"]

ANCHORS = (128, 256, 512, 1024)
QUERIES = (192, 384, 768)


def _shape(q) -> tuple[int, int, int]:
    """A query/anchor: an int n (the cube n^3) or an (nx, ny, nz) tuple."""
    return (q, q, q) if isinstance(q, int) else tuple(q)


def _label(q) -> str:
    return f"{q}^3" if isinstance(q, int) else "x".join(map(str, q))


def _tune(kernel, precision, n, ctx, wdir, evals, log):
    """Per-shape optimum the way the wisdom files are made: an exhaustive
    session over the focused TMA sub-space plus a short random DIRECT one
    (keep-best merges them into ``wdir``)."""
    from .autotune import FOCUSED_TMA, tune_problem

    sessions = []
    for family, strategy, restrict, budget in (("TMA", "exhaustive", FOCUSED_TMA, Budget(4000, 900.0)),
                                               ("DIRECT", "random", None, Budget(max(4, evals // 4), 300.0))):
        s, summary = tune_problem(kernel, precision, _shape(n), ctx, strategy=strategy, budget=budget,
                                  seed=_shape(n)[0],
                                  wisdom_dir=wdir, family=family, restrict=restrict, log=lambda *_: None)
        sessions.append(s)
        log(f"  tuned {kernel} {precision} {_label(n)} {family}: {summary.get('best_gbs', 0):.0f} GB/s "
            f"({summary['evaluations']} evaluations)")
    return sessions


def _measure(kernel, precision, n, ctx, configs):
    from .cuda.executor import CudaReplayExecutor
    from .stencils.layout import GridLayout
    from .stencils.problem import StencilProblem

    lay = GridLayout(*_shape(n), precision)
    prob = StencilProblem(kernel, lay, ctx)
    ex = CudaReplayExecutor(None, ctx, definition=prob.definition, args=prob.args(), output_layout=lay, verify=False)
    out = [ex.measure(c) for c in configs]
    ex.close()
    prob.close()
    return out


def sweep(ctx, kernels=("advec_u", "diff_uvw"), precisions=("fp32", "fp64"), anchors=ANCHORS, queries=QUERIES,
          evals=60, log=print, anchor_wisdom: str | Path | None = None) -> dict:
    """Selection from anchor wisdom vs the per-shape tuned optimum.  With
    ``anchor_wisdom`` the anchors are the records of an existing wisdom
    directory (e.g. the committed ``wisdom/``) instead of fresh sessions."""
    from .stencils.definitions import definition_for

    results = {"anchors": "wisdom:" + str(anchor_wisdom) if anchor_wisdom else [_label(a) for a in anchors],
               "queries": [_label(q) for q in queries], "rows": []}
    with tempfile.TemporaryDirectory() as tmp:
        for precision in precisions:
            for kernel in kernels:
                d = definition_for(kernel, precision)
                if anchor_wisdom:
                    wfile = WisdomFile.load(wisdom_path(anchor_wisdom, d.kernel_key()))
                else:
                    wdir = Path(tmp) / f"{kernel}_{precision}"
                    wdir.mkdir()
                    for n in anchors:
                        _tune(kernel, precision, n, ctx, wdir, evals, log)
                    wfile = WisdomFile.load(wisdom_path(wdir, d.kernel_key()))
                default = d.space.default_config()[0]
                for q in queries:
                    qdir = Path(tmp) / f"q_{kernel}_{precision}_{_label(q)}"
                    qdir.mkdir()
                    sessions = _tune(kernel, precision, q, ctx, qdir, evals, log)
                    best = min((s for s in sessions if s.best is not None), key=lambda s: s.best_objective)
                    choice = select(wfile, ctx.ident, _shape(q), default)
                    m_sel, m_def = _measure(kernel, precision, q, ctx, [choice.config, default])
                    row = {"kernel": kernel, "precision": precision, "query": q if isinstance(q, int) else list(q),
                           "match_kind": choice.match_kind,
                           "selected_from": list(choice.record.problem) if choice.record else None,
                           "optimum_us": best.best_objective * 1e6}
                    for tag, m, cfg in (("selected", m_sel, choice.config), ("default", m_def, default)):
                        if m.status == STATUS_OK:
                            row[f"{tag}_us"] = m.objective * 1e6
                            row[f"{tag}_fraction"] = fraction_of_optimum(best, cfg, lambda c, m=m: m)
                    results["rows"].append(row)
                    log(f"{kernel} {precision} {_label(q)}: selected {row.get('selected_fraction', 0):.3f} of optimum "
                        f"(from {row['selected_from']}), default {row.get('default_fraction', 0):.3f}")
    for tag in ("selected", "default"):
        effs = [r.get(f"{tag}_fraction") for r in results["rows"]]
        res = ppm(effs)
        results[f"ppm_{tag}"] = {"ppm": res.ppm, "best": res.best, "worst": res.worst}
    return results


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2303_12374_b200.portability")
    ap.add_argument("--out", default="portability.json")
    ap.add_argument("--evals", type=int, default=60)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--anchors", default=",".join(map(str, ANCHORS)))
    ap.add_argument("--queries", default=",".join(map(str, QUERIES)),
                    help="comma-separated; n for n^3 or NXxNYxNZ")
    ap.add_argument("--anchor-wisdom", default=None, help="use this wisdom directory's records as the anchors")
    a = ap.parse_args(argv)
    from .cuda import open_device

    ctx = open_device(a.device)
    t0 = time.time()
    def parse(text):
        out = []
        for tok in text.split(","):
            dims = [int(x) for x in tok.lower().split("x")]
            out.append(dims[0] if len(dims) == 1 else tuple(dims))
        return tuple(out)

    res = sweep(ctx, anchors=parse(a.anchors), queries=parse(a.queries), evals=a.evals,
                anchor_wisdom=a.anchor_wisdom)
    res["seconds"] = round(time.time() - t0, 1)
    res["device"] = ctx.ident.to_json_obj()
    Path(a.out).write_text(json.dumps(res, indent=1, sort_keys=True))
    print(json.dumps({k: v for k, v in res.items() if k.startswith("ppm")}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
