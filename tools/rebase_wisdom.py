"""Head-to-head re-measurement of wisdom candidates on ONE box.

Objectives recorded on different boxes (or days) are not comparable — the
same configuration measured 70.8 us on one B200 and 77.9 us on another — so
the keep-best merge of a new session into an older record can keep the
slower configuration.  This tool re-times the current record's config and
the best configurations of the given sessions interleaved for several rounds
in one process (L2 flushed, verified against the default configuration),
and rewrites the problem's record with the winner and its objective measured
here (provenance notes the rebase).

    python tools/rebase_wisdom.py --kernel advec_u --precision fp32 --grid 256,256,256 \
        --sessions gpurun_out/r02g_sessions/*.klsession --top 6 --rounds 5
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
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", required=True)
    ap.add_argument("--sessions", nargs="*", default=[])
    ap.add_argument("--top", type=int, default=6)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
    ap.add_argument("--json-out")
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.backend import STATUS_OK
    from paper_2303_12374_b200.cuda import open_device
    from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem
    from paper_2303_12374_b200.tuner import load_session
    from paper_2303_12374_b200.wisdom import Provenance, WisdomRecord, load_or_create, select, wisdom_path

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    d = prob.definition
    ex = CudaReplayExecutor(None, ctx, definition=d, args=prob.args(), repetitions=9, flush_l2=True, verify=True,
                            output_layout=lay)
    wfile = load_or_create(a.wisdom, d.kernel_key())
    current = select(wfile, ctx.ident, ex.problem, d.space.default_config()[0])
    cands = [("current", dict(current.config))]
    for path in a.sessions:
        s = load_session(path)
        if s.kernel_key != d.kernel_key():
            continue
        ok = sorted(s.ok_evaluations(), key=lambda e: e.measurement.objective)
        for e in ok[: a.top]:
            if all(e.config != c for _, c in cands):
                cands.append((Path(path).name, dict(e.config)))
    ex.prefetch([c for _, c in cands])
    times = {i: [] for i in range(len(cands))}
    for r in range(a.rounds):
        for i, (_, cfg) in enumerate(cands):
            m = ex.measure(cfg)
            if m.status == STATUS_OK:
                times[i].append(m.objective)
    rows = []
    for i, (src, cfg) in enumerate(cands):
        if times[i]:
            rows.append((statistics.median(times[i]), i, src, cfg))
    rows.sort(key=lambda x: x[0])
    for t, i, src, cfg in rows:
        print(f"{t * 1e6:9.2f} us  {src:40s} {json.dumps(cfg, sort_keys=True)}", flush=True)
    best_t, _, best_src, best_cfg = rows[0]
    prov = Provenance(device_properties=dict(ctx.ident.attributes))
    prov.versions["rebased_by"] = "tools/rebase_wisdom.py (head-to-head, one box)"
    rec = WisdomRecord(ctx.ident, ex.problem, best_cfg, best_t, prov)
    wfile.records = [r for r in wfile.records if not (r.device.name == ctx.ident.name and r.problem == ex.problem)]
    wfile.records.append(rec)
    wfile.save(wisdom_path(a.wisdom, d.kernel_key()))
    out = {"kernel": a.kernel, "precision": a.precision, "grid": list(grid), "winner": best_src,
           "winner_us": best_t * 1e6, "current_was": dict(current.config),
           "candidates": [{"source": s, "us": t * 1e6, "config": c} for t, _, s, c in rows]}
    if a.json_out:
        with open(a.json_out, "a") as fh:
            fh.write(json.dumps(out, sort_keys=True) + "\n")
    ex.close()
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
