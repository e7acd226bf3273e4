"""Time to a near-optimal configuration per search strategy (the paper's
tuning-session figure, §5: "Bayesian optimization takes, on average,
3.4 minutes ... to find a configuration 10% away from the optimum and 7.5
minutes ... for a 5% difference").

Reads ``.klsession`` files of the same scenario(s) run with different
strategies; per scenario the optimum is the best objective over all of its
sessions; per session it reports the wall-clock seconds (the evaluation's
``wall_offset``, the session lines' ``t``) at which the best-so-far came within 10 % and 5 % of that optimum, and
the best-so-far curve.  No GPU.

    python tools/convergence.py profiles/convergence_b200/*.klsession > convergence.json
"""

from __future__ import annotations

import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(paths) -> int:
    from paper_2303_12374_b200.tuner import load_session

    by = defaultdict(list)
    for p in paths:
        s = load_session(p)
        by[(s.kernel_key.rsplit("-", 1)[0], tuple(s.problem))].append((Path(p).name, s))
    out = {}
    for (name, problem), sess in sorted(by.items()):
        best = min(e.measurement.objective for _, s in sess for e in s.evaluations if e.measurement.status == "ok")
        rows = {}
        for fname, s in sess:
            cur, curve, hit = float("inf"), [], {}
            for e in s.evaluations:
                if e.measurement.status == "ok" and e.measurement.objective < cur:
                    cur = e.measurement.objective
                    curve.append([round(e.wall_offset, 1), round(best / cur, 4)])
                    for tol in (0.10, 0.05):
                        if tol not in hit and cur <= best * (1 + tol):
                            hit[tol] = round(e.wall_offset, 1)
            rows[s.strategy] = {"session": fname, "evaluations": len(s.evaluations),
                                "seconds_to_within_10pct": hit.get(0.10), "seconds_to_within_5pct": hit.get(0.05),
                                "final_fraction": round(best / cur, 4), "best_so_far": curve}
        out[f"{name} {'x'.join(map(str, problem))}"] = {"optimum_us": round(best * 1e6, 2), "strategies": rows}
    print(json.dumps(out, indent=1, sort_keys=True))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
