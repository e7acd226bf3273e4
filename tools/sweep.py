"""Measure an explicit cartesian sweep of stencil configurations (GPU).

Used to study one knob at a time around a tuned point (the tuner samples the
space; this isolates effects).  Configurations need not lie inside the
space's restrictions — the executor measures whatever it is given (a launch
that exceeds the device's limits reports launch_failed).

    python tools/sweep.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 \
        --base wisdom --vary unravel=XZY,XYZ --vary block_y=1,2,4 --json-out gpurun_out/sweep.jsonl
"""

from __future__ import annotations

import argparse
import itertools
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _parse_value(text: str):
    if text in ("true", "false"):
        return text == "true"
    try:
        return int(text)
    except ValueError:
        return text


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="1024,1024,1024")
    ap.add_argument("--base", default="wisdom", help="'wisdom' (selected config), 'default', or a JSON object")
    ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
    ap.add_argument("--vary", action="append", default=[], help="knob=v1,v2,... (cartesian product)")
    ap.add_argument("--set", action="append", default=[], help="knob=value applied to the base")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--json-out", default=None)
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.backend import STATUS_OK
    from paper_2303_12374_b200.cuda import open_device
    from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem
    from paper_2303_12374_b200.wisdom import load_or_create, select

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    layout = GridLayout(*grid, a.precision)
    prob = StencilProblem(a.kernel, layout, ctx)
    args = prob.args()
    ex = CudaReplayExecutor(None, ctx, definition=prob.definition, args=args, repetitions=a.reps,
                            flush_l2=True, verify=not a.no_verify, output_layout=layout)
    space = prob.definition.space
    default, _ = space.default_config()
    if a.base == "default":
        base = dict(default)
    elif a.base == "wisdom":
        wfile = load_or_create(a.wisdom, prob.definition.kernel_key())
        base = dict(select(wfile, ctx.ident, ex.problem, default).config)
    else:
        base = dict(default, **json.loads(a.base))
    for item in a.set:
        k, v = item.split("=", 1)
        base[k] = _parse_value(v)
    knobs = []
    for item in a.vary:
        k, vs = item.split("=", 1)
        knobs.append((k, [_parse_value(v) for v in vs.split(",")]))
    cells = grid[0] * grid[1] * grid[2]
    from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS

    words = BYTES_PER_CELL_WORDS[a.kernel]
    configs = []
    for combo in itertools.product(*[vs for _, vs in knobs]):
        cfg = dict(base)
        cfg.update({k: v for (k, _), v in zip(knobs, combo)})
        configs.append(cfg)
    ex.prefetch(configs)
    out = open(a.json_out, "a") if a.json_out else None
    print(f"base {json.dumps(base, sort_keys=True)}", flush=True)
    for cfg in configs:
        m = ex.measure(cfg)
        tag = " ".join(f"{k}={cfg[k]}" for k, _ in knobs)
        if m.status == STATUS_OK:
            us = m.objective * 1e6
            gbs = cells * words * layout.elem_bytes / m.objective / 1e9
            print(f"{tag:60s} {us:10.1f} us {cells / m.objective / 1e9:8.2f} Gcells/s {gbs:8.1f} GB/s", flush=True)
        else:
            us = gbs = None
            print(f"{tag:60s} {m.status}", flush=True)
        if out:
            out.write(json.dumps({"kernel": a.kernel, "precision": a.precision, "grid": list(grid), "config": cfg,
                                  "status": m.status, "us": us, "gbs": gbs}, sort_keys=True) + "\n")
            out.flush()
    ex.close()
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
