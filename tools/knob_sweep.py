"""One-knob-at-a-time variants of a wisdom record, each evidenced by its
achieved HBM bandwidth (north star: "each tunable variant evidenced by ncu
achieved-HBM GB/s against the B200's ~8 TB/s").

For ``--kernel/--precision/--grid`` the record's configuration is varied one
Table-2 / B200 knob at a time (block shape, thread tiling along x/y, loop
unrolling and the staging family with its z-chunk and prefetch depth; only
points of the tuning space are kept).  ``--mode time`` event-times every
variant interleaved (L2 flushed, klb_time_launches) and writes JSON lines;
``--mode ncu`` launches each variant ``4`` times (3 warm-up + 1) for an ncu
capture, in the same order; ``--merge`` joins an ncu CSV (dram bytes,
gpu__time_duration) onto the timed lines.  GPU only (except ``--merge``).

    python tools/knob_sweep.py --kernel diff_uvw --precision fp32 --grid 512,512,512 --mode time --out t.jsonl
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file n.csv \\
        python tools/knob_sweep.py ... --mode ncu
    python tools/knob_sweep.py ... --merge n.csv --out t.jsonl > knobs.json
"""

from __future__ import annotations

import argparse
import csv
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def variants(space, record: dict) -> list[tuple[str, dict]]:
    """(label, config) pairs: the record, then one knob changed at a time."""
    out = [("record", dict(record))]
    default, _ = space.default_config()
    tries = [("staging", "DIRECT (Table-2 default)", dict(default))]
    tries.append(("staging", "ZMARCH", dict(record, staging="ZMARCH", depth=0)))
    zm = dict(default, staging="ZMARCH", block_x=32, block_y=8, tile_y=2, zchunk=32, unroll_x=False, unroll_y=False)
    tries.append(("staging", "ZMARCH (32x8, tile_y 2, zchunk 32)", zm))
    for v in (16, 32, 64, 128):
        tries.append(("block_x", v, dict(record, block_x=v)))
    for v in (1, 2, 4, 8):
        tries.append(("block_y", v, dict(record, block_y=v)))
    for v in (1, 2, 4):
        tries.append(("tile_x", v, dict(record, tile_x=v)))
        tries.append(("tile_y", v, dict(record, tile_y=v)))
    for v in (16, 32, 64, 128):
        tries.append(("zchunk", v, dict(record, zchunk=v)))
    for v in (1, 2, 3):
        tries.append(("depth", v, dict(record, depth=v)))
    tries.append(("unravel", "YXZ", dict(record, unravel="YXZ")))
    tries.append(("min_blocks", 2, dict(record, min_blocks=2)))
    # loop unrolling is a DIRECT-family knob (the marching families unroll their tiles)
    tiled = dict(default, tile_x=2, tile_y=2, contiguous_x=True)
    tries.append(("unroll (DIRECT 2x2 tile)", "none", dict(tiled)))
    tries.append(("unroll (DIRECT 2x2 tile)", "x,y", dict(tiled, unroll_x=True, unroll_y=True)))
    seen = {json.dumps(record, sort_keys=True)}
    for knob, val, cfg in tries:
        key = json.dumps(cfg, sort_keys=True)
        if key in seen or not space.is_valid(cfg):
            continue
        seen.add(key)
        out.append((f"{knob}={val}", cfg))
    return out


def merge(lines: list[dict], ncu_csv: str, peak: float) -> list[dict]:
    rows = [r for r in csv.DictReader(ln for ln in open(ncu_csv) if not ln.startswith("=="))]
    by: dict[int, dict] = {}
    for r in rows:
        by.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ids = sorted(by)
    if len(ids) != 4 * len(lines):
        raise SystemExit(f"{len(ids)} ncu launches for {len(lines)} variants (expected 4 each)")
    for i, line in enumerate(lines):
        m = by[ids[4 * i + 3]]
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        secs = m["gpu__time_duration.sum"] * 1e-9
        line["ncu"] = {"us": round(secs * 1e6, 2), "dram_bytes": dram, "dram_gbs": round(dram / secs / 1e9, 1),
                       "dram_over_algorithmic": round(dram / line["algorithmic_bytes"], 4),
                       "dram_frac_of_8tbs": round(dram / secs / 8e12, 4),
                       "algorithmic_gbs": round(line["algorithmic_bytes"] / secs / 1e9, 1),
                       "algorithmic_frac_of_measured_peak": round(line["algorithmic_bytes"] / secs / 1e9 / peak, 4)}
    return lines


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="diff_uvw")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="512,512,512")
    ap.add_argument("--mode", choices=("time", "ncu"), default="time")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", help="JSON lines (time mode writes, merge reads)")
    ap.add_argument("--merge", help="ncu CSV to join onto --out (no GPU)")
    a = ap.parse_args(argv)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    if a.merge:
        lines = [json.loads(x) for x in open(a.out)]
        print(json.dumps({"kernel": a.kernel, "precision": a.precision, "grid": a.grid, "measured_peak_gbs": peak,
                          "variants": merge(lines, a.merge, peak)}, indent=1))
        return 0

    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.dispatch import WisdomKernel
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
    _, record, _ = wk.resolve(ctx.ident, problem, env)
    from paper_2303_12374_b200.backend import CompileError

    runs = []
    for label, cfg in variants(d.space, record):
        try:  # (a space point a kernel does not implement — e.g. ZMARCH of the family — fails to compile)
            exe = comp.compile(d.render_compile_request(cfg, problem, env), ctx.ident)
        except CompileError:
            continue
        exe.load()
        runs.append((label, cfg, exe, d.derive_geometry(cfg, problem, env)))
    args = prob.args()
    flush = ctx.flush_buffer()
    if a.mode == "ncu":
        for _, _, exe, geom in runs:
            exe.time_launches(geom, args, 3, 1, flush=flush)
        return 0
    times = [[] for _ in runs]
    for _ in range(a.rounds):
        for i, (_, _, exe, geom) in enumerate(runs):
            times[i].append(statistics.median(exe.time_launches(geom, args, 3, a.reps, flush=flush)))
    nbytes = BYTES_PER_CELL_WORDS[a.kernel] * lay.elem_bytes * lay.cells
    with open(a.out, "w") as fh:
        for i, (label, cfg, _, geom) in enumerate(runs):
            t = statistics.median(times[i])
            line = {"variant": label, "config": cfg, "blocks": geom.grid[0], "threads": geom.threads_per_block,
                    "smem": geom.shared_mem_bytes, "algorithmic_bytes": nbytes,
                    "event": {"us": round(t * 1e6, 2), "algorithmic_gbs": round(nbytes / t / 1e9, 1),
                              "frac_of_measured_peak": round(nbytes / t / 1e9 / peak, 4)}}
            fh.write(json.dumps(line, sort_keys=True) + "\n")
            print(json.dumps(line, sort_keys=True), flush=True)
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
