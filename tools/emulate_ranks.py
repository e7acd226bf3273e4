"""Per-rank compute of the BASELINE config 4 slab decomposition, emulated on ONE GPU.

For N in 1, 2, 4, 8 the SlabDriver of an interior rank (both neighbours,
so the interior / lower / upper sub-range launches of the real N-GPU step)
is built on the one visible B200 and its step timed with CUDA events — the
compute part of an N-GPU step, halo exchange excluded (no second GPU here).
The compute-only strong-scaling efficiency t_1 / (N * t_N) bounds what the
N-GPU run can reach; the exchange (NCCL, overlapped with the interior
sub-range) comes on top.

    python tools/emulate_ranks.py [--steps 20] [--precision fp32]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2303_12374_b200.cuda import Event, NvrtcCompiler, open_device  # noqa: E402
from paper_2303_12374_b200.slab import SlabDriver  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="diff_uvw")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="1024,1024,1024")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
    a = ap.parse_args()
    grid = tuple(int(x) for x in a.grid.split(","))
    ctx = open_device(0)
    comp = NvrtcCompiler(ctx)
    rows = []
    for n in (1, 2, 4, 8):
        rank = n // 2  # an interior rank when n > 2 (both neighbours)
        drv = SlabDriver(a.kernel, a.precision, grid, ctx, rank=rank, nranks=n, compiler=comp, wisdom_dir=a.wisdom)
        sel = drv.resolve()
        for _ in range(3):
            drv.step()
        ctx.synchronize()
        times = []
        for _ in range(a.steps):
            e0, e1 = Event(), Event()
            e0.record(drv.compute)
            drv.step()
            e1.record(drv.compute)
            e1.synchronize()
            times.append(e0.elapsed_ms(e1))
        t = statistics.median(times)
        cells = grid[0] * grid[1] * drv.slab.count
        rows.append({"n": n, "rank": rank, "planes": drv.slab.count, "subranges": sorted(drv.ranges),
                     "ms_per_step": round(t, 4), "gcells_per_gpu": round(cells / (t * 1e-3) / 1e9, 2),
                     "selection": {k: v[1] if isinstance(v, tuple) else str(v) for k, v in sel.items()}})
        drv.close()
    t1 = rows[0]["ms_per_step"]
    for r in rows:
        r["compute_only_efficiency"] = round(t1 / (r["n"] * r["ms_per_step"]), 4)
    print(json.dumps({"kernel": a.kernel, "precision": a.precision, "grid": list(grid), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
