"""Per-rank step of the z-slab decomposition on ONE GPU: the exchange variant
(interior launch + the two boundary launches; the plane copies overlap the
interior on a real multi-GPU box, so they are not on this clock) against the
fused halo (one diff_uvw_peer / advec_u_peer launch over the whole slab
reading the planes outside it from the neighbours' fields).  The middle rank of an N-way split
is built with its two neighbours as virtual ranks (LocalPeers), its step timed
with CUDA events (L2 flushed between steps), and its outputs checked against
the exchange variant's.  GPU only.

    python tools/fused_halo_probe.py --precision fp32 --grid 1024,1024,1024 --ranks 2,4,8
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
    ap.add_argument("--kernel", default="diff_uvw", choices=("diff_uvw", "advec_u"))
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="1024,1024,1024")
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--json-out")
    a = ap.parse_args(argv)

    import numpy as np

    from paper_2303_12374_b200.cuda import Event, NvrtcCompiler, open_device
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.halo import CopyExchanger, HALO_REACH, LocalPeers
    from paper_2303_12374_b200.slab import FUSED_HALO, SlabDriver
    from paper_2303_12374_b200.stencils.problem import PEER_KERNELS

    ctx = open_device(0)
    comp = NvrtcCompiler(ctx)
    grid = tuple(int(x) for x in a.grid.split(","))
    flush = ctx.flush_buffer()
    out = open(a.json_out, "a") if a.json_out else None

    def timed(fn) -> float:
        secs = []
        for _ in range(3):
            fn()
        for _ in range(a.reps):
            check(lib().klb_memset_d8(flush.ptr, 0, flush.nbytes, ctx.stream.handle))
            e0, e1 = Event(), Event()
            e0.record(ctx.stream)
            fn()
            e1.record(ctx.stream)
            e1.synchronize()
            secs.append(e0.elapsed_ms(e1) * 1e-3)
        return statistics.median(secs)

    for n in (int(x) for x in a.ranks.split(",")):
        mid = n // 2
        ids = [r for r in (mid - 1, mid, mid + 1) if 0 <= r < n]
        rec = {"kernel": a.kernel, "precision": a.precision, "grid": list(grid), "nranks": n, "rank": mid}
        for halo in ("exchange", "fused"):
            peers = LocalPeers([])
            drivers = {r: SlabDriver(a.kernel, a.precision, grid, ctx, rank=r, nranks=n, compiler=comp,
                                     wisdom_dir=ROOT / "wisdom", halo=halo,
                                     exchanger=peers.for_rank(ids.index(r)) if halo == "fused" else None)
                       for r in ids}
            peers.ranks = [({f: drivers[r].problem.field_ptr(f) for f in PEER_KERNELS[FUSED_HALO[a.kernel]]},
                            drivers[r].layout.kstart, drivers[r].layout.kend) for r in ids]
            if halo == "exchange":  # fill the middle rank's ghost planes once (its own copies, untimed)
                lay = drivers[mid].layout
                ex = CopyExchanger([{f: drivers[r].problem.field_ptr(f) for f in HALO_REACH[a.kernel]}
                                    for r in ids])
                ex.exchange_all(ctx.stream, HALO_REACH[a.kernel], lay.elem_bytes, lay.kk,
                                [(drivers[r].layout.kstart, drivers[r].layout.kend) for r in ids])
            d = drivers[mid]
            sel = d.resolve()
            t = timed(d.step)
            cells = grid[0] * grid[1] * d.slab.count
            rec[halo] = {"us_per_step": round(t * 1e6, 1), "launches": len(d.ranges),
                         "gcells_per_rank": round(cells / t / 1e9, 2),
                         "selection": {k: v[0] for k, v in sel.items()}}
            d.problem.regenerate(d.problem.outputs())
            d.step()
            ctx.synchronize()
            rec[halo]["_out"] = {name: d.problem.download(name)[d.layout.kstart:d.layout.kend].copy()
                                 for name in d.problem.outputs()}
            for r in ids:
                drivers[r].close()
        worst = 0.0
        for name, want in rec["exchange"].pop("_out").items():
            got = rec["fused"]["_out"][name]
            worst = max(worst, float(np.max(np.abs(got - want)) / np.max(np.abs(want))))
        rec["fused"].pop("_out")
        rec["fused_vs_exchange_max_rel_diff"] = worst
        rec["fused_speedup"] = round(rec["exchange"]["us_per_step"] / rec["fused"]["us_per_step"], 4)
        print(json.dumps(rec, sort_keys=True), flush=True)
        if out:
            out.write(json.dumps(rec, sort_keys=True) + "\n")
            out.flush()
    return 0


if __name__ == "__main__":
    sys.exit(main())
