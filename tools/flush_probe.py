"""How much of a small kernel's time is the L2 flush's dirty write-back?

Times the wisdom-selected kernel of a problem with (a) the bench's flush (a
memset of 2x L2 right before the launch: L2 left full of dirty lines),
(b) the memset followed by a read pass over another 2x L2 buffer (L2 left
clean and cold), (c) no flush; and D2D copies of several sizes after the
memset flush (the achievable-bandwidth floor per transfer size).  GPU only.
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
    ap.add_argument("--kernel", default="advec_u")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="256,256,256")
    ap.add_argument("--reps", type=int, default=15)
    a = ap.parse_args(argv)

    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import DeviceArray, Event, NvrtcCompiler, open_device
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.cuda.capture_device import device_crc32
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    ctx = open_device(0)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    wk = WisdomKernel(prob.definition, NvrtcCompiler(ctx), wisdom_dir=ROOT / "wisdom", capture_policy=CapturePolicy())
    run = wk.bind(ctx.ident, prob.args(), stream=ctx.stream)
    flush = ctx.flush_buffer()
    clean = DeviceArray(flush.nbytes)
    s = ctx.stream

    def timed(prep):
        out = []
        for i in range(a.reps + 3):
            prep(i)
            e0, e1 = Event(), Event()
            e0.record(s)
            run()
            e1.record(s)
            e1.synchronize()
            out.append(e0.elapsed_ms(e1) * 1e3)
        return statistics.median(out[3:])

    def dirty(i):
        check(lib().klb_memset_d8(flush.ptr, i & 0xFF, flush.nbytes, s.handle))

    def cleaned(i):
        dirty(i)
        device_crc32(clean.ptr, clean.nbytes, s)  # reads 2x L2: evicts (writes back) the dirty lines

    res = {"kernel": a.kernel, "grid": list(grid), "algorithmic_bytes": prob.algorithmic_bytes,
           "dirty_flush_us": timed(dirty), "clean_flush_us": timed(cleaned), "no_flush_us": timed(lambda i: None)}
    # copy floors: D2D copy of n bytes (n read + n written) after the dirty flush
    floors = {}
    for mb in (32, 64, 128, 168, 256, 512, 1024, 4096):
        n = mb << 20
        src, dst = DeviceArray(n), DeviceArray(n)
        ts = []
        for i in range(8):
            dirty(i)
            e0, e1 = Event(), Event()
            e0.record(s)
            check(lib().klb_memcpy_dtod(dst.ptr, src.ptr, n, s.handle))
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_ms(e1) * 1e-3)
        t = statistics.median(ts[2:])
        floors[f"{2 * mb}MB_moved"] = {"us": round(t * 1e6, 2), "gbs": round(2 * n / t / 1e9, 1)}
        src.free()
        dst.free()
    res["copy_floor_after_dirty_flush"] = floors
    print(json.dumps(res))
    prob.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
