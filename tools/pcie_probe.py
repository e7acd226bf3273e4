"""Host-link ceiling for the e2e step: pinned H2D / D2H / both directions at
once, one and two streams per direction, on buffers the size of the bench's
per-step traffic (1024^3 fp32 diff_uvw: 7 fields in, 3 out).  GPU only."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> int:
    from paper_2303_12374_b200.cuda import DeviceArray, Event, HostPinned, Stream, open_device
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.stencils.layout import GridLayout

    ctx = open_device(0)
    field = GridLayout(1024, 1024, 1024, "fp32").alloc_bytes
    nin, nout = 7, 3
    host = [HostPinned(field) for _ in range(nin)]
    dev = [DeviceArray(field) for _ in range(nin)]
    streams = [Stream.create() for _ in range(4)]
    chunk = 256 << 20
    res = {"field_bytes": field, "h2d_bytes": nin * field, "d2h_bytes": nout * field}

    def run(h2d_streams, d2h_streams, do_h2d=True, do_d2h=True):
        up, down = streams[:h2d_streams], streams[2:2 + d2h_streams]
        ctx.synchronize()
        e0 = Event().record(streams[0])
        for s in streams[1:]:
            s.wait(e0)
        i = 0
        if do_h2d:
            for f in range(nin):
                for lo in range(0, field, chunk):
                    n = min(chunk, field - lo)
                    check(lib().klb_memcpy_htod(dev[f].ptr + lo, host[f].ptr + lo, n, up[i % len(up)].handle))
                    i += 1
        i = 0
        if do_d2h:
            for f in range(nout):
                for lo in range(0, field, chunk):
                    n = min(chunk, field - lo)
                    check(lib().klb_memcpy_dtoh(host[f].ptr + lo, dev[f].ptr + lo, n, down[i % len(down)].handle))
                    i += 1
        t0 = time.perf_counter()
        ctx.synchronize()
        return time.perf_counter() - t0

    for name, kw in (("h2d_1", dict(h2d_streams=1, d2h_streams=1, do_d2h=False)),
                     ("h2d_2", dict(h2d_streams=2, d2h_streams=1, do_d2h=False)),
                     ("d2h_1", dict(h2d_streams=1, d2h_streams=1, do_h2d=False)),
                     ("both_1_1", dict(h2d_streams=1, d2h_streams=1)),
                     ("both_2_2", dict(h2d_streams=2, d2h_streams=2))):
        run(**kw)
        best = None
        for _ in range(3):
            ctx.synchronize()
            t0 = time.perf_counter()
            run(**kw)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        moved = (nin * field if kw.get("do_h2d", True) else 0) + (nout * field if kw.get("do_d2h", True) else 0)
        res[name] = {"ms": round(best * 1e3, 1), "gbs": round(moved / best / 1e9, 1)}
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
