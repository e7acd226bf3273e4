"""NVRTC-compile one configuration (no GPU needed) and write the cubin, for
cuobjdump / tools/sass_loops.py.

    python tools/dump_cubin.py --kernel advec_u --precision fp32 --grid 512,512,512 \
        --config wisdom/advec_u_fp32-*.wisdom  (best record for the grid) | '{"staging": "TMA", ...}'
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2303_12374_b200.backend import DeviceIdent  # noqa: E402
from paper_2303_12374_b200.cuda.compiler import NvrtcCompiler  # noqa: E402
from paper_2303_12374_b200.stencils.definitions import definition_for  # noqa: E402
from paper_2303_12374_b200.stencils.layout import GridLayout  # noqa: E402
from paper_2303_12374_b200.wisdom import WisdomFile, select  # noqa: E402

B200 = DeviceIdent("NVIDIA B200", "Blackwell", {"compute_capability": "10.0"})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--precision", required=True)
    ap.add_argument("--grid", required=True)
    ap.add_argument("--config", required=True, help="JSON config (merged over the default) or a .wisdom file")
    ap.add_argument("--out", default="/tmp/k.cubin")
    ap.add_argument("--define", action="append", default=[], help="extra NAME=VALUE compile-time switch")
    a = ap.parse_args()
    d = definition_for(a.kernel, a.precision)
    grid = tuple(int(x) for x in a.grid.split(","))
    lay = GridLayout(*grid, a.precision)
    from paper_2303_12374_b200.stencils.definitions import ARG_LAYOUT
    nb = len(ARG_LAYOUT[a.kernel]["buffers"])
    vals = dict(dxi=1.0, dyi=1.0, tpri=3.0, cs=0.23, rk_a=-5 / 9, rk_bdt=0.01, peer_klo=-(1 << 30), peer_khi=1 << 30,
                peer_shift_lo=0, peer_shift_hi=0, jj=lay.jj, kk=lay.kk, istart=lay.istart, jstart=lay.jstart, kstart=lay.kstart,
                iend=lay.iend, jend=lay.jend, kend=lay.kend)
    env = {f"arg{nb + i}": vals[n] for i, n in enumerate(ARG_LAYOUT[a.kernel]["scalars"])}
    problem = d.derive_problem_size(env)
    default = d.space.default_config()[0]
    if a.config.endswith(".wisdom"):
        w = WisdomFile.load(Path(a.config))
        cfg = select(w, B200, problem, default).config
    else:
        cfg = dict(default, **json.loads(a.config))
    print(json.dumps(cfg, sort_keys=True))
    req = d.render_compile_request(cfg, problem, env)
    if a.define:
        from paper_2303_12374_b200.kerneldef import CompileRequest
        names = tuple(f"-D {x.split('=')[0]}=" for x in a.define)
        req = CompileRequest(req.source, req.entry, tuple(x for x in req.defines if not x.startswith(names)) +
                             tuple(f"-D {x}" for x in a.define), req.flags)
    img = NvrtcCompiler().compile_many([req], B200)[0].result()
    Path(a.out).write_bytes(img.cubin)
    print(a.out, len(img.cubin))


if __name__ == "__main__":
    main()
