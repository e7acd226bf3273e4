"""Launch one stencil configuration a few times (target for ncu -k regex:<kernel>).

    python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 512,512,512 \
        --config '{"staging":"ZMARCH",...}' --launches 3
--config accepts JSON (merged over the default) or 'default' or 'wisdom'
(runtime selection from ./wisdom).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="diff_uvw")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--grid", default="512,512,512")
    ap.add_argument("--config", default="default")
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--wisdom", default="wisdom")
    a = ap.parse_args()
    from paper_2303_12374_b200.capture import CapturePolicy
    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    ctx = open_device(0)
    lay = GridLayout(*(int(x) for x in a.grid.split(",")), a.precision)
    prob = StencilProblem(a.kernel, lay, ctx)
    d = prob.definition
    env = prob.scalar_env()
    problem = d.derive_problem_size(env)
    comp = NvrtcCompiler(ctx)
    if a.config == "wisdom":
        wk = WisdomKernel(d, comp, wisdom_dir=a.wisdom, capture_policy=CapturePolicy())
        handle, cfg, kind = wk.resolve(ctx.ident, problem, env)
    else:
        cfg = d.space.default_config()[0]
        if a.config != "default":
            cfg.update(json.loads(a.config))
        handle = comp.compile(d.render_compile_request(cfg, problem, env), ctx.ident)
        handle.load()
    geom = d.derive_geometry(cfg, problem, env)
    for _ in range(a.launches):
        secs = handle.launch(geom, prob.args(), timed=True)
        print(f"{a.kernel}_{a.precision} {a.grid} {secs * 1e6:.1f} us  {json.dumps(cfg, sort_keys=True)}")
    prob.close()


if __name__ == "__main__":
    main()
