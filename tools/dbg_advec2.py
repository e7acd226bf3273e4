import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
from paper_2303_12374_b200.stencils.layout import GridLayout
from paper_2303_12374_b200.stencils.problem import StencilProblem
from stencil_helpers import oracle_outputs, rel_error, run_config

ctx = open_device(0)
comp = NvrtcCompiler(ctx)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
lay = GridLayout(n, n, n, "fp32")
prob = StencilProblem("advec_u", lay, ctx)
d = prob.definition
base = d.space.default_config()[0]
cases = [dict(block_x=32, block_y=1, tile_y=1, depth=1, zchunk=8, min_blocks=2),
         dict(block_x=128, block_y=1, tile_y=1, depth=2, zchunk=8, min_blocks=2),
         dict(block_x=32, block_y=1, tile_y=4, depth=2, zchunk=16, min_blocks=1),
         dict(block_x=64, block_y=4, tile_y=4, depth=1, zchunk=64, min_blocks=2)]
ex = CudaReplayExecutor(None, ctx, definition=d, args=prob.args(), output_layout=lay, compiler=comp)
for c in cases:
    cfg = dict(base, staging="TMA", **c)
    m = ex.measure(cfg)
    print("replay", c, m.status, m.stage_timings.get("verify_error"))
    m = ex.measure(cfg)
    print("replay again", m.status, m.stage_timings.get("verify_error"))
ex.close()
prob.close()
ref, _ = oracle_outputs("advec_u", lay)
for c in cases:
    cfg = dict(base, staging="TMA", **c)
    got = run_config(ctx, comp, "advec_u", lay, cfg)
    print("oracle", c, rel_error(got["ut"], ref["ut"], lay))
