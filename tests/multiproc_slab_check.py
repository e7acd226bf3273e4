"""One rank of the z-slab decomposition on the GPU, checked against the oracle.

Run under ``torch.distributed.run`` (tests/test_gpu_multiproc.py): every rank
drives its ``SlabDriver`` slab with the host-relayed ``StagedExchanger`` (all
ranks may share one device, which NCCL refuses), steps once and compares its
planes of every output with the NumPy oracle of the undecomposed grid.
Prints ``rank <r> ok <max rel err>``; exits nonzero on a mismatch.
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> int:
    import numpy as np
    import torch.distributed as dist

    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.halo import StagedExchanger
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from stencil_helpers import oracle_outputs

    kernel, precision, grid = sys.argv[1], sys.argv[2], tuple(int(x) for x in sys.argv[3].split(","))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = open_device(int(os.environ.get("KL_DEVICE_ORDINAL", "0")))
    drv = SlabDriver(kernel, precision, grid, ctx, rank=rank, nranks=world, exchanger=StagedExchanger(rank, world),
                     compiler=NvrtcCompiler(ctx), wisdom_dir=str(ROOT / "wisdom"))
    drv.resolve()
    drv.step()
    ctx.synchronize()
    ref, _ = oracle_outputs(kernel, GridLayout(*grid, precision))
    g = drv.layout.kgc
    off, count = drv.slab.offset, drv.slab.count
    worst = 0.0
    for name in ref:
        got = drv.problem.download(name)[g:g + count, g:-g, g:g + grid[0]].astype(np.float64)
        want = ref[name][g + off:g + off + count, g:-g, g:g + grid[0]]
        worst = max(worst, float(np.max(np.abs(got - want)) / np.max(np.abs(ref[name][g:-g, g:-g, g:g + grid[0]]))))
    drv.close()
    dist.barrier()
    dist.destroy_process_group()
    tol = 1e-5 if precision == "fp32" else 1e-12
    print(f"rank {rank} {'ok' if worst <= tol else 'FAIL'} {worst:.3e}", flush=True)
    return 0 if worst <= tol else 1


if __name__ == "__main__":
    sys.exit(main())
