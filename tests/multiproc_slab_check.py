"""One rank of the z-slab decomposition on the GPU, checked against the oracle.

Launched N times (tests/test_gpu_multiproc.py: by torchrun or by a plain
spawner — RANK / WORLD_SIZE from the environment, no torch in this process):
every rank opens the ``ProcessGroup``, drives its ``SlabDriver`` slab with the
production halo transport (``IpcExchanger`` by default: neighbours map each
other's fields with CUDA IPC and pull the halo planes; all ranks may share
one device), POISONS every ghost plane the exchange must fill (NaN), steps,
and compares its planes of every output with the oracle of the undecomposed
grid — twice, so the per-step event protocol is exercised with reused
events.  Prints ``rank <r> ok <max rel err>``; exits nonzero on a mismatch.
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def poison_halo(drv) -> int:
    """NaN-fill the ghost planes a neighbour provides; returns planes poisoned."""
    from paper_2303_12374_b200.cuda._abi import check, lib
    from paper_2303_12374_b200.halo import HALO_REACH

    lay = drv.layout
    plane = lay.kk * lay.elem_bytes
    n = 0
    for field, (down, up) in HALO_REACH[drv.kernel].items():
        base = drv.problem.field_ptr(field)
        if drv.below >= 0 and up:
            check(lib().klb_memset_d8(base + (lay.kstart - up) * plane, 0xFF, up * plane, drv.compute.handle))
            n += up
        if drv.above >= 0 and down:
            check(lib().klb_memset_d8(base + lay.kend * plane, 0xFF, down * plane, drv.compute.handle))
            n += down
    return n


def main() -> int:
    import numpy as np

    from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
    from paper_2303_12374_b200.group import ProcessGroup
    from paper_2303_12374_b200.halo import IpcExchanger, NcclExchanger
    from paper_2303_12374_b200.slab import SlabDriver
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from stencil_helpers import oracle_outputs

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    group = ProcessGroup(rank, world, timeout=300)
    ctx = open_device(int(os.environ.get("KL_DEVICE_ORDINAL", os.environ.get("LOCAL_RANK", "0"))))
    if sys.argv[1] == "probe":  # the collective transport probe bench.py runs before choosing IPC
        ok, why = IpcExchanger.probe(group)
        group.close()
        print(f"rank {rank} {'ok' if ok else 'FAIL'} probe {why}", flush=True)
        return 0 if ok else 1
    kernel, precision, grid = sys.argv[1], sys.argv[2], tuple(int(x) for x in sys.argv[3].split(","))
    transport = os.environ.get("KL_HALO_TRANSPORT", "ipc")
    if transport == "nccl":
        uid = group.broadcast(NcclExchanger.unique_id() if rank == 0 else None, size=128)
        ex = NcclExchanger(rank, world, uid)
    else:
        ex = IpcExchanger(group)
    # "fused": no exchange at all — diff_uvw_peer reads the planes outside the
    # slab from the neighbours' IPC-mapped fields (the poisoned ghost planes
    # below are then never read)
    drv = SlabDriver(kernel, precision, grid, ctx, rank=rank, nranks=world, exchanger=ex,
                     compiler=NvrtcCompiler(ctx), wisdom_dir=str(ROOT / "wisdom"),
                     halo="fused" if transport == "fused" else "exchange")
    if kernel == "diff_uvw_rk3":  # the RK3 time loop: 4 substeps, fused halo, vs the oracle's loop
        return rk3_loop_check(drv, ctx, group, ex, rank, grid, precision)
    drv.resolve()
    if os.environ.get("KL_CHECK_SHARED"):
        # another driver on the same exchanger, stepped and closed: closing it
        # must unmap only its own field set, not drv's peer mappings
        extra = SlabDriver(kernel, precision, grid, ctx, rank=rank, nranks=world, exchanger=ex,
                           compiler=NvrtcCompiler(ctx), wisdom_dir=str(ROOT / "wisdom"))
        extra.resolve()
        extra.step()
        extra.close()
    ref, _ = oracle_outputs(kernel, GridLayout(*grid, precision))
    g = drv.layout.kgc
    off, count = drv.slab.offset, drv.slab.count
    worst, poisoned = 0.0, 0
    for _ in range(2):
        drv.problem.regenerate(drv.problem.outputs())
        poisoned = poison_halo(drv)
        ctx.synchronize()
        group.barrier()  # every rank's halo is poisoned before anyone pulls
        drv.step()
        ctx.synchronize()
        for name in ref:
            got = drv.problem.download(name)[g:g + count, g:-g, g:g + grid[0]].astype(np.float64)
            want = ref[name][g + off:g + off + count, g:-g, g:g + grid[0]]
            err = float(np.max(np.abs(got - want)) / np.max(np.abs(ref[name][g:-g, g:-g, g:g + grid[0]])))
            worst = max(worst, err if np.isfinite(err) else float("inf"))
    drv.close()
    ex.close()
    group.close()
    tol = 1e-5 if precision == "fp32" else 1e-12
    ok = worst <= tol and (poisoned > 0 or world == 1)
    print(f"rank {rank} {'ok' if ok else 'FAIL'} {worst:.3e} poisoned_planes={poisoned}", flush=True)
    return 0 if ok else 1


def rk3_loop_check(drv, ctx, group, ex, rank, grid, precision) -> int:
    import numpy as np

    from stencil_helpers import oracle_rk3_loop

    nsub, dt = 4, 0.05
    poisoned = poison_halo(drv)
    ctx.synchronize()
    group.barrier()
    for s in range(nsub):
        drv.rk3_substep(s, dt)
    ctx.synchronize()
    want_t, want_u = oracle_rk3_loop(drv.global_layout, nsub, dt)
    g = drv.layout.kgc
    off, count = drv.slab.offset, drv.slab.count
    worst = 0.0
    for name, ref in list(want_t.items()) + list(want_u.items()):
        got = drv.problem.download(name)[g:g + count, g:-g, g:g + grid[0]].astype(np.float64)
        r = ref[g + off:g + off + count, g:-g, g:g + grid[0]]
        err = float(np.max(np.abs(got - r)) / np.max(np.abs(ref[g:-g, g:-g, g:g + grid[0]])))
        worst = max(worst, err if np.isfinite(err) else float("inf"))
    drv.close()
    ex.close()
    group.close()
    tol = 1e-5 if precision == "fp32" else 1e-12
    ok = worst <= tol
    print(f"rank {rank} {'ok' if ok else 'FAIL'} {worst:.3e} rk3 substeps={nsub} poisoned_planes={poisoned}", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
