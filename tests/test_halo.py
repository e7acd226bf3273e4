"""Multi-GPU z-slab logic on CPU: decomposition, the halo plan, and a
world_size-2 gloo run of the exchange protocol feeding the NumPy oracle."""

import os
import socket

import numpy as np
import pytest

from paper_2303_12374_b200.halo import HALO_REACH, SlabDecomposition, SlabRank, halo_plan, kernel_reach


def test_decomposition_covers_grid():
    for ktot, n in ((1024, 8), (1024, 3), (17, 4), (5, 5)):
        dec = SlabDecomposition(ktot, n)
        spans = [dec.planes(r) for r in range(n)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == ktot
        assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(n - 1))
        assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    assert SlabDecomposition(8, 3).neighbours(0) == (-1, 1) and SlabDecomposition(8, 3).neighbours(2) == (1, -1)


def test_plan_pairs_match():
    """Every send of rank r has a recv of the same plane count on the peer."""
    for kernel, fields in HALO_REACH.items():
        for name, (down, up) in fields.items():
            dec = SlabDecomposition(40, 4)
            for r in range(3):
                a, b = SlabRank(dec, r, 3, kernel), SlabRank(dec, r + 1, 3, kernel)
                ops_a = halo_plan(a.kstart, a.kend, down, up, *dec.neighbours(r))
                ops_b = halo_plan(b.kstart, b.kend, down, up, *dec.neighbours(r + 1))
                sent_up = [n for op, peer, _, n in ops_a if op == "send" and peer == r + 1]
                recv_from_below = [n for op, peer, _, n in ops_b if op == "recv" and peer == r]
                assert sent_up == recv_from_below
                sent_down = [n for op, peer, _, n in ops_b if op == "send" and peer == r]
                recv_from_above = [n for op, peer, _, n in ops_a if op == "recv" and peer == r + 1]
                assert sent_down == recv_from_above


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
def test_subranges_partition_slab(kernel):
    dec = SlabDecomposition(64, 4)
    down, up = kernel_reach(kernel)
    for r in range(4):
        sr = SlabRank(dec, r, 3, kernel)
        ranges = sr.subranges()
        planes = sorted(k for lo, hi in ranges.values() for k in range(lo, hi))
        assert planes == list(range(sr.kstart, sr.kend))
        lo, hi = ranges["interior"]
        below, above = dec.neighbours(r)
        # the interior launch never reads a ghost plane that the exchange writes
        if below >= 0:
            assert lo - up >= sr.kstart
        if above >= 0:
            assert hi - 1 + down < sr.kend


def _slab_fields(kernel, itot, jtot, ktot, rank, nranks, g=3):
    from oracle.synth import synth_field
    from paper_2303_12374_b200.stencils.problem import KERNEL_FIELDS
    from paper_2303_12374_b200.stencils.profiles import FIELD_SEED_BASE, FIELD_SPECS

    dec = SlabDecomposition(ktot, nranks)
    off, count = dec.planes(rank)
    out = {}
    for name in KERNEL_FIELDS[kernel]:
        s, lo, hi = FIELD_SPECS[name]
        out[name] = synth_field(FIELD_SEED_BASE + s, lo, hi, itot + 2 * g, jtot + 2 * g, count + 2 * g, g, g,
                                k_offset=off)
    return out, off, count


def _oracle(kernel, f, prof, interior):
    from oracle import stencil_oracle

    if kernel == "advec_u":
        return {"ut": stencil_oracle.advec_u(f["ut"], f["u"], f["v"], f["w"], prof.rhoref, prof.rhorefh, prof.dzi, 1.0,
                                             1.0, interior=interior)}
    ut, vt, wt = stencil_oracle.diff_uvw(f["ut"], f["vt"], f["wt"], f["evisc"], f["u"], f["v"], f["w"], prof.dzi,
                                         prof.dzhi, prof.rhoref, prof.rhorefh, 1.0, 1.0, interior=interior)
    return {"ut": ut, "vt": vt, "wt": wt}


class HostExchanger:
    """The halo plan over torch.distributed (gloo) on NumPy (kcells, jcells, icells)
    arrays — the CPU-test transport of the same ``halo_plan`` the C-ABI
    transports (NCCL send/recv, CUDA-IPC pull) run on the GPU."""

    def __init__(self, rank: int, nranks: int) -> None:
        self.rank, self.nranks = rank, nranks

    def exchange(self, arrays, kstart: int, kend: int, down: int, up: int, below: int, above: int) -> None:
        import numpy as np
        import torch
        import torch.distributed as dist

        reqs, sinks = [], []
        for arr in arrays:
            for op, peer, first, count in halo_plan(kstart, kend, down, up, below, above):
                if op == "send":
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr[first:first + count])), peer))
                else:
                    buf = torch.empty(arr[first:first + count].shape, dtype=torch.from_numpy(arr[:1]).dtype)
                    reqs.append(dist.irecv(buf, peer))
                    sinks.append((arr, first, count, buf))
        for req in reqs:
            req.wait()
        for arr, first, count, buf in sinks:
            arr[first:first + count] = buf.numpy()


def _rank_main(rank, nranks, port, kernel, queue):
    import torch.distributed as dist

    from paper_2303_12374_b200.stencils.profiles import make_profiles

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    itot, jtot, ktot, g = 12, 10, 16, 3
    f, off, count = _slab_fields(kernel, itot, jtot, ktot, rank, nranks)
    # poison the ghost planes that the exchange must fill
    dec = SlabDecomposition(ktot, nranks)
    below, above = dec.neighbours(rank)
    for name, (down, up) in HALO_REACH[kernel].items():
        if below >= 0:
            f[name][g - up:g] = np.nan
        if above >= 0:
            f[name][g + count:g + count + down] = np.nan
    ex = HostExchanger(rank, nranks)
    for name, (down, up) in HALO_REACH[kernel].items():
        ex.exchange([f[name]], g, g + count, down, up, below, above)
    prof = make_profiles(ktot + 2 * g, g).window(off, count + 2 * g)
    res = _oracle(kernel, f, prof, (itot, jtot, count))
    queue.put((rank, off, count, {k: v[g:g + count] for k, v in res.items()}))
    dist.destroy_process_group()


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
def test_gloo_world2_slabs_equal_global(kernel):
    import torch.multiprocessing as mp

    from paper_2303_12374_b200.stencils.profiles import make_profiles

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, kernel, queue)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [queue.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    itot, jtot, ktot, g = 12, 10, 16, 3
    f, _, _ = _slab_fields(kernel, itot, jtot, ktot, 0, 1)
    ref = _oracle(kernel, f, make_profiles(ktot + 2 * g, g), (itot, jtot, ktot))
    for rank, off, count, res in parts:
        for name, arr in res.items():
            assert np.array_equal(arr, ref[name][g + off:g + off + count]), (rank, name)
