"""``ProcessGroup`` (klb_group_*, POSIX shared memory): the torch-free rank
rendezvous of the multi-rank driver, exercised with real processes on CPU
(the group needs no GPU)."""

import multiprocessing as mp
import os
import time

import pytest

from paper_2303_12374_b200.cuda._abi import KlbError, library_path

pytestmark = pytest.mark.skipif(not library_path().exists(), reason="libklb200.so not built")


def _rank(rank, nranks, name, queue):
    from paper_2303_12374_b200.group import ProcessGroup

    with ProcessGroup(rank, nranks, name=name, timeout=60) as g:
        got = g.allgather(bytes([rank]) * 100)
        seq = []
        for step in range(50):  # barriers keep the ranks in lockstep
            seq.append(g.max(rank * 1000 + step))
        total = g.sum(rank + 1)
        uid = g.broadcast(os.urandom(128) if rank == 0 else None, size=128)
        uids = g.allgather(uid)
        g.barrier()
    queue.put((rank, [b[0] for b in got], seq, total, len(set(uids))))


@pytest.mark.parametrize("nranks", [2, 3])
def test_group_barrier_allgather_reductions(nranks):
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    name = f"/klb_test_{os.getpid()}_{nranks}_{time.monotonic_ns()}"
    procs = [ctx.Process(target=_rank, args=(r, nranks, name, queue)) for r in range(nranks)]
    for p in procs:
        p.start()
    out = sorted(queue.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, gathered, seq, total, distinct in out:
        assert gathered == list(range(nranks))
        assert seq == [(nranks - 1) * 1000 + s for s in range(50)]
        assert total == nranks * (nranks + 1) / 2
        assert distinct == 1  # everyone holds rank 0's id
    assert not os.path.exists("/dev/shm" + name)  # unlinked once everyone attached


def test_group_times_out_when_a_peer_never_arrives():
    from paper_2303_12374_b200.group import ProcessGroup

    t0 = time.monotonic()
    with pytest.raises(KlbError, match="timed out"):
        ProcessGroup(0, 2, name=f"/klb_test_alone_{os.getpid()}", timeout=1.0)
    assert time.monotonic() - t0 < 30
    os.unlink(f"/dev/shm/klb_test_alone_{os.getpid()}")


def test_group_name_is_per_launcher():
    from paper_2303_12374_b200.group import group_name

    a = group_name({"MASTER_PORT": "29500", "TORCHELASTIC_RUN_ID": "abc"})
    assert a.startswith("/klb_") and "/" not in a[1:] and a.endswith("_29500_abc")
    assert group_name({"KLB_GROUP": "/x/y"}) == "/x_y"
