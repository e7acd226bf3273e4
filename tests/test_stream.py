"""Host-streamed step plan (stream.py): every plane a stage's stencil reads is
uploaded by that stage or an earlier one, exactly once per step, never a ghost
plane the halo exchange owns; outputs are downloaded once."""

import pytest

from paper_2303_12374_b200.halo import HALO_REACH, SlabDecomposition, SlabRank
from paper_2303_12374_b200.stencils.problem import KERNEL_FIELDS
from paper_2303_12374_b200.stencils.definitions import ARG_LAYOUT
from paper_2303_12374_b200.stream import chunk_ranges, stream_plan


def test_chunk_ranges():
    assert chunk_ranges(3, 1027, 16) == [(3 + 64 * i, 67 + 64 * i) for i in range(16)]
    assert chunk_ranges(3, 13, 4) == [(3, 6), (6, 9), (9, 12), (12, 13)]
    assert chunk_ranges(3, 5, 16) == [(3, 4), (4, 5)]
    assert chunk_ranges(5, 5, 4) == []


def _outputs(kernel):
    return tuple(n for n, role in ARG_LAYOUT[kernel]["buffers"] if role == "output")


@pytest.mark.parametrize("kernel", ["advec_u", "diff_uvw"])
@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
@pytest.mark.parametrize("chunks", [1, 3, 16])
def test_plan_covers_reads_once(kernel, nranks, chunks):
    ktot, g = 20, 3
    dec = SlabDecomposition(ktot, nranks)
    fields, outputs = tuple(KERNEL_FIELDS[kernel]), _outputs(kernel)
    for rank in range(nranks):
        slab = SlabRank(dec, rank, g, kernel)
        below, above = dec.neighbours(rank)
        kcells = slab.count + 2 * g
        ranges = slab.subranges()
        plan = stream_plan(kernel, fields, outputs, ranges, kcells, slab.kstart, slab.kend, below, above, chunks)
        # the stages tile the launch ranges exactly
        covered = sorted(st.k_range for st in plan)
        assert covered[0][0] == slab.kstart and covered[-1][1] == slab.kend
        assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
        assert len([s for s in plan if s.name.startswith("interior")]) <= chunks
        uploaded = {f: [] for f in fields}
        for st in plan:
            for c in st.uploads:
                uploaded[c.field].extend(range(c.p0, c.p1))
                # never a ghost plane on a side the exchange fills
                if below >= 0:
                    assert c.p0 >= slab.kstart
                if above >= 0:
                    assert c.p1 <= slab.kend
            k0, k1 = st.k_range
            for f in fields:
                down, up = HALO_REACH[kernel].get(f, (0, 0))
                have = set(uploaded[f])
                for p in range(k0 - up, k1 + down):
                    ghost_from_exchange = (p < slab.kstart and below >= 0) or (p >= slab.kend and above >= 0)
                    assert ghost_from_exchange or p in have, (rank, st.name, f, p)
                    if ghost_from_exchange:
                        assert st.after_halo
            assert [(c.field, c.p0, c.p1) for c in st.downloads] == [(f, k0, k1) for f in outputs]
        for f, planes in uploaded.items():
            assert len(planes) == len(set(planes)), f  # exactly once
        # boundary stages (whose uploads hold the exchange's send planes) come first
        flags = [st.after_halo for st in plan]
        assert flags == sorted(flags, reverse=True)


def test_single_rank_has_no_halo_wait():
    kernel = "diff_uvw"
    dec = SlabDecomposition(64, 1)
    slab = SlabRank(dec, 0, 3, kernel)
    plan = stream_plan(kernel, tuple(KERNEL_FIELDS[kernel]), _outputs(kernel), slab.subranges(), 70, 3, 67, -1, -1, 4)
    assert [st.k_range for st in plan] == [(3, 19), (19, 35), (35, 51), (51, 67)]
    assert not any(st.after_halo for st in plan)
    # first chunk brings the bottom physical ghost plane, last the top one; plain fields: no ghosts
    u = [(c.p0, c.p1) for st in plan for c in st.uploads if c.field == "u"]
    assert u[0] == (2, 20) and u[-1] == (52, 68)
    ut = [(c.p0, c.p1) for st in plan for c in st.uploads if c.field == "ut"]
    assert ut == [(3, 19), (19, 35), (35, 51), (51, 67)]
