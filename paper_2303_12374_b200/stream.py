"""Host-streamed stencil step: fields live in pinned host memory, the GPU
pulls them in z-chunks, so PCIe uploads, kernels and downloads overlap.

The end-to-end use of the hot path (BASELINE e2e: inputs in host memory,
tendencies back to the host every step) is bound by the host link, not HBM:
a 1024^3 fp32 ``diff_uvw`` step moves 7 fields in and 3 out (~31 GB + 13 GB).
Issued as whole-field copies around one launch the two directions serialise;
here the slab is cut into chunks of planes and each chunk's

    h2d stream     : upload the planes its stencil reads that no earlier
                     chunk uploaded (inputs with their z reach, RMW outputs)
    compute stream : wait(upload) ; launch the chunk's sub-range
    d2h stream     : wait(launch) ; download the chunk's output planes

so downloads of chunk c run on the second copy engine while chunk c+1 is
uploaded; the step costs ~ max(upload, download) + one chunk, not the sum.

Every chunk is a k sub-range launched through ``WisdomKernel.launch`` (its
own problem size -> its own wisdom selection), exactly like the slab
sub-ranges of ``halo.py``.  With neighbours (z-slab ranks) the boundary
stages come first: their uploads include the planes the halo exchange sends,
the exchange is issued on the comm stream right after them, and their
launches wait for it; uploads never touch ghost planes the exchange owns.

``stream_plan`` is pure (no CUDA) so the plan is unit-tested on CPU;
``SlabDriver.step_host`` executes it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .halo import HALO_REACH

__all__ = ["PlaneCopy", "StreamStage", "stream_plan", "chunk_ranges"]


@dataclass(frozen=True)
class PlaneCopy:
    """Planes ``[p0, p1)`` of one field (local plane indices)."""

    field: str
    p0: int
    p1: int


@dataclass
class StreamStage:
    name: str
    k_range: tuple[int, int]
    after_halo: bool
    uploads: list[PlaneCopy] = field(default_factory=list)
    downloads: list[PlaneCopy] = field(default_factory=list)


def chunk_ranges(kb: int, ke: int, chunks: int) -> list[tuple[int, int]]:
    """Split ``[kb, ke)`` into at most ``chunks`` pieces of ceil size (the last
    may be shorter) — at most two distinct problem sizes to compile."""
    n = ke - kb
    if n <= 0:
        return []
    size = -(-n // max(1, min(chunks, n)))
    return [(k, min(k + size, ke)) for k in range(kb, ke, size)]


def _runs(flags: list[bool], lo: int, hi: int):
    """Maximal runs of False in flags[lo:hi] as (p0, p1)."""
    p = lo
    while p < hi:
        if flags[p]:
            p += 1
            continue
        q = p
        while q < hi and not flags[q]:
            q += 1
        yield p, q
        p = q


def stream_plan(kernel: str, fields: tuple[str, ...], outputs: tuple[str, ...], ranges: dict[str, tuple[int, int]],
                kcells: int, kstart: int, kend: int, below: int, above: int, chunks: int) -> list[StreamStage]:
    """Stages in upload order: boundary sub-ranges (lower/upper), then the
    interior sub-range cut into ``chunks`` pieces.

    ``ranges`` are ``SlabRank.subranges()``; planes a stage's stencil reads
    for field f with reach (down, up) = ``HALO_REACH`` are
    ``[k0 - up, k1 + down)`` (fields without an entry: ``[k0, k1)``),
    clipped to the host-owned planes — all of ``[0, kcells)`` on a side
    without a neighbour, only ``[kstart, kend)`` on a side the exchange fills.
    Each plane of each field is uploaded exactly once per step.
    """
    reach = HALO_REACH[kernel]
    own_lo = kstart if below >= 0 else 0
    own_hi = kend if above >= 0 else kcells
    stages = [StreamStage(n, ranges[n], True) for n in ("lower", "upper") if n in ranges]
    if "interior" in ranges:
        kb, ke = ranges["interior"]
        pieces = chunk_ranges(kb, ke, chunks)
        stages += [StreamStage(f"interior.{i}", r, False) for i, r in enumerate(pieces)]
    done = {f: [False] * kcells for f in fields}
    for st in stages:
        k0, k1 = st.k_range
        for f in fields:
            down, up = reach.get(f, (0, 0))
            lo, hi = max(k0 - up, own_lo), min(k1 + down, own_hi)
            for p0, p1 in _runs(done[f], lo, hi):
                st.uploads.append(PlaneCopy(f, p0, p1))
                for p in range(p0, p1):
                    done[f][p] = True
        st.downloads = [PlaneCopy(f, k0, k1) for f in outputs]
    if any(s.after_halo for s in stages) and below < 0 and above < 0:
        for s in stages:  # no neighbours: nothing to wait for
            s.after_halo = False
    return stages
