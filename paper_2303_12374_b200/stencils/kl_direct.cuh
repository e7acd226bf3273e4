// kl_direct.cuh — the paper's DIRECT kernel structure (Table-2 knobs) as a
// reusable tile loop for the per-cell stencils of the MicroHH family
// (advec_v/w/s, diff_c, evisc_smag).
//
// Every thread covers TILE_X*TILE_Y*TILE_Z cells of its block (block-strided
// or CONTIG_* consecutive), loops unrolled or not per UNROLL_*, blocks
// unravelled from a 1-D id in UNRAVEL order (SURVEY.md
// Appendix A.4).  `plane(k)` is evaluated once per tile plane (per-level
// factors hoisted out of the x/y loops), `cell(ijk, i, j, k, p)` per cell.

#ifndef KL_DIRECT_CUH
#define KL_DIRECT_CUH

namespace kl {

template <class Plane, class Cell>
__device__ __forceinline__ void direct_tiles(int istart, int jstart, int kstart, int iend, int jend, int kend,
                                             Plane&& plane, Cell&& cell) {
  const unsigned nbx = ceil_div(iend - istart, BLOCK_X * TILE_X);
  const unsigned nby = ceil_div(jend - jstart, BLOCK_Y * TILE_Y);
  const unsigned nbz = ceil_div(kend - kstart, BLOCK_Z * TILE_Z);
  int bx, by, bz;
  unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  KL_UNROLL_Z
  for (int tz = 0; tz < TILE_Z; ++tz) {
    const int k = kstart + tile_index<BLOCK_Z, TILE_Z, CONTIG_Z>(bz, threadIdx.z, tz);
    if (k >= kend) continue;
    const auto p = plane(k);
    KL_UNROLL_Y
    for (int ty = 0; ty < TILE_Y; ++ty) {
      const int j = jstart + tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(by, threadIdx.y, ty);
      if (j >= jend) continue;
      KL_UNROLL_X
      for (int tx = 0; tx < TILE_X; ++tx) {
        const int i = istart + tile_index<BLOCK_X, TILE_X, CONTIG_X>(bx, threadIdx.x, tx);
        if (i >= iend) continue;
        const long long ijk = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k) * KL_KK;
        cell(ijk, p);
      }
    }
  }
}

}  // namespace kl

#endif  // KL_DIRECT_CUH
