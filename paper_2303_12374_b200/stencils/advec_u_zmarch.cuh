// advec_u_zmarch.cuh — STAGING == ZMARCH variant of advec_u (included by
// advec_u.cu): flux-form, z-marching, shared-memory staged.
//
// The DIRECT kernel evaluates both faces of every cell in all three
// directions (6 upwind fluxes per cell, each ~16 FP ops plus its 6 loads).
// Here every face flux is evaluated once:
//   * z: a thread keeps the 7-point z-stencil of u for each of its cells in a
//     register window and carries F[k+1/2] to the next plane as F[k-1/2];
//   * y: a thread owns a contiguous strip of TILE_Y rows; F[j+1/2] of row j is
//     reused as F[j-1/2] of row j+1 (one extra flux per strip);
//   * x: both faces of a cell are evaluated (sharing the west face through a
//     warp shuffle was measured slower: lane 0's own evaluation runs as a
//     divergent branch in every warp, costing as many issue slots as it saves).
// u is staged per plane into a double-buffered shared-memory tile with a
// 3-cell halo (the x/y stencil reads), the next plane is prefetched into
// registers before the compute and stored after it — one __syncthreads per
// plane.

#if BLOCK_Z != 1 || TILE_Z != 1 || TILE_X != 1
#error "advec_u ZMARCH requires BLOCK_Z == TILE_Z == TILE_X == 1"
#endif

#define KL_TYT (BLOCK_Y * TILE_Y)
#define KL_SW (BLOCK_X + 6)
#define KL_SH (KL_TYT + 6)
#define KL_PLANE (KL_SW * KL_SH)
#define KL_FILL ((KL_PLANE + KL_THREADS - 1) / KL_THREADS)

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
         const real* __restrict__ dzi, const real dxi, const real dyi, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  extern __shared__ __align__(16) unsigned char kl_smem_raw[];
  real* const tiles = reinterpret_cast<real*>(kl_smem_raw);  // [2][KL_SH][KL_SW]

  const unsigned nbx = kl::ceil_div(iend - istart, BLOCK_X);
  const unsigned nby = kl::ceil_div(jend - jstart, KL_TYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * BLOCK_X;
  const int j0 = jstart + by * KL_TYT;
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  const real dxi60 = dxi * real(1.0 / 60.0);
  const real dyi60 = dyi * real(1.0 / 60.0);
  constexpr long long K1 = KL_KK;
  constexpr long long J1 = KL_JJ;

  // plane-fill mapping (clamped into the ghost box)
  long long goff[KL_FILL];
  int soff[KL_FILL];
#pragma unroll
  for (int n = 0; n < KL_FILL; ++n) {
    const int idx = tid + n * KL_THREADS;
    const int r = idx / KL_SW, c = idx - r * KL_SW;
    goff[n] = min(i0 - 3 + c, iend + 2) + static_cast<long long>(min(j0 - 3 + r, jend + 2)) * KL_JJ;
    soff[n] = idx < KL_PLANE ? idx : -1;
  }

  // this thread's column and strip (clamped for cells outside the grid; never stored)
  const int i = min(i0 + static_cast<int>(threadIdx.x), iend - 1);
  const int lj0 = threadIdx.y * TILE_Y;
  long long base[TILE_Y];  // (i, j, k0)
  real uq[TILE_Y][7];      // u[k-3 .. k+3]
  real fz_bot[TILE_Y];
  const real rh0 = rhorefh[k0];
#pragma unroll
  for (int t = 0; t < TILE_Y; ++t) {
    const int j = min(j0 + lj0 + t, jend - 1);
    base[t] = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
#pragma unroll
    for (int m = 0; m < 7; ++m) uq[t][m] = u[base[t] + (m - 3) * K1];
    const real wb = kl::interp2(w[base[t] - 1], w[base[t]]);
    fz_bot[t] = rh0 * kl::flux5x60(wb, uq[t][0], uq[t][1], uq[t][2], uq[t][3], uq[t][4], uq[t][5]);
  }
  {
    real* tile = tiles + (k0 & 1) * KL_PLANE;
    const long long kofs = static_cast<long long>(k0) * KL_KK;
#pragma unroll
    for (int n = 0; n < KL_FILL; ++n)
      if (soff[n] >= 0) tile[soff[n]] = u[goff[n] + kofs];
  }

  for (int k = k0; k < k1; ++k) {
    __syncthreads();
    const bool more = k + 1 < k1;
    // prefetch: next plane tile and the next window values
    real nxt[KL_FILL];
    real unext[TILE_Y];
    {
      const long long kofs = static_cast<long long>(k + 1) * KL_KK;
#pragma unroll
      for (int n = 0; n < KL_FILL; ++n) nxt[n] = (more && soff[n] >= 0) ? u[goff[n] + kofs] : real(0);
#pragma unroll
      for (int t = 0; t < TILE_Y; ++t) unext[t] = more ? u[base[t] + (k - k0 + 4) * K1] : real(0);
    }
    const real* tile = tiles + (k & 1) * KL_PLANE;
    const real* col = tile + (lj0 + 3) * KL_SW + (threadIdx.x + 3);  // (i, j0+lj0) in the tile
    const real rh_top = rhorefh[k + 1];
    const real zfac60 = dzi[k] / (rhoref[k] * real(60));
    const long long kofs = static_cast<long long>(k - k0) * K1;

    // u along y in this column: rows lj0-3 .. lj0+TILE_Y+2
    real ucol[TILE_Y + 6];
#pragma unroll
    for (int m = 0; m < TILE_Y + 6; ++m) ucol[m] = col[(m - 3) * KL_SW];

    // lower y-face of the strip (row j0+lj0-1/2)
    real fy_lo;
    {
      const long long b = base[0] + kofs;
      const real vs = kl::interp2(v[b - 1], v[b]);
      fy_lo = kl::flux5x60(vs, ucol[0], ucol[1], ucol[2], ucol[3], ucol[4], ucol[5]);
    }
#pragma unroll
    for (int t = 0; t < TILE_Y; ++t) {
      const long long ijk = base[t] + kofs;
      const real* row = col + t * KL_SW;
      const real* q = uq[t];
      // x: east and west faces of this cell
      const real xm2 = row[-2], xm1 = row[-1], x0 = ucol[t + 3], xp1 = row[1], xp2 = row[2], xp3 = row[3];
      const real fx_e = kl::flux5x60(kl::interp2(x0, xp1), xm2, xm1, x0, xp1, xp2, xp3);
      const real fx_w = kl::flux5x60(kl::interp2(xm1, x0), row[-3], xm2, xm1, x0, xp1, xp2);
      // y: north face of this row; south face carried from the previous row
      const real vn = kl::interp2(v[ijk - 1 + J1], v[ijk + J1]);
      const real fy_hi = kl::flux5x60(vn, ucol[t + 1], ucol[t + 2], ucol[t + 3], ucol[t + 4], ucol[t + 5], ucol[t + 6]);
      // z: top face of this plane; bottom face carried from the previous plane
      const real wtop = kl::interp2(w[ijk - 1 + K1], w[ijk + K1]);
      const real fz_top = rh_top * kl::flux5x60(wtop, q[1], q[2], q[3], q[4], q[5], q[6]);
      const int j = j0 + lj0 + t;
      if (i0 + static_cast<int>(threadIdx.x) < iend && j < jend)
        ut[ijk] -= (fx_e - fx_w) * dxi60 + (fy_hi - fy_lo) * dyi60 + (fz_top - fz_bot[t]) * zfac60;
      fy_lo = fy_hi;
      fz_bot[t] = fz_top;
#pragma unroll
      for (int m = 0; m < 6; ++m) uq[t][m] = uq[t][m + 1];
      uq[t][6] = unext[t];
    }
    if (more) {
      real* dst = tiles + ((k + 1) & 1) * KL_PLANE;
#pragma unroll
      for (int n = 0; n < KL_FILL; ++n)
        if (soff[n] >= 0) dst[soff[n]] = nxt[n];
    }
  }
}

#undef KL_TYT
#undef KL_SW
#undef KL_SH
#undef KL_PLANE
#undef KL_FILL
