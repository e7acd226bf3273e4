// advec_u_zmarch.cuh — STAGING == ZMARCH variant of advec_u (included by
// advec_u.cu).  A block owns a (BLOCK_X*TILE_X) x (BLOCK_Y*TILE_Y) column of
// cells and marches up ZCHUNK planes:
//
//   * the 7-point z-stencil of u for each owned cell lives in a register
//     window uq[0..6] = u[k-3 .. k+3]; one new plane value is loaded per step;
//   * the x/y neighbours come from a halo'd (3-cell) shared-memory copy of
//     plane k, double-buffered so one __syncthreads per plane suffices;
//   * the bottom z-face flux and the bottom face velocity are carried from
//     the previous plane (Fz[k-1/2] of plane k == Fz[k+1/2] of plane k-1),
//     so each plane computes 1 z-flux instead of 2.
// HBM traffic stays at the compulsory 5 words/cell (+ the 6 z-halo planes per
// chunk); the x/y halo re-reads are served by L2/shared memory.

#if BLOCK_Z != 1 || TILE_Z != 1
#error "ZMARCH requires BLOCK_Z == 1 and TILE_Z == 1"
#endif

#define KL_TXT (BLOCK_X * TILE_X)
#define KL_TYT (BLOCK_Y * TILE_Y)
#define KL_SW (KL_TXT + 6)
#define KL_SH (KL_TYT + 6)
#define KL_PLANE (KL_SW * KL_SH)

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
         const real* __restrict__ dzi, const real dxi, const real dyi, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  extern __shared__ __align__(16) unsigned char kl_smem_raw[];
  real* const splanes = reinterpret_cast<real*>(kl_smem_raw);  // [2][KL_SH][KL_SW]

  const unsigned nbx = kl::ceil_div(iend - istart, KL_TXT);
  const unsigned nby = kl::ceil_div(jend - jstart, KL_TYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * KL_TXT;
  const int j0 = jstart + by * KL_TYT;
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  const real dxi60 = dxi * real(1.0 / 60.0);
  const real dyi60 = dyi * real(1.0 / 60.0);
  constexpr long long K1 = KL_KK;

  real uq[TILE_Y][TILE_X][7];
  real fz_bot[TILE_Y][TILE_X];
  long long base[TILE_Y][TILE_X];  // index of (i, j, k0) (clamped for out-of-range cells)

  const real rh0 = rhorefh[k0];
#pragma unroll
  for (int ty = 0; ty < TILE_Y; ++ty) {
#pragma unroll
    for (int tx = 0; tx < TILE_X; ++tx) {
      const int i = min(i0 + kl::tile_index<BLOCK_X, TILE_X, CONTIG_X>(0, threadIdx.x, tx), iend - 1);
      const int j = min(j0 + kl::tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(0, threadIdx.y, ty), jend - 1);
      const long long ijk = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
      base[ty][tx] = ijk;
#pragma unroll
      for (int m = 0; m < 7; ++m) uq[ty][tx][m] = u[ijk + (m - 3) * K1];
      const real wb = kl::interp2(w[ijk - 1], w[ijk]);
      fz_bot[ty][tx] = rh0 * kl::flux5x60(wb, uq[ty][tx][0], uq[ty][tx][1], uq[ty][tx][2], uq[ty][tx][3],
                                         uq[ty][tx][4], uq[ty][tx][5]);
    }
  }

  for (int k = k0; k < k1; ++k) {
    real* const plane = splanes + (k & 1) * KL_PLANE;
    const long long kofs = static_cast<long long>(k) * KL_KK;
    // Cooperative halo'd plane fill (coalesced along x; clamped to the ghost box).
    for (int idx = tid; idx < KL_PLANE; idx += KL_THREADS) {
      const int r = idx / KL_SW;
      const int c = idx - r * KL_SW;
      const int gj = min(j0 - 3 + r, jend + 2);
      const int gi = min(i0 - 3 + c, iend + 2);
      plane[idx] = u[gi + static_cast<long long>(gj) * KL_JJ + kofs];
    }
    // Next-plane window values, issued before the barrier to overlap latency.
    real unext[TILE_Y][TILE_X];
    const bool more = k + 1 < k1;
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty)
#pragma unroll
      for (int tx = 0; tx < TILE_X; ++tx)
        unext[ty][tx] = more ? u[base[ty][tx] + (k - k0 + 4) * K1] : real(0);
    __syncthreads();

    const real rh_top = rhorefh[k + 1];
    const real zfac60 = dzi[k] / (rhoref[k] * real(60));
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty) {
      const int lj = kl::tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(0, threadIdx.y, ty);
#pragma unroll
      for (int tx = 0; tx < TILE_X; ++tx) {
        const int li = kl::tile_index<BLOCK_X, TILE_X, CONTIG_X>(0, threadIdx.x, tx);
        const real* p = plane + (lj + 3) * KL_SW + (li + 3);
        const long long ijk = base[ty][tx] + (k - k0) * K1;
        real* q = uq[ty][tx];

        const real xa = p[-3], xb = p[-2], xc = p[-1], xd = p[0], xe = p[1], xf = p[2], xg = p[3];
        const real fx = kl::flux5x60(kl::interp2(xd, xe), xb, xc, xd, xe, xf, xg) -
                        kl::flux5x60(kl::interp2(xc, xd), xa, xb, xc, xd, xe, xf);

        const real ya = p[-3 * KL_SW], yb = p[-2 * KL_SW], yc = p[-KL_SW];
        const real ye = p[KL_SW], yf = p[2 * KL_SW], yg = p[3 * KL_SW];
        const real vn = kl::interp2(v[ijk - 1 + KL_JJ], v[ijk + KL_JJ]);
        const real vs = kl::interp2(v[ijk - 1], v[ijk]);
        const real fy = kl::flux5x60(vn, yb, yc, xd, ye, yf, yg) - kl::flux5x60(vs, ya, yb, yc, xd, ye, yf);

        const real wt_face = kl::interp2(w[ijk - 1 + K1], w[ijk + K1]);
        const real fz_top = rh_top * kl::flux5x60(wt_face, q[1], q[2], q[3], q[4], q[5], q[6]);

        const int i = i0 + li, j = j0 + lj;
        if (i < iend && j < jend) ut[ijk] -= fx * dxi60 + fy * dyi60 + (fz_top - fz_bot[ty][tx]) * zfac60;
        fz_bot[ty][tx] = fz_top;
#pragma unroll
        for (int m = 0; m < 6; ++m) q[m] = q[m + 1];
        q[6] = unext[ty][tx];
      }
    }
  }
}

#undef KL_TXT
#undef KL_TYT
#undef KL_SW
#undef KL_SH
#undef KL_PLANE
