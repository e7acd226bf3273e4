// diff_uvw_zmarch.cuh — STAGING == ZMARCH variant of diff_uvw (included by
// diff_uvw.cu): flux-form, z-marching, shared-memory staged.
//
// The DIRECT kernel evaluates the A.3 formulas per cell: every face flux and
// every 4-point viscosity average is computed twice (once by each cell that
// shares the face) and ~54 neighbour loads go through L1 (ncu: L1 90% busy,
// ~380 SASS instructions per cell).  Here each face quantity is computed
// once:
//   * a block owns BLOCK_X columns x (BLOCK_Y*TILE_Y) rows and marches up
//     ZCHUNK planes; each thread owns one column and a contiguous strip of
//     TILE_Y rows;
//   * quantities on the upper y-face of row j (y-fluxes, xy/yz edge
//     viscosities, the row's +1 neighbours) are kept in registers and reused
//     as the lower y-face of row j+1;
//   * quantities on the upper z-face of plane k (z-fluxes, and the x/y fluxes
//     of w which live at k+1/2) are carried in registers to plane k+1;
//   * evisc, u, v, w are staged plane by plane into a 3-slot shared-memory
//     ring with a 1-cell x/y halo; the next plane is prefetched into registers
//     before the compute and stored after it, so one __syncthreads per plane.
// Identical arithmetic to the formulas (reassociated): parity vs the oracle is
// checked at 1e-5 (fp32) / 1e-12 (fp64) in tests/test_gpu_stencils.py.

#if BLOCK_Z != 1 || TILE_Z != 1 || TILE_X != 1
#error "diff_uvw ZMARCH requires BLOCK_Z == TILE_Z == TILE_X == 1"
#endif

#include "diff_uvw_flux.cuh"

#define KL_TYT (BLOCK_Y * TILE_Y)
#define KL_SW (BLOCK_X + 2)
#define KL_SH (KL_TYT + 2)
#define KL_PLANE (KL_SW * KL_SH)
#define KL_FILL ((KL_PLANE + KL_THREADS - 1) / KL_THREADS)


extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, const real* __restrict__ evisc,
         const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh KL_RK3_BUFFERS, const real dxi, const real dyi KL_RK3_SCALARS,
         const int jj, const int kk, const int istart, const int jstart, const int kstart, const int iend,
         const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  extern __shared__ __align__(16) unsigned char kl_smem_raw[];
  real* const ring = reinterpret_cast<real*>(kl_smem_raw);  // [3 slots][4 fields][KL_SH][KL_SW]
  constexpr int FS = KL_PLANE;        // field stride inside a slot
  constexpr int SLOT = 4 * KL_PLANE;  // slot stride

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
  const real* const src[4] = {evisc, u, v, w};

  // Plane fill: element idx of the halo'd tile -> global offset (clamped to the ghost box).
  long long goff[KL_FILL];
  int soff[KL_FILL];
#pragma unroll
  for (int n = 0; n < KL_FILL; ++n) {
    const int idx = tid + n * KL_THREADS;
    const int r = idx / KL_SW, col = idx - r * KL_SW;
    const int gj = min(j0 - 1 + r, jend);
    const int gi = min(i0 - 1 + col, iend);
    goff[n] = gi + static_cast<long long>(gj) * KL_JJ;
    soff[n] = idx < KL_PLANE ? idx : -1;
  }
  auto load_plane = [&](int kp, real (&buf)[KL_FILL][4]) {
    const long long kofs = static_cast<long long>(kp) * KL_KK;
#pragma unroll
    for (int n = 0; n < KL_FILL; ++n)
#pragma unroll
      for (int f = 0; f < 4; ++f) buf[n][f] = soff[n] >= 0 ? src[f][goff[n] + kofs] : real(0);
  };
  auto store_plane = [&](int kp, const real (&buf)[KL_FILL][4]) {
    real* slot = ring + (kp % 3) * SLOT;
#pragma unroll
    for (int n = 0; n < KL_FILL; ++n)
      if (soff[n] >= 0) {
#pragma unroll
        for (int f = 0; f < 4; ++f) slot[f * FS + soff[n]] = buf[n][f];
      }
  };

  const real c2x = real(2) * dxi * dxi;
  const real c2y = real(2) * dyi * dyi;
  const real qsx = real(0.25) * dxi, qsy = real(0.25) * dyi;
  const int lj0 = threadIdx.y * TILE_Y;  // first strip row (tile-local)
  const int col = threadIdx.x + 1;
  const int i = i0 + threadIdx.x;
  DiffCarry carry;
  auto no_store = [](int, real, real, real) {};

  {
    real buf[KL_FILL][4];
    load_plane(k0 - 1, buf);
    store_plane(k0 - 1, buf);
    load_plane(k0, buf);
    store_plane(k0, buf);
  }
  __syncthreads();
  {
    const int kp = k0 - 1;
    const real* p0 = ring + (kp % 3) * SLOT + lj0 * KL_SW + col;
    const real* p1 = ring + ((kp + 1) % 3) * SLOT + lj0 * KL_SW + col;
    diff_step<false, KL_SW>(p0, p1, FS, carry, dxi, dyi, qsx, qsy, c2x, c2y, rhorefh[kp + 1], dzhi[kp + 1],
                            rhoref[kp] * dzi[kp], real(0), real(0), no_store);
  }
  {
    real buf[KL_FILL][4];
    load_plane(k0 + 1, buf);
    store_plane(k0 + 1, buf);
  }

  for (int k = k0; k < k1; ++k) {
    __syncthreads();
    real buf[KL_FILL][4];
    const bool more = k + 2 <= k1;
    if (more) load_plane(k + 2, buf);  // prefetch; stored after the compute
    const real* p0 = ring + (k % 3) * SLOT + lj0 * KL_SW + col;
    const real* p1 = ring + ((k + 1) % 3) * SLOT + lj0 * KL_SW + col;
    const real qfac = real(0.25) * dzi[k] / rhoref[k];
    const real fac_w = real(2) * dzhi[k] / rhorefh[k];
    const long long kofs = static_cast<long long>(k) * KL_KK;
    auto store = [&](int t, real dut, real dvt, real dwt) {
      const int j = j0 + lj0 + t;
      if (i < iend && j < jend) {
        const long long ijk = i + static_cast<long long>(j) * KL_JJ + kofs;
#if KL_RK3
        // centre values of u, v, w at (row t, plane k) in the staged plane
        const real* c = p0 + (t + 1) * KL_SW;
        const real tu = ut[ijk] + dut, tv = vt[ijk] + dvt, tw = wt[ijk] + dwt;
        un[ijk] = c[FS] + rk_bdt * tu;
        vn[ijk] = c[2 * FS] + rk_bdt * tv;
        wn[ijk] = c[3 * FS] + rk_bdt * tw;
        ut[ijk] = rk_a * tu;
        vt[ijk] = rk_a * tv;
        wt[ijk] = rk_a * tw;
#else
        ut[ijk] += dut;
        vt[ijk] += dvt;
        wt[ijk] += dwt;
#endif
      }
    };
    diff_step<true, KL_SW>(p0, p1, FS, carry, dxi, dyi, qsx, qsy, c2x, c2y, rhorefh[k + 1], dzhi[k + 1], rhoref[k] * dzi[k],
                           qfac, fac_w, store);
    if (more) store_plane(k + 2, buf);
  }
}

#undef KL_TYT
#undef KL_SW
#undef KL_SH
#undef KL_PLANE
#undef KL_FILL
