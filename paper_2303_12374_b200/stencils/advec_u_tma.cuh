// advec_u_tma.cuh — STAGING == TMA variant of advec_u (included by
// advec_u.cu).  Same flux-form z-march as ZMARCH (advec_u_zmarch.cuh), with
// every operand fetched by the Tensor Memory Accelerator into a shared-memory
// ring of DEPTH+4 slots (one mbarrier each).  Slot p holds plane p of
//   * u with a 3-cell x/y halo — plane k feeds the x/y stencil of step k and
//     plane k+3 the z-window (so u[k+3] of every cell comes from the ring);
//   * v (columns i-1..i, rows j..j+1), w (columns i-1..i) and ut (no halo):
//     step k reads v and ut of plane k and w of plane k+1;
// so the compute warps issue no global loads, only the final ut stores.  One
// elected thread refills the slot vacated by plane k-1 at the start of step
// k, keeping DEPTH planes beyond the ones being read in flight.  Box starts
// are rounded down to 16-byte aligned x (TMA requires it).  Requires
// BLOCK_X % 32 == 0 (warps along x; west fluxes via __shfl_up_sync).

#if BLOCK_Z != 1 || TILE_Z != 1 || TILE_X != 1
#error "advec_u TMA requires BLOCK_Z == TILE_Z == TILE_X == 1"
#endif
#if BLOCK_X % 32 != 0
#error "advec_u TMA requires BLOCK_X to be a multiple of the warp size"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif

#include "kl_tma.cuh"

namespace {
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;
constexpr int kTYT = BLOCK_Y * TILE_Y;
constexpr int kBW = (((BLOCK_X + 6) * kS + 16 - kS + 15) / 16) * 16 / kS;  // u: 3-halo + alignment slack
constexpr int kBH = kTYT + 6;
constexpr int kVW = (((BLOCK_X + 1) * kS + 16 - kS + 15) / 16) * 16 / kS;  // v, w: column i-1 + slack
constexpr int kTW = ((BLOCK_X * kS + 16 - kS + 15) / 16) * 16 / kS;        // ut: no halo
constexpr int kUB = ((kBW * kBH * kS + 127) / 128) * 128;
constexpr int kVB = ((kVW * (kTYT + 1) * kS + 127) / 128) * 128;
constexpr int kWB = ((kVW * kTYT * kS + 127) / 128) * 128;
constexpr int kTB = ((kTW * kTYT * kS + 127) / 128) * 128;
constexpr int kPB = kUB + kVB + kWB + kTB;  // bytes per plane slot
constexpr int kPS = kPB / kS;
constexpr int kVO = kUB / kS, kWO = (kUB + kVB) / kS, kTO = (kUB + kVB + kWB) / kS;  // field offsets in a slot
constexpr int kNS = DEPTH + 4;
constexpr unsigned kTxBytes =
    static_cast<unsigned>((kBW * kBH + kVW * (kTYT + 1) + kVW * kTYT + kTW * kTYT) * kS);
static_assert(kBW <= 256 && kBH <= 256, "TMA box extents are limited to 256");
}  // namespace

// positions: ut=0 u=1 v=2 w=3, jj=9 kk=10 (definitions.ARG_LAYOUT["advec_u"])
extern "C" __device__ const int kl_tma_spec[1 + 5 * 4] = {4, 1, 9, 10, kBW, kBH, 2, 9, 10, kVW, kTYT + 1,
                                                          3, 9, 10, kVW, kTYT, 0, 9, 10, kTW, kTYT};
struct __align__(64) KlTmaParams {
  TmaDesc map[4];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
         const real* __restrict__ dzi, const real dxi, const real dyi, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  // param-space address of the descriptors (__grid_constant__: no local copy)
  const TmaDesc* const maps = &tma.map[0];
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* sbase = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sbase);
  real* const ring = reinterpret_cast<real*>(sbase + 128);  // [kNS][kPS]

  const unsigned nbx = kl::ceil_div(iend - istart, BLOCK_X);
  const unsigned nby = kl::ceil_div(jend - jstart, kTYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * BLOCK_X;
  const int j0 = jstart + by * kTYT;
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int kmax = k1 + 2;  // last plane the z-window reads
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  const int lane = threadIdx.x & 31;
  const int xu = i0 - 3 + kl::tma_xoff(u);  // tensor x of column i0-3
  const int xu0 = xu & ~(kE - 1);            // 16-byte aligned box starts
  const int xv0 = (xu + 2) & ~(kE - 1);      // column i0-1
  const int xt0 = (xu + 3) & ~(kE - 1);      // column i0
  const int ushift = xu - xu0, vshift = xu + 2 - xv0, tshift = xu + 3 - xt0;
  const real dxi60 = dxi * real(1.0 / 60.0);
  const real dyi60 = dyi * real(1.0 / 60.0);
  constexpr long long K1 = KL_KK;

  auto slot = [&](int p) { return (p - k0) % kNS; };
  auto issue = [&](int p) {
    unsigned long long* bar = full + slot(p);
    real* dst = ring + slot(p) * kPS;
    kl::mbar_expect_tx(bar, kTxBytes);
    kl::tma_load_3d(dst, maps + 0, bar, xu0, j0 - 3, p);
    kl::tma_load_3d(dst + kVO, maps + 1, bar, xv0, j0, p);
    kl::tma_load_3d(dst + kWO, maps + 2, bar, xv0, j0, p);
    kl::tma_load_3d(dst + kTO, maps + 3, bar, xt0, j0, p);
  };
  auto wait = [&](int p) { kl::mbar_wait(full + slot(p), ((p - k0) / kNS) & 1); };

  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) kl::mbar_init(full + s, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    for (int p = k0; p <= min(k0 + kNS - 1, kmax); ++p) issue(p);
  }

  const int i = min(i0 + static_cast<int>(threadIdx.x), iend - 1);
  const bool col_ok = i0 + static_cast<int>(threadIdx.x) < iend;
  const int lj0 = threadIdx.y * TILE_Y;
  const int colofs = (lj0 + 3) * kBW + threadIdx.x + 3 + ushift;  // (i, j0+lj0) in the u box
  const int vofs = lj0 * kVW + threadIdx.x + vshift;             // (i-1, j0+lj0) in the v / w boxes
  const int tofs = lj0 * kTW + threadIdx.x + tshift;             // (i, j0+lj0) in the ut box
  real uq[TILE_Y][7];
  real fz_bot[TILE_Y];
  // planes k0..k0+2 are first read as the x/y plane (k) or the w plane (k+1)
  // of the first steps; every later plane is first read as the z-window
  // plane (k+3) and waited for there
  wait(k0);
  wait(k0 + 1);
  wait(k0 + 2);
  {
    const real* ring0 = ring + slot(k0) * kPS;
    const real rh0 = rhorefh[k0];
#pragma unroll
    for (int t = 0; t < TILE_Y; ++t) {
      const int j = min(j0 + lj0 + t, jend - 1);
      const long long b = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
#pragma unroll
      for (int m = 0; m < 3; ++m) uq[t][m] = u[b + (m - 3) * K1];  // planes below the chunk: not staged
#pragma unroll
      for (int m = 3; m < 6; ++m) uq[t][m] = u[b + (m - 3) * K1];
      const real* wp = ring0 + kWO + vofs + t * kVW;
      const real wb = kl::interp2(wp[0], wp[1]);
      fz_bot[t] = rh0 * kl::flux5x60(wb, uq[t][0], uq[t][1], uq[t][2], uq[t][3], uq[t][4], uq[t][5]);
    }
  }

  for (int k = k0; k < k1; ++k) {
    __syncthreads();  // plane k-1's slot is free
    if (tid == 0) {
      const int p = k - 1 + kNS;
      if (k > k0 && p <= kmax) {
        kl::fence_proxy_async_smem();
        issue(p);
      }
    }
    wait(k + 3);
    const real* sk = ring + slot(k) * kPS;
    const real* xy = sk + colofs;                          // u, plane k at (i, j0+lj0)
    const real* zf = ring + slot(k + 3) * kPS + colofs;    // u, plane k+3
    const real* vp = sk + kVO + vofs;                      // v, plane k at (i-1, j0+lj0)
    const real* wp = ring + slot(k + 1) * kPS + kWO + vofs;  // w, plane k+1 at (i-1, j0+lj0)
    const real* tp = sk + kTO + tofs;                      // ut, plane k
    const real rh_top = rhorefh[k + 1];
    const real zfac60 = dzi[k] / (rhoref[k] * real(60));
    const long long kofs = static_cast<long long>(k) * K1;

    real ucol[TILE_Y + 6];
#pragma unroll
    for (int m = 0; m < TILE_Y + 6; ++m) ucol[m] = xy[(m - 3) * kBW];
    real fy_lo = kl::flux5x60(kl::interp2(vp[0], vp[1]), ucol[0], ucol[1], ucol[2], ucol[3], ucol[4], ucol[5]);

#pragma unroll
    for (int t = 0; t < TILE_Y; ++t) {
      const real* row = xy + t * kBW;
      real* q = uq[t];
      q[6] = zf[t * kBW];
      const real xm2 = row[-2], xm1 = row[-1], x0v = ucol[t + 3], xp1 = row[1], xp2 = row[2], xp3 = row[3];
      const real fx_e = kl::flux5x60(kl::interp2(x0v, xp1), xm2, xm1, x0v, xp1, xp2, xp3);
      real fx_w = __shfl_up_sync(0xffffffffu, fx_e, 1);
      if (lane == 0) fx_w = kl::flux5x60(kl::interp2(xm1, x0v), row[-3], xm2, xm1, x0v, xp1, xp2);
      const real* vn = vp + (t + 1) * kVW;
      const real fy_hi = kl::flux5x60(kl::interp2(vn[0], vn[1]), ucol[t + 1], ucol[t + 2], ucol[t + 3],
                                      ucol[t + 4], ucol[t + 5], ucol[t + 6]);
      const real* wt_ = wp + t * kVW;
      const real fz_top = rh_top * kl::flux5x60(kl::interp2(wt_[0], wt_[1]), q[1], q[2], q[3], q[4], q[5], q[6]);
      const int j = j0 + lj0 + t;
      if (col_ok && j < jend) {
        const long long ijk = i + static_cast<long long>(j) * KL_JJ + kofs;
        ut[ijk] = tp[t * kTW] - ((fx_e - fx_w) * dxi60 + (fy_hi - fy_lo) * dyi60 + (fz_top - fz_bot[t]) * zfac60);
      }
      fy_lo = fy_hi;
      fz_bot[t] = fz_top;
#pragma unroll
      for (int m = 0; m < 6; ++m) q[m] = q[m + 1];
    }
  }
}
