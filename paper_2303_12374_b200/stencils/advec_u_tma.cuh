// advec_u_tma.cuh — STAGING == TMA variant of advec_u (included by
// advec_u.cu).  Same flux-form z-march as ZMARCH (advec_u_zmarch.cuh), with
// the halo'd u planes fetched by the Tensor Memory Accelerator into a
// shared-memory ring of DEPTH+4 slots (one mbarrier each):
//   * plane k feeds the x/y stencil of step k, plane k+3 feeds the z-window
//     (the u[k+3] of every cell comes from the ring instead of a global load);
//   * one elected thread refills the slot vacated by plane k-1 at the start of
//     step k, so DEPTH planes beyond the ones being read are in flight;
//   * v, w and ut of the next plane are prefetched into registers one step
//     ahead, so their latency overlaps the current plane's compute.
// Requires BLOCK_X % 32 == 0 (warps along x; west fluxes via __shfl_up_sync).

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
constexpr int kTYT = BLOCK_Y * TILE_Y;
// Box width: BLOCK_X + 6 halo columns from a 16-byte aligned x start (TMA
// requires it), rounded to a 16-byte multiple.
constexpr int kBW = (((BLOCK_X + 6) * kS + 16 - kS + 15) / 16) * 16 / kS;
constexpr int kBH = kTYT + 6;
constexpr int kPB = ((kBW * kBH * kS + 127) / 128) * 128;  // bytes per plane slot
constexpr int kPS = kPB / kS;
constexpr int kNS = DEPTH + 4;
constexpr unsigned kTxBytes = static_cast<unsigned>(kBW * kBH * kS);
static_assert(kBW <= 256 && kBH <= 256, "TMA box extents are limited to 256");
}  // namespace

// position of u = 1, jj = 9, kk = 10 (definitions.ARG_LAYOUT["advec_u"])
extern "C" __device__ const int kl_tma_spec[1 + 5] = {1, 1, 9, 10, kBW, kBH};
struct __align__(64) KlTmaParams {
  TmaDesc map[1];
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
  const int xfirst = i0 - 3 + kl::tma_xoff(u);  // tensor x of column i0-3
  const int x0 = xfirst & ~(16 / kS - 1);       // 16-byte aligned box start
  const int cshift = xfirst - x0;
  const real dxi60 = dxi * real(1.0 / 60.0);
  const real dyi60 = dyi * real(1.0 / 60.0);
  constexpr long long K1 = KL_KK;
  constexpr long long J1 = KL_JJ;

  auto slot = [&](int p) { return (p - k0) % kNS; };
  auto issue = [&](int p) {
    unsigned long long* bar = full + slot(p);
    kl::mbar_expect_tx(bar, kTxBytes);
    kl::tma_load_3d(ring + slot(p) * kPS, maps, bar, x0, j0 - 3, p);
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
  const int colofs = (lj0 + 3) * kBW + threadIdx.x + 3 + cshift;  // (i, j0+lj0) inside a plane slot
  long long base[TILE_Y];
  real uq[TILE_Y][7];
  real fz_bot[TILE_Y];
  // next-plane operands (prefetched one step ahead)
  real nv_n0[TILE_Y], nv_n1[TILE_Y], nw_t0[TILE_Y], nw_t1[TILE_Y], nut[TILE_Y];
  real nv_s0, nv_s1;
  const real rh0 = rhorefh[k0];
#pragma unroll
  for (int t = 0; t < TILE_Y; ++t) {
    const int j = min(j0 + lj0 + t, jend - 1);
    base[t] = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
#pragma unroll
    for (int m = 0; m < 6; ++m) uq[t][m] = u[base[t] + (m - 3) * K1];
    const real wb = kl::interp2(w[base[t] - 1], w[base[t]]);
    fz_bot[t] = rh0 * kl::flux5x60(wb, uq[t][0], uq[t][1], uq[t][2], uq[t][3], uq[t][4], uq[t][5]);
    nv_n0[t] = v[base[t] - 1 + J1];
    nv_n1[t] = v[base[t] + J1];
    nw_t0[t] = w[base[t] - 1 + K1];
    nw_t1[t] = w[base[t] + K1];
    nut[t] = col_ok ? ut[base[t]] : real(0);
  }
  nv_s0 = v[base[0] - 1];
  nv_s1 = v[base[0]];

  for (int k = k0; k < k1; ++k) {
    __syncthreads();  // plane k-1's slot is free
    if (tid == 0) {
      const int p = k - 1 + kNS;
      if (k > k0 && p <= kmax) {
        kl::fence_proxy_async_smem();
        issue(p);
      }
    }
    const long long kofs = static_cast<long long>(k - k0) * K1;
    // this plane's operands, then prefetch the next plane's
    real cv_n0[TILE_Y], cv_n1[TILE_Y], cw_t0[TILE_Y], cw_t1[TILE_Y], cut[TILE_Y];
    const real cv_s0 = nv_s0, cv_s1 = nv_s1;
#pragma unroll
    for (int t = 0; t < TILE_Y; ++t) {
      cv_n0[t] = nv_n0[t];
      cv_n1[t] = nv_n1[t];
      cw_t0[t] = nw_t0[t];
      cw_t1[t] = nw_t1[t];
      cut[t] = nut[t];
    }
    if (k + 1 < k1) {
#pragma unroll
      for (int t = 0; t < TILE_Y; ++t) {
        const long long b = base[t] + kofs + K1;
        nv_n0[t] = v[b - 1 + J1];
        nv_n1[t] = v[b + J1];
        nw_t0[t] = w[b - 1 + K1];
        nw_t1[t] = w[b + K1];
        nut[t] = col_ok ? ut[b] : real(0);
      }
      nv_s0 = v[base[0] + kofs + K1 - 1];
      nv_s1 = v[base[0] + kofs + K1];
    }
    if (k < k0 + 3) wait(k);
    wait(k + 3);
    const real* xy = ring + slot(k) * kPS + colofs;    // plane k at (i, j0+lj0)
    const real* zf = ring + slot(k + 3) * kPS + colofs;  // plane k+3
    const real rh_top = rhorefh[k + 1];
    const real zfac60 = dzi[k] / (rhoref[k] * real(60));

    real ucol[TILE_Y + 6];
#pragma unroll
    for (int m = 0; m < TILE_Y + 6; ++m) ucol[m] = xy[(m - 3) * kBW];
    real fy_lo = kl::flux5x60(kl::interp2(cv_s0, cv_s1), ucol[0], ucol[1], ucol[2], ucol[3], ucol[4], ucol[5]);

#pragma unroll
    for (int t = 0; t < TILE_Y; ++t) {
      const real* row = xy + t * kBW;
      real* q = uq[t];
      q[6] = zf[t * kBW];
      const real xm2 = row[-2], xm1 = row[-1], x0v = ucol[t + 3], xp1 = row[1], xp2 = row[2], xp3 = row[3];
      const real fx_e = kl::flux5x60(kl::interp2(x0v, xp1), xm2, xm1, x0v, xp1, xp2, xp3);
      real fx_w = __shfl_up_sync(0xffffffffu, fx_e, 1);
      if (lane == 0) fx_w = kl::flux5x60(kl::interp2(xm1, x0v), row[-3], xm2, xm1, x0v, xp1, xp2);
      const real fy_hi = kl::flux5x60(kl::interp2(cv_n0[t], cv_n1[t]), ucol[t + 1], ucol[t + 2], ucol[t + 3],
                                      ucol[t + 4], ucol[t + 5], ucol[t + 6]);
      const real fz_top = rh_top * kl::flux5x60(kl::interp2(cw_t0[t], cw_t1[t]), q[1], q[2], q[3], q[4], q[5], q[6]);
      const int j = j0 + lj0 + t;
      if (col_ok && j < jend)
        ut[base[t] + kofs] = cut[t] - ((fx_e - fx_w) * dxi60 + (fy_hi - fy_lo) * dyi60 + (fz_top - fz_bot[t]) * zfac60);
      fy_lo = fy_hi;
      fz_bot[t] = fz_top;
#pragma unroll
      for (int m = 0; m < 6; ++m) q[m] = q[m + 1];
    }
  }
}
