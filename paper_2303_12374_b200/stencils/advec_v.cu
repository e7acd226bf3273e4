// advec_v — MicroHH advec_2i5 v-tendency (2nd-order advection, 5th-order
// upwind face interpolation) on the Arakawa-C grid; restated on the CPU in
// oracle/family_oracle.py:advec_v.  v sits at
// (i, j-1/2, k): x faces carry u summed over rows j-1, j; y faces v summed
// to the centres j-1, j; z faces w summed over rows j-1, j, times rhorefh.
//
//   vt -= dxi (Fx+ - Fx-) + dyi (Fy+ - Fy-) + dzi[k]/rhoref[k] (Fz+ - Fz-)
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh) or
// TMA staging (flux-form z-march fed by the Tensor Memory Accelerator,
// advec_family_tma.cuh).
// Algorithmic HBM traffic: read u, v, w, vt; write vt = 5 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING == 1
#error "advec_v: DIRECT or TMA staging (no ZMARCH variant)"
#endif
#define ADV_V 1
#define ADV_W 2
#define ADV_S 3
#define ADV_KIND ADV_V

#if STAGING == 0

namespace {
struct Plane {
  real rh_top, rh_bot, zfac;  // rhorefh[k+1], rhorefh[k], dzi[k] / (120 rhoref[k])
};
}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ vt, const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ rhoref, const real* __restrict__ rhorefh, const real* __restrict__ dzi,
         const real dxi, const real dyi, const int jj, const int kk, const int istart, const int jstart,
         const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  constexpr long long I1 = 1, J1 = KL_JJ, K1 = KL_KK;
  // velocities enter as two-point sums: the 1/2 of interp2 is in the 1/120
  const real dx120 = dxi * real(1.0 / 120.0), dy120 = dyi * real(1.0 / 120.0);
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend,
      [&](int k) { return Plane{rhorefh[k + 1], rhorefh[k], dzi[k] / (rhoref[k] * real(120))}; },
      [&](long long ijk, const Plane& p) {
        const real* c = v + ijk;
        const real ue = u[ijk + I1 - J1] + u[ijk + I1], uw = u[ijk - J1] + u[ijk];
        const real fx = kl::flux5x60(ue, c[-2], c[-1], c[0], c[1], c[2], c[3]) -
                        kl::flux5x60(uw, c[-3], c[-2], c[-1], c[0], c[1], c[2]);
        const real vn = c[0] + c[J1], vs = c[-J1] + c[0];
        const real fy = kl::flux5x60(vn, c[-2 * J1], c[-J1], c[0], c[J1], c[2 * J1], c[3 * J1]) -
                        kl::flux5x60(vs, c[-3 * J1], c[-2 * J1], c[-J1], c[0], c[J1], c[2 * J1]);
        const real wt = w[ijk - J1 + K1] + w[ijk + K1], wb = w[ijk - J1] + w[ijk];
        const real fz = p.rh_top * kl::flux5x60(wt, c[-2 * K1], c[-K1], c[0], c[K1], c[2 * K1], c[3 * K1]) -
                        p.rh_bot * kl::flux5x60(wb, c[-3 * K1], c[-2 * K1], c[-K1], c[0], c[K1], c[2 * K1]);
        vt[ijk] -= fx * dx120 + fy * dy120 + fz * p.zfac;
      });
}

#else
#include "advec_family_tma.cuh"
#endif
