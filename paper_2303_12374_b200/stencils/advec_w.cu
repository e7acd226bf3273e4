// advec_w — MicroHH advec_2i5 w-tendency on the Arakawa-C grid; restated on
// the CPU in oracle/family_oracle.py:advec_w.  w sits
// at (i, j, k-1/2): x faces carry u summed over levels k-1, k; y faces v
// likewise; z faces (at the centres k-1, k) w summed, times rhoref; the
// divergence is divided by rhorefh[k] and scaled by dzhi[k].  Every interior
// level is evaluated (builder decision, as for diff_uvw's wt).
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh) or
// TMA staging (flux-form z-march fed by the Tensor Memory Accelerator,
// advec_family_tma.cuh).
// Algorithmic HBM traffic: read u, v, w, wt; write wt = 5 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING == 1
#error "advec_w: DIRECT or TMA staging (no ZMARCH variant)"
#endif
#define ADV_V 1
#define ADV_W 2
#define ADV_S 3
#define ADV_KIND ADV_W

#if STAGING == 0

namespace {
struct Plane {
  real rho_top, rho_bot, zfac;  // rhoref[k], rhoref[k-1], dzhi[k] / (120 rhorefh[k])
};
}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ wt, const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ rhoref, const real* __restrict__ rhorefh, const real* __restrict__ dzhi,
         const real dxi, const real dyi, const int jj, const int kk, const int istart, const int jstart,
         const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  constexpr long long I1 = 1, J1 = KL_JJ, K1 = KL_KK;
  const real dx120 = dxi * real(1.0 / 120.0), dy120 = dyi * real(1.0 / 120.0);
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend,
      [&](int k) { return Plane{rhoref[k], rhoref[k - 1], dzhi[k] / (rhorefh[k] * real(120))}; },
      [&](long long ijk, const Plane& p) {
        const real* c = w + ijk;
        const real ue = u[ijk + I1 - K1] + u[ijk + I1], uw = u[ijk - K1] + u[ijk];
        const real fx = kl::flux5x60(ue, c[-2], c[-1], c[0], c[1], c[2], c[3]) -
                        kl::flux5x60(uw, c[-3], c[-2], c[-1], c[0], c[1], c[2]);
        const real vn = v[ijk + J1 - K1] + v[ijk + J1], vs = v[ijk - K1] + v[ijk];
        const real fy = kl::flux5x60(vn, c[-2 * J1], c[-J1], c[0], c[J1], c[2 * J1], c[3 * J1]) -
                        kl::flux5x60(vs, c[-3 * J1], c[-2 * J1], c[-J1], c[0], c[J1], c[2 * J1]);
        const real wtop = c[0] + c[K1], wbot = c[-K1] + c[0];
        const real fz = p.rho_top * kl::flux5x60(wtop, c[-2 * K1], c[-K1], c[0], c[K1], c[2 * K1], c[3 * K1]) -
                        p.rho_bot * kl::flux5x60(wbot, c[-3 * K1], c[-2 * K1], c[-K1], c[0], c[K1], c[2 * K1]);
        wt[ijk] -= fx * dx120 + fy * dy120 + fz * p.zfac;
      });
}

#else
#include "advec_family_tma.cuh"
#endif
