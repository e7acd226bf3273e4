// advec_s — MicroHH advec_2i5 tendency of a cell-centred scalar s on the
// Arakawa-C grid; restated on the CPU in oracle/family_oracle.py:advec_s
// (SURVEY.md §8f row 2).  The face velocities are the staggered components
// themselves (u[i], u[i+1], v[j], v[j+1], w[k], w[k+1]) — no interpolation.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh) or
// TMA staging (flux-form z-march fed by the Tensor Memory Accelerator,
// advec_family_tma.cuh).
// Algorithmic HBM traffic: read s, u, v, w, st; write st = 6 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING == 1
#error "advec_s: DIRECT or TMA staging (no ZMARCH variant)"
#endif
#define ADV_V 1
#define ADV_W 2
#define ADV_S 3
#define ADV_KIND ADV_S

#if STAGING == 0

namespace {
struct Plane {
  real rh_top, rh_bot, zfac;  // rhorefh[k+1], rhorefh[k], dzi[k] / (60 rhoref[k])
};
}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ st, const real* __restrict__ s, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
         const real* __restrict__ dzi, const real dxi, const real dyi, const int jj, const int kk, const int istart,
         const int jstart, const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  constexpr long long I1 = 1, J1 = KL_JJ, K1 = KL_KK;
  const real dx60 = dxi * real(1.0 / 60.0), dy60 = dyi * real(1.0 / 60.0);
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend,
      [&](int k) { return Plane{rhorefh[k + 1], rhorefh[k], dzi[k] / (rhoref[k] * real(60))}; },
      [&](long long ijk, const Plane& p) {
        const real* c = s + ijk;
        const real fx = kl::flux5x60(u[ijk + I1], c[-2], c[-1], c[0], c[1], c[2], c[3]) -
                        kl::flux5x60(u[ijk], c[-3], c[-2], c[-1], c[0], c[1], c[2]);
        const real fy = kl::flux5x60(v[ijk + J1], c[-2 * J1], c[-J1], c[0], c[J1], c[2 * J1], c[3 * J1]) -
                        kl::flux5x60(v[ijk], c[-3 * J1], c[-2 * J1], c[-J1], c[0], c[J1], c[2 * J1]);
        const real fz =
            p.rh_top * kl::flux5x60(w[ijk + K1], c[-2 * K1], c[-K1], c[0], c[K1], c[2 * K1], c[3 * K1]) -
            p.rh_bot * kl::flux5x60(w[ijk], c[-3 * K1], c[-2 * K1], c[-K1], c[0], c[K1], c[2 * K1]);
        st[ijk] -= fx * dx60 + fy * dy60 + fz * p.zfac;
      });
}

#else
#include "advec_family_tma.cuh"
#endif
