// diff_c — MicroHH diff_smag2 diffusion of a cell-centred scalar with the
// eddy diffusivity evisc / Pr_t (tPri = 1 / Pr_t); restated on the CPU in
// oracle/family_oracle.py:diff_c.  Face diffusivities
// are two-point means of evisc; z faces are weighted by rhorefh * dzhi and
// the divergence divided by rhoref and scaled by dzi.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh).
// Algorithmic HBM traffic: read s, evisc, st; write st = 4 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING != 0
#error "diff_c has the DIRECT staging only"
#endif

namespace {
struct Plane {
  real top, bot;  // rhorefh[k+1] dzhi[k+1] and rhorefh[k] dzhi[k], times dzi[k] / rhoref[k]
};
}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ st, const real* __restrict__ s, const real* __restrict__ evisc,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh, const real dxi, const real dyi, const real tpri, const int jj,
         const int kk, const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  constexpr long long I1 = 1, J1 = KL_JJ, K1 = KL_KK;
  // the 1/2 of the two-point means and 1/Pr_t folded into the metric factors
  const real h = real(0.5) * tpri;
  const real cx = h * dxi * dxi, cy = h * dyi * dyi;
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend,
      [&](int k) {
        const real f = h * dzi[k] / rhoref[k];
        return Plane{f * rhorefh[k + 1] * dzhi[k + 1], f * rhorefh[k] * dzhi[k]};
      },
      [&](long long ijk, const Plane& p) {
        const real* a = s + ijk;
        const real* e = evisc + ijk;
        const real a0 = a[0], e0 = e[0];
        st[ijk] += ((e0 + e[I1]) * (a[I1] - a0) - (e[-I1] + e0) * (a0 - a[-I1])) * cx +
                   ((e0 + e[J1]) * (a[J1] - a0) - (e[-J1] + e0) * (a0 - a[-J1])) * cy +
                   (e0 + e[K1]) * (a[K1] - a0) * p.top - (e[-K1] + e0) * (a0 - a[-K1]) * p.bot;
      });
}
