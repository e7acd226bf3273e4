// rk3_uvw — one substep of MicroHH's low-storage third-order Runge-Kutta
// scheme for u, v, w as a separate pass over HBM (the unfused baseline the
// diff_uvw_rk3 epilogue is measured against):
//     a <- a + rk_bdt * at ;  at <- rk_a * at      for (a, at) in (u,ut) (v,vt) (w,wt)
// Restated on the CPU in oracle/family_oracle.py:rk3_uvw.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh).
// Algorithmic HBM traffic: read + write u, v, w, ut, vt, wt = 12 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING != 0
#error "rk3_uvw has the DIRECT staging only"
#endif

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, real* __restrict__ u,
         real* __restrict__ v, real* __restrict__ w, const real rk_a, const real rk_bdt, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend, [](int) { return 0; },
      [&](long long ijk, int) {
        const real tu = ut[ijk], tv = vt[ijk], tw = wt[ijk];
        u[ijk] += rk_bdt * tu;
        v[ijk] += rk_bdt * tv;
        w[ijk] += rk_bdt * tw;
        ut[ijk] = rk_a * tu;
        vt[ijk] = rk_a * tv;
        wt[ijk] = rk_a * tw;
      });
}
