// evisc_smag — MicroHH diff_smag2 eddy viscosity, neutral Smagorinsky model:
// the squared strain rate 2 S_ij S_ij at cell centres (diagonal terms at the
// centre, every off-diagonal term the mean of its four surrounding edges,
// MicroHH calc_strain2) and evisc = (cs * (dx dy dz)^(1/3))^2 * sqrt(2 S_ij S_ij)
// — the step that produces diff_uvw's evisc.  Restated on the CPU in
// oracle/family_oracle.py:strain2 / evisc_smag.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh).
// Algorithmic HBM traffic: read u, v, w; write evisc = 4 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING != 0
#error "evisc_smag has the DIRECT staging only"
#endif

namespace {
struct Plane {
  real dz, dzh, dzh1, fac;  // dzi[k], dzhi[k], dzhi[k+1], (cs mlen)^2
};

__device__ __forceinline__ real sq(real a) { return a * a; }
}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ evisc, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ dzi, const real* __restrict__ dzhi, const real dxi,
         const real dyi, const real cs, const int jj, const int kk, const int istart, const int jstart,
         const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  constexpr long long I1 = 1, J1 = KL_JJ, K1 = KL_KK;
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend,
      [&](int k) {
        const real mlen = cbrt(real(1) / (dxi * dyi * dzi[k]));
        return Plane{dzi[k], dzhi[k], dzhi[k + 1], sq(cs * mlen)};
      },
      [&](long long ijk, const Plane& p) {
        const real* U = u + ijk;
        const real* V = v + ijk;
        const real* W = w + ijk;
        const real diag = sq((U[I1] - U[0]) * dxi) + sq((V[J1] - V[0]) * dyi) + sq((W[K1] - W[0]) * p.dz);
        // du/dy + dv/dx on the four xy edges around the centre
        const real sxy = sq((U[0] - U[-J1]) * dyi + (V[0] - V[-I1]) * dxi) +
                         sq((U[J1] - U[0]) * dyi + (V[J1] - V[J1 - I1]) * dxi) +
                         sq((U[I1] - U[I1 - J1]) * dyi + (V[I1] - V[0]) * dxi) +
                         sq((U[I1 + J1] - U[I1]) * dyi + (V[I1 + J1] - V[J1]) * dxi);
        // du/dz + dw/dx on the four xz edges
        const real sxz = sq((U[0] - U[-K1]) * p.dzh + (W[0] - W[-I1]) * dxi) +
                         sq((U[K1] - U[0]) * p.dzh1 + (W[K1] - W[K1 - I1]) * dxi) +
                         sq((U[I1] - U[I1 - K1]) * p.dzh + (W[I1] - W[0]) * dxi) +
                         sq((U[I1 + K1] - U[I1]) * p.dzh1 + (W[I1 + K1] - W[K1]) * dxi);
        // dv/dz + dw/dy on the four yz edges
        const real syz = sq((V[0] - V[-K1]) * p.dzh + (W[0] - W[-J1]) * dyi) +
                         sq((V[K1] - V[0]) * p.dzh1 + (W[K1] - W[K1 - J1]) * dyi) +
                         sq((V[J1] - V[J1 - K1]) * p.dzh + (W[J1] - W[0]) * dyi) +
                         sq((V[J1 + K1] - V[J1]) * p.dzh1 + (W[J1 + K1] - W[K1]) * dyi);
        const real strain2 = real(2) * diag + real(0.25) * (sxy + sxz + syz);
        evisc[ijk] = p.fac * sqrt(strain2);
      });
}
