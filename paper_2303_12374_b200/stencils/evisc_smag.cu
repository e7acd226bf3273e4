// evisc_smag — MicroHH diff_smag2 eddy viscosity, neutral Smagorinsky model:
// the squared strain rate 2 S_ij S_ij at cell centres (diagonal terms at the
// centre, every off-diagonal term the mean of its four surrounding edges,
// MicroHH calc_strain2) and evisc = (cs * (dx dy dz)^(1/3))^2 * sqrt(2 S_ij S_ij)
// — the step that produces diff_uvw's evisc.  Restated on the CPU in
// oracle/family_oracle.py:strain2 / evisc_smag.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh) or
// TMA staging (edge-reusing z-march over a shared-memory ring of u / v / w
// planes with a 1-cell halo, evisc_smag_tma.cuh).
// Algorithmic HBM traffic: read u, v, w; write evisc = 4 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"
#include "kl_pack.cuh"

#if STAGING == 1
#error "evisc_smag: DIRECT or TMA staging (no ZMARCH variant)"
#endif

namespace {
template <class T>
__device__ __forceinline__ T sq(T a) { return a * a; }

struct Smag {
  static constexpr int NH = 3, HAS_T = 0;  // halo'd inputs: 0 = u, 1 = v, 2 = w; evisc written
  const real *dzi, *dzhi;
  real dxi, dyi, cs;
  struct Plane {
    real dz, dzh, dzh1, fac;  // dzi[k], dzhi[k], dzhi[k+1], (cs mlen)^2
  };
  __device__ __forceinline__ Plane plane(int k) const {
    const real mlen = cbrt(real(1) / (dxi * dyi * dzi[k]));
    return Plane{dzi[k], dzhi[k], dzhi[k + 1], sq(cs * mlen)};
  }
  // T = real, or a pair of neighbouring cells (kl::f2 / kl::d2) under the TMA march
  template <class T, class A>
  __device__ __forceinline__ T cell(const A& at, const Plane& pl, T) const {
    auto U = [&](int di, int dj, int dk) { return at(0, di, dj, dk); };
    auto V = [&](int di, int dj, int dk) { return at(1, di, dj, dk); };
    auto W = [&](int di, int dj, int dk) { return at(2, di, dj, dk); };
    const T dxi = T(this->dxi), dyi = T(this->dyi);
    struct {
      T dz, dzh, dzh1;
    } p{T(pl.dz), T(pl.dzh), T(pl.dzh1)};
    const T diag = sq((U(1, 0, 0) - U(0, 0, 0)) * dxi) + sq((V(0, 1, 0) - V(0, 0, 0)) * dyi) +
                      sq((W(0, 0, 1) - W(0, 0, 0)) * p.dz);
    // du/dy + dv/dx on the four xy edges around the centre
    const T sxy = sq((U(0, 0, 0) - U(0, -1, 0)) * dyi + (V(0, 0, 0) - V(-1, 0, 0)) * dxi) +
                     sq((U(0, 1, 0) - U(0, 0, 0)) * dyi + (V(0, 1, 0) - V(-1, 1, 0)) * dxi) +
                     sq((U(1, 0, 0) - U(1, -1, 0)) * dyi + (V(1, 0, 0) - V(0, 0, 0)) * dxi) +
                     sq((U(1, 1, 0) - U(1, 0, 0)) * dyi + (V(1, 1, 0) - V(0, 1, 0)) * dxi);
    // du/dz + dw/dx on the four xz edges
    const T sxz = sq((U(0, 0, 0) - U(0, 0, -1)) * p.dzh + (W(0, 0, 0) - W(-1, 0, 0)) * dxi) +
                     sq((U(0, 0, 1) - U(0, 0, 0)) * p.dzh1 + (W(0, 0, 1) - W(-1, 0, 1)) * dxi) +
                     sq((U(1, 0, 0) - U(1, 0, -1)) * p.dzh + (W(1, 0, 0) - W(0, 0, 0)) * dxi) +
                     sq((U(1, 0, 1) - U(1, 0, 0)) * p.dzh1 + (W(1, 0, 1) - W(0, 0, 1)) * dxi);
    // dv/dz + dw/dy on the four yz edges
    const T syz = sq((V(0, 0, 0) - V(0, 0, -1)) * p.dzh + (W(0, 0, 0) - W(0, -1, 0)) * dyi) +
                     sq((V(0, 0, 1) - V(0, 0, 0)) * p.dzh1 + (W(0, 0, 1) - W(0, -1, 1)) * dyi) +
                     sq((V(0, 1, 0) - V(0, 1, -1)) * p.dzh + (W(0, 1, 0) - W(0, 0, 0)) * dyi) +
                     sq((V(0, 1, 1) - V(0, 1, 0)) * p.dzh1 + (W(0, 1, 1) - W(0, 0, 1)) * dyi);
    const T strain2 = T(real(2)) * diag + T(real(0.25)) * (sxy + sxz + syz);
    return T(pl.fac) * kl::sqrt2(strain2);
  }
};

struct GlobalAt {
  const real* f[3];
  __device__ __forceinline__ real operator()(int fi, int di, int dj, int dk) const {
    return f[fi][di + dj * static_cast<long long>(KL_JJ) + dk * static_cast<long long>(KL_KK)];
  }
};
}  // namespace

#if STAGING == 0

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ evisc, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ dzi, const real* __restrict__ dzhi, const real dxi,
         const real dyi, const real cs, const int jj, const int kk, const int istart, const int jstart,
         const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  const Smag tr{dzi, dzhi, dxi, dyi, cs};
  kl::direct_tiles(istart, jstart, kstart, iend, jend, kend, [&](int k) { return tr.plane(k); },
                   [&](long long ijk, const Smag::Plane& p) {
                     evisc[ijk] = tr.cell<real>(GlobalAt{{u + ijk, v + ijk, w + ijk}}, p, real(0));
                   });
}

#else
#include "evisc_smag_tma.cuh"
#endif
