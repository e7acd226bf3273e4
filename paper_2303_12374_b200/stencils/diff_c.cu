// diff_c — MicroHH diff_smag2 diffusion of a cell-centred scalar with the
// eddy diffusivity evisc / Pr_t (tPri = 1 / Pr_t); restated on the CPU in
// oracle/family_oracle.py:diff_c.  Face diffusivities
// are two-point means of evisc; z faces are weighted by rhorefh * dzhi and
// the divergence divided by rhoref and scaled by dzi.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh) or
// TMA staging (z-march over a shared-memory ring of s / evisc planes with a
// 1-cell halo, kl_plane_tma.cuh); one cell formula serves both.
// Algorithmic HBM traffic: read s, evisc, st; write st = 4 words per cell.

#include "kl_common.cuh"
#include "kl_direct.cuh"
#include "kl_pack.cuh"

#if STAGING == 1
#error "diff_c: DIRECT or TMA staging (no ZMARCH variant)"
#endif

namespace {
struct DiffC {
  static constexpr int NH = 2, HAS_T = 1;  // halo'd inputs: 0 = s, 1 = evisc; st read-modify-written
  const real *dzi, *dzhi, *rhoref, *rhorefh;
  real h, cx, cy;  // 1/2 of the two-point means x 1/Pr_t folded into the metric factors
  struct Plane {
    real top, bot;  // rhorefh[k+1] dzhi[k+1] and rhorefh[k] dzhi[k], times h dzi[k] / rhoref[k]
  };
  __device__ __forceinline__ Plane plane(int k) const {
    const real f = h * dzi[k] / rhoref[k];
    return Plane{f * rhorefh[k + 1] * dzhi[k + 1], f * rhorefh[k] * dzhi[k]};
  }
  // at(f, di, dj, dk): field f at the offset from the cell; T = real, or a
  // pair of neighbouring cells (kl::f2 / kl::d2) under the TMA march
  template <class T, class A>
  __device__ __forceinline__ T cell(const A& at, const Plane& p, T t_old) const {
    const T a0 = at(0, 0, 0, 0), e0 = at(1, 0, 0, 0);
    return t_old +
           ((e0 + at(1, 1, 0, 0)) * (at(0, 1, 0, 0) - a0) - (at(1, -1, 0, 0) + e0) * (a0 - at(0, -1, 0, 0))) * T(cx) +
           ((e0 + at(1, 0, 1, 0)) * (at(0, 0, 1, 0) - a0) - (at(1, 0, -1, 0) + e0) * (a0 - at(0, 0, -1, 0))) * T(cy) +
           (e0 + at(1, 0, 0, 1)) * (at(0, 0, 0, 1) - a0) * T(p.top) -
           (at(1, 0, 0, -1) + e0) * (a0 - at(0, 0, 0, -1)) * T(p.bot);
  }
};

struct GlobalAt {
  const real* f[2];
  __device__ __forceinline__ real operator()(int fi, int di, int dj, int dk) const {
    return f[fi][di + dj * static_cast<long long>(KL_JJ) + dk * static_cast<long long>(KL_KK)];
  }
};

__device__ __forceinline__ DiffC make_traits(const real* dzi, const real* dzhi, const real* rhoref,
                                             const real* rhorefh, real dxi, real dyi, real tpri) {
  const real h = real(0.5) * tpri;
  return DiffC{dzi, dzhi, rhoref, rhorefh, h, h * dxi * dxi, h * dyi * dyi};
}
}  // namespace

#if STAGING == 0

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ st, const real* __restrict__ s, const real* __restrict__ evisc,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh, const real dxi, const real dyi, const real tpri, const int jj,
         const int kk, const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  const DiffC tr = make_traits(dzi, dzhi, rhoref, rhorefh, dxi, dyi, tpri);
  kl::direct_tiles(istart, jstart, kstart, iend, jend, kend, [&](int k) { return tr.plane(k); },
                   [&](long long ijk, const DiffC::Plane& p) {
                     st[ijk] = tr.cell<real>(GlobalAt{{s + ijk, evisc + ijk}}, p, st[ijk]);
                   });
}

#else
#include "kl_plane_tma.cuh"

// positions: st 0, s 1, evisc 2, jj 10, kk 11 (definitions.ARG_LAYOUT["diff_c"]); maps: s, evisc, st
extern "C" __device__ const int kl_tma_spec[1 + 5 * 3] = {3, 1, 10, 11, ps::kBW, ps::kBH, 2, 10, 11, ps::kBW, ps::kBH,
                                                          0, 10, 11, ps::kTW, ps::kTYT};
struct __align__(64) KlTmaParams {
  TmaDesc map[3];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ st, const real* __restrict__ s, const real* __restrict__ evisc,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh, const real dxi, const real dyi, const real tpri, const int jj,
         const int kk, const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  const DiffC tr = make_traits(dzi, dzhi, rhoref, rhorefh, dxi, dyi, tpri);
  const real* const hp[2] = {s, evisc};
  ps::march(tr, st, &tma.map[0], istart, jstart, kstart, iend, jend, kend, hp);
}
#endif
