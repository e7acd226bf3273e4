// diff_uvw — MicroHH diff_smag2 momentum diffusion: divergence of the
// eddy-viscosity stress tensor for u, v and w in one pass (SURVEY.md
// Appendix A.3; restated in oracle/stencil_oracle.py:diff_uvw).
//
// Signature follows MicroHH's diff_uvw_g: tendencies first, then evisc and
// the velocity fields, the 1-D profiles, grid spacings, pitches and bounds.
// Problem size = (iend-istart, jend-jstart, kend-kstart) from args 18..20
// minus 15..17.  Algorithmic HBM traffic: read evisc, u, v, w, ut, vt, wt;
// write ut, vt, wt = 10 words per cell.
//
// STAGING 0: direct global loads (paper kernel, Table-2 knobs);
// STAGING 1 (ZMARCH): flux-form z-march, planes staged through registers into
//            a shared-memory ring (diff_uvw_zmarch.cuh);
// STAGING 2 (TMA): same compute, planes staged by the Tensor Memory
//            Accelerator DEPTH planes ahead (diff_uvw_tma.cuh).

#include "kl_common.cuh"

#ifndef STAGING
#define STAGING 0
#endif

// KL_RK3 (kernel diff_uvw_rk3): the epilogue fuses the
// MicroHH low-storage RK3 time step into the tendency store.  With the final
// tendency T = t + d of every component,
//     t <- rk_a * T          (the tendency carried into the next substep)
//     next <- cur + rk_bdt * T   (u/v/w of the next substep, double-buffered:
//                                 neighbours still read cur)
// — 13 words per cell instead of diff_uvw (10) + a separate RK3 pass (12).
#ifndef KL_RK3
#define KL_RK3 0
#endif
#if KL_RK3
#define KL_RK3_BUFFERS , real* __restrict__ un, real* __restrict__ vn, real* __restrict__ wn
#define KL_RK3_SCALARS , const real rk_a, const real rk_bdt
#else
#define KL_RK3_BUFFERS
#define KL_RK3_SCALARS
#endif
// KL_PEER (kernel diff_uvw_peer, SURVEY §5's B200 option for the z-slab
// halo): the planes just outside the rank's slab are not exchanged into ghost
// planes first — the TMA loads of every plane p < peer_klo (p >= peer_khi)
// read plane p + peer_shift_lo (p + peer_shift_hi) of the neighbour's field
// through a peer-mapped pointer (CUDA IPC over NVLink), so one launch covers
// the whole slab and the exchange is fused into the stencil's staging.  The
// peer pointers have the local fields' layout; a rank without a neighbour on
// a side passes its own fields and a bound no plane reaches.
#ifndef KL_PEER
#define KL_PEER 0
#endif
#if KL_PEER
#if STAGING != 2
#error "KL_PEER (diff_uvw_peer) reads the neighbours' planes in the TMA staging only"
#endif
#define KL_PEER_BUFFERS                                                                                 \
  , const real* __restrict__ evisc_lo, const real* __restrict__ u_lo, const real* __restrict__ v_lo,  \
      const real* __restrict__ w_lo, const real* __restrict__ evisc_hi, const real* __restrict__ u_hi, \
      const real* __restrict__ v_hi, const real* __restrict__ w_hi
#define KL_PEER_SCALARS , const int peer_klo, const int peer_khi, const int peer_shift_lo, const int peer_shift_hi
#else
#define KL_PEER_BUFFERS
#define KL_PEER_SCALARS
#endif
// argument positions of jj / kk (definitions.ARG_LAYOUT) for the TMA spec:
// 11 buffers (+3 RK3, +8 peer), dxi, dyi (+2 RK3, +4 peer scalars), jj, kk
#define KL_POS_JJ (13 + 5 * KL_RK3 + 12 * KL_PEER)
#define KL_POS_KK (KL_POS_JJ + 1)
// first peer buffer (evisc_lo) and the peer count of the TMA spec
#define KL_POS_PEER (11 + 3 * KL_RK3)

namespace {

struct ZFactors {
  real rh_top, rh_bot;  // rhorefh[k+1], rhorefh[k]
  real dzhi_top, dzhi_bot;  // dzhi[k+1], dzhi[k]
  real fac_uv;  // dzi[k] / rhoref[k]
  real w_top, w_bot;  // rhoref[k]*dzi[k], rhoref[k-1]*dzi[k-1]
  real fac_w;  // 2*dzhi[k] / rhorefh[k]
};

__device__ __forceinline__ ZFactors z_factors(const real* __restrict__ dzi, const real* __restrict__ dzhi,
                                              const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
                                              int k) {
  ZFactors f;
  f.rh_top = rhorefh[k + 1];
  f.rh_bot = rhorefh[k];
  f.dzhi_top = dzhi[k + 1];
  f.dzhi_bot = dzhi[k];
  f.fac_uv = dzi[k] / rhoref[k];
  f.w_top = rhoref[k] * dzi[k];
  f.w_bot = rhoref[k - 1] * dzi[k - 1];
  f.fac_w = real(2) * dzhi[k] / rhorefh[k];
  return f;
}

// Tendency increments of one cell.  `A(f, di, dj, dk)` returns field f
// (0=evisc, 1=u, 2=v, 3=w) at offset (di, dj, dk) from the cell — global
// memory in the DIRECT variant, shared-memory planes in ZMARCH.
template <class Acc>
__device__ __forceinline__ void diff_uvw_tend(const Acc& A, real dxi, real dyi, const ZFactors& z, real& dut,
                                              real& dvt, real& dwt) {
  const real q = real(0.25);
  const real e0 = A(0, 0, 0, 0);
  // ---- ut ----
  {
    const real en = q * (A(0, -1, 0, 0) + e0 + A(0, -1, 1, 0) + A(0, 0, 1, 0));
    const real es = q * (A(0, -1, -1, 0) + A(0, 0, -1, 0) + A(0, -1, 0, 0) + e0);
    const real et = q * (A(0, -1, 0, 0) + e0 + A(0, -1, 0, 1) + A(0, 0, 0, 1));
    const real eb = q * (A(0, -1, 0, -1) + A(0, 0, 0, -1) + A(0, -1, 0, 0) + e0);
    const real u0 = A(1, 0, 0, 0);
    const real tx = (e0 * (A(1, 1, 0, 0) - u0) * dxi - A(0, -1, 0, 0) * (u0 - A(1, -1, 0, 0)) * dxi) * real(2) * dxi;
    const real ty = (en * ((A(1, 0, 1, 0) - u0) * dyi + (A(2, 0, 1, 0) - A(2, -1, 1, 0)) * dxi) -
                     es * ((u0 - A(1, 0, -1, 0)) * dyi + (A(2, 0, 0, 0) - A(2, -1, 0, 0)) * dxi)) * dyi;
    const real tz = (z.rh_top * et * ((A(1, 0, 0, 1) - u0) * z.dzhi_top + (A(3, 0, 0, 1) - A(3, -1, 0, 1)) * dxi) -
                     z.rh_bot * eb * ((u0 - A(1, 0, 0, -1)) * z.dzhi_bot + (A(3, 0, 0, 0) - A(3, -1, 0, 0)) * dxi)) *
                    z.fac_uv;
    dut = tx + ty + tz;
  }
  // ---- vt ----
  {
    const real ee = q * (A(0, 0, -1, 0) + e0 + A(0, 1, -1, 0) + A(0, 1, 0, 0));
    const real ew = q * (A(0, -1, -1, 0) + A(0, -1, 0, 0) + A(0, 0, -1, 0) + e0);
    const real et = q * (A(0, 0, -1, 0) + e0 + A(0, 0, -1, 1) + A(0, 0, 0, 1));
    const real eb = q * (A(0, 0, -1, -1) + A(0, 0, 0, -1) + A(0, 0, -1, 0) + e0);
    const real v0 = A(2, 0, 0, 0);
    const real tx = (ee * ((A(2, 1, 0, 0) - v0) * dxi + (A(1, 1, 0, 0) - A(1, 1, -1, 0)) * dyi) -
                     ew * ((v0 - A(2, -1, 0, 0)) * dxi + (A(1, 0, 0, 0) - A(1, 0, -1, 0)) * dyi)) * dxi;
    const real ty = (e0 * (A(2, 0, 1, 0) - v0) * dyi - A(0, 0, -1, 0) * (v0 - A(2, 0, -1, 0)) * dyi) * real(2) * dyi;
    const real tz = (z.rh_top * et * ((A(2, 0, 0, 1) - v0) * z.dzhi_top + (A(3, 0, 0, 1) - A(3, 0, -1, 1)) * dyi) -
                     z.rh_bot * eb * ((v0 - A(2, 0, 0, -1)) * z.dzhi_bot + (A(3, 0, 0, 0) - A(3, 0, -1, 0)) * dyi)) *
                    z.fac_uv;
    dvt = tx + ty + tz;
  }
  // ---- wt ----
  {
    const real ee = q * (A(0, 0, 0, -1) + e0 + A(0, 1, 0, -1) + A(0, 1, 0, 0));
    const real ew = q * (A(0, -1, 0, -1) + A(0, -1, 0, 0) + A(0, 0, 0, -1) + e0);
    const real en = q * (A(0, 0, 0, -1) + e0 + A(0, 0, 1, -1) + A(0, 0, 1, 0));
    const real es = q * (A(0, 0, -1, -1) + A(0, 0, -1, 0) + A(0, 0, 0, -1) + e0);
    const real w0 = A(3, 0, 0, 0);
    const real tx = (ee * ((A(3, 1, 0, 0) - w0) * dxi + (A(1, 1, 0, 0) - A(1, 1, 0, -1)) * z.dzhi_bot) -
                     ew * ((w0 - A(3, -1, 0, 0)) * dxi + (A(1, 0, 0, 0) - A(1, 0, 0, -1)) * z.dzhi_bot)) * dxi;
    const real ty = (en * ((A(3, 0, 1, 0) - w0) * dyi + (A(2, 0, 1, 0) - A(2, 0, 1, -1)) * z.dzhi_bot) -
                     es * ((w0 - A(3, 0, -1, 0)) * dyi + (A(2, 0, 0, 0) - A(2, 0, 0, -1)) * z.dzhi_bot)) * dyi;
    const real tz = (z.w_top * e0 * (A(3, 0, 0, 1) - w0) - z.w_bot * A(0, 0, 0, -1) * (w0 - A(3, 0, 0, -1))) * z.fac_w;
    dwt = tx + ty + tz;
  }
}

// Global-memory accessor (DIRECT): neighbour offsets fold into immediates.
struct GlobalAcc {
  const real* __restrict__ f[4];
  __device__ __forceinline__ real operator()(int field, int di, int dj, int dk) const {
    return f[field][di + dj * static_cast<long long>(KL_JJ) + dk * static_cast<long long>(KL_KK)];
  }
};

}  // namespace

#if STAGING == 0

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, const real* __restrict__ evisc,
         const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh KL_RK3_BUFFERS KL_PEER_BUFFERS, const real dxi,
         const real dyi KL_RK3_SCALARS KL_PEER_SCALARS,
         const int jj, const int kk, const int istart, const int jstart, const int kstart, const int iend,
         const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  const unsigned nbx = kl::ceil_div(iend - istart, BLOCK_X * TILE_X);
  const unsigned nby = kl::ceil_div(jend - jstart, BLOCK_Y * TILE_Y);
  const unsigned nbz = kl::ceil_div(kend - kstart, BLOCK_Z * TILE_Z);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);

  KL_UNROLL_Z
  for (int tz = 0; tz < TILE_Z; ++tz) {
    const int k = kstart + kl::tile_index<BLOCK_Z, TILE_Z, CONTIG_Z>(bz, threadIdx.z, tz);
    if (k >= kend) continue;
    const ZFactors zf = z_factors(dzi, dzhi, rhoref, rhorefh, k);
    KL_UNROLL_Y
    for (int ty = 0; ty < TILE_Y; ++ty) {
      const int j = jstart + kl::tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(by, threadIdx.y, ty);
      if (j >= jend) continue;
      KL_UNROLL_X
      for (int tx = 0; tx < TILE_X; ++tx) {
        const int i = istart + kl::tile_index<BLOCK_X, TILE_X, CONTIG_X>(bx, threadIdx.x, tx);
        if (i >= iend) continue;
        const long long ijk = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k) * KL_KK;
        const GlobalAcc acc{{evisc + ijk, u + ijk, v + ijk, w + ijk}};
        real dut, dvt, dwt;
        diff_uvw_tend(acc, dxi, dyi, zf, dut, dvt, dwt);
#if KL_RK3
        const real tu = ut[ijk] + dut, tv = vt[ijk] + dvt, tw = wt[ijk] + dwt;
        un[ijk] = u[ijk] + rk_bdt * tu;
        vn[ijk] = v[ijk] + rk_bdt * tv;
        wn[ijk] = w[ijk] + rk_bdt * tw;
        ut[ijk] = rk_a * tu;
        vt[ijk] = rk_a * tv;
        wt[ijk] = rk_a * tw;
#else
        ut[ijk] += dut;
        vt[ijk] += dvt;
        wt[ijk] += dwt;
#endif
      }
    }
  }
}

#elif STAGING == 1
#include "diff_uvw_zmarch.cuh"
#else
#include "diff_uvw_tma.cuh"
#endif
