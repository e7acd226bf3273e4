// advec_u — MicroHH advec_2i5 u-tendency: 2nd-order advection with
// 5th-order upwind face interpolation on an Arakawa-C grid (SURVEY.md
// Appendix A.2; restated on the CPU in oracle/stencil_oracle.py:advec_u).
//
//   ut -= dxi (Fx[i+1/2] - Fx[i-1/2]) + dyi (Fy[j+1/2] - Fy[j-1/2])
//         + dzi[k]/rhoref[k] (Fz[k+1/2] - Fz[k-1/2])
//   F  = vel * interp6_ws(u...) - |vel| * interp5_ws(u...)
//
// Signature follows MicroHH's advec_u_g (jj/kk pitches, istart..kend bounds),
// so the problem size of the reference KernelDefinition is
// (iend-istart, jend-jstart, kend-kstart) over args 14..16 minus 11..13.
// Algorithmic HBM traffic: read u, v, w, ut; write ut = 5 words per cell.
//
// Variant selected by STAGING (a B200 knob added to the Table-2 space):
//   0  direct: every thread covers a TILE_X*TILE_Y*TILE_Z tile with global
//      loads (the paper's kernel; neighbours come from L1/L2);
//   1  ZMARCH: flux-form z-march; every face flux evaluated once (z carried,
//      y reused along a TILE_Y strip, x via warp shuffles); u planes staged
//      through registers into shared memory (advec_u_zmarch.cuh);
//   2  TMA: the same compute with u planes staged by the Tensor Memory
//      Accelerator DEPTH planes ahead (advec_u_tma.cuh).

#include "kl_common.cuh"

#ifndef STAGING
#define STAGING 0
#endif

// KL_PEER (kernel advec_u_peer): the z-slab halo fused into the TMA staging,
// as diff_uvw_peer (diff_uvw.cu) — planes p < peer_klo of u (the chunk
// prologue's loads) come from u_lo, planes p >= peer_khi of u and w (the
// rings) from u_hi / w_hi, at the neighbour's plane p + peer_shift_lo/hi.
// (w_lo is never read: w's reach is one plane up.)
#ifndef KL_PEER
#define KL_PEER 0
#endif
#if KL_PEER
#if STAGING != 2
#error "KL_PEER (advec_u_peer) reads the neighbours' planes in the TMA staging only"
#endif
#define KL_PEER_BUFFERS                                                                                \
  , const real* __restrict__ u_lo, const real* __restrict__ w_lo, const real* __restrict__ u_hi,     \
      const real* __restrict__ w_hi
#define KL_PEER_SCALARS , const int peer_klo, const int peer_khi, const int peer_shift_lo, const int peer_shift_hi
#else
#define KL_PEER_BUFFERS
#define KL_PEER_SCALARS
#endif
// argument positions (definitions.ARG_LAYOUT): 7 buffers (+4 peer), dxi, dyi (+4 peer scalars), jj, kk
#define KL_POS_JJ (9 + 8 * KL_PEER)
#define KL_POS_KK (KL_POS_JJ + 1)

namespace {

template <bool kTrap>
__device__ __forceinline__ void check_pitch(int jj, int kk) {
  if (kTrap && (jj != KL_JJ || kk != KL_KK)) __trap();
}

// One cell of the direct variant.  xy/z scale factors are hoisted by the caller.
__device__ __forceinline__ void advec_u_cell(real* __restrict__ ut, const real* __restrict__ u,
                                             const real* __restrict__ v, const real* __restrict__ w,
                                             long long ijk, real dxi60, real dyi60, real rh_top, real rh_bot,
                                             real zfac60) {
  constexpr long long I1 = 1, I2 = 2, I3 = 3;
  constexpr long long J1 = KL_JJ, J2 = 2LL * KL_JJ, J3 = 3LL * KL_JJ;
  constexpr long long K1 = KL_KK, K2 = 2LL * KL_KK, K3 = 3LL * KL_KK;
  const real* __restrict__ c = u + ijk;

  const real ue = kl::interp2(c[0], c[I1]);
  const real uw = kl::interp2(c[-I1], c[0]);
  const real fx = kl::flux5x60(ue, c[-I2], c[-I1], c[0], c[I1], c[I2], c[I3]) -
                  kl::flux5x60(uw, c[-I3], c[-I2], c[-I1], c[0], c[I1], c[I2]);

  const real vn = kl::interp2(v[ijk - I1 + J1], v[ijk + J1]);
  const real vs = kl::interp2(v[ijk - I1], v[ijk]);
  const real fy = kl::flux5x60(vn, c[-J2], c[-J1], c[0], c[J1], c[J2], c[J3]) -
                  kl::flux5x60(vs, c[-J3], c[-J2], c[-J1], c[0], c[J1], c[J2]);

  const real wtop = kl::interp2(w[ijk - I1 + K1], w[ijk + K1]);
  const real wbot = kl::interp2(w[ijk - I1], w[ijk]);
  const real fz = rh_top * kl::flux5x60(wtop, c[-K2], c[-K1], c[0], c[K1], c[K2], c[K3]) -
                  rh_bot * kl::flux5x60(wbot, c[-K3], c[-K2], c[-K1], c[0], c[K1], c[K2]);

  ut[ijk] -= fx * dxi60 + fy * dyi60 + fz * zfac60;
}

}  // namespace

#if STAGING == 0

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
         const real* __restrict__ dzi, const real dxi, const real dyi, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend,
         const int kend) {
  check_pitch<true>(jj, kk);
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  const unsigned nbx = kl::ceil_div(iend - istart, BLOCK_X * TILE_X);
  const unsigned nby = kl::ceil_div(jend - jstart, BLOCK_Y * TILE_Y);
  const unsigned nbz = kl::ceil_div(kend - kstart, BLOCK_Z * TILE_Z);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const real dxi60 = dxi * real(1.0 / 60.0);
  const real dyi60 = dyi * real(1.0 / 60.0);

  KL_UNROLL_Z
  for (int tz = 0; tz < TILE_Z; ++tz) {
    const int k = kstart + kl::tile_index<BLOCK_Z, TILE_Z, CONTIG_Z>(bz, threadIdx.z, tz);
    if (k >= kend) continue;
    const real rh_top = rhorefh[k + 1];
    const real rh_bot = rhorefh[k];
    const real zfac60 = dzi[k] / (rhoref[k] * real(60));
    KL_UNROLL_Y
    for (int ty = 0; ty < TILE_Y; ++ty) {
      const int j = jstart + kl::tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(by, threadIdx.y, ty);
      if (j >= jend) continue;
      KL_UNROLL_X
      for (int tx = 0; tx < TILE_X; ++tx) {
        const int i = istart + kl::tile_index<BLOCK_X, TILE_X, CONTIG_X>(bx, threadIdx.x, tx);
        if (i >= iend) continue;
        const long long ijk = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k) * KL_KK;
        advec_u_cell(ut, u, v, w, ijk, dxi60, dyi60, rh_top, rh_bot, zfac60);
      }
    }
  }
}

#elif STAGING == 1
#include "advec_u_zmarch.cuh"
#else
#include "advec_u_tma.cuh"
#endif
