// rk3_uvw — one substep of MicroHH's low-storage third-order Runge-Kutta
// scheme for u, v, w as a separate pass over HBM (the unfused baseline the
// diff_uvw_rk3 epilogue is measured against):
//     a <- a + rk_bdt * at ;  at <- rk_a * at      for (a, at) in (u,ut) (v,vt) (w,wt)
// Restated on the CPU in oracle/family_oracle.py:rk3_uvw.
//
// DIRECT staging (the paper's kernel, every Table-2 knob; kl_direct.cuh).
// Algorithmic HBM traffic: read + write u, v, w, ut, vt, wt = 12 words per cell.
//
// Vector path: with consecutive columns per thread (CONTIG_X, TILE_X >= 2)
// a thread's cells of one row are TILE_X adjacent elements starting at a
// multiple of TILE_X from istart, so when the six fields' row starts are
// aligned to the vector width (always, for the GridLayout pitches; checked
// uniformly: pointers at run time, pitches at compile time) each row of the
// tile is read and written with VA-element vector accesses (VA =
// min(TILE_X, 16 B)) — 12 / VA memory
// instructions per cell instead of 12, which is what keeps an fp32
// elementwise pass on the HBM roofline.  Any other alignment takes the
// scalar loop of direct_tiles.

#include "kl_common.cuh"
#include "kl_direct.cuh"

#if STAGING != 0
#error "rk3_uvw has the DIRECT staging only"
#endif

namespace {
constexpr int kVE = 16 / static_cast<int>(sizeof(real));           // elements per 16 bytes
constexpr int kVA = (CONTIG_X && TILE_X >= 2) ? (TILE_X < kVE ? TILE_X : kVE) : 1;

template <int N>
struct __align__(N * sizeof(real)) Vec {
  real v[N];
};

// every row start (i = istart) of the field is VA-element aligned: the
// pointer at istart, and the row / plane pitches (compile-time) in VA steps
__device__ __forceinline__ bool aligned_rows(const void* p, int istart) {
  return KL_JJ % kVA == 0 && KL_KK % kVA == 0 &&
         ((reinterpret_cast<unsigned long long>(p) + static_cast<unsigned long long>(istart) * sizeof(real)) %
          (kVA * sizeof(real))) == 0;
}

struct Rk3 {
  real *ut, *vt, *wt, *u, *v, *w;
  real rk_a, rk_bdt;

  __device__ __forceinline__ void cell(long long ijk) const {
    const real tu = ut[ijk], tv = vt[ijk], tw = wt[ijk];
    u[ijk] += rk_bdt * tu;
    v[ijk] += rk_bdt * tv;
    w[ijk] += rk_bdt * tw;
    ut[ijk] = rk_a * tu;
    vt[ijk] = rk_a * tv;
    wt[ijk] = rk_a * tw;
  }

  template <int VA>
  __device__ __forceinline__ void vec(real* a, real* at, long long ijk) const {
    using V = Vec<VA>;
    V t = *reinterpret_cast<const V*>(at + ijk);
    V x = *reinterpret_cast<const V*>(a + ijk);
#pragma unroll
    for (int q = 0; q < VA; ++q) {
      x.v[q] += rk_bdt * t.v[q];
      t.v[q] *= rk_a;
    }
    *reinterpret_cast<V*>(a + ijk) = x;
    *reinterpret_cast<V*>(at + ijk) = t;
  }

  // the direct_tiles loop with each row of TILE_X consecutive cells in VA-wide
  // chunks (a chunk that crosses iend falls back to scalar cells)
  template <int VA>
  __device__ __forceinline__ void tiles(int istart, int jstart, int kstart, int iend, int jend, int kend) const {
    const unsigned nbx = kl::ceil_div(iend - istart, BLOCK_X * TILE_X);
    const unsigned nby = kl::ceil_div(jend - jstart, BLOCK_Y * TILE_Y);
    const unsigned nbz = kl::ceil_div(kend - kstart, BLOCK_Z * TILE_Z);
    int bx, by, bz;
    kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
    const int i0 = istart + kl::tile_index<BLOCK_X, TILE_X, true>(bx, threadIdx.x, 0);
    KL_UNROLL_Z
    for (int tz = 0; tz < TILE_Z; ++tz) {
      const int k = kstart + kl::tile_index<BLOCK_Z, TILE_Z, CONTIG_Z>(bz, threadIdx.z, tz);
      if (k >= kend) continue;
      KL_UNROLL_Y
      for (int ty = 0; ty < TILE_Y; ++ty) {
        const int j = jstart + kl::tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(by, threadIdx.y, ty);
        if (j >= jend) continue;
        const long long row = static_cast<long long>(j) * KL_JJ + static_cast<long long>(k) * KL_KK;
#pragma unroll
        for (int e = 0; e < TILE_X; e += VA) {
          const int i = i0 + e;
          const long long ijk = i + row;
          if (i + VA <= iend) {
            vec<VA>(u, ut, ijk);
            vec<VA>(v, vt, ijk);
            vec<VA>(w, wt, ijk);
          } else {
#pragma unroll
            for (int q = 0; q < VA; ++q)
              if (i + q < iend) cell(ijk + q);
          }
        }
      }
    }
  }
};
}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, real* __restrict__ u,
         real* __restrict__ v, real* __restrict__ w, const real rk_a, const real rk_bdt, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  const Rk3 r{ut, vt, wt, u, v, w, rk_a, rk_bdt};
  if (kVA > 1 && aligned_rows(ut, istart) && aligned_rows(vt, istart) && aligned_rows(wt, istart) &&
      aligned_rows(u, istart) && aligned_rows(v, istart) && aligned_rows(w, istart)) {
    r.tiles<kVA>(istart, jstart, kstart, iend, jend, kend);
    return;
  }
  kl::direct_tiles(
      istart, jstart, kstart, iend, jend, kend, [](int) { return 0; }, [&](long long ijk, int) { r.cell(ijk); });
}
