// diff_uvw_zmarch.cuh — STAGING == ZMARCH variant of diff_uvw (included by
// diff_uvw.cu).  A block owns a (BLOCK_X*TILE_X) x (BLOCK_Y*TILE_Y) column of
// cells and marches up ZCHUNK planes.  evisc, u, v and w are staged plane by
// plane into a 4-slot shared-memory ring (1-cell x/y halo): the stencil
// reads planes k-1, k, k+1 while plane k+2's slot is being refilled, so one
// __syncthreads per plane is enough.  Every field value is fetched from HBM
// once per block (plus the 2 z-halo planes of the chunk); all 40+ neighbour
// reads per cell are shared-memory loads.

#if BLOCK_Z != 1 || TILE_Z != 1
#error "ZMARCH requires BLOCK_Z == 1 and TILE_Z == 1"
#endif

#define KL_TXT (BLOCK_X * TILE_X)
#define KL_TYT (BLOCK_Y * TILE_Y)
#define KL_SW (KL_TXT + 2)
#define KL_SH (KL_TYT + 2)
#define KL_PLANE (KL_SW * KL_SH)
#define KL_SLOTS 4

namespace {

// Shared-memory accessor: ring slot of plane k+dk, local (li, lj) + (di, dj).
struct SmemAcc {
  const real* s;  // &ring[field 0][slot of plane k][lj+1][li+1]
  const real* s_lo;  // same, slot of plane k-1
  const real* s_hi;  // same, slot of plane k+1
  __device__ __forceinline__ real operator()(int field, int di, int dj, int dk) const {
    const real* p = dk < 0 ? s_lo : (dk > 0 ? s_hi : s);
    return p[field * (KL_SLOTS * KL_PLANE) + dj * KL_SW + di];
  }
};

}  // namespace

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, const real* __restrict__ evisc,
         const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh, const real dxi, const real dyi, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend, const int kend) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  extern __shared__ __align__(16) unsigned char kl_smem_raw[];
  real* const ring = reinterpret_cast<real*>(kl_smem_raw);  // [4 fields][4 slots][KL_SH][KL_SW]

  const unsigned nbx = kl::ceil_div(iend - istart, KL_TXT);
  const unsigned nby = kl::ceil_div(jend - jstart, KL_TYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * KL_TXT;
  const int j0 = jstart + by * KL_TYT;
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  const real* const src[4] = {evisc, u, v, w};

  auto fill = [&](int kp) {
    const long long kofs = static_cast<long long>(kp) * KL_KK;
    const int slot = kp & (KL_SLOTS - 1);
    for (int idx = tid; idx < KL_PLANE; idx += KL_THREADS) {
      const int r = idx / KL_SW;
      const int c = idx - r * KL_SW;
      const int gj = min(j0 - 1 + r, jend);
      const int gi = min(i0 - 1 + c, iend);
      const long long g = gi + static_cast<long long>(gj) * KL_JJ + kofs;
#pragma unroll
      for (int f = 0; f < 4; ++f) ring[(f * KL_SLOTS + slot) * KL_PLANE + idx] = src[f][g];
    }
  };

  fill(k0 - 1);
  fill(k0);
  for (int k = k0; k < k1; ++k) {
    fill(k + 1);
    __syncthreads();
    const ZFactors zf = z_factors(dzi, dzhi, rhoref, rhorefh, k);
    const int s0 = (k & (KL_SLOTS - 1)) * KL_PLANE;
    const int sm = ((k - 1) & (KL_SLOTS - 1)) * KL_PLANE;
    const int sp = ((k + 1) & (KL_SLOTS - 1)) * KL_PLANE;
#pragma unroll
    for (int ty = 0; ty < TILE_Y; ++ty) {
      const int lj = kl::tile_index<BLOCK_Y, TILE_Y, CONTIG_Y>(0, threadIdx.y, ty);
#pragma unroll
      for (int tx = 0; tx < TILE_X; ++tx) {
        const int li = kl::tile_index<BLOCK_X, TILE_X, CONTIG_X>(0, threadIdx.x, tx);
        const int local = (lj + 1) * KL_SW + (li + 1);
        const SmemAcc acc{ring + s0 + local, ring + sm + local, ring + sp + local};
        real dut, dvt, dwt;
        diff_uvw_tend(acc, dxi, dyi, zf, dut, dvt, dwt);
        const int i = i0 + li, j = j0 + lj;
        if (i < iend && j < jend) {
          const long long ijk = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k) * KL_KK;
          ut[ijk] += dut;
          vt[ijk] += dvt;
          wt[ijk] += dwt;
        }
      }
    }
  }
}

#undef KL_TXT
#undef KL_TYT
#undef KL_SW
#undef KL_SH
#undef KL_PLANE
#undef KL_SLOTS
