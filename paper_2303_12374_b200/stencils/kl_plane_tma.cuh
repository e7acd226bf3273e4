// kl_plane_tma.cuh — TMA z-march for the point-wise 1-halo stencils of the
// family (diff_c, evisc_smag; STAGING == TMA).  The including kernel provides
//   struct Traits { static constexpr int NH, HAS_T;         // halo'd inputs, RMW output?
//                   struct Plane; Plane plane(int k) const;   // per-level factors
//                   template <class A> real cell(const A& at, const Plane&, real t_old) const; };
// exports kl_tma_spec with the NH halo'd inputs first and (HAS_T) the output
// last, and calls ps::march from its entry point.
//
// A ring of DEPTH+3 shared-memory slots holds, per plane p, the NH input
// fields with a 1-cell x/y halo (and the output's pre-launch plane when the
// kernel reads-modifies-writes it); step k reads planes k-1, k, k+1 and one
// elected thread refills the slot plane k-2 vacated, DEPTH planes ahead, each
// slot completing on its own mbarrier.  Threads evaluate the DIRECT formula
// of their TILE_X consecutive columns x TILE_Y rows with a shared-memory
// accessor at(f, di, dj, dk) — every neighbour offset an immediate — so the
// compute warps issue no global loads, only the (vectorised, when aligned)
// output stores.

#ifndef KL_PLANE_TMA_CUH
#define KL_PLANE_TMA_CUH

#if BLOCK_Z != 1 || TILE_Z != 1
#error "plane-stencil TMA requires BLOCK_Z == TILE_Z == 1"
#endif
#if TILE_X > 1 && !CONTIG_X
#error "plane-stencil TMA: TILE_X > 1 needs consecutive columns (CONTIG_X)"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif

#include "kl_pack.cuh"
#include "kl_tma.cuh"

namespace ps {
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;
constexpr int kTX = TILE_X, kTY = TILE_Y;
constexpr int kXT = BLOCK_X * kTX;
constexpr int kTYT = BLOCK_Y * kTY;
constexpr int kVA = kTX < kE ? kTX : kE;
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }
constexpr int kBW = rup(kXT + 2 + kE - 1, kE);  // columns i0-1 .. i0+kXT (start rounded down)
constexpr int kBH = kTYT + 2;
constexpr int kTW = rup(kXT + kE - 1, kE);
constexpr int kFS = rup(kBW * kBH * kS, 128) / kS;
constexpr int kTS = rup(kTW * kTYT * kS, 128) / kS;
constexpr int kNS = DEPTH + 3;
static_assert(kBW <= 256 && kBH <= 256, "TMA box extents are limited to 256");
static_assert(kNS <= 16, "mbarriers must fit the 128-byte header");

template <int N>
struct __align__(N * sizeof(real)) Pack {
  real v[N];
};

// shared-memory accessor of one cell: field f at offset (di, dj, dk)
template <int NH>
struct At {
  const real* p[3][NH];  // field f of planes k-1, k, k+1 at the cell
  __device__ __forceinline__ real operator()(int f, int di, int dj, int dk) const {
    return p[dk + 1][f][dj * kBW + di];
  }
};
// the same for two neighbouring cells (columns c, c+1) as a pair: the cell
// formula then runs on kl::f2 (packed FADD2/FMUL2/FFMA2 in fp32) / kl::d2
using P2 = typename kl::pair_of<real>::type;
template <int NH, bool AL>
struct At2 {
  const real* p[3][NH];
  __device__ __forceinline__ P2 operator()(int f, int di, int dj, int dk) const {
    const real* q = p[dk + 1][f] + dj * kBW + di;
    if (AL && (di & 1) == 0) {  // even column of an aligned layout: one 2-element shared load
      const Pack<2> v = *reinterpret_cast<const Pack<2>*>(q);
      return P2(v.v[0], v.v[1]);
    }
    return P2(q[0], q[1]);
  }
};

template <bool AL, class Traits>
__device__ __forceinline__ void march_impl(const Traits& tr, real* __restrict__ out, const TmaDesc* maps, int istart,
                                           int jstart, int kstart, int iend, int jend, int kend,
                                           const real* const (&hp)[Traits::NH]) {
  constexpr int NH = Traits::NH;
  constexpr int kSlot = NH * kFS + (Traits::HAS_T ? kTS : 0);
  constexpr unsigned kTx = static_cast<unsigned>((NH * kBW * kBH + (Traits::HAS_T ? kTW * kTYT : 0)) * kS);
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* sbase = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sbase);
  real* const ring = reinterpret_cast<real*>(sbase + 128);

  const unsigned nbx = kl::ceil_div(iend - istart, kXT);
  const unsigned nby = kl::ceil_div(jend - jstart, kTYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * kXT;
  const int j0 = jstart + by * kTYT;
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  const int lj0 = threadIdx.y * kTY;
  const int cx = kTX * static_cast<int>(threadIdx.x);
  const int ic = i0 + cx;
  // per-field box starts (column i0-1 / i0 rounded down to 16 B) and the
  // offset of (strip row 0, column ic) inside each box
  int xh[NH], hof[NH];
#pragma unroll
  for (int f = 0; f < NH; ++f) {
    const int x = i0 - 1 + kl::tma_xoff(hp[f]);
    xh[f] = x & ~(kE - 1);
    hof[f] = f * kFS + (lj0 + 1) * kBW + (x - xh[f]) + 1 + cx;
  }
  const int xt0 = i0 + kl::tma_xoff(out);
  const int xt = xt0 & ~(kE - 1);
  const int tof = NH * kFS + lj0 * kTW + (xt0 - xt) + cx;
  const bool vec = kVA > 1 && xt0 == xt;

  const int kfirst = k0 - 1;
  auto issue = [&](int slot, int p) {
    unsigned long long* bar = bars + slot;
    real* dst = ring + slot * kSlot;
    kl::mbar_expect_tx(bar, kTx);
#pragma unroll
    for (int f = 0; f < NH; ++f) kl::tma_load_3d(dst + f * kFS, maps + f, bar, xh[f], j0 - 1, p);
    if (Traits::HAS_T) kl::tma_load_3d(dst + NH * kFS, maps + NH, bar, xt, j0, p);
  };
  if (tid == 0) {
    for (int q = 0; q < kNS; ++q) kl::mbar_init(bars + q, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0)
    for (int p = kfirst; p <= min(kfirst + kNS - 1, k1); ++p) issue(p - kfirst, p);
  kl::mbar_wait(bars + 0, 0);  // plane k0-1
  kl::mbar_wait(bars + 1, 0);  // plane k0

  int sm = 0, s0 = 1, s1 = 2 % kNS, sfree = kNS - 1;  // slots of planes k-1, k, k+1, k-2
  unsigned ph1 = 0;
  for (int k = k0; k < k1; ++k) {
    __syncthreads();  // every thread is done with plane k-2's slot
    if (tid == 0 && k > k0) {
      const int p = k - 2 + kNS;
      if (p <= k1) {
        kl::fence_proxy_async_smem();
        issue(sfree, p);
      }
    }
    kl::mbar_wait(bars + s1, ph1);
    const typename Traits::Plane pl = tr.plane(k);
    const real* base[3] = {ring + sm * kSlot, ring + s0 * kSlot, ring + s1 * kSlot};
    const real* tend = ring + s0 * kSlot + tof;
    // (strip row 0, column ic) of this plane in the output: rows are immediate offsets
    real* const orow = out + ic + static_cast<long long>(j0 + lj0) * KL_JJ + static_cast<long long>(k) * KL_KK;
    const real* pb[3][NH];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int f = 0; f < NH; ++f) pb[d][f] = base[d] + hof[f];
#pragma unroll
    for (int t = 0; t < kTY; ++t) {
      const int j = j0 + lj0 + t;
      real o[kTX];
      if (kTX >= 2) {
#pragma unroll
        for (int c = 0; c < kTX; c += 2) {
          At2<NH, AL> at;
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int f = 0; f < NH; ++f) at.p[d][f] = pb[d][f] + (t * kBW + c);
          const P2 t_old = Traits::HAS_T ? P2(tend[t * kTW + c], tend[t * kTW + c + 1]) : P2(real(0));
          const P2 r = tr.template cell<P2>(at, pl, t_old);
          o[c] = r.lo();
          o[c + 1] = r.hi();
        }
      } else {
        At<NH> at;
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int f = 0; f < NH; ++f) at.p[d][f] = pb[d][f] + t * kBW;
        const real t_old = Traits::HAS_T ? tend[t * kTW] : real(0);
        o[0] = tr.template cell<real>(at, pl, t_old);
      }
      if (j < jend) {
        real* dst = orow + t * KL_JJ;
        if (vec && ic + kTX <= iend) {
#pragma unroll
          for (int e = 0; e < kTX; e += kVA) {
            Pack<kVA> pk;
#pragma unroll
            for (int q = 0; q < kVA; ++q) pk.v[q] = o[e + q];
            *reinterpret_cast<Pack<kVA>*>(dst + e) = pk;
          }
        } else {
#pragma unroll
          for (int c = 0; c < kTX; ++c)
            if (ic + c < iend) dst[c] = o[c];
        }
      }
    }
    sfree = sm;
    sm = s0;
    s0 = s1;
    s1 = s1 + 1 == kNS ? 0 : s1 + 1;
    ph1 ^= s1 == 0 ? 1u : 0u;
  }
}

// Aligned layouts (column i0 16-byte aligned in every field — always, for
// GridLayout) read even-column operand pairs with one shared load; any other
// alignment takes the scalar-pair instantiation (uniform branch per launch).
template <class Traits>
__device__ __forceinline__ void march(const Traits& tr, real* __restrict__ out, const TmaDesc* maps, int istart,
                                      int jstart, int kstart, int iend, int jend, int kend,
                                      const real* const (&hp)[Traits::NH]) {
  bool al = kl::tma_xoff(out) == 0;
#pragma unroll
  for (int f = 0; f < Traits::NH; ++f) al = al && kl::tma_xoff(hp[f]) == 0;
  const int i0 = istart;  // block starts are multiples of kXT from istart
  al = al && (i0 & (kE - 1)) == 0;
  if (kTX >= 2 && al)
    march_impl<true>(tr, out, maps, istart, jstart, kstart, iend, jend, kend, hp);
  else
    march_impl<false>(tr, out, maps, istart, jstart, kstart, iend, jend, kend, hp);
}
}  // namespace ps

#endif  // KL_PLANE_TMA_CUH
