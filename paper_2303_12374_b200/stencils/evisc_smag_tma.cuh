// evisc_smag_tma.cuh — STAGING == TMA variant of evisc_smag (included by
// evisc_smag.cu): an edge-reusing z-march.  The strain rate sums, per cell,
// the squared shear of its 12 surrounding edges (4 xy, 4 xz, 4 yz) — each
// edge shared by four cells.  Here every edge is evaluated once per thread
// tile and carried:
//   * xy edges of plane k at the (TILE_X+1) x (TILE_Y+1) corners of the tile,
//     summed in x pairs and shared by the rows above/below;
//   * xz / yz edges on the top face k+1/2 of the tile, summed in x / y pairs
//     and carried up the march as the next plane's bottom-face sums.
// u, v, w planes with a 1-cell x/y halo are fetched by TMA DEPTH planes ahead
// into a (DEPTH+2)-slot ring (step k reads planes k and k+1; a prologue
// evaluates the bottom faces of the chunk from planes k0-1, k0), so the
// compute warps issue no global loads, only the evisc stores.  ~3x fewer
// floating-point operations per cell than the per-cell formula.  The
// per-level factors (a cube root each) are evaluated once per 32 levels per
// warp and broadcast by shuffle.  (Handing slots back per warp through
// "empty" mbarriers instead of the per-step __syncthreads was measured
// slower: 397 vs 383 us at 512^3 fp32.)

#if BLOCK_Z != 1 || TILE_Z != 1
#error "evisc_smag TMA requires BLOCK_Z == TILE_Z == 1"
#endif
#if TILE_X > 1 && !CONTIG_X
#error "evisc_smag TMA: TILE_X > 1 needs consecutive columns (CONTIG_X)"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif
#ifndef KL_XSHARE
#define KL_XSHARE 0
#endif
#ifndef KL_SKEL
#define KL_SKEL 0  // diagnostic only (tools/ysplit_probe.py defines): 1 = keep the TMA ring, barriers and
                   // evisc stores, replace the strain-rate arithmetic by one read of u — the data-movement floor
#endif
#if KL_XSHARE && (TILE_X != 1 || BLOCK_X % 32 != 0)
#error "evisc_smag x-edge sharing needs TILE_X == 1 and whole warps along x"
#endif

#include "kl_pack.cuh"
#include "kl_tma.cuh"

namespace {
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;
constexpr int kTX = TILE_X, kTY = TILE_Y;
// KL_XSHARE (xshare knob): lane 31 of every warp is a helper that evaluates
// only the west-face edges of the column after the warp's 31 output columns;
// every lane's east-face edges are its right neighbour's west-face edges (a
// shuffle) instead of a second evaluation — 32 edge evaluations per 31
// columns instead of 62 along x.
constexpr bool kXS = KL_XSHARE != 0;
constexpr int kXT = kXS ? BLOCK_X / 32 * 31 : BLOCK_X * kTX;  // output columns per block
constexpr int kTYT = BLOCK_Y * kTY;
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }
constexpr int kBW = rup(kXT + 2 + kE - 1, kE);  // columns i0-1 .. i0+kXT (start rounded down to 16 B)
constexpr int kBH = kTYT + 2;                    // rows j0-1 .. j0+kTYT
constexpr int kFS = rup(kBW * kBH * kS, 128) / kS;
constexpr int kSlot = 3 * kFS;                   // u, v, w
constexpr int kNS = DEPTH + 2;
constexpr unsigned kTx = static_cast<unsigned>(3 * kBW * kBH * kS);
static_assert(kBW <= 256 && kBH <= 256, "TMA box extents are limited to 256");

template <int N>
struct __align__(N * sizeof(real)) Pack {
  real v[N];
};

// Top-face (k+1/2) edge pair sums of a tile: xz summed over the two x-edges of
// each cell, yz over the two y-edges.  Carried to the next plane.
struct Faces {
  real xz[kTY][kTX], yz[kTY][kTX];
};

// Column pairs (TILE_X >= 2): the same quantities of cells (c, c+1) in
// kl::f2 (packed FADD2/FMUL2/FFMA2, fp32) / kl::d2 (fp64).  Operands of
// even columns are aligned register pairs (one shared load on aligned
// layouts); x-face operands one column to the left, and the x-pair sums of
// edge values, straddle the pairs and stay scalar.
using P2 = typename kl::pair_of<real>::type;
constexpr int kP = kTX / 2 > 0 ? kTX / 2 : 1;
struct Faces2 {
  P2 xz[kTY][kP], yz[kTY][kP];
};
template <bool AL>
__device__ __forceinline__ P2 ld2(const real* q) {
  if (AL) {
    const Pack<2> v = *reinterpret_cast<const Pack<2>*>(q);
    return P2(v.v[0], v.v[1]);
  }
  return P2(q[0], q[1]);
}
// x-pair sums s[c] = e[c] + e[c+1] (c = 0..kTX-1) of kTX+1 edge values held
// as kP pairs + the last one, returned as pairs
__device__ __forceinline__ void xpair_sums(const P2 (&e)[kP], real last, P2 (&s)[kP]) {
#pragma unroll
  for (int p = 0; p < kP; ++p) {
    const real next = p + 1 < kP ? e[p + 1].lo() : last;
    s[p] = P2(e[p].lo() + e[p].hi(), e[p].hi() + next);
  }
}

// Per-level factors of the march (dzi[k], dzhi[k+1], the squared Smagorinsky
// length (cs * mlen)^2 — a cube root per level): lane l of every warp
// evaluates them for level k+l once per 32 steps, the steps in between read
// them with one shuffle each instead of every thread recomputing them.
struct Levels {
  real dz, dzh1, fac;
};
struct LevelCache {
  real dz = 0, dzh1 = 0, fac = 0;
  __device__ __forceinline__ Levels at(int k, int k0, int k1, int lane, const real* dzi, const real* dzhi,
                                       real dxi, real dyi, real cs) {
    const int r = (k - k0) & 31;
    if (r == 0) {  // warp-uniform
      const int kq = min(k + lane, k1 - 1);
      dz = dzi[kq];
      dzh1 = dzhi[kq + 1];
      const real mlen = cbrt(real(1) / (dxi * dyi * dz));
      fac = (cs * mlen) * (cs * mlen);
    }
    Levels l;
    l.dz = __shfl_sync(0xffffffffu, dz, r);
    l.dzh1 = __shfl_sync(0xffffffffu, dzh1, r);
    l.fac = __shfl_sync(0xffffffffu, fac, r);
    return l;
  }
};

struct EviscTma {
  real* evisc;
  const real *dzi, *dzhi;
  real* ring;
  unsigned long long* bars;
  const TmaDesc* maps;
  real dxi, dyi, cs;
  int j0, k0, k1, tid, iend, jend, ic, lj0;
  bool helper;  // KL_XSHARE: lane 31 evaluates edges only, stores nothing
  int xh[3], hof[3];  // per-field box starts / (strip row 0, column ic) offsets in a slot

  __device__ __forceinline__ void issue(int slot, int p) const {
    unsigned long long* bar = bars + slot;
    real* dst = ring + slot * kSlot;
    kl::mbar_expect_tx(bar, kTx);
#pragma unroll
    for (int f = 0; f < 3; ++f) kl::tma_load_3d(dst + f * kFS, maps + f, bar, xh[f], j0 - 1, p);
  }

  // Top-face edge pair sums from planes k (lo) and k+1 (hi) of u, v, w:
  //   xz edge (i-1/2+a, k+1/2): (u[i+a,k+1]-u[i+a,k]) dzh1 + (w[i+a,k+1]-w[i+a-1,k+1]) dxi
  //   yz edge (j-1/2+b, k+1/2): (v[j+b,k+1]-v[j+b,k]) dzh1 + (w[j+b,k+1]-w[j+b-1,k+1]) dyi
  __device__ __forceinline__ void top_faces(const real* lo, const real* hi, real dzh1, Faces& out) const {
    const real *ul = lo + hof[0], *uh = hi + hof[0], *vl = lo + hof[1], *vh = hi + hof[1], *wh = hi + hof[2];
#pragma unroll
    for (int t = 0; t < kTY; ++t) {
      real ex[kTX + 1];
#pragma unroll
      for (int a = 0; a <= (kXS ? 0 : kTX); ++a) {
        const int o = t * kBW + a;
        const real s = (uh[o] - ul[o]) * dzh1 + (wh[o] - wh[o - 1]) * dxi;
        ex[a] = s * s;
      }
      if constexpr (kXS) ex[1] = __shfl_down_sync(0xffffffffu, ex[0], 1);  // the right neighbour's west edge
#pragma unroll
      for (int c = 0; c < kTX; ++c) out.xz[t][c] = ex[c] + ex[c + 1];
    }
    real ey[kTY + 1][kTX];
#pragma unroll
    for (int b = 0; b <= kTY; ++b)
#pragma unroll
      for (int c = 0; c < kTX; ++c) {
        const int o = b * kBW + c;
        const real s = (vh[o] - vl[o]) * dzh1 + (wh[o] - wh[o - kBW]) * dyi;
        ey[b][c] = s * s;
      }
#pragma unroll
    for (int t = 0; t < kTY; ++t)
#pragma unroll
      for (int c = 0; c < kTX; ++c) out.yz[t][c] = ey[t][c] + ey[t + 1][c];
  }

  template <bool AL>
  __device__ __forceinline__ void top_faces2(const real* lo, const real* hi, real dzh1_, Faces2& out) const {
    const real *ul = lo + hof[0], *uh = hi + hof[0], *vl = lo + hof[1], *vh = hi + hof[1], *wh = hi + hof[2];
    const P2 dzh1(dzh1_), dx(dxi), dy(dyi);
#pragma unroll
    for (int t = 0; t < kTY; ++t) {
      const int o = t * kBW;
      P2 ex[kP];
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        const int a = o + 2 * p;
        const P2 s = kl::fma2(ld2<AL>(uh + a) - ld2<AL>(ul + a), dzh1, (ld2<AL>(wh + a) - ld2<false>(wh + a - 1)) * dx);
        ex[p] = s * s;
      }
      const real sl = (uh[o + kTX] - ul[o + kTX]) * dzh1_ + (wh[o + kTX] - wh[o + kTX - 1]) * dxi;
      xpair_sums(ex, sl * sl, out.xz[t]);
    }
    P2 ey[kTY + 1][kP];
#pragma unroll
    for (int b = 0; b <= kTY; ++b)
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        const int o = b * kBW + 2 * p;
        const P2 s = kl::fma2(ld2<AL>(vh + o) - ld2<AL>(vl + o), dzh1, (ld2<AL>(wh + o) - ld2<AL>(wh + o - kBW)) * dy);
        ey[b][p] = s * s;
      }
#pragma unroll
    for (int t = 0; t < kTY; ++t)
#pragma unroll
      for (int p = 0; p < kP; ++p) out.yz[t][p] = ey[t][p] + ey[t + 1][p];
  }

  template <bool VEC>
  __device__ __forceinline__ void march2() const {
    Faces2 bot;
    kl::mbar_wait(bars + 0, 0);  // plane k0-1
    kl::mbar_wait(bars + 1, 0);  // plane k0
    top_faces2<VEC>(ring, ring + kSlot, dzhi[k0], bot);
    const P2 dx(dxi), dy(dyi), two(real(2)), quarter(real(0.25));

    int sprev = 0, sk = 1, sk1 = 2 % kNS;  // slots of planes k-1, k, k+1
    unsigned ph1 = 0;
    LevelCache lc;
    for (int k = k0; k < k1; ++k) {
      __syncthreads();  // every thread is done with plane k-1's slot
      if (tid == 0) {
        const int p = k - 1 + kNS;
        if (p <= k1) {
          kl::fence_proxy_async_smem();
          issue(sprev, p);
        }
      }
      const Levels lv = lc.at(k, k0, k1, tid & 31, dzi, dzhi, dxi, dyi, cs);
      kl::mbar_wait(bars + sk1, ph1);
      const real* pk = ring + sk * kSlot;
      const real* pk1 = ring + sk1 * kSlot;
      const P2 fac(lv.fac), dz(lv.dz);
      Faces2 top;
      top_faces2<VEC>(pk, pk1, lv.dzh1, top);

      const real *u = pk + hof[0], *v = pk + hof[1], *w = pk + hof[2], *w1 = pk1 + hof[2];
      P2 pxy[kTY + 1][kP];
#pragma unroll
      for (int t = 0; t <= kTY; ++t) {
        const int o = t * kBW;
        P2 e[kP];
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int a = o + 2 * p;
          const P2 s = kl::fma2(ld2<VEC>(u + a) - ld2<VEC>(u + a - kBW), dy, (ld2<VEC>(v + a) - ld2<false>(v + a - 1)) * dx);
          e[p] = s * s;
        }
        const real sl = (u[o + kTX] - u[o + kTX - kBW]) * dyi + (v[o + kTX] - v[o + kTX - 1]) * dxi;
        xpair_sums(e, sl * sl, pxy[t]);
      }
      real* const orow = evisc + ic + static_cast<long long>(j0 + lj0) * KL_JJ + static_cast<long long>(k) * KL_KK;
#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        real out[kTX];
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int o = t * kBW + 2 * p;
          const P2 ddx = (ld2<false>(u + o + 1) - ld2<VEC>(u + o)) * dx;
          const P2 ddy = (ld2<VEC>(v + o + kBW) - ld2<VEC>(v + o)) * dy;
          const P2 ddz = (ld2<VEC>(w1 + o) - ld2<VEC>(w + o)) * dz;
          const P2 diag = kl::fma2(ddx, ddx, kl::fma2(ddy, ddy, ddz * ddz));
          const P2 off = (pxy[t][p] + pxy[t + 1][p]) + (bot.xz[t][p] + top.xz[t][p]) + (bot.yz[t][p] + top.yz[t][p]);
          const P2 r = fac * kl::sqrt2(kl::fma2(two, diag, quarter * off));
          out[2 * p] = r.lo();
          out[2 * p + 1] = r.hi();
        }
        if (j0 + lj0 + t < jend) {
          real* dst = orow + t * KL_JJ;
          if (VEC && ic + kTX <= iend) {
            constexpr int VA = kTX < kE ? kTX : kE;
#pragma unroll
            for (int e = 0; e < kTX; e += VA) {
              Pack<VA> pk;
#pragma unroll
              for (int q = 0; q < VA; ++q) pk.v[q] = out[e + q];
              *reinterpret_cast<Pack<VA>*>(dst + e) = pk;
            }
          } else {
#pragma unroll
            for (int c = 0; c < kTX; ++c)
              if (ic + c < iend) dst[c] = out[c];
          }
        }
      }
      bot = top;
      sprev = sk;
      sk = sk1;
      sk1 = sk1 + 1 == kNS ? 0 : sk1 + 1;
      ph1 ^= sk1 == 0 ? 1u : 0u;
    }
  }

  template <bool VEC>
  __device__ __forceinline__ void march() const {
    Faces bot;
    kl::mbar_wait(bars + 0, 0);  // plane k0-1
    kl::mbar_wait(bars + 1, 0);  // plane k0
    top_faces(ring, ring + kSlot, dzhi[k0], bot);  // the bottom faces k0-1/2 of the chunk

    int sprev = 0, sk = 1, sk1 = 2 % kNS;  // slots of planes k-1, k, k+1
    unsigned ph1 = 0;
    LevelCache lc;
    for (int k = k0; k < k1; ++k) {
      __syncthreads();  // every thread is done with plane k-1's slot
      if (tid == 0) {
        const int p = k - 1 + kNS;
        if (p <= k1) {
          kl::fence_proxy_async_smem();
          issue(sprev, p);
        }
      }
      const Levels lv = lc.at(k, k0, k1, tid & 31, dzi, dzhi, dxi, dyi, cs);
      kl::mbar_wait(bars + sk1, ph1);
      const real* pk = ring + sk * kSlot;
      const real* pk1 = ring + sk1 * kSlot;
      const real dz = lv.dz, dzh1 = lv.dzh1, fac = lv.fac;
      if (KL_SKEL) {
        real* const srow = evisc + ic + static_cast<long long>(j0 + lj0) * KL_JJ + static_cast<long long>(k) * KL_KK;
#pragma unroll
        for (int t = 0; t < kTY; ++t)
#pragma unroll
          for (int c = 0; c < kTX; ++c)
            if (j0 + lj0 + t < jend && ic + c < iend && !(kXS && helper)) srow[t * KL_JJ + c] = pk1[hof[0] + t * kBW + c];
        sprev = sk;
        sk = sk1;
        sk1 = sk1 + 1 == kNS ? 0 : sk1 + 1;
        ph1 ^= sk1 == 0 ? 1u : 0u;
        continue;
      }
      Faces top;
      top_faces(pk, pk1, dzh1, top);

      const real *u = pk + hof[0], *v = pk + hof[1], *w = pk + hof[2], *w1 = pk1 + hof[2];
      // east u of each cell; the helper lane (no output, computes along with
      // its warp) reads its own column so the last warp's stays in the box
      const real* ue = u + ((kXS && helper) ? 0 : 1);
      // xy edges at the tile's corners (rows t = 0..kTY, columns a = 0..kTX), x-pair sums
      //   edge (i-1/2+a, j-1/2+t): (u[i+a,j+t]-u[i+a,j+t-1]) dyi + (v[i+a,j+t]-v[i+a-1,j+t]) dxi
      real pxy[kTY + 1][kTX];
#pragma unroll
      for (int t = 0; t <= kTY; ++t) {
        real e[kTX + 1];
#pragma unroll
        for (int a = 0; a <= (kXS ? 0 : kTX); ++a) {
          const int o = t * kBW + a;
          const real s = (u[o] - u[o - kBW]) * dyi + (v[o] - v[o - 1]) * dxi;
          e[a] = s * s;
        }
        if constexpr (kXS) e[1] = __shfl_down_sync(0xffffffffu, e[0], 1);
#pragma unroll
        for (int c = 0; c < kTX; ++c) pxy[t][c] = e[c] + e[c + 1];
      }

      real* const orow = evisc + ic + static_cast<long long>(j0 + lj0) * KL_JJ + static_cast<long long>(k) * KL_KK;
#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        real out[kTX];
#pragma unroll
        for (int c = 0; c < kTX; ++c) {
          const int o = t * kBW + c;
          const real dx = (ue[o] - u[o]) * dxi, dy = (v[o + kBW] - v[o]) * dyi, dzz = (w1[o] - w[o]) * dz;
          const real diag = dx * dx + dy * dy + dzz * dzz;
          const real off = (pxy[t][c] + pxy[t + 1][c]) + (bot.xz[t][c] + top.xz[t][c]) + (bot.yz[t][c] + top.yz[t][c]);
          out[c] = fac * kl::sqrt_fast(real(2) * diag + real(0.25) * off);
        }
        if (j0 + lj0 + t < jend && !(kXS && helper)) {
          real* dst = orow + t * KL_JJ;
          if (VEC && ic + kTX <= iend) {
            constexpr int VA = kTX < kE ? kTX : kE;
#pragma unroll
            for (int e = 0; e < kTX; e += VA) {
              Pack<VA> pk;
#pragma unroll
              for (int q = 0; q < VA; ++q) pk.v[q] = out[e + q];
              *reinterpret_cast<Pack<VA>*>(dst + e) = pk;
            }
          } else {
#pragma unroll
            for (int c = 0; c < kTX; ++c)
              if (ic + c < iend) dst[c] = out[c];
          }
        }
      }
      bot = top;
      sprev = sk;
      sk = sk1;
      sk1 = sk1 + 1 == kNS ? 0 : sk1 + 1;
      ph1 ^= sk1 == 0 ? 1u : 0u;
    }
  }
};
// selects the pair march for TILE_X >= 2 without instantiating it otherwise
template <bool kPairs>
struct Marcher {
  template <bool VEC>
  static __device__ __forceinline__ void run(const EviscTma& m) { m.march<VEC>(); }
};
template <>
struct Marcher<true> {
  template <bool VEC>
  static __device__ __forceinline__ void run(const EviscTma& m) { m.march2<VEC>(); }
};
}  // namespace

// positions: evisc 0, u 1, v 2, w 3, jj 9, kk 10 (definitions.ARG_LAYOUT["evisc_smag"]); maps: u, v, w
extern "C" __device__ const int kl_tma_spec[1 + 5 * 3] = {3, 1, 9, 10, kBW, kBH, 2, 9, 10, kBW, kBH,
                                                          3, 9, 10, kBW, kBH};
struct __align__(64) KlTmaParams {
  TmaDesc map[3];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ evisc, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ dzi, const real* __restrict__ dzhi, const real dxi,
         const real dyi, const real cs, const int jj, const int kk, const int istart, const int jstart,
         const int kstart, const int iend, const int jend, const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* sbase = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);

  const unsigned nbx = kl::ceil_div(iend - istart, kXT);
  const unsigned nby = kl::ceil_div(jend - jstart, kTYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * kXT;

  EviscTma m;
  m.evisc = evisc;
  m.dzi = dzi;
  m.dzhi = dzhi;
  m.bars = reinterpret_cast<unsigned long long*>(sbase);
  m.ring = reinterpret_cast<real*>(sbase + 128);
  m.maps = &tma.map[0];
  m.dxi = dxi;
  m.dyi = dyi;
  m.cs = cs;
  m.j0 = jstart + by * kTYT;
  m.k0 = kstart + bz * ZCHUNK;
  m.k1 = min(m.k0 + ZCHUNK, kend);
  m.tid = threadIdx.x + threadIdx.y * BLOCK_X;
  m.iend = iend;
  m.jend = jend;
  m.lj0 = threadIdx.y * kTY;
  // column of this thread within the block: kTX per thread, or (KL_XSHARE)
  // 31 per warp with lane 31 on the next warp's first column (the helper)
  const int lane = static_cast<int>(threadIdx.x) & 31;
  const int cx = kXS ? static_cast<int>(threadIdx.x) / 32 * 31 + lane : kTX * static_cast<int>(threadIdx.x);
  m.helper = kXS && lane == 31;
  m.ic = i0 + cx;
  const real* const hp[3] = {u, v, w};
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    const int x = i0 - 1 + kl::tma_xoff(hp[f]);
    m.xh[f] = x & ~(kE - 1);
    m.hof[f] = f * kFS + (m.lj0 + 1) * kBW + (x - m.xh[f]) + 1 + cx;  // (strip row 0, column ic)
  }
  if (m.tid == 0) {
    for (int q = 0; q < kNS; ++q) kl::mbar_init(m.bars + q, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (m.tid == 0)
    for (int p = m.k0 - 1; p <= min(m.k0 - 1 + kNS - 1, m.k1); ++p) m.issue(p - (m.k0 - 1), p);
  bool aligned = kl::tma_xoff(evisc) == 0 && (i0 & (kE - 1)) == 0;
#pragma unroll
  for (int f = 0; f < 3; ++f) aligned = aligned && kl::tma_xoff(hp[f]) == 0;
  if (kTX > 1 && aligned)
    Marcher<(kTX >= 2)>::template run<true>(m);
  else
    Marcher<(kTX >= 2)>::template run<false>(m);
}
