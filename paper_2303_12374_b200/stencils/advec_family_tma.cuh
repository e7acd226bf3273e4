// advec_family_tma.cuh — STAGING == TMA variant of advec_v / advec_w /
// advec_s (included by those sources with ADV_KIND set): the flux-form
// z-march of advec_u_tma.cuh generalised over the staggering of the advected
// field phi (oracle/family_oracle.py).
//
// Rings (one mbarrier per slot, refilled by one elected thread):
//   * phi with a 3-cell x/y halo in DEPTH+4 slots: plane k feeds the x/y
//     stencils of step k, plane k+3 the register z-window;
//   * the velocity boxes + the tendency box of plane p in DEPTH+2 slots:
//       kind  phi  x face velocity (u)        y face velocity (v)        z face velocity (w)
//       V     v    u rows j-1, j   (box A)    phi (v[j] + v[j+1])        w rows j-1, j of plane k+1 (B)
//       S     s    u               (box A)    v               (box C)    w of plane k+1 (B)
//       W     w    u planes k-1, k (box A)    v planes k-1, k (box C)    phi (w[k] + w[k+1])
//     (for W a slot of plane p holds u, v of plane p-1 and wt of plane p, so
//     step k reads only the slots of planes k and k+1, as for V and S).
// The compute warps issue no global loads, only the final tendency stores.
//
// A thread owns TILE_X in {2, 4} consecutive columns x a strip of TILE_Y rows
// and evaluates the arithmetic of column pairs in kl::f2 (fp32: packed
// FADD2/FMUL2/FFMA2) or kl::d2 (fp64: two scalar instructions) — one source
// for both precisions; face fluxes are evaluated once per face (x: TILE_X+1
// per TILE_X cells, y carried along the strip, z carried up the march).
// Boxes of the halo'd phi start at column i0-4, the others at i0; with
// 16-byte aligned rows the shared reads and tendency stores are vectorised,
// any other alignment takes a uniform scalar-access branch.

#if BLOCK_Z != 1 || TILE_Z != 1
#error "family TMA advection requires BLOCK_Z == TILE_Z == 1"
#endif
#if TILE_X != 2 && TILE_X != 4
#error "family TMA advection requires TILE_X in {2, 4} (column pairs)"
#endif
#if !CONTIG_X
#error "family TMA advection needs consecutive columns (CONTIG_X)"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif

#include "kl_pack.cuh"
#include "kl_tma.cuh"

namespace {
using P2 = typename kl::pair_of<real>::type;
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;
constexpr int kTX = TILE_X, kTY = TILE_Y;
constexpr int kXT = BLOCK_X * kTX;
constexpr int kTYT = BLOCK_Y * kTY;
constexpr int kVA = kTX < kE ? kTX : kE;
constexpr int kP = kTX / 2;
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }

constexpr bool kV = ADV_KIND == ADV_V, kW = ADV_KIND == ADV_W, kSc = ADV_KIND == ADV_S;
// phi: columns i0-4 .. i0+kXT+3 (start rounded down to 16 B), rows j0-3 .. j0+kTYT+2
constexpr int kBW = rup(kXT + 8 + kE - 1, kE);
constexpr int kBH = kTYT + 6;
constexpr int kUB = rup(kBW * kBH * kS, 128);
// velocity / tendency boxes start at column i0 (+ up to kE-1 alignment slack)
constexpr int kFW = rup(kXT + 1 + kE - 1, kE);  // x faces: columns i0 .. i0+kXT
constexpr int kCW = rup(kXT + kE - 1, kE);      // cells: columns i0 .. i0+kXT-1
constexpr bool kHasB = !kW, kHasC = !kV;
constexpr int kAR = kV ? kTYT + 1 : kTYT;  // A rows (V: from j0-1)
constexpr int kBR = kV ? kTYT + 1 : kTYT;  // B rows (V: from j0-1)
constexpr int kCR = kTYT + 1;              // C rows j0 .. j0+kTYT
constexpr int kAB = rup(kFW * kAR * kS, 128);
constexpr int kBB = kHasB ? rup(kCW * kBR * kS, 128) : 0;
constexpr int kCB = kHasC ? rup(kCW * kCR * kS, 128) : 0;
constexpr int kTB = rup(kCW * kTYT * kS, 128);
constexpr int kUS = kUB / kS;
constexpr int kVS = (kAB + kBB + kCB + kTB) / kS;
constexpr int kAO = 0, kBO = kAB / kS, kCO = (kAB + kBB) / kS, kTO = (kAB + kBB + kCB) / kS;
constexpr int kNU = DEPTH + 4;
constexpr int kNV = DEPTH + 2;
constexpr unsigned kTxU = static_cast<unsigned>(kBW * kBH * kS);
constexpr unsigned kTxV = static_cast<unsigned>(
    (kFW * kAR + (kHasB ? kCW * kBR : 0) + (kHasC ? kCW * kCR : 0) + kCW * kTYT) * kS);
constexpr int kNMaps = 2 + (kHasB ? 1 : 0) + (kHasC ? 1 : 0) + 1;  // phi, A, [B], [C], T
static_assert(kBW <= 256 && kBH <= 256, "TMA box extents are limited to 256");
static_assert(kNU + kNV <= 16, "mbarriers must fit the 128-byte header");
// velocities enter as two-point sums (V, W; the 1/2 folded into the scale) or single values (S)
constexpr double kScale = kSc ? 60.0 : 120.0;

template <int N>
struct __align__(N * sizeof(real)) Pack {
  real v[N];
};

template <int VA, int LO, int HI, int N>
__device__ __forceinline__ void ld_span(real (&d)[N], const real* s) {
  constexpr int lo = LO / VA * VA, hi = (HI + VA - 1) / VA * VA;
  static_assert(hi <= N, "span exceeds the destination");
#pragma unroll
  for (int e = lo; e < hi; e += VA) {
    const Pack<VA> p = *reinterpret_cast<const Pack<VA>*>(s + e);
#pragma unroll
    for (int q = 0; q < VA; ++q) d[e + q] = p.v[q];
  }
}

template <int VA>
__device__ __forceinline__ void st_span(real* d, const real (&s)[kTX]) {
#pragma unroll
  for (int e = 0; e < kTX; e += VA) {
    Pack<VA> p;
#pragma unroll
    for (int q = 0; q < VA; ++q) p.v[q] = s[e + q];
    *reinterpret_cast<Pack<VA>*>(d + e) = p;
  }
}

struct AdvFam {
  real* tend;
  const real* phi;
  real* ring_u;
  real* ring_v;
  const real* zprof;  // [ZCHUNK][2]: z-face rho of the top face, metric / scale
  unsigned long long* bar_u;
  unsigned long long* bar_v;
  const TmaDesc* maps;
  real dxs, dys;   // dxi / scale, dyi / scale
  real rho_bot0;   // rho of the bottom face of plane k0
  int j0, k0, k1, tid, iend, jend;
  int xp, xa, xb, xc, xt;  // 16-byte aligned box starts (phi, A, B, C, T)
  int ic, lj0, uofs, aofs, bofs, cofs, tofs;

  __device__ __forceinline__ void issue_u(int slot, int p) const {
    kl::mbar_expect_tx(bar_u + slot, kTxU);
    kl::tma_load_3d(ring_u + slot * kUS, maps + 0, bar_u + slot, xp, j0 - 3, p);
  }
  __device__ __forceinline__ void issue_v(int slot, int p) const {
    unsigned long long* bar = bar_v + slot;
    real* dst = ring_v + slot * kVS;
    kl::mbar_expect_tx(bar, kTxV);
    int m = 1;
    kl::tma_load_3d(dst + kAO, maps + m++, bar, xa, kV ? j0 - 1 : j0, kW ? p - 1 : p);
    if (kHasB) kl::tma_load_3d(dst + kBO, maps + m++, bar, xb, kV ? j0 - 1 : j0, p);
    if (kHasC) kl::tma_load_3d(dst + kCO, maps + m++, bar, xc, j0, kW ? p - 1 : p);
    kl::tma_load_3d(dst + kTO, maps + m, bar, xt, j0, p);
  }
  __device__ __forceinline__ void prime() const {
    for (int p = k0; p <= min(k0 + kNU - 1, k1 + 2); ++p) issue_u(p - k0, p);
    for (int p = k0; p <= min(k0 + kNV - 1, k1); ++p) issue_v(p - k0, p);
  }

  struct Cursor {
    int u0 = 0, u3 = 3, uprev = kNU - 1;
    int v0 = 0, v1 = 1, vprev = kNV - 1;
    unsigned ph_u3 = 0, ph_v1 = 0;
  };
  struct Planes {
    const real *xy, *zf, *s0, *s1;  // phi plane k / k+3; velocity slots of planes k, k+1
  };

  __device__ __forceinline__ void wait_first() const {
    kl::mbar_wait(bar_u + 0, 0);
    kl::mbar_wait(bar_u + 1, 0);
    kl::mbar_wait(bar_u + 2, 0);
    kl::mbar_wait(bar_v + 0, 0);
  }

  __device__ __forceinline__ Planes begin_step(int k, Cursor& c) const {
    __syncthreads();  // every thread is done with plane k-1's slots
    if (tid == 0 && k > k0) {
      const int pu = k - 1 + kNU, pv = k - 1 + kNV;
      kl::fence_proxy_async_smem();
      if (pu <= k1 + 2) issue_u(c.uprev, pu);
      if (pv <= k1) issue_v(c.vprev, pv);
    }
    kl::mbar_wait(bar_u + c.u3, c.ph_u3);
    kl::mbar_wait(bar_v + c.v1, c.ph_v1);
    Planes pl;
    pl.xy = ring_u + c.u0 * kUS + uofs;
    pl.zf = ring_u + c.u3 * kUS + uofs + 4;
    pl.s0 = ring_v + c.v0 * kVS;
    pl.s1 = ring_v + c.v1 * kVS;
    c.uprev = c.u0;
    c.u0 = c.u0 + 1 == kNU ? 0 : c.u0 + 1;
    c.u3 = c.u3 + 1 == kNU ? 0 : c.u3 + 1;
    c.ph_u3 ^= c.u3 == 0 ? 1u : 0u;
    c.vprev = c.v0;
    c.v0 = c.v1;
    c.v1 = c.v1 + 1 == kNV ? 0 : c.v1 + 1;
    c.ph_v1 ^= c.v1 == 0 ? 1u : 0u;
    return pl;
  }

  // z-face velocity pairs of the cells (t, c..c+1): bottom of plane k0 from
  // slot k0 (V, S) or the phi window (W), top of plane k from slot k+1
  template <int VA>
  __device__ __forceinline__ P2 zvel_box(const real* slot, int t, int c) const {
    real r0[kTX], r1[kTX];
    ld_span<VA, 0, kTX>(r0, slot + kBO + bofs + t * kCW);
    if (kV) {
      ld_span<VA, 0, kTX>(r1, slot + kBO + bofs + (t + 1) * kCW);
      return P2(r0[c], r0[c + 1]) + P2(r1[c], r1[c + 1]);
    }
    return P2(r0[c], r0[c + 1]);
  }

  template <int VA>
  __device__ __forceinline__ void march() const {
    constexpr long long K1 = KL_KK;
    P2 uq[kTY][kP][6];  // phi[k-2 .. k+3] of every column pair
    P2 fz_bot[kTY][kP];
    wait_first();
    {
      const P2 rb(rho_bot0);
#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        const int j = min(j0 + lj0 + t, jend - 1);
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int c = 2 * p;
          const long long rowk = static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
          const long long b0 = min(ic + c, iend - 1) + rowk, b1 = min(ic + c + 1, iend - 1) + rowk;
          const P2 um3(phi[b0 - 3 * K1], phi[b1 - 3 * K1]);  // planes below the chunk: not staged
#pragma unroll
          for (int m = 0; m < 5; ++m) uq[t][p][m] = P2(phi[b0 + (m - 2) * K1], phi[b1 + (m - 2) * K1]);
          const P2 vel = kW ? uq[t][p][1] + uq[t][p][2] : zvel_box<VA>(ring_v, t, c);
          fz_bot[t][p] = rb * kl::flux5x60(vel, um3, uq[t][p][0], uq[t][p][1], uq[t][p][2], uq[t][p][3],
                                            uq[t][p][4]);
        }
      }
    }
    const P2 dx2(dxs), dy2(dys);

    Cursor cur;
    for (int k = k0; k < k1; ++k) {
      const Planes pl = begin_step(k, cur);
      const real *xy = pl.xy, *zf = pl.zf;
      const real* tp = pl.s0 + kTO + tofs;  // tendency, plane k at (ic, j0+lj0)
      const P2 rh_top(zprof[2 * (k - k0)]);
      const P2 zfac(zprof[2 * (k - k0) + 1]);
      const long long kofs = static_cast<long long>(k) * K1;

      // phi along y in this thread's columns: rows lj0-3 .. lj0+kTY+2
      real ucol[kTY + 6][kTX];
#pragma unroll
      for (int m = 0; m < kTY + 6; ++m) {
        if (m >= 3 && m < kTY + 3) continue;
        real r[kTX + 8];
        ld_span<VA, 4, 4 + kTX>(r, xy + (m - 3) * kBW);
#pragma unroll
        for (int c = 0; c < kTX; ++c) ucol[m][c] = r[4 + c];
      }
      real xr[kTY][kTX + 8];  // x rows of the strip: columns ic-4 .. ic+kTX+3
#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        ld_span<VA, 1, kTX + 7>(xr[t], xy + t * kBW);
#pragma unroll
        for (int c = 0; c < kTX; ++c) ucol[t + 3][c] = xr[t][4 + c];
      }
      auto ucp = [&](int m, int p) { return P2(ucol[m][2 * p], ucol[m][2 * p + 1]); };
      // y face velocities of the box rows r = lj0 + t (north faces of row t-1)
      auto yvel = [&](int t, int c) -> P2 {
        if (kV) return P2(ucol[t + 2][c], ucol[t + 2][c + 1]) + P2(ucol[t + 3][c], ucol[t + 3][c + 1]);
        real r0[kTX];
        ld_span<VA, 0, kTX>(r0, pl.s0 + kCO + cofs + t * kCW);
        if (kSc) return P2(r0[c], r0[c + 1]);
        real r1[kTX];
        ld_span<VA, 0, kTX>(r1, pl.s1 + kCO + cofs + t * kCW);
        return P2(r0[c], r0[c + 1]) + P2(r1[c], r1[c + 1]);
      };
      P2 fy_lo[kP];
#pragma unroll
      for (int p = 0; p < kP; ++p)
        fy_lo[p] = kl::flux5x60(yvel(0, 2 * p), ucp(0, p), ucp(1, p), ucp(2, p), ucp(3, p), ucp(4, p), ucp(5, p));

#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        // x face velocities (faces 0..kTX of row t)
        real av[kTX + 1];
        {
          real a0[kFW];
          ld_span<VA, 0, kTX + 1>(a0, pl.s0 + kAO + aofs + t * kFW);
          if (kV || kW) {
            real a1[kFW];
            ld_span<VA, 0, kTX + 1>(a1, kV ? pl.s0 + kAO + aofs + (t + 1) * kFW : pl.s1 + kAO + aofs + t * kFW);
#pragma unroll
            for (int f = 0; f <= kTX; ++f) av[f] = a0[f] + a1[f];
          } else {
#pragma unroll
            for (int f = 0; f <= kTX; ++f) av[f] = a0[f];
          }
        }
        const real* r = xr[t];
        real fx[kTX + 1];
#pragma unroll
        for (int f = 0; f < kTX; f += 2) {
          const P2 s_cd(r[f + 3] + r[f + 4], r[f + 4] + r[f + 5]);
          const P2 s_be(r[f + 2] + r[f + 5], r[f + 3] + r[f + 6]);
          const P2 s_af(r[f + 1] + r[f + 6], r[f + 2] + r[f + 7]);
          const P2 d_dc(r[f + 4] - r[f + 3], r[f + 5] - r[f + 4]);
          const P2 d_eb(r[f + 5] - r[f + 2], r[f + 6] - r[f + 3]);
          const P2 d_fa(r[f + 6] - r[f + 1], r[f + 7] - r[f + 2]);
          const P2 fl = kl::flux5x60_sd(P2(av[f], av[f + 1]), s_cd, s_be, s_af, d_dc, d_eb, d_fa);
          fx[f] = fl.lo();
          fx[f + 1] = fl.hi();
        }
        fx[kTX] = kl::flux5x60(av[kTX], r[kTX + 1], r[kTX + 2], r[kTX + 3], r[kTX + 4], r[kTX + 5], r[kTX + 6]);
        real zr[kTX + 8], tr[kTX + 8], out[kTX];
        ld_span<VA, 0, kTX>(zr, zf + t * kBW);
        ld_span<VA, 0, kTX>(tr, tp + t * kCW);
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int c = 2 * p;
          P2* q = uq[t][p];
          q[5] = P2(zr[c], zr[c + 1]);
          const P2 fy_hi = kl::flux5x60(yvel(t + 1, c), ucp(t + 1, p), ucp(t + 2, p), ucp(t + 3, p),
                                        ucp(t + 4, p), ucp(t + 5, p), ucp(t + 6, p));
          const P2 vel_t = kW ? q[2] + q[3] : zvel_box<VA>(pl.s1, t, c);
          const P2 fz_top = rh_top * kl::flux5x60(vel_t, q[0], q[1], q[2], q[3], q[4], q[5]);
          const P2 dfx(fx[c + 1] - fx[c], fx[c + 2] - fx[c + 1]);
          const P2 o = P2(tr[c], tr[c + 1]) -
                       kl::fma2(fz_top - fz_bot[t][p], zfac, kl::fma2(fy_hi - fy_lo[p], dy2, dfx * dx2));
          out[c] = o.lo();
          out[c + 1] = o.hi();
          fy_lo[p] = fy_hi;
          fz_bot[t][p] = fz_top;
#pragma unroll
          for (int m = 0; m < 5; ++m) q[m] = q[m + 1];
        }
        const int j = j0 + lj0 + t;
        if (j < jend) {
          real* dst = tend + ic + static_cast<long long>(j) * KL_JJ + kofs;
          if (ic + kTX <= iend) {
            st_span<VA>(dst, out);
          } else {
#pragma unroll
            for (int c = 0; c < kTX; ++c)
              if (ic + c < iend) dst[c] = out[c];
          }
        }
      }
    }
  }
};
}  // namespace

// positions (definitions.ARG_LAYOUT): tendency 0; advec_v/_w: u 1, v 2, w 3, jj 9, kk 10;
// advec_s: s 1, u 2, v 3, w 4, jj 10, kk 11.  Map order: phi, A (u), [B (w)], [C (v)], T.
#if ADV_KIND == ADV_S
#define KL_PU 2
#define KL_PV 3
#define KL_PW 4
#define KL_PPHI 1
#define KL_J 10
#define KL_K 11
#else
#define KL_PU 1
#define KL_PV 2
#define KL_PW 3
#define KL_PPHI (ADV_KIND == ADV_V ? 2 : 3)
#define KL_J 9
#define KL_K 10
#endif
extern "C" __device__ const int kl_tma_spec[1 + 5 * kNMaps] = {
    kNMaps,
    KL_PPHI, KL_J, KL_K, kBW, kBH,
    KL_PU, KL_J, KL_K, kFW, kAR,
#if ADV_KIND != ADV_W
    KL_PW, KL_J, KL_K, kCW, kBR,
#endif
#if ADV_KIND != ADV_V
    KL_PV, KL_J, KL_K, kCW, kCR,
#endif
    0, KL_J, KL_K, kCW, kTYT};
struct __align__(64) KlTmaParams {
  TmaDesc map[kNMaps];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ tend,
#if ADV_KIND == ADV_S
         const real* __restrict__ s,
#endif
         const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ rhoref, const real* __restrict__ rhorefh, const real* __restrict__ dz1,
         const real dxi, const real dyi, const int jj, const int kk, const int istart, const int jstart,
         const int kstart, const int iend, const int jend, const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
#if ADV_KIND == ADV_S
  const real* phi = s;
#elif ADV_KIND == ADV_V
  const real* phi = v;
#else
  const real* phi = w;
#endif
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* sbase = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sbase);
  real* const ring_u = reinterpret_cast<real*>(sbase + 128);
  real* const ring_v = ring_u + kNU * kUS;
  real* const zprof = ring_v + kNV * kVS;

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
  // box starts: tensor x of column i0-4 (phi) / i0 (the rest) rounded down to 16 B
  const int xp = i0 - 4 + kl::tma_xoff(phi), xa = i0 + kl::tma_xoff(u), xb = i0 + kl::tma_xoff(w),
            xc = i0 + kl::tma_xoff(v), xt = i0 + kl::tma_xoff(tend);
  const int sp = xp & (kE - 1), sa = xa & (kE - 1), sb = xb & (kE - 1), sc = xc & (kE - 1), st = xt & (kE - 1);

  AdvFam m;
  m.tend = tend;
  m.phi = phi;
  m.ring_u = ring_u;
  m.ring_v = ring_v;
  m.zprof = zprof;
  m.bar_u = bars;
  m.bar_v = bars + kNU;
  m.maps = &tma.map[0];
  m.dxs = dxi * real(1.0 / kScale);
  m.dys = dyi * real(1.0 / kScale);
  m.rho_bot0 = kW ? rhoref[k0 - 1] : rhorefh[k0];
  m.j0 = j0;
  m.k0 = k0;
  m.k1 = k1;
  m.tid = tid;
  m.iend = iend;
  m.jend = jend;
  m.xp = xp - sp;
  m.xa = xa - sa;
  m.xb = xb - sb;
  m.xc = xc - sc;
  m.xt = xt - st;
  m.ic = i0 + kTX * static_cast<int>(threadIdx.x);
  m.lj0 = threadIdx.y * kTY;
  const int cx = kTX * static_cast<int>(threadIdx.x);
  m.uofs = sp + (m.lj0 + 3) * kBW + cx;  // phi at (ic-4, j0+lj0)
  m.aofs = sa + m.lj0 * kFW + cx;        // A row lj0 (V: row j0+lj0-1)
  m.bofs = sb + m.lj0 * kCW + cx;        // B row lj0 (V: row j0+lj0-1)
  m.cofs = sc + m.lj0 * kCW + cx;        // C row lj0
  m.tofs = st + m.lj0 * kCW + cx;        // T row lj0

  if (tid == 0) {
    for (int q = 0; q < kNU + kNV; ++q) kl::mbar_init(bars + q, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) m.prime();
  for (int q = tid; q < k1 - k0; q += KL_THREADS) {
    const int k = k0 + q;
    if (kW) {
      zprof[2 * q] = rhoref[k];
      zprof[2 * q + 1] = dz1[k] / (rhorefh[k] * real(kScale));
    } else {
      zprof[2 * q] = rhorefh[k + 1];
      zprof[2 * q + 1] = dz1[k] / (rhoref[k] * real(kScale));
    }
  }
  // (the march's first __syncthreads publishes zprof)
  const bool aligned = sp == 0 && sa == 0 && st == 0 && (!kHasB || sb == 0) && (!kHasC || sc == 0);
  if (kVA > 1 && aligned) {
    m.march<kVA>();
  } else {
    m.march<1>();
  }
}

#undef KL_PU
#undef KL_PV
#undef KL_PW
#undef KL_PPHI
#undef KL_J
#undef KL_K
