// advec_u_tma.cuh — STAGING == TMA variant of advec_u (included by
// advec_u.cu).  Flux-form z-march (see advec_u_zmarch.cuh) with every operand
// fetched by the Tensor Memory Accelerator into two shared-memory rings, one
// mbarrier per slot:
//   * u, with a 3-cell x/y halo, in DEPTH+4 slots — plane k feeds the x/y
//     stencil of step k and plane k+3 the z-window (so u[k+3] of every cell
//     comes from the ring);
//   * v (columns i-1..i, rows j..j+1), w (columns i-1..i) and ut (no halo)
//     in DEPTH+2 slots — step k reads v and ut of plane k and w of plane k+1;
// so the compute warps issue no global loads, only the final ut stores.  One
// elected thread refills the slots vacated by plane k-1 at the start of step
// k, keeping DEPTH planes beyond the ones being read in flight in both rings
// (the halo-free fields do not occupy the three extra slots the z-window
// needs, which leaves the shared memory for deeper prefetch or more blocks).
//
// A thread owns TILE_X consecutive columns (TILE_X in {1, 2, 4}; CONTIG_X)
// times a strip of TILE_Y rows.  Per plane it evaluates TILE_X+1 x-faces
// (the shared faces of its own cells once), TILE_X y-faces per row (the
// south face carried from the row below) and TILE_X z-faces per row (the
// bottom face carried from the plane below): 3 + 1/TILE_X + 1/TILE_Y face
// fluxes per cell.  The advection work is issue-bound in fp32, so the
// operand reads are vectorised: boxes start at column i0-4, so when the
// tensor's x alignment makes column i0 16-byte aligned (always, for the
// GridLayout pitches) every thread's cells sit at vector-aligned shared
// offsets and a row of TILE_X+8 values is TILE_X+8 / VA loads of VA
// elements (VA = min(TILE_X, 16 B)), the ut stores VA-wide too; a uniform
// branch falls back to scalar accesses for any other alignment.  Face
// velocities are passed as sums (the 1/2 of interp2 is folded into the 1/120
// scale factors).

#if BLOCK_Z != 1 || TILE_Z != 1
#error "advec_u TMA requires BLOCK_Z == TILE_Z == 1"
#endif
#if TILE_X != 1 && TILE_X != 2 && TILE_X != 4
#error "advec_u TMA requires TILE_X in {1, 2, 4}"
#endif
#if TILE_X > 1 && !CONTIG_X
#error "advec_u TMA: TILE_X > 1 needs consecutive columns (CONTIG_X)"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif
#ifndef KL_YBAL
#define KL_YBAL 0  // 0: blocks of kTYT rows; > 0: near-equal row runs, as many as the grid holds (entry)
#endif
#ifndef KL_SKEL
#define KL_SKEL 0  // diagnostic only (tools/skeleton_probe.py): 1 = keep the TMA rings, barriers and ut
                   // stores but replace the stencil by ut += 1 — the data-movement floor of the tiling;
                   // 2 = that with u boxes stripped of their x/y halo, 3 = v/w boxes too (what the
                   // halos cost in bytes and time)
#endif

#ifndef KL_L2PF
#define KL_L2PF 0  // > 0: also prefetch plane p + KL_L2PF into L2 when plane p is loaded into a ring
#endif
#ifndef KL_L2HINT
#define KL_L2HINT 0  // experiment: L2 eviction priorities, bit 1 = ut loads evict_first, 2 = v/w loads
                     // evict_first, 4 = u loads evict_last, 8 = ut stores evict_first
#endif

#include "kl_pack.cuh"
#include "kl_tma.cuh"

namespace {
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;                // elements per 16 bytes
constexpr int kTX = TILE_X, kTY = TILE_Y;
constexpr int kXT = BLOCK_X * kTX;          // columns per block
constexpr int kTYT = BLOCK_Y * kTY;         // rows per block
constexpr int kVA = kTX < kE ? kTX : kE;    // vector width (elements) of aligned reads
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }
// box widths: start column i0-4 rounded down to 16 B (up to kE-1 slack)
constexpr int kTW = rup(kXT + kE - 1, kE);      // ut: columns i0 .. i0+kXT-1
#if KL_SKEL >= 2  // diagnostic floors: u boxes without the x/y halo (2), v/w boxes too (3)
constexpr int kBW = kTW, kBH = kTYT;
#else
constexpr int kBW = rup(kXT + 8 + kE - 1, kE);  // u: columns i0-4 .. i0+kXT+3
constexpr int kBH = kTYT + 6;
#endif
#if KL_SKEL >= 3
constexpr int kVW = kTW, kVH = kTYT;
#else
constexpr int kVW = rup(kXT + 4 + kE - 1, kE);  // v, w: columns i0-4 .. i0+kXT-1
constexpr int kVH = kTYT + 1;                   // v: rows j0 .. j0+kTYT
#endif
constexpr int kUB = rup(kBW * kBH * kS, 128);
constexpr int kVB = rup(kVW * kVH * kS, 128);
constexpr int kWB = rup(kVW * kTYT * kS, 128);
constexpr int kTB = rup(kTW * kTYT * kS, 128);
// two rings: u planes (kNU slots: plane k feeds the x/y stencil of step k,
// plane k+3 the z-window) and v/w/ut planes (kNV slots: step k reads v, ut
// of plane k and w of plane k+1) — the halo-free fields are not kept for the
// three extra planes the z-window needs
constexpr int kNU = DEPTH + 4;
constexpr int kNV = DEPTH + 2;
constexpr int kUS = kUB / kS;                 // elements per u slot
constexpr int kVS = (kVB + kWB + kTB) / kS;   // elements per v/w/ut slot
constexpr int kVO = 0, kWO = kVB / kS, kTO = (kVB + kWB) / kS;  // field offsets in a v/w/ut slot
// fp32 with column tiles: pairs of neighbouring columns share packed
// FADD2/FMUL2/FFMA2 instructions (kl_pack.cuh)
constexpr bool kPack = sizeof(real) == 4 && kTX >= 2;
constexpr int kP = kTX / 2 > 0 ? kTX / 2 : 1;  // column pairs per thread
constexpr unsigned kTxU = static_cast<unsigned>(kBW * kBH * kS);
constexpr unsigned kTxV = static_cast<unsigned>((kVW * kVH + kVW * kTYT + kTW * kTYT) * kS);
static_assert(kBW <= 256 && kBH <= 256, "TMA box extents are limited to 256");
static_assert(kNU + kNV <= 16, "mbarriers must fit the 128-byte header");

template <int N>
struct __align__(N * sizeof(real)) Pack {
  real v[N];
};

// d[e] = s[e] for e in [LO, HI), widened to VA-aligned loads of VA elements
// (s must be VA-element aligned).
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

// one VA-element store with an L2 evict_first policy (KL_L2HINT & 8)
template <int VA>
__device__ __forceinline__ void st_hint(real* d, const Pack<VA>& p, unsigned long long pol) {
  if constexpr (sizeof(real) == 4 && VA == 4) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(d), "f"(p.v[0]), "f"(p.v[1]),
                 "f"(p.v[2]), "f"(p.v[3]), "l"(pol) : "memory");
  } else if constexpr (sizeof(real) == 4 && VA == 2) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(d), "f"(p.v[0]), "f"(p.v[1]), "l"(pol)
                 : "memory");
  } else if constexpr (sizeof(real) == 8 && VA == 2) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(d), "d"(p.v[0]), "d"(p.v[1]), "l"(pol)
                 : "memory");
  } else {
    *reinterpret_cast<Pack<VA>*>(d) = p;
  }
}

template <int VA>
__device__ __forceinline__ void st_span(real* d, const real (&s)[kTX]) {
#if KL_L2HINT & 8
  const unsigned long long pol = kl::l2_evict_first();
#endif
#pragma unroll
  for (int e = 0; e < kTX; e += VA) {
    Pack<VA> p;
#pragma unroll
    for (int q = 0; q < VA; ++q) p.v[q] = s[e + q];
#if KL_L2HINT & 8
    st_hint<VA>(d + e, p, pol);
#else
    *reinterpret_cast<Pack<VA>*>(d + e) = p;
#endif
  }
}

// Per-block state of the march (a struct with a member template rather than
// a generic lambda: NVRTC has no extended device lambdas).
struct AdvecTma {
  real* ut;
  const real* u;
#if KL_PEER
  const real *u_lo, *u_hi;  // the neighbours' u (the prologue's planes outside the slab)
  int peer_klo, peer_khi, peer_shift_lo, peer_shift_hi;
#endif
  const real* rhoref;
  const real* rhorefh;
  const real* dzi;
  real* ring_u;  // [kNU][kUS]
  real* ring_v;  // [kNV][kVS]
  const real* zprof;  // [ZCHUNK][2]: rhorefh[k+1], dzi[k] / (120 rhoref[k])
  unsigned long long* bar_u;  // kNU mbarriers
  unsigned long long* bar_v;  // kNV mbarriers
  const TmaDesc* maps;
  real dxi120, dyi120;
  int j0, k0, k1, tid, iend, jend;
  int xu, xv, xw, xt;  // 16-byte aligned box starts
  int ic, lj0, uofs, vofs, wofs, tofs;

  __device__ __forceinline__ void issue_u(int slot, int p) const {
    kl::mbar_expect_tx(bar_u + slot, kTxU);
#if KL_PEER
    if (p >= peer_khi) {  // above the slab: the neighbour's u (map 4)
      kl::tma_load_3d(ring_u + slot * kUS, maps + 4, bar_u + slot, xu, j0 - 3, p + peer_shift_hi);
      return;
    }
#endif
#if KL_L2HINT & 4
    kl::tma_load_3d_hint(ring_u + slot * kUS, maps + 0, bar_u + slot, xu, j0 - 3, p, kl::l2_evict_last());
#else
    kl::tma_load_3d(ring_u + slot * kUS, maps + 0, bar_u + slot, xu, j0 - 3, p);
#endif
  }
  __device__ __forceinline__ void issue_v(int slot, int p) const {
    unsigned long long* bar = bar_v + slot;
    real* dst = ring_v + slot * kVS;
    kl::mbar_expect_tx(bar, kTxV);
#if KL_L2HINT & 2
    kl::tma_load_3d_hint(dst + kVO, maps + 1, bar, xv, j0, p, kl::l2_evict_first());
#else
    kl::tma_load_3d(dst + kVO, maps + 1, bar, xv, j0, p);
#endif
#if KL_PEER
    if (p >= peer_khi)  // above the slab: the neighbour's w (map 5); v / ut of that plane are never read
      kl::tma_load_3d(dst + kWO, maps + 5, bar, xw, j0, p + peer_shift_hi);
    else
#endif
#if KL_L2HINT & 2
      kl::tma_load_3d_hint(dst + kWO, maps + 2, bar, xw, j0, p, kl::l2_evict_first());
#else
      kl::tma_load_3d(dst + kWO, maps + 2, bar, xw, j0, p);
#endif
#if KL_L2HINT & 1
    kl::tma_load_3d_hint(dst + kTO, maps + 3, bar, xt, j0, p, kl::l2_evict_first());
#else
    kl::tma_load_3d(dst + kTO, maps + 3, bar, xt, j0, p);
#endif
  }
  // L2 prefetches (KL_L2PF): DRAM reads of planes beyond the rings start
  // early without costing shared memory
  __device__ __forceinline__ void prefetch_u(int p) const { kl::tma_prefetch_3d(maps + 0, xu, j0 - 3, p); }
  __device__ __forceinline__ void prefetch_v(int p) const {
    kl::tma_prefetch_3d(maps + 1, xv, j0, p);
    kl::tma_prefetch_3d(maps + 2, xw, j0, p);
    kl::tma_prefetch_3d(maps + 3, xt, j0, p);
  }
  // u of plane k0 + d at element offset b of plane k0 (the chunk prologue's
  // unstaged loads, planes k0-3 .. k0+2: below the slab for the first chunk,
  // above it for a last chunk shorter than 3 planes — from the neighbours)
  __device__ __forceinline__ real u_at(long long b, int d) const {
#if KL_PEER
    if (k0 + d < peer_klo) return u_lo[b + static_cast<long long>(d + peer_shift_lo) * KL_KK];
    if (k0 + d >= peer_khi) return u_hi[b + static_cast<long long>(d + peer_shift_hi) * KL_KK];
#endif
    return u[b + static_cast<long long>(d) * KL_KK];
  }
  // first fills: u planes k0 .. k1+2 (the last the z-window reads), v/w/ut
  // planes k0 .. k1 (w of plane k1 feeds the last step's top face)
  __device__ __forceinline__ void prime() const {
    for (int p = k0; p <= min(k0 + kNU - 1, k1 + 2); ++p) issue_u(p - k0, p);
    for (int p = k0; p <= min(k0 + kNV - 1, k1); ++p) issue_v(p - k0, p);
#if KL_L2PF > 0 && !KL_PEER
    for (int p = k0 + kNU; p < min(k0 + kNU + KL_L2PF, k1 + 3); ++p) prefetch_u(p);
    for (int p = k0 + kNV; p < min(k0 + kNV + KL_L2PF, k1 + 1); ++p) prefetch_v(p);
#endif
  }

  // Ring positions at step k: slots of u planes k, k+3, k-1 and of v/w/ut
  // planes k, k+1, k-1, with the barrier parities of the planes waited for.
  struct Cursor {
    int u0 = 0, u3 = 3, uprev = kNU - 1;
    int v0 = 0, v1 = 1, vprev = kNV - 1;
    unsigned ph_u3 = 0, ph_v1 = 0;
  };
  // Planes of step k: u (x/y stencil), u k+3 (z-window), v, w (plane k+1), ut.
  struct Planes {
    const real *xy, *zf, *vp, *wp, *tp;
  };

  // Planes read before the march: u k0..k0+2 (first read as x/y planes) and
  // v/w/ut k0 (w of plane k0 feeds the prologue); every later u plane is
  // first read as the z-window plane (k+3), every later v/w/ut plane as the
  // w plane (k+1), and waited for there.
  __device__ __forceinline__ void wait_first() const {
    kl::mbar_wait(bar_u + 0, 0);
    kl::mbar_wait(bar_u + 1, 0);
    kl::mbar_wait(bar_u + 2, 0);
    kl::mbar_wait(bar_v + 0, 0);
  }

  // Start of step k: refill the slots plane k-1 vacated, wait for the planes
  // this step reads first, advance the cursor.
  __device__ __forceinline__ Planes begin_step(int k, Cursor& c) const {
    __syncthreads();  // every thread is done with plane k-1's slots
    if (tid == 0 && k > k0) {
      const int pu = k - 1 + kNU, pv = k - 1 + kNV;
      kl::fence_proxy_async_smem();
      if (pu <= k1 + 2) issue_u(c.uprev, pu);
      if (pv <= k1) issue_v(c.vprev, pv);
#if KL_L2PF > 0 && !KL_PEER
      if (pu + KL_L2PF <= k1 + 2) prefetch_u(pu + KL_L2PF);
      if (pv + KL_L2PF <= k1) prefetch_v(pv + KL_L2PF);
#endif
    }
    kl::mbar_wait(bar_u + c.u3, c.ph_u3);
    kl::mbar_wait(bar_v + c.v1, c.ph_v1);
    Planes pl;
    pl.xy = ring_u + c.u0 * kUS + uofs;             // u, plane k at (ic-4, j0+lj0)
    pl.zf = ring_u + c.u3 * kUS + uofs + 4;         // u, plane k+3 at (ic, j0+lj0)
    pl.vp = ring_v + c.v0 * kVS + kVO + vofs;       // v, plane k at (ic-4, j0+lj0)
    pl.wp = ring_v + c.v1 * kVS + kWO + wofs;       // w, plane k+1 at (ic-4, j0+lj0)
    pl.tp = ring_v + c.v0 * kVS + kTO + tofs;       // ut, plane k at (ic, j0+lj0)
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

  // main loop, VA = vector width of the shared-memory reads / ut stores
  template <int VA>
  __device__ __forceinline__ void march() const {
    constexpr long long K1 = KL_KK;
    real uq[kTY][kTX][6];  // u[k-2 .. k+3] of every cell (k+3 loaded at step k)
    real fz_bot[kTY][kTX];
    wait_first();
    {
      const real rh0 = rhorefh[k0];
      const real* wp = ring_v + kWO + wofs;  // v/w/ut slot 0 = plane k0
#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        const int j = min(j0 + lj0 + t, jend - 1);
        real wr[kTX + 8];
        wr[3] = wp[t * kVW + 3];
        ld_span<VA, 4, 4 + kTX>(wr, wp + t * kVW);
#pragma unroll
        for (int c = 0; c < kTX; ++c) {
          const int i = min(ic + c, iend - 1);
          const long long b = i + static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
          const real um3 = u_at(b, -3);  // planes below the chunk: not staged
#pragma unroll
          for (int m = 0; m < 5; ++m) uq[t][c][m] = u_at(b, m - 2);
          fz_bot[t][c] = rh0 * kl::flux5x60(wr[3 + c] + wr[4 + c], um3, uq[t][c][0], uq[t][c][1], uq[t][c][2],
                                            uq[t][c][3], uq[t][c][4]);
        }
      }
    }

    Cursor cur;
    const bool active = j0 + lj0 < jend;  // a strip past the block's last row only keeps the barriers
    for (int k = k0; k < k1; ++k) {
      const Planes pl = begin_step(k, cur);
      if (!active) continue;
      if (KL_SKEL) {
        const long long kofs = static_cast<long long>(k) * K1;
#pragma unroll
        for (int t = 0; t < kTY; ++t) {
          real tr[kTX], out[kTX];
          ld_span<VA, 0, kTX>(tr, pl.tp + t * kTW);
#pragma unroll
          for (int c = 0; c < kTX; ++c) out[c] = tr[c] + real(1);
          const int j = j0 + lj0 + t;
          if (j < jend && ic + kTX <= iend) st_span<VA>(ut + ic + static_cast<long long>(j) * KL_JJ + kofs, out);
        }
        continue;
      }
      const real *xy = pl.xy, *zf = pl.zf, *vp = pl.vp, *wp = pl.wp, *tp = pl.tp;
      const real rh_top = zprof[2 * (k - k0)];
      const real zfac120 = zprof[2 * (k - k0) + 1];
      const long long kofs = static_cast<long long>(k) * K1;

      // u along y in this thread's columns: rows lj0-3 .. lj0+kTY+2
      real ucol[kTY + 6][kTX];
#pragma unroll
      for (int m = 0; m < kTY + 6; ++m) {
        if (m >= 3 && m < kTY + 3) continue;  // strip rows: taken from the x rows below
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
      // south faces of the strip (row j0+lj0-1/2)
      real fy_lo[kTX];
      {
        real vr[kTX + 8];
        vr[3] = vp[3];
        ld_span<VA, 4, 4 + kTX>(vr, vp);
#pragma unroll
        for (int c = 0; c < kTX; ++c)
          fy_lo[c] = kl::flux5x60(vr[3 + c] + vr[4 + c], ucol[0][c], ucol[1][c], ucol[2][c], ucol[3][c], ucol[4][c],
                                  ucol[5][c]);
      }

#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        // x: faces f = 0..kTX sit between columns ic+f-1 and ic+f
        real fx[kTX + 1];
#pragma unroll
        for (int f = 0; f <= kTX; ++f)
          fx[f] = kl::flux5x60(xr[t][f + 3] + xr[t][f + 4], xr[t][f + 1], xr[t][f + 2], xr[t][f + 3],
                               xr[t][f + 4], xr[t][f + 5], xr[t][f + 6]);
        real vr[kTX + 8], wr[kTX + 8], zr[kTX + 8], tr[kTX + 8], out[kTX];
        const real* vn = vp + (t + 1) * kVW;
        vr[3] = vn[3];
        ld_span<VA, 4, 4 + kTX>(vr, vn);
        const real* wrow = wp + t * kVW;
        wr[3] = wrow[3];
        ld_span<VA, 4, 4 + kTX>(wr, wrow);
        ld_span<VA, 0, kTX>(zr, zf + t * kBW);
        ld_span<VA, 0, kTX>(tr, tp + t * kTW);
#pragma unroll
        for (int c = 0; c < kTX; ++c) {
          real* q = uq[t][c];
          q[5] = zr[c];
          // y: north face of this row; south face carried from the previous row
          const real fy_hi = kl::flux5x60(vr[3 + c] + vr[4 + c], ucol[t + 1][c], ucol[t + 2][c], ucol[t + 3][c],
                                          ucol[t + 4][c], ucol[t + 5][c], ucol[t + 6][c]);
          // z: top face of this plane; bottom face carried from the previous plane
          const real fz_top = rh_top * kl::flux5x60(wr[3 + c] + wr[4 + c], q[0], q[1], q[2], q[3], q[4], q[5]);
          out[c] = tr[c] - ((fx[c + 1] - fx[c]) * dxi120 + (fy_hi - fy_lo[c]) * dyi120 +
                            (fz_top - fz_bot[t][c]) * zfac120);
          fy_lo[c] = fy_hi;
          fz_bot[t][c] = fz_top;
#pragma unroll
          for (int m = 0; m < 5; ++m) q[m] = q[m + 1];
        }
        const int j = j0 + lj0 + t;
        if (j < jend) {
          real* dst = ut + ic + static_cast<long long>(j) * KL_JJ + kofs;
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

  // main loop of the packed variant (fp32, TILE_X in {2, 4}, aligned layout):
  // the same flux-form march with the arithmetic of column pairs (c, c+1)
  // in f2 registers.  x faces: the first-level operand sums of a face pair
  // mix even- and odd-aligned columns, so they are scalar FADDs whose results
  // pair up freely; everything after them is packed.  y and z faces read
  // operands of the same column pair, which the vectorised shared loads
  // already hold as aligned register pairs.
  template <int VA>
  __device__ __forceinline__ void march2() const {
    using kl::f2;
    constexpr long long K1 = KL_KK;
    f2 uq[kTY][kP][6];  // u[k-2 .. k+3] of every column pair
    f2 fz_bot[kTY][kP];
    wait_first();
    {
      const f2 rh0(rhorefh[k0]);
      const real* wp = ring_v + kWO + wofs;  // v/w/ut slot 0 = plane k0
#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        const int j = min(j0 + lj0 + t, jend - 1);
        real wr[kTX + 8];
        wr[3] = wp[t * kVW + 3];
        ld_span<VA, 4, 4 + kTX>(wr, wp + t * kVW);
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int c = 2 * p;
          const long long rowk = static_cast<long long>(j) * KL_JJ + static_cast<long long>(k0) * KL_KK;
          const long long b0 = min(ic + c, iend - 1) + rowk, b1 = min(ic + c + 1, iend - 1) + rowk;
          const f2 um3(u_at(b0, -3), u_at(b1, -3));  // planes below the chunk: not staged
#pragma unroll
          for (int m = 0; m < 5; ++m) uq[t][p][m] = f2(u_at(b0, m - 2), u_at(b1, m - 2));
          const f2 vel(wr[3 + c] + wr[4 + c], wr[4 + c] + wr[5 + c]);
          fz_bot[t][p] = rh0 * kl::flux5x60(vel, um3, uq[t][p][0], uq[t][p][1], uq[t][p][2], uq[t][p][3],
                                             uq[t][p][4]);
        }
      }
    }
    const f2 dx2(dxi120), dy2(dyi120);

    Cursor cur;
    const bool active = j0 + lj0 < jend;  // a strip past the block's last row only keeps the barriers
    for (int k = k0; k < k1; ++k) {
      const Planes pl = begin_step(k, cur);
      if (!active) continue;
      if (KL_SKEL) {
        const long long kofs = static_cast<long long>(k) * K1;
#pragma unroll
        for (int t = 0; t < kTY; ++t) {
          real tr[kTX], out[kTX];
          ld_span<VA, 0, kTX>(tr, pl.tp + t * kTW);
#pragma unroll
          for (int c = 0; c < kTX; ++c) out[c] = tr[c] + real(1);
          const int j = j0 + lj0 + t;
          if (j < jend && ic + kTX <= iend) st_span<VA>(ut + ic + static_cast<long long>(j) * KL_JJ + kofs, out);
        }
        continue;
      }
      const real *xy = pl.xy, *zf = pl.zf, *vp = pl.vp, *wp = pl.wp, *tp = pl.tp;
      const f2 rh_top(zprof[2 * (k - k0)]);
      const f2 zfac(zprof[2 * (k - k0) + 1]);
      const long long kofs = static_cast<long long>(k) * K1;

      // u along y in this thread's columns: rows lj0-3 .. lj0+kTY+2
      real ucol[kTY + 6][kTX];
#pragma unroll
      for (int m = 0; m < kTY + 6; ++m) {
        if (m >= 3 && m < kTY + 3) continue;  // strip rows: taken from the x rows below
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
      auto ucp = [&](int m, int p) { return f2(ucol[m][2 * p], ucol[m][2 * p + 1]); };
      // south faces of the strip (row j0+lj0-1/2)
      f2 fy_lo[kP];
      {
        real vr[kTX + 8];
        vr[3] = vp[3];
        ld_span<VA, 4, 4 + kTX>(vr, vp);
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int c = 2 * p;
          const f2 vel(vr[3 + c] + vr[4 + c], vr[4 + c] + vr[5 + c]);
          fy_lo[p] = kl::flux5x60(vel, ucp(0, p), ucp(1, p), ucp(2, p), ucp(3, p), ucp(4, p), ucp(5, p));
        }
      }

#pragma unroll
      for (int t = 0; t < kTY; ++t) {
        // x: faces f = 0..kTX sit between columns ic+f-1 and ic+f; face pairs
        // (f, f+1) from scalar first-level sums, the last face alone
        const real* r = xr[t];
        real fx[kTX + 1];
#pragma unroll
        for (int f = 0; f < kTX; f += 2) {
          const f2 s_cd(r[f + 3] + r[f + 4], r[f + 4] + r[f + 5]);
          const f2 s_be(r[f + 2] + r[f + 5], r[f + 3] + r[f + 6]);
          const f2 s_af(r[f + 1] + r[f + 6], r[f + 2] + r[f + 7]);
          const f2 d_dc(r[f + 4] - r[f + 3], r[f + 5] - r[f + 4]);
          const f2 d_eb(r[f + 5] - r[f + 2], r[f + 6] - r[f + 3]);
          const f2 d_fa(r[f + 6] - r[f + 1], r[f + 7] - r[f + 2]);
          const f2 fl = kl::flux5x60_sd(s_cd, s_cd, s_be, s_af, d_dc, d_eb, d_fa);
          fx[f] = fl.lo();
          fx[f + 1] = fl.hi();
        }
        fx[kTX] = kl::flux5x60(r[kTX + 3] + r[kTX + 4], r[kTX + 1], r[kTX + 2], r[kTX + 3], r[kTX + 4],
                               r[kTX + 5], r[kTX + 6]);
        real vr[kTX + 8], wr[kTX + 8], zr[kTX + 8], tr[kTX + 8], out[kTX];
        const real* vn = vp + (t + 1) * kVW;
        vr[3] = vn[3];
        ld_span<VA, 4, 4 + kTX>(vr, vn);
        const real* wrow = wp + t * kVW;
        wr[3] = wrow[3];
        ld_span<VA, 4, 4 + kTX>(wr, wrow);
        ld_span<VA, 0, kTX>(zr, zf + t * kBW);
        ld_span<VA, 0, kTX>(tr, tp + t * kTW);
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int c = 2 * p;
          f2* q = uq[t][p];
          q[5] = f2(zr[c], zr[c + 1]);
          // y: north face of this row; south face carried from the previous row
          const f2 vel_n(vr[3 + c] + vr[4 + c], vr[4 + c] + vr[5 + c]);
          const f2 fy_hi = kl::flux5x60(vel_n, ucp(t + 1, p), ucp(t + 2, p), ucp(t + 3, p), ucp(t + 4, p),
                                        ucp(t + 5, p), ucp(t + 6, p));
          // z: top face of this plane; bottom face carried from the previous plane
          const f2 vel_t(wr[3 + c] + wr[4 + c], wr[4 + c] + wr[5 + c]);
          const f2 fz_top = rh_top * kl::flux5x60(vel_t, q[0], q[1], q[2], q[3], q[4], q[5]);
          const f2 dfx(fx[c + 1] - fx[c], fx[c + 2] - fx[c + 1]);
          const f2 o = f2(tr[c], tr[c + 1]) -
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
          real* dst = ut + ic + static_cast<long long>(j) * KL_JJ + kofs;
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

namespace {
// selects the packed main loop without instantiating it for fp64 / TILE_X == 1
template <bool kPacked>
struct Marcher {
  template <int VA>
  static __device__ __forceinline__ void run(const AdvecTma& m) { m.march<VA>(); }
};
template <>
struct Marcher<true> {
  template <int VA>
  static __device__ __forceinline__ void run(const AdvecTma& m) { m.march2<VA>(); }
};
}  // namespace

// positions: ut=0 u=1 v=2 w=3, jj / kk = KL_POS_JJ / KL_POS_KK (definitions.ARG_LAYOUT["advec_u"],
// ["advec_u_peer"]: + u_hi = 9, w_hi = 10 as maps 4, 5)
#define KL_J KL_POS_JJ
#define KL_K KL_POS_KK
#define KL_NMAPS (4 + 2 * KL_PEER)
extern "C" __device__ const int kl_tma_spec[1 + 5 * KL_NMAPS] = {
    KL_NMAPS, 1, KL_J, KL_K, kBW, kBH, 2, KL_J, KL_K, kVW, kVH, 3, KL_J, KL_K, kVW, kTYT, 0, KL_J, KL_K, kTW, kTYT
#if KL_PEER
    , 9, KL_J, KL_K, kBW, kBH, 10, KL_J, KL_K, kVW, kTYT
#endif
};
#undef KL_J
#undef KL_K
struct __align__(64) KlTmaParams {
  TmaDesc map[KL_NMAPS];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, const real* __restrict__ u, const real* __restrict__ v,
         const real* __restrict__ w, const real* __restrict__ rhoref, const real* __restrict__ rhorefh,
         const real* __restrict__ dzi KL_PEER_BUFFERS, const real dxi, const real dyi KL_PEER_SCALARS,
         const int jj, const int kk, const int istart, const int jstart, const int kstart, const int iend,
         const int jend, const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  // param-space address of the descriptors (__grid_constant__: no local copy)
  const TmaDesc* const maps = &tma.map[0];
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* sbase = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sbase);  // kNU + kNV <= 16 mbarriers
  real* const ring_u = reinterpret_cast<real*>(sbase + 128);                 // [kNU][kUS]
  real* const ring_v = ring_u + kNU * kUS;                                    // [kNV][kVS]
  real* const zprof = ring_v + kNV * kVS;                                     // [ZCHUNK][2]

  const unsigned nbx = kl::ceil_div(iend - istart, kXT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  // rows of this block: tiles of kTYT rows, or (ysplit > 0, KL_YBAL) the y
  // extent cut into nby near-equal runs of at most kTYT rows, nby taken from
  // the launched grid — the definition sizes it to whole waves of the SMs
  // (definitions.YSPLIT_VALUES), whatever jtot / kTYT is
  const int jt = jend - jstart;
  const unsigned nby = KL_YBAL > 0 ? gridDim.x / (nbx * nbz) : kl::ceil_div(jt, kTYT);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * kXT;
  const int j0 = KL_YBAL > 0 ? jstart + static_cast<int>((static_cast<long long>(by) * jt) / nby)
                             : jstart + by * kTYT;
  const int jhi = KL_YBAL > 0 ? jstart + static_cast<int>((static_cast<long long>(by + 1) * jt) / nby) : jend;
  if (KL_YBAL > 0 && jhi - j0 > kTYT) __trap();  // the grid must hold >= ceil(jt / kTYT) row runs
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  // box starts: tensor x of column i0-4 (u, v, w) / i0 (ut) rounded down to
  // 16 B; the rounding shifts the columns by sh_* within the boxes
  const int xu = i0 - 4 + kl::tma_xoff(u), xv = i0 - 4 + kl::tma_xoff(v), xw = i0 - 4 + kl::tma_xoff(w);
  const int xt = i0 + kl::tma_xoff(ut);
  const int sh_u = xu & (kE - 1), sh_v = xv & (kE - 1), sh_w = xw & (kE - 1), sh_t = xt & (kE - 1);

  AdvecTma m;
  m.ut = ut;
  m.u = u;
#if KL_PEER
  m.u_lo = u_lo;
  m.u_hi = u_hi;
  m.peer_klo = peer_klo;
  m.peer_khi = peer_khi;
  m.peer_shift_lo = peer_shift_lo;
  m.peer_shift_hi = peer_shift_hi;
#endif
  m.rhoref = rhoref;
  m.rhorefh = rhorefh;
  m.dzi = dzi;
  m.ring_u = ring_u;
  m.ring_v = ring_v;
  m.zprof = zprof;
  m.bar_u = bars;
  m.bar_v = bars + kNU;
  m.maps = maps;
  m.dxi120 = dxi * real(1.0 / 120.0);
  m.dyi120 = dyi * real(1.0 / 120.0);
  m.j0 = j0;
  m.k0 = k0;
  m.k1 = k1;
  m.tid = tid;
  m.iend = iend;
  m.jend = jhi;
  m.xu = xu - sh_u;
  m.xv = xv - sh_v;
  m.xw = xw - sh_w;
  m.xt = xt - sh_t;
  m.ic = i0 + kTX * static_cast<int>(threadIdx.x);  // first column of this thread
  m.lj0 = threadIdx.y * kTY;
  m.uofs = sh_u + (m.lj0 + 3) * kBW + kTX * threadIdx.x;  // (ic-4, j0+lj0) in the u box
  m.vofs = sh_v + m.lj0 * kVW + kTX * threadIdx.x;        // (ic-4, j0+lj0) in the v box
  m.wofs = sh_w + m.lj0 * kVW + kTX * threadIdx.x;        // (ic-4, j0+lj0) in the w box
  m.tofs = sh_t + m.lj0 * kTW + kTX * threadIdx.x;        // (ic, j0+lj0) in the ut box

  if (tid == 0) {
    for (int s = 0; s < kNU + kNV; ++s) kl::mbar_init(bars + s, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) m.prime();
  for (int q = tid; q < k1 - k0; q += KL_THREADS) {
    zprof[2 * q] = rhorefh[k0 + q + 1];
    zprof[2 * q + 1] = dzi[k0 + q] / (rhoref[k0 + q] * real(120));
  }
  // (the march's first __syncthreads publishes zprof)
  if (kVA > 1 && (sh_u | sh_v | sh_w | sh_t) == 0) {
    Marcher<kPack>::template run<kVA>(m);
  } else {
    m.march<1>();
  }
}
