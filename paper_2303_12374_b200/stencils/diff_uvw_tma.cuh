// diff_uvw_tma.cuh — STAGING == TMA variant of diff_uvw (included by
// diff_uvw.cu).  Flux-form z-march (the reuse scheme of diff_uvw_flux.cuh)
// with every operand fetched by the Tensor Memory Accelerator: one elected
// thread issues cp.async.bulk.tensor.3d copies DEPTH planes ahead of the
// compute into a (DEPTH+2)-slot shared-memory ring, each slot completing on
// its own mbarrier (expect_tx bytes).  A slot holds plane p of
//   * evisc, u, v, w with a 1-cell x/y halo (the stencil reads planes k, k+1),
//   * ut, vt, wt without halo (the read half of the read-modify-write),
// so the compute warps issue no global loads — only the final stores of the
// updated tendencies.  Staging costs no registers, and DEPTH planes x 7
// fields of every block are in flight.
//
// A thread owns TILE_X consecutive columns (TILE_X in {1, 2, 4}; CONTIG_X)
// times a strip of TILE_Y rows.  Every face quantity of A.3 is evaluated
// once per thread: x-faces (the x fluxes, the xy/xz edge viscosities) TILE_X+1
// times per row for TILE_X cells, y-faces carried from the row below, z-faces
// carried from the plane below.  Halo'd boxes start at column i0-kE (kE =
// elements per 16 bytes), so when column i0 is 16-byte aligned in every field
// (always, for GridLayout pitches) a thread's cells sit at vector-aligned
// shared offsets: a row of TILE_X+2 values is TILE_X/VA + 2 loads of VA
// elements (VA = min(TILE_X, kE)), and the tendency reads and stores are
// VA-wide too.  A uniform branch falls back to scalar shared reads (and
// global tendency reads) for any other alignment.  Out-of-box rows/columns
// are zero-filled by TMA and only feed cells that are never stored.

#if BLOCK_Z != 1 || TILE_Z != 1
#error "diff_uvw TMA requires BLOCK_Z == TILE_Z == 1"
#endif
#if TILE_X != 1 && TILE_X != 2 && TILE_X != 4
#error "diff_uvw TMA requires TILE_X in {1, 2, 4}"
#endif
#if TILE_X > 1 && !CONTIG_X
#error "diff_uvw TMA: TILE_X > 1 needs consecutive columns (CONTIG_X)"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif
#ifndef KL_L2PF
#define KL_L2PF 0  // > 0: also prefetch plane p + KL_L2PF into L2 when plane p is loaded into the ring
#endif

#include "kl_pack.cuh"
#include "kl_tma.cuh"

namespace {
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;  // elements per 16 bytes
constexpr int kTX = TILE_X, kTY = TILE_Y;
constexpr int kXT = BLOCK_X * kTX;   // columns per block
constexpr int kTYT = BLOCK_Y * kTY;  // rows per block
constexpr int kVA = kTX < kE ? kTX : kE;
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }
// halo'd box: columns from (i0 - kE) rounded down to 16 B, kXT + 2 kE wide
constexpr int kBW = rup(kXT + 2 * kE, kE);
constexpr int kBH = kTYT + 2;
constexpr int kTW = rup(kXT, kE);  // tendency box: columns i0 .. i0+kXT-1 (start rounded down)
constexpr int kFSB = rup(kBW * kBH * kS, 128);   // bytes per halo'd field-plane
constexpr int kTSB = rup(kTW * kTYT * kS, 128);  // bytes per tendency field-plane
constexpr int kFS = kFSB / kS;
constexpr int kTS = kTSB / kS;
constexpr int kSlot = 4 * kFS + 3 * kTS;
constexpr int kNS = DEPTH + 2;
constexpr unsigned kTxBytes = 4u * kBW * kBH * kS + 3u * kTW * kTYT * kS;
// fp32 with column tiles: the arithmetic of column pairs runs on packed
// FADD2/FMUL2/FFMA2 (kl_pack.cuh)
constexpr bool kPack = sizeof(real) == 4 && kTX >= 2;
constexpr int kP = kTX / 2 > 0 ? kTX / 2 : 1;  // column pairs per thread
static_assert(kBW <= 256 && kBH <= 256 && kTW <= 256, "TMA box extents are limited to 256");

template <int N>
struct __align__(N * sizeof(real)) Pack {
  real v[N];
};

// d[m] = s[m - 1] for m in [0, kTX + 2): columns -1 .. kTX of a thread's cells
// (s points at its first column; VA-element aligned when VA > 1).
template <int VA>
__device__ __forceinline__ void ld_row(real (&d)[kTX + 2], const real* s) {
  if (VA == 1) {
#pragma unroll
    for (int m = 0; m < kTX + 2; ++m) d[m] = s[m - 1];
  } else {
    real b[kTX + 2 * VA];
#pragma unroll
    for (int e = 0; e < kTX + 2 * VA; e += VA) {
      const Pack<VA> p = *reinterpret_cast<const Pack<VA>*>(s - VA + e);
#pragma unroll
      for (int q = 0; q < VA; ++q) b[e + q] = p.v[q];
    }
#pragma unroll
    for (int m = 0; m < kTX + 2; ++m) d[m] = b[VA - 1 + m];
  }
}

// d[m] = s[m] for m in [0, N), N in {kTX, kTX + 1}
template <int VA, int N>
__device__ __forceinline__ void ld_span(real (&d)[N], const real* s) {
  if (VA == 1) {
#pragma unroll
    for (int m = 0; m < N; ++m) d[m] = s[m];
  } else {
    constexpr int R = rup(N, VA);
    real b[R];
#pragma unroll
    for (int e = 0; e < R; e += VA) {
      const Pack<VA> p = *reinterpret_cast<const Pack<VA>*>(s + e);
#pragma unroll
      for (int q = 0; q < VA; ++q) b[e + q] = p.v[q];
    }
#pragma unroll
    for (int m = 0; m < N; ++m) d[m] = b[m];
  }
}

// One shared-memory row of the strip: e/u/v at plane k, f = evisc, w,
// y = v, x = u at plane k+1, z = w at plane k; index m <-> column m-1 for the
// (kTX+2)-wide rows, column m for y, x (kTX+1 wide) and z.
struct Row {
  real e[kTX + 2], u[kTX + 2], v[kTX + 2], f[kTX + 2], w[kTX + 2];
  real y[kTX], x[kTX + 1], z[kTX];
};

// Quantities on the z-face k+1/2 carried to the next plane (per strip row
// and column; FXW per x-face).  The south y-face flux of w at row t is the
// north one of row t-1, so only the strip's lowest (fyw_lo) is stored apart.
struct Carry {
  real fzu[kTY][kTX], fzv[kTY][kTX], gz[kTY][kTX], fyw_p[kTY][kTX];
  real fxw[kTY][kTX + 1];
  real fyw_lo[kTX];
};

struct Scales {
  real sx, sy, qsx, qsy, c2x, c2y;
};

// Per-plane factors: rh1 = rhorefh[k+1], dzhi1 = dzhi[k+1], rdz =
// rhoref[k]*dzi[k], qfac = dzi[k]/(4 rhoref[k]), fac_w = 2 dzhi[k]/rhorefh[k].
struct PlaneFactors {
  real rh1, dzhi1, rdz, qfac, fac_w;
};

// One plane step.  h0/h1: plane k / k+1 slots, pointing at (strip row -1,
// first column) of field 0 with field f at +hof[f]; with OUT=false only the
// carried upper-z quantities are produced (the prologue at plane k0-1).
template <bool OUT, int VA, class Store>
__device__ __forceinline__ void plane_step(const real* h0, const real* h1, const int (&hof)[4], Carry& c,
                                           const Scales& s, const PlaneFactors& z, Store&& store) {
  Row cur, nrt;
  auto load = [&](Row& r, int row) {
    const int ro = row * kBW;
    ld_row<VA>(r.e, h0 + hof[0] + ro);
    ld_row<VA>(r.u, h0 + hof[1] + ro);
    ld_row<VA>(r.v, h0 + hof[2] + ro);
    ld_row<VA>(r.f, h1 + hof[0] + ro);
    ld_row<VA>(r.w, h1 + hof[3] + ro);
    ld_span<VA, kTX>(r.y, h1 + hof[2] + ro);
    ld_span<VA, kTX + 1>(r.x, h1 + hof[1] + ro);
    ld_span<VA, kTX>(r.z, h0 + hof[3] + ro);
  };
  load(cur, 0);
  // y-face quantities of the current row's lower face (from the previous row)
  real sxy[kTX + 1], fyu[kTX], gy[kTX], fyw[kTX], ulo[kTX + 1], fyw_prev[kTX];
#pragma unroll
  for (int q = 0; q < kTX; ++q) fyw_prev[q] = real(0);

#pragma unroll
  for (int t = -1; t < kTY; ++t) {
    load(nrt, t + 2);
    // upper y-face quantities of this row (4 x the edge viscosities)
    real sxy_up[kTX + 1], fyu_up[kTX], gy_up[kTX], syz_up[kTX], fyw_up[kTX];
#pragma unroll
    for (int f = 0; f <= kTX; ++f) sxy_up[f] = (cur.e[f] + cur.e[f + 1]) + (nrt.e[f] + nrt.e[f + 1]);
#pragma unroll
    for (int q = 0; q < kTX; ++q) {
      fyu_up[q] = sxy_up[q] * ((nrt.u[q + 1] - cur.u[q + 1]) * s.sy + (nrt.v[q + 1] - nrt.v[q]) * s.sx);
      gy_up[q] = cur.e[q + 1] * (nrt.v[q + 1] - cur.v[q + 1]);
      syz_up[q] = (cur.e[q + 1] + nrt.e[q + 1]) + (cur.f[q + 1] + nrt.f[q + 1]);
      fyw_up[q] = syz_up[q] * ((nrt.w[q + 1] - cur.w[q + 1]) * s.sy + (nrt.y[q] - nrt.v[q + 1]) * z.dzhi1);
    }

    if (t >= 0) {
      // x-faces f (between columns f-1 and f) of the xz edge viscosity and w's x flux
      real sxz[kTX + 1], fxw[kTX + 1];
#pragma unroll
      for (int f = 0; f <= kTX; ++f) {
        sxz[f] = (cur.e[f] + cur.e[f + 1]) + (cur.f[f] + cur.f[f + 1]);
        fxw[f] = sxz[f] * ((cur.w[f + 1] - cur.w[f]) * s.sx + (cur.x[f] - cur.u[f + 1]) * z.dzhi1);
      }
      real fzu[kTX], fzv[kTX], gz[kTX];
#pragma unroll
      for (int q = 0; q < kTX; ++q) {
        // the stress tensor is symmetric: u's z flux through the top face is
        // rhorefh[k+1] x w's x flux through the west face of the cell above
        // (both tau_xz at (i-1/2, k+1/2)), and v's z flux is rhorefh[k+1] x
        // w's y flux through the south face (tau_yz at (j-1/2, k+1/2), the
        // previous row's fyw_up) — evaluated once, reused
        fzu[q] = z.rh1 * fxw[q];
        fzv[q] = z.rh1 * fyw[q];
        gz[q] = z.rdz * cur.e[q + 1] * (cur.w[q + 1] - cur.z[q]);
      }
      if (OUT) {
        real gx[kTX + 1], fxv[kTX + 1];
#pragma unroll
        for (int f = 0; f <= kTX; ++f) {
          gx[f] = cur.e[f] * (cur.u[f + 1] - cur.u[f]);
          fxv[f] = sxy[f] * ((cur.v[f + 1] - cur.v[f]) * s.sx + (cur.u[f + 1] - ulo[f]) * s.sy);
        }
        real dut[kTX], dvt[kTX], dwt[kTX];
#pragma unroll
        for (int q = 0; q < kTX; ++q) {
          const real fyw_s = t == 0 ? c.fyw_lo[q] : fyw_prev[q];  // previous plane's south face of this row
          dut[q] = s.c2x * (gx[q + 1] - gx[q]) + (fyu_up[q] - fyu[q]) * s.qsy + (fzu[q] - c.fzu[t][q]) * z.qfac;
          dvt[q] = (fxv[q + 1] - fxv[q]) * s.qsx + s.c2y * (gy_up[q] - gy[q]) + (fzv[q] - c.fzv[t][q]) * z.qfac;
          dwt[q] = (c.fxw[t][q + 1] - c.fxw[t][q]) * s.qsx + (c.fyw_p[t][q] - fyw_s) * s.qsy +
                   (gz[q] - c.gz[t][q]) * z.fac_w;
        }
        store(t, dut, dvt, dwt);
      }
#pragma unroll
      for (int q = 0; q < kTX; ++q) {
        c.fzu[t][q] = fzu[q];
        c.fzv[t][q] = fzv[q];
        c.gz[t][q] = gz[q];
        if (t == 0) c.fyw_lo[q] = fyw[q];
        fyw_prev[q] = c.fyw_p[t][q];  // previous plane's north face of row t = south face of row t+1
        c.fyw_p[t][q] = fyw_up[q];
      }
#pragma unroll
      for (int f = 0; f <= kTX; ++f) c.fxw[t][f] = fxw[f];
    }

    // slide the strip: the north row becomes the current row
#pragma unroll
    for (int f = 0; f <= kTX; ++f) {
      ulo[f] = cur.u[f + 1];
      sxy[f] = sxy_up[f];
    }
#pragma unroll
    for (int q = 0; q < kTX; ++q) {
      fyu[q] = fyu_up[q];
      gy[q] = gy_up[q];
      fyw[q] = fyw_up[q];
    }
    cur = nrt;
  }
}

// Carried z-face quantities of the packed variant (column pairs in f2; the
// x-face flux of w stays per face, its differences mix column parities).
struct Carry2 {
  kl::f2 fzu[kTY][kP], fzv[kTY][kP], gz[kTY][kP], fyw_p[kTY][kP];
  real fxw[kTY][kTX + 1];
  kl::f2 fyw_lo[kP];
};

// Packed plane step (fp32, kTX in {2, 4}): plane_step's arithmetic with the
// quantities of column pairs (c, c+1) in f2 registers.  x-face quantities
// need columns (f-1, f), whose pairs straddle the aligned register pairs the
// vectorised shared loads produce, so their first-level sums/differences are
// scalar (their results pair up freely) and the rest is packed for face pairs
// (0,1), (2,3) with the last face scalar.  Cell-centred and y/z quantities
// read aligned pairs directly.
template <bool OUT, int VA, class Store>
__device__ __forceinline__ void plane_step2(const real* h0, const real* h1, const int (&hof)[4], Carry2& c,
                                            const Scales& s, const PlaneFactors& z, Store&& store) {
  using kl::f2;
  Row cur, nrt;
  auto load = [&](Row& r, int row) {
    const int ro = row * kBW;
    ld_row<VA>(r.e, h0 + hof[0] + ro);
    ld_row<VA>(r.u, h0 + hof[1] + ro);
    ld_row<VA>(r.v, h0 + hof[2] + ro);
    ld_row<VA>(r.f, h1 + hof[0] + ro);
    ld_row<VA>(r.w, h1 + hof[3] + ro);
    ld_span<VA, kTX>(r.y, h1 + hof[2] + ro);
    ld_span<VA, kTX + 1>(r.x, h1 + hof[1] + ro);
    ld_span<VA, kTX>(r.z, h0 + hof[3] + ro);
  };
  // (T[1+c], T[2+c]) = columns (c, c+1) of a (kTX+2)-wide row; (T[c], T[c+1]) of y/x/z
  auto pr = [](const real* a, int c) { return f2(a[1 + c], a[2 + c]); };
  auto pc = [](const real* a, int c) { return f2(a[c], a[c + 1]); };
  const f2 sx(s.sx), sy(s.sy), dz1(z.dzhi1), rh1(z.rh1), rdz(z.rdz);
  load(cur, 0);
  // per-face sums of the current row's lower face, carried from the row below
  real eS[kTX + 1], dv[kTX + 1], sxy_l[kTX + 1];  // e pair sums, v differences, 4x edge viscosity
  f2 fyu[kP], gy[kP], fyw[kP], ulo[kP];
  real ulo_last = 0;
  f2 fyw_prev[kP];
#pragma unroll
  for (int f = 0; f <= kTX; ++f) eS[f] = cur.e[f] + cur.e[f + 1];

#pragma unroll
  for (int t = -1; t < kTY; ++t) {
    load(nrt, t + 2);
    // north row: e pair sums and v differences per face (scalar)
    real eN[kTX + 1], dvn[kTX + 1], sxy_up[kTX + 1];
#pragma unroll
    for (int f = 0; f <= kTX; ++f) {
      eN[f] = nrt.e[f] + nrt.e[f + 1];
      dvn[f] = nrt.v[f + 1] - nrt.v[f];
      sxy_up[f] = eS[f] + eN[f];
    }
    f2 fyu_up[kP], gy_up[kP], syz_up[kP], fyw_up[kP];
#pragma unroll
    for (int p = 0; p < kP; ++p) {
      const int q = 2 * p;
      const f2 e = pr(cur.e, q), en = pr(nrt.e, q), v = pr(cur.v, q), vn = pr(nrt.v, q);
      fyu_up[p] = f2(sxy_up[q], sxy_up[q + 1]) * kl::fma2(pr(nrt.u, q) - pr(cur.u, q), sy, f2(dvn[q], dvn[q + 1]) * sx);
      gy_up[p] = e * (vn - v);
      syz_up[p] = (e + en) + (pr(cur.f, q) + pr(nrt.f, q));
      fyw_up[p] = syz_up[p] * kl::fma2(pr(nrt.w, q) - pr(cur.w, q), sy, (pc(nrt.y, q) - vn) * dz1);
    }

    if (t >= 0) {
      // x-faces: sxz (4x the xz edge viscosity) and w's x flux (= tau_xz)
      real fxw[kTX + 1];
#pragma unroll
      for (int f = 0; f < kTX; f += 2) {
        const f2 sxz = f2(eS[f], eS[f + 1]) + f2(cur.f[f] + cur.f[f + 1], cur.f[f + 1] + cur.f[f + 2]);
        const f2 dw(cur.w[f + 1] - cur.w[f], cur.w[f + 2] - cur.w[f + 1]);
        const f2 fl = sxz * kl::fma2(dw, sx, (pc(cur.x, f) - pr(cur.u, f)) * dz1);
        fxw[f] = fl.lo();
        fxw[f + 1] = fl.hi();
      }
      {
        constexpr int f = kTX;
        const real sxz = eS[f] + (cur.f[f] + cur.f[f + 1]);
        fxw[f] = sxz * ((cur.w[f + 1] - cur.w[f]) * s.sx + (cur.x[f] - cur.u[f + 1]) * z.dzhi1);
      }
      f2 fzu[kP], fzv[kP], gz[kP];
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        const int q = 2 * p;
        // symmetric stress: u's z flux = rhorefh[k+1] tau_xz (w's west-face x
        // flux), v's z flux = rhorefh[k+1] tau_yz (the previous row's fyw_up)
        fzu[p] = rh1 * f2(fxw[q], fxw[q + 1]);
        fzv[p] = rh1 * fyw[p];
        gz[p] = rdz * pr(cur.e, q) * (pr(cur.w, q) - pc(cur.z, q));
      }
      if (OUT) {
        real gx[kTX + 1], fxv[kTX + 1];
#pragma unroll
        for (int f = 0; f <= kTX; ++f) gx[f] = cur.e[f] * (cur.u[f + 1] - cur.u[f]);
#pragma unroll
        for (int f = 0; f < kTX; f += 2) {
          const f2 dul = pr(cur.u, f) - ulo[f / 2];
          const f2 fl = f2(sxy_l[f], sxy_l[f + 1]) * kl::fma2(f2(dv[f], dv[f + 1]), sx, dul * sy);
          fxv[f] = fl.lo();
          fxv[f + 1] = fl.hi();
        }
        fxv[kTX] = sxy_l[kTX] * (dv[kTX] * s.sx + (cur.u[kTX + 1] - ulo_last) * s.sy);
        const f2 c2x(s.c2x), c2y(s.c2y), qsx(s.qsx), qsy(s.qsy), qfac(z.qfac), facw(z.fac_w);
        real dut[kTX], dvt[kTX], dwt[kTX];
#pragma unroll
        for (int p = 0; p < kP; ++p) {
          const int q = 2 * p;
          const f2 fyw_s = t == 0 ? c.fyw_lo[p] : fyw_prev[p];  // previous plane's south face of this row
          const f2 dgx(gx[q + 1] - gx[q], gx[q + 2] - gx[q + 1]);
          const f2 dfxv(fxv[q + 1] - fxv[q], fxv[q + 2] - fxv[q + 1]);
          const f2 dfxw(c.fxw[t][q + 1] - c.fxw[t][q], c.fxw[t][q + 2] - c.fxw[t][q + 1]);
          const f2 a = kl::fma2(c2x, dgx, kl::fma2(fyu_up[p] - fyu[p], qsy, (fzu[p] - c.fzu[t][p]) * qfac));
          const f2 b = kl::fma2(dfxv, qsx, kl::fma2(c2y, gy_up[p] - gy[p], (fzv[p] - c.fzv[t][p]) * qfac));
          const f2 d = kl::fma2(dfxw, qsx, kl::fma2(c.fyw_p[t][p] - fyw_s, qsy, (gz[p] - c.gz[t][p]) * facw));
          dut[q] = a.lo();
          dut[q + 1] = a.hi();
          dvt[q] = b.lo();
          dvt[q + 1] = b.hi();
          dwt[q] = d.lo();
          dwt[q + 1] = d.hi();
        }
        store(t, dut, dvt, dwt);
      }
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        c.fzu[t][p] = fzu[p];
        c.fzv[t][p] = fzv[p];
        c.gz[t][p] = gz[p];
        if (t == 0) c.fyw_lo[p] = fyw[p];
        fyw_prev[p] = c.fyw_p[t][p];  // previous plane's north face of row t = south face of row t+1
        c.fyw_p[t][p] = fyw_up[p];
      }
#pragma unroll
      for (int f = 0; f <= kTX; ++f) c.fxw[t][f] = fxw[f];
    }

    // slide the strip: the north row becomes the current row
#pragma unroll
    for (int f = 0; f <= kTX; ++f) {
      eS[f] = eN[f];
      dv[f] = dvn[f];
      sxy_l[f] = sxy_up[f];
    }
#pragma unroll
    for (int p = 0; p < kP; ++p) {
      ulo[p] = pr(cur.u, 2 * p);
      fyu[p] = fyu_up[p];
      gy[p] = gy_up[p];
      fyw[p] = fyw_up[p];
    }
    ulo_last = cur.u[kTX + 1];
    cur = nrt;
  }
}

template <bool kPacked>
struct Step {
  using CarryT = Carry;
  template <bool OUT, int VA, class Store>
  static __device__ __forceinline__ void run(const real* h0, const real* h1, const int (&hof)[4], CarryT& c,
                                             const Scales& s, const PlaneFactors& z, Store&& store) {
    plane_step<OUT, VA>(h0, h1, hof, c, s, z, store);
  }
};
template <>
struct Step<true> {
  using CarryT = Carry2;
  template <bool OUT, int VA, class Store>
  static __device__ __forceinline__ void run(const real* h0, const real* h1, const int (&hof)[4], CarryT& c,
                                             const Scales& s, const PlaneFactors& z, Store&& store) {
    plane_step2<OUT, VA>(h0, h1, hof, c, s, z, store);
  }
};

// Per-block state of the march (member template instead of a generic lambda:
// NVRTC has no extended device lambdas).
struct DiffTma {
  real *ut, *vt, *wt;
#if KL_RK3
  real *un, *vn, *wn;  // u, v, w of the next RK3 substep
  real rk_a, rk_bdt;
#endif
#if KL_PEER
  int peer_klo, peer_khi, peer_shift_lo, peer_shift_hi;  // planes read from the neighbours (diff_uvw.cu)
#endif
  const real* zprof;  // [ZCHUNK][5] per-plane factors
  real* ring;
  unsigned long long* full;
  const TmaDesc* maps;
  Scales sc;
  PlaneFactors pro;  // factors of the prologue plane k0-1
  int j0, k0, k1, tid, iend, jend, ic, lj0;
  int xh[4], xt;  // 16-byte aligned box starts (halo'd fields / tendencies)
  int hof[4];     // (strip row -1, column ic) of each halo'd field inside a slot
  int tofs;       // (strip row 0, column ic) inside a tendency plane

  __device__ __forceinline__ void issue(int slot, int p) const {
    unsigned long long* bar = full + slot;
    real* dst = ring + slot * kSlot;
    kl::mbar_expect_tx(bar, kTxBytes);
#if KL_PEER
    // a plane outside the slab comes from the neighbour's field (maps 7..10
    // below, 11..14 above) at the neighbour's own plane index
    const TmaDesc* hm = maps;
    int hp = p;
    if (p < peer_klo) {
      hm = maps + 7;
      hp = p + peer_shift_lo;
    } else if (p >= peer_khi) {
      hm = maps + 11;
      hp = p + peer_shift_hi;
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) kl::tma_load_3d(dst + f * kFS, hm + f, bar, xh[f], j0 - 1, hp);
#else
#pragma unroll
    for (int f = 0; f < 4; ++f) kl::tma_load_3d(dst + f * kFS, maps + f, bar, xh[f], j0 - 1, p);
#endif
#pragma unroll
    for (int f = 0; f < 3; ++f) kl::tma_load_3d(dst + 4 * kFS + f * kTS, maps + 4 + f, bar, xt, j0, p);
  }
  // L2 prefetch of plane p (KL_L2PF): DRAM reads of the planes beyond the
  // ring start early without costing shared memory
  __device__ __forceinline__ void prefetch(int p) const {
#pragma unroll
    for (int f = 0; f < 4; ++f) kl::tma_prefetch_3d(maps + f, xh[f], j0 - 1, p);
#pragma unroll
    for (int f = 0; f < 3; ++f) kl::tma_prefetch_3d(maps + 4 + f, xt, j0, p);
  }

  template <int VA, bool PK = false>
  __device__ __forceinline__ void march() const {
    using S = Step<PK>;
    typename S::CarryT carry;
    auto no_store = [](int, const real(&)[kTX], const real(&)[kTX], const real(&)[kTX]) {};
    const int kfirst = k0 - 1;
    kl::mbar_wait(full + 0, 0);  // plane kfirst
    kl::mbar_wait(full + 1, 0);  // plane k0
    S::template run<false, VA>(ring, ring + kSlot, hof, carry, sc, pro, no_store);

    int sprev = 0, sk = 1, sk1 = 2 % kNS;  // slots of planes k-1, k, k+1
    unsigned ph1 = 0;                      // barrier parity of plane k+1
    for (int k = k0; k < k1; ++k) {
      __syncthreads();  // everyone is done with plane k-1's slot
      if (tid == 0) {
        const int p = k - 1 + kNS;  // refill the slot plane k-1 vacated
        if (p <= k1) {
          kl::fence_proxy_async_smem();
          issue(sprev, p);
        }
#if KL_L2PF > 0 && !KL_PEER
        if (p + KL_L2PF <= k1) prefetch(p + KL_L2PF);
#endif
      }
      kl::mbar_wait(full + sk1, ph1);
      const real* zp = zprof + 5 * (k - k0);
      const PlaneFactors pf{zp[0], zp[1], zp[2], zp[3], zp[4]};
      const real* pk = ring + sk * kSlot;
      const real* pk1 = ring + sk1 * kSlot;
      const real* tend = pk + 4 * kFS + tofs;
      const long long kofs = static_cast<long long>(k) * KL_KK;
      // this plane's (strip row 0, first column) in each tendency: rows are
      // then immediate offsets (t * KL_JJ) from three per-plane pointers
      const long long base = ic + static_cast<long long>(j0 + lj0) * KL_JJ + kofs;
      real* const up = ut + base;
      real* const vp = vt + base;
      real* const wp = wt + base;
      const bool full_x = ic + kTX <= iend;
      auto store = [&](int t, const real(&dut)[kTX], const real(&dvt)[kTX], const real(&dwt)[kTX]) {
        if (j0 + lj0 + t >= jend) return;
        real* const ur = up + t * KL_JJ;
        real* const vr = vp + t * KL_JJ;
        real* const wr = wp + t * KL_JJ;
        real o[3][kTX];
        if (VA > 1) {
          ld_span<VA, kTX>(o[0], tend + t * kTW);
          ld_span<VA, kTX>(o[1], tend + kTS + t * kTW);
          ld_span<VA, kTX>(o[2], tend + 2 * kTS + t * kTW);
        } else {  // unaligned layout: the tendency boxes may not cover the columns
#pragma unroll
          for (int q = 0; q < kTX; ++q) {
            const bool in = ic + q < iend;
            o[0][q] = in ? ur[q] : real(0);
            o[1][q] = in ? vr[q] : real(0);
            o[2][q] = in ? wr[q] : real(0);
          }
        }
#pragma unroll
        for (int q = 0; q < kTX; ++q) {
          o[0][q] += dut[q];
          o[1][q] += dvt[q];
          o[2][q] += dwt[q];
        }
#if KL_RK3
        // fused RK3 substep: next = centre + rk_bdt T (centre u/v/w of row t
        // from the staged plane), t = rk_a T
        real nx[3][kTX];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const real* c = pk + hof[1 + f] + (t + 1) * kBW;
#pragma unroll
          for (int q = 0; q < kTX; ++q) {
            nx[f][q] = c[q] + rk_bdt * o[f][q];
            o[f][q] *= rk_a;
          }
        }
        real* const nr[3] = {un + (ur - ut), vn + (vr - vt), wn + (wr - wt)};
        if (VA > 1 && full_x) {
#pragma unroll
          for (int f = 0; f < 3; ++f)
#pragma unroll
            for (int e = 0; e < kTX; e += VA) {
              Pack<VA> a;
#pragma unroll
              for (int q = 0; q < VA; ++q) a.v[q] = nx[f][e + q];
              *reinterpret_cast<Pack<VA>*>(nr[f] + e) = a;
            }
        } else {
#pragma unroll
          for (int f = 0; f < 3; ++f)
#pragma unroll
            for (int q = 0; q < kTX; ++q)
              if (ic + q < iend) nr[f][q] = nx[f][q];
        }
#endif
        if (VA > 1 && full_x) {
#pragma unroll
          for (int e = 0; e < kTX; e += VA) {
            Pack<VA> a, b, d;
#pragma unroll
            for (int q = 0; q < VA; ++q) {
              a.v[q] = o[0][e + q];
              b.v[q] = o[1][e + q];
              d.v[q] = o[2][e + q];
            }
            *reinterpret_cast<Pack<VA>*>(ur + e) = a;
            *reinterpret_cast<Pack<VA>*>(vr + e) = b;
            *reinterpret_cast<Pack<VA>*>(wr + e) = d;
          }
        } else {
#pragma unroll
          for (int q = 0; q < kTX; ++q) {
            if (ic + q < iend) {
              ur[q] = o[0][q];
              vr[q] = o[1][q];
              wr[q] = o[2][q];
            }
          }
        }
      };
      S::template run<true, VA>(pk, pk1, hof, carry, sc, pf, store);
      sprev = sk;
      sk = sk1;
      sk1 = sk1 + 1 == kNS ? 0 : sk1 + 1;
      ph1 ^= sk1 == 0 ? 1u : 0u;
    }
  }
};
}  // namespace

// positions: ut=0 vt=1 wt=2 evisc=3 u=4 v=5 w=6, jj / kk = KL_POS_JJ / KL_POS_KK
// (definitions.ARG_LAYOUT["diff_uvw"] / ["diff_uvw_rk3"])
#define KL_J KL_POS_JJ
#define KL_K KL_POS_KK
#define KL_NMAPS (7 + 8 * KL_PEER)
extern "C" __device__ const int kl_tma_spec[1 + 5 * KL_NMAPS] = {
    KL_NMAPS, 3, KL_J, KL_K, kBW, kBH, 4, KL_J, KL_K, kBW, kBH, 5, KL_J, KL_K, kBW, kBH, 6, KL_J, KL_K, kBW, kBH,
    0, KL_J, KL_K, kTW, kTYT, 1, KL_J, KL_K, kTW, kTYT, 2, KL_J, KL_K, kTW, kTYT
#if KL_PEER
    // the neighbours' evisc, u, v, w (below, then above), same boxes as the local ones
    , KL_POS_PEER + 0, KL_J, KL_K, kBW, kBH, KL_POS_PEER + 1, KL_J, KL_K, kBW, kBH,
    KL_POS_PEER + 2, KL_J, KL_K, kBW, kBH, KL_POS_PEER + 3, KL_J, KL_K, kBW, kBH,
    KL_POS_PEER + 4, KL_J, KL_K, kBW, kBH, KL_POS_PEER + 5, KL_J, KL_K, kBW, kBH,
    KL_POS_PEER + 6, KL_J, KL_K, kBW, kBH, KL_POS_PEER + 7, KL_J, KL_K, kBW, kBH
#endif
};
#undef KL_J
#undef KL_K
struct __align__(64) KlTmaParams {
  TmaDesc map[KL_NMAPS];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, const real* __restrict__ evisc,
         const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh KL_RK3_BUFFERS KL_PEER_BUFFERS, const real dxi,
         const real dyi KL_RK3_SCALARS KL_PEER_SCALARS,
         const int jj, const int kk, const int istart, const int jstart, const int kstart, const int iend,
         const int jend, const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  const kl::PdlTriggerAtExit kl_pdl_exit;  // programmatic dependent launch (kl_common.cuh)
  kl::pdl_wait();     // no global access before the previous kernel on the stream has completed
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* base = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base);  // kNS mbarriers
  real* const ring = reinterpret_cast<real*>(base + 128);                  // [kNS][kSlot]

  const unsigned nbx = kl::ceil_div(iend - istart, kXT);
  const unsigned nby = kl::ceil_div(jend - jstart, kTYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * kXT;
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;

  DiffTma m;
  m.ut = ut;
  m.vt = vt;
  m.wt = wt;
#if KL_RK3
  m.un = un;
  m.vn = vn;
  m.wn = wn;
  m.rk_a = rk_a;
  m.rk_bdt = rk_bdt;
#endif
#if KL_PEER
  m.peer_klo = peer_klo;
  m.peer_khi = peer_khi;
  m.peer_shift_lo = peer_shift_lo;
  m.peer_shift_hi = peer_shift_hi;
  // (the peer fields share the local layout, so their boxes start at the
  // local x coordinates; the host checks the 16-byte phase of each pointer)
#endif
  m.ring = ring;
  m.full = full;
  m.maps = &tma.map[0];  // param-space address of the descriptors (__grid_constant__: no local copy)
  m.j0 = jstart + by * kTYT;
  m.k0 = kstart + bz * ZCHUNK;
  m.k1 = min(m.k0 + ZCHUNK, kend);
  m.tid = tid;
  m.iend = iend;
  m.jend = jend;
  m.ic = i0 + kTX * static_cast<int>(threadIdx.x);
  m.lj0 = threadIdx.y * kTY;
  // box starts: tensor x of column i0-kE (halo'd) / i0 (tendencies) rounded
  // down to 16 B (each base pointer may carry its own sub-16-byte offset,
  // tma_xoff); the fast path needs column i0 at box column kE (halo'd) / 0
  const real* hp[4] = {evisc, u, v, w};
  const int xt = i0 + kl::tma_xoff(ut);
  m.xt = xt & ~(kE - 1);
  bool aligned = xt == m.xt && kl::tma_xoff(vt) == kl::tma_xoff(ut) && kl::tma_xoff(wt) == kl::tma_xoff(ut);
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int x = i0 - kE + kl::tma_xoff(hp[f]);
    m.xh[f] = x & ~(kE - 1);
    aligned = aligned && x == m.xh[f];
    m.hof[f] = f * kFS + m.lj0 * kBW + (x - m.xh[f]) + kE + kTX * static_cast<int>(threadIdx.x);
  }
  m.tofs = m.lj0 * kTW + (xt - m.xt) + kTX * static_cast<int>(threadIdx.x);
  m.sc.sx = dxi;
  m.sc.sy = dyi;
  m.sc.qsx = real(0.25) * dxi;
  m.sc.qsy = real(0.25) * dyi;
  m.sc.c2x = real(2) * dxi * dxi;
  m.sc.c2y = real(2) * dyi * dyi;
  const int kfirst = m.k0 - 1;
  m.pro = PlaneFactors{rhorefh[m.k0], dzhi[m.k0], rhoref[kfirst] * dzi[kfirst], real(0), real(0)};

  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) kl::mbar_init(full + s, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    for (int p = kfirst; p <= min(kfirst + kNS - 1, m.k1); ++p) m.issue(p - kfirst, p);
#if KL_L2PF > 0 && !KL_PEER
    for (int p = kfirst + kNS; p < min(kfirst + kNS + KL_L2PF, m.k1 + 1); ++p) m.prefetch(p);
#endif
  }
  // per-plane factors of the chunk (one division per plane and block instead
  // of two per thread and plane; published by the march's first __syncthreads)
  real* const zprof = ring + kNS * kSlot;  // [ZCHUNK][5]
  for (int q = tid; q < m.k1 - m.k0; q += KL_THREADS) {
    const int k = m.k0 + q;
    zprof[5 * q + 0] = rhorefh[k + 1];
    zprof[5 * q + 1] = dzhi[k + 1];
    zprof[5 * q + 2] = rhoref[k] * dzi[k];
    zprof[5 * q + 3] = real(0.25) * dzi[k] / rhoref[k];
    zprof[5 * q + 4] = real(2) * dzhi[k] / rhorefh[k];
  }
  m.zprof = zprof;
  if (kVA > 1 && aligned) {
    m.march<kVA, kPack>();
  } else {
    m.march<1>();
  }
}
