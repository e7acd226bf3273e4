// diff_uvw_tma.cuh — STAGING == TMA variant of diff_uvw (included by
// diff_uvw.cu).  Same flux-form plane step as ZMARCH (diff_uvw_flux.cuh), but
// every operand is fetched by the Tensor Memory Accelerator: one elected
// thread issues cp.async.bulk.tensor.3d copies DEPTH planes ahead of the
// compute into a (DEPTH+2)-slot shared-memory ring, each slot completing on
// its own mbarrier (expect_tx bytes).  A slot holds plane p of
//   * evisc, u, v, w with a 1-cell x/y halo (the stencil reads planes k, k+1),
//   * ut, vt, wt without halo (the read half of the read-modify-write),
// so the compute warps issue no global loads at all — only the final
// stores of the updated tendencies.  Staging costs no registers, and DEPTH
// planes x 7 fields of every block are in flight (ncu on the register-staged
// ZMARCH variant: long_scoreboard-bound at 25% occupancy).  Box starts are
// rounded down to 16-byte aligned x (TMA faults otherwise); out-of-box
// rows/columns are zero-filled and only feed cells that are never stored.

#if BLOCK_Z != 1 || TILE_Z != 1 || TILE_X != 1
#error "diff_uvw TMA requires BLOCK_Z == TILE_Z == TILE_X == 1"
#endif
#ifndef DEPTH
#define DEPTH 2
#endif

#include "diff_uvw_flux.cuh"
#include "kl_tma.cuh"

namespace {
constexpr int kS = static_cast<int>(sizeof(real));
constexpr int kE = 16 / kS;  // elements per 16 bytes
constexpr int kTYT = BLOCK_Y * TILE_Y;
// halo'd box: BLOCK_X + 2 columns plus up to kE-1 alignment columns, 16-B multiple
constexpr int kBW = (((BLOCK_X + 2) * kS + 16 - kS + 15) / 16) * 16 / kS;
constexpr int kBH = kTYT + 2;
// tendency box: BLOCK_X columns (+ alignment slack), no halo
constexpr int kTW = ((BLOCK_X * kS + 16 - kS + 15) / 16) * 16 / kS;
constexpr int kFSB = ((kBW * kBH * kS + 127) / 128) * 128;   // bytes per halo'd field-plane
constexpr int kTSB = ((kTW * kTYT * kS + 127) / 128) * 128;  // bytes per tendency field-plane
constexpr int kFS = kFSB / kS;
constexpr int kTS = kTSB / kS;
constexpr int kSlot = 4 * kFS + 3 * kTS;
constexpr int kNS = DEPTH + 2;
constexpr unsigned kTxBytes = 4u * kBW * kBH * kS + 3u * kTW * kTYT * kS;
static_assert(kBW <= 256 && kBH <= 256 && kTW <= 256, "TMA box extents are limited to 256");
}  // namespace

// positions: ut=0 vt=1 wt=2 evisc=3 u=4 v=5 w=6, jj=13 kk=14 (definitions.ARG_LAYOUT["diff_uvw"])
extern "C" __device__ const int kl_tma_spec[1 + 5 * 7] = {
    7, 3, 13, 14, kBW, kBH, 4, 13, 14, kBW, kBH, 5, 13, 14, kBW, kBH, 6, 13, 14, kBW, kBH,
    0, 13, 14, kTW, kTYT, 1, 13, 14, kTW, kTYT, 2, 13, 14, kTW, kTYT};
struct __align__(64) KlTmaParams {
  TmaDesc map[7];
};

extern "C" __global__ void __launch_bounds__(KL_THREADS, MIN_BLOCKS)
KL_ENTRY(real* __restrict__ ut, real* __restrict__ vt, real* __restrict__ wt, const real* __restrict__ evisc,
         const real* __restrict__ u, const real* __restrict__ v, const real* __restrict__ w,
         const real* __restrict__ dzi, const real* __restrict__ dzhi, const real* __restrict__ rhoref,
         const real* __restrict__ rhorefh, const real dxi, const real dyi, const int jj, const int kk,
         const int istart, const int jstart, const int kstart, const int iend, const int jend, const int kend, const __grid_constant__ KlTmaParams tma) {
  if (jj != KL_JJ || kk != KL_KK) __trap();
  // param-space address of the descriptors (__grid_constant__: no local copy)
  const TmaDesc* const maps = &tma.map[0];
  extern __shared__ __align__(128) unsigned char kl_smem_raw[];
  unsigned char* base = kl_smem_raw + ((128u - (kl::smem_u32(kl_smem_raw) & 127u)) & 127u);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base);  // kNS mbarriers
  real* const ring = reinterpret_cast<real*>(base + 128);                  // [kNS][4][kFS]

  const unsigned nbx = kl::ceil_div(iend - istart, BLOCK_X);
  const unsigned nby = kl::ceil_div(jend - jstart, kTYT);
  const unsigned nbz = kl::ceil_div(kend - kstart, ZCHUNK);
  int bx, by, bz;
  kl::unravel(blockIdx.x, nbx, nby, nbz, bx, by, bz);
  const int i0 = istart + bx * BLOCK_X;
  const int j0 = jstart + by * kTYT;
  const int k0 = kstart + bz * ZCHUNK;
  const int k1 = min(k0 + ZCHUNK, kend);
  const int tid = threadIdx.x + threadIdx.y * BLOCK_X;
  const int xfirst = i0 - 1 + kl::tma_xoff(evisc);  // tensor x of column i0-1 (all fields share the layout)
  const int x0 = xfirst & ~(kE - 1);               // 16-byte aligned box start
  const int cshift = xfirst - x0;                  // extra leading columns in the tile
  const int xt0 = (xfirst + 1) & ~(kE - 1);        // tendency box start (column i0)
  const int tshift = xfirst + 1 - xt0;
  const int kfirst = k0 - 1;                     // first staged plane

  // plane p lives in slot (p - kfirst) % kNS; its mbarrier phase is ((p - kfirst) / kNS) & 1
  auto issue = [&](int slot, int p) {
    unsigned long long* bar = full + slot;
    real* dst = ring + slot * kSlot;
    kl::mbar_expect_tx(bar, kTxBytes);
#pragma unroll
    for (int f = 0; f < 4; ++f) kl::tma_load_3d(dst + f * kFS, maps + f, bar, x0, j0 - 1, p);
#pragma unroll
    for (int f = 0; f < 3; ++f) kl::tma_load_3d(dst + 4 * kFS + f * kTS, maps + 4 + f, bar, xt0, j0, p);
  };

  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) kl::mbar_init(full + s, 1);
    kl::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    for (int p = kfirst; p <= min(kfirst + kNS - 1, k1); ++p) issue(p - kfirst, p);
  }
  // per-plane factors of the chunk (one division per plane and block instead
  // of two per thread and plane; published by the loop's first __syncthreads)
  real* const zprof = ring + kNS * kSlot;  // [ZCHUNK][5]
  for (int q = tid; q < k1 - k0; q += KL_THREADS) {
    const int k = k0 + q;
    zprof[5 * q + 0] = rhorefh[k + 1];
    zprof[5 * q + 1] = dzhi[k + 1];
    zprof[5 * q + 2] = rhoref[k] * dzi[k];
    zprof[5 * q + 3] = real(0.25) * dzi[k] / rhoref[k];
    zprof[5 * q + 4] = real(2) * dzhi[k] / rhorefh[k];
  }

  const real c2x = real(2) * dxi * dxi;
  const real c2y = real(2) * dyi * dyi;
  const real qsx = real(0.25) * dxi, qsy = real(0.25) * dyi;
  const int lj0 = threadIdx.y * TILE_Y;
  const int off = lj0 * kBW + threadIdx.x + 1 + cshift;  // (strip row -1, this column) inside a field-plane
  const int i = i0 + threadIdx.x;
  DiffCarry carry;
  auto no_store = [](int, real, real, real) {};

  kl::mbar_wait(full + 0, 0);  // plane kfirst
  kl::mbar_wait(full + 1, 0);  // plane k0
  diff_step<false, kBW>(ring + off, ring + kSlot + off, kFS, carry, dxi, dyi, qsx, qsy, c2x, c2y,
                        rhorefh[k0], dzhi[k0], rhoref[kfirst] * dzi[kfirst], real(0), real(0), no_store);

  const int toff = lj0 * kTW + threadIdx.x + tshift;  // (strip row 0, this column) in a tendency plane
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
    }
    kl::mbar_wait(full + sk1, ph1);
    const real* zp = zprof + 5 * (k - k0);
    const real* pk = ring + sk * kSlot;
    const real* pk1 = ring + sk1 * kSlot;
    const real* tend = pk + 4 * kFS + toff;
    const long long kofs = static_cast<long long>(k) * KL_KK;
    auto store = [&](int t, real dut, real dvt, real dwt) {
      const int j = j0 + lj0 + t;
      if (i < iend && j < jend) {
        const long long ijk = i + static_cast<long long>(j) * KL_JJ + kofs;
        ut[ijk] = tend[t * kTW] + dut;
        vt[ijk] = tend[kTS + t * kTW] + dvt;
        wt[ijk] = tend[2 * kTS + t * kTW] + dwt;
      }
    };
    diff_step<true, kBW>(pk + off, pk1 + off, kFS, carry, dxi, dyi, qsx, qsy, c2x, c2y, zp[0], zp[1], zp[2], zp[3],
                         zp[4], store);
    sprev = sk;
    sk = sk1;
    sk1 = sk1 + 1 == kNS ? 0 : sk1 + 1;
    ph1 ^= sk1 == 0 ? 1u : 0u;
  }
}
