// diff_uvw_flux.cuh — flux-form plane step shared by the ZMARCH and TMA
// variants of diff_uvw (see diff_uvw_zmarch.cuh for the reuse scheme).
// Every face quantity of A.3 is evaluated once: upper-y quantities of row j
// are reused by row j+1 inside a thread's TILE_Y strip, upper-z quantities
// (z fluxes and the x/y fluxes of w, which live at k+1/2) are carried to the
// next plane in `DiffCarry`.

#ifndef DIFF_UVW_FLUX_CUH
#define DIFF_UVW_FLUX_CUH

namespace {

// Quantities on the z-face k+1/2 carried to the next plane.  The south y-face
// flux of w at row t is the north one of row t-1, so only the strip's
// lowest (fyw_lo) is stored separately.
struct DiffCarry {
  real fzu[TILE_Y], fzv[TILE_Y], gz[TILE_Y];
  real fxw_p[TILE_Y], fxw_m[TILE_Y], fyw_p[TILE_Y];
  real fyw_lo;
};

// One plane step.  p0/p1 point at (strip row -1, this column) of planes k and
// k+1 of field 0 (evisc) in the shared-memory ring; fields are `fs` elements
// apart, rows SW elements.  With OUT=false only the carried upper-z
// quantities are produced (the prologue at plane k0-1).
// West-face value from the lane on the left: with warps laid along x
// (BLOCK_X % 32 == 0) every x-face quantity is evaluated once per face — lane
// l's east value is lane l+1's west value — and only lane 0 evaluates its own.
#define KL_XSHFL ((BLOCK_X % 32) == 0)

template <class F>
__device__ __forceinline__ real from_west(real east, F&& own) {
#if KL_XSHFL
  real v = __shfl_up_sync(0xffffffffu, east, 1);
  if ((threadIdx.x & 31) == 0) v = own();
  return v;
#else
  (void)east;
  return own();
#endif
}

template <bool OUT, int SW, class Store>
__device__ __forceinline__ void diff_step(const real* __restrict__ p0, const real* __restrict__ p1, int fs,
                                          DiffCarry& c, real dxi, real dyi, real c2x, real c2y, real rh1,
                                          real dzhi1, real rdz, real fac_uv, real fac_w, Store&& store) {
  const real q = real(0.25);
  // field accessors on the planes: f = 0 evisc, 1 u, 2 v, 3 w; row offset r (0 = strip row -1), column di
#define P0(f, r, di) p0[(f) * fs + (r) * SW + (di)]
#define P1(f, r, di) p1[(f) * fs + (r) * SW + (di)]
  // registers of the current row (starts at strip row -1)
  real e_0 = P0(0, 0, 0), e_p = P0(0, 0, 1);
  real u_0 = P0(1, 0, 0), u_p = P0(1, 0, 1);
  real v_0 = P0(2, 0, 0);
  real e1_0 = P1(0, 0, 0), w1_0 = P1(3, 0, 0), v1_0 = P1(2, 0, 0);
  // upper-y quantities of the previous row (row -1 computes them first)
  real exy_i = 0, exy_i1 = 0, fyu = 0, gy = 0, eyz = 0, fyw = 0;
  real u_lo0 = 0, u_lop = 0, w1_lo = 0;
  real fyw_prev = 0;

#pragma unroll
  for (int t = -1; t < TILE_Y; ++t) {
    const int r = t + 1;
    // upper neighbours (row j+1)
    const real e_01 = P0(0, r + 1, 0), e_p1 = P0(0, r + 1, 1);
    const real u_01 = P0(1, r + 1, 0), v_01 = P0(2, r + 1, 0);
    const real e1_01 = P1(0, r + 1, 0), w1_01 = P1(3, r + 1, 0), v1_01 = P1(2, r + 1, 0);
    // upper y-face quantities of row j
    const real exy_i1_up = q * (e_0 + e_p + e_01 + e_p1);
    const real exy_i_up = from_west(exy_i1_up, [&] { return q * (P0(0, r, -1) + e_0 + P0(0, r + 1, -1) + e_01); });
    const real fyu_up = exy_i_up * ((u_01 - u_0) * dyi + (v_01 - P0(2, r + 1, -1)) * dxi);
    const real gy_up = e_0 * (v_01 - v_0);
    const real eyz_up = q * (e_0 + e_01 + e1_0 + e1_01);
    const real fyw_up = eyz_up * ((w1_01 - w1_0) * dyi + (v1_01 - v_01) * dzhi1);

    if (t >= 0) {
      // z-face quantities at k+1/2 (the prologue needs them too)
      const real e1_p = P1(0, r, 1), u1_0 = P1(1, r, 0), u1_p = P1(1, r, 1), w1_p = P1(3, r, 1);
      const real w1_m = P1(3, r, -1);
      const real exz_i1 = q * (e_0 + e_p + e1_0 + e1_p);
      const real exz_i = from_west(exz_i1, [&] { return q * (P0(0, r, -1) + e_0 + P1(0, r, -1) + e1_0); });
      const real fzu = rh1 * exz_i * ((u1_0 - u_0) * dzhi1 + (w1_0 - w1_m) * dxi);
      const real fzv = rh1 * eyz * ((v1_0 - v_0) * dzhi1 + (w1_0 - w1_lo) * dyi);
      const real gz = rdz * e_0 * (w1_0 - P0(3, r, 0));
      const real fxw_p = exz_i1 * ((w1_p - w1_0) * dxi + (u1_p - u_p) * dzhi1);
      const real fxw_m = from_west(fxw_p, [&] { return exz_i * ((w1_0 - w1_m) * dxi + (u1_0 - u_0) * dzhi1); });

      if (OUT) {
        const real v_p = P0(2, r, 1);
        const real gx_i = e_0 * (u_p - u_0);
        const real gx_im = from_west(gx_i, [&] { return P0(0, r, -1) * (u_0 - P0(1, r, -1)); });
        const real fxv_p = exy_i1 * ((v_p - v_0) * dxi + (u_p - u_lop) * dyi);
        const real fxv_m =
            from_west(fxv_p, [&] { return exy_i * ((v_0 - P0(2, r, -1)) * dxi + (u_0 - u_lo0) * dyi); });
        const real fyw_s = t == 0 ? c.fyw_lo : fyw_prev;  // previous plane's south face of this row
        store(t, c2x * (gx_i - gx_im) + (fyu_up - fyu) * dyi + (fzu - c.fzu[t]) * fac_uv,
              (fxv_p - fxv_m) * dxi + c2y * (gy_up - gy) + (fzv - c.fzv[t]) * fac_uv,
              (c.fxw_p[t] - c.fxw_m[t]) * dxi + (c.fyw_p[t] - fyw_s) * dyi + (gz - c.gz[t]) * fac_w);
      }
      c.fzu[t] = fzu;
      c.fzv[t] = fzv;
      c.gz[t] = gz;
      c.fxw_m[t] = fxw_m;
      if (t == 0) c.fyw_lo = fyw;
      fyw_prev = c.fyw_p[t];  // previous plane's north face of row t = south face of row t+1
      c.fyw_p[t] = fyw_up;
      c.fxw_p[t] = fxw_p;
    }

    // slide the strip: row j+1 becomes row j
    u_lo0 = u_0;
    u_lop = u_p;
    w1_lo = w1_0;
    exy_i = exy_i_up;
    exy_i1 = exy_i1_up;
    fyu = fyu_up;
    gy = gy_up;
    eyz = eyz_up;
    fyw = fyw_up;
    e_0 = e_01;
    e_p = e_p1;
    u_0 = u_01;
    u_p = P0(1, r + 1, 1);
    v_0 = v_01;
    e1_0 = e1_01;
    w1_0 = w1_01;
    v1_0 = v1_01;
  }
#undef P0
#undef P1
}

}  // namespace

#endif  // DIFF_UVW_FLUX_CUH
