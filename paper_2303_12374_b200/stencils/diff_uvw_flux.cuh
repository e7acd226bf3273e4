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
//
// Register discipline: every value of the strip's next row (19 loads) is read
// once and slides down to become the current row, so each shared-memory
// element is loaded once per thread; the 1/4 of the edge viscosity averages is
// folded into the scale factors qsx = dxi/4, qsy = dyi/4, qfac = fac_uv/4.
// (x-faces are evaluated by both neighbouring cells: sharing them through
// warp shuffles costs more issue slots than it saves — lane 0's own
// evaluation runs as a divergent branch in every warp.)
template <bool OUT, int SW, class Store>
__device__ __forceinline__ void diff_step(const real* __restrict__ p0, const real* __restrict__ p1, int fs,
                                          DiffCarry& c, real sx, real sy, real qsx, real qsy, real c2x, real c2y,
                                          real rh1, real dzhi1, real rdz, real qfac, real fac_w, Store&& store) {
#define P0(f, r, di) p0[(f) * fs + (r) * SW + (di)]
#define P1(f, r, di) p1[(f) * fs + (r) * SW + (di)]
  // current row (starts at strip row -1): e/u/v at plane k; f = evisc, w, y = v, x = u at
  // plane k+1; z = w at plane k
  real e_m = P0(0, 0, -1), e_0 = P0(0, 0, 0), e_p = P0(0, 0, 1);
  real u_m = P0(1, 0, -1), u_0 = P0(1, 0, 0), u_p = P0(1, 0, 1);
  real v_m = P0(2, 0, -1), v_0 = P0(2, 0, 0), v_p = P0(2, 0, 1);
  real f_m = P1(0, 0, -1), f_0 = P1(0, 0, 0), f_p = P1(0, 0, 1);
  real w_m = P1(3, 0, -1), w_0 = P1(3, 0, 0), w_p = P1(3, 0, 1);
  real y_0 = P1(2, 0, 0), x_0 = P1(1, 0, 0), x_p = P1(1, 0, 1), z_0 = P0(3, 0, 0);
  // upper-y quantities of the previous row
  real sxy_i = 0, sxy_i1 = 0, fyu = 0, gy = 0, syz = 0, fyw = 0;
  real u_lo0 = 0, u_lop = 0, w_lo = 0, fyw_prev = 0;

#pragma unroll
  for (int t = -1; t < TILE_Y; ++t) {
    const int rn = t + 2;  // ring row of the north neighbour row
    const real en_m = P0(0, rn, -1), en_0 = P0(0, rn, 0), en_p = P0(0, rn, 1);
    const real un_m = P0(1, rn, -1), un_0 = P0(1, rn, 0), un_p = P0(1, rn, 1);
    const real vn_m = P0(2, rn, -1), vn_0 = P0(2, rn, 0), vn_p = P0(2, rn, 1);
    const real fn_m = P1(0, rn, -1), fn_0 = P1(0, rn, 0), fn_p = P1(0, rn, 1);
    const real wn_m = P1(3, rn, -1), wn_0 = P1(3, rn, 0), wn_p = P1(3, rn, 1);
    const real yn_0 = P1(2, rn, 0), xn_0 = P1(1, rn, 0), xn_p = P1(1, rn, 1), zn_0 = P0(3, rn, 0);

    // upper y-face quantities of this row (4 x the edge viscosities)
    const real sxy_i_up = e_m + e_0 + en_m + en_0;
    const real sxy_i1_up = e_0 + e_p + en_0 + en_p;
    const real fyu_up = sxy_i_up * ((un_0 - u_0) * sy + (vn_0 - vn_m) * sx);
    const real gy_up = e_0 * (vn_0 - v_0);
    const real syz_up = e_0 + en_0 + f_0 + fn_0;
    const real fyw_up = syz_up * ((wn_0 - w_0) * sy + (yn_0 - vn_0) * dzhi1);

    if (t >= 0) {
      // z-face quantities at k+1/2 (the prologue needs them too)
      const real sxz_i = e_m + e_0 + f_m + f_0;
      const real sxz_i1 = e_0 + e_p + f_0 + f_p;
      const real fzu = rh1 * sxz_i * ((x_0 - u_0) * dzhi1 + (w_0 - w_m) * sx);
      const real fzv = rh1 * syz * ((y_0 - v_0) * dzhi1 + (w_0 - w_lo) * sy);
      const real gz = rdz * e_0 * (w_0 - z_0);
      const real fxw_p = sxz_i1 * ((w_p - w_0) * sx + (x_p - u_p) * dzhi1);
      const real fxw_m = sxz_i * ((w_0 - w_m) * sx + (x_0 - u_0) * dzhi1);
      if (OUT) {
        const real gx_i = e_0 * (u_p - u_0);
        const real gx_im = e_m * (u_0 - u_m);
        const real fxv_p = sxy_i1 * ((v_p - v_0) * sx + (u_p - u_lop) * sy);
        const real fxv_m = sxy_i * ((v_0 - v_m) * sx + (u_0 - u_lo0) * sy);
        const real fyw_s = t == 0 ? c.fyw_lo : fyw_prev;  // previous plane's south face of this row
        store(t, c2x * (gx_i - gx_im) + (fyu_up - fyu) * qsy + (fzu - c.fzu[t]) * qfac,
              (fxv_p - fxv_m) * qsx + c2y * (gy_up - gy) + (fzv - c.fzv[t]) * qfac,
              (c.fxw_p[t] - c.fxw_m[t]) * qsx + (c.fyw_p[t] - fyw_s) * qsy + (gz - c.gz[t]) * fac_w);
      }
      c.fzu[t] = fzu;
      c.fzv[t] = fzv;
      c.gz[t] = gz;
      c.fxw_m[t] = fxw_m;
      c.fxw_p[t] = fxw_p;
      if (t == 0) c.fyw_lo = fyw;
      fyw_prev = c.fyw_p[t];  // previous plane's north face of row t = south face of row t+1
      c.fyw_p[t] = fyw_up;
    }

    // slide the strip: the north row becomes the current row
    u_lo0 = u_0;
    u_lop = u_p;
    w_lo = w_0;
    sxy_i = sxy_i_up;
    sxy_i1 = sxy_i1_up;
    fyu = fyu_up;
    gy = gy_up;
    syz = syz_up;
    fyw = fyw_up;
    e_m = en_m; e_0 = en_0; e_p = en_p;
    u_m = un_m; u_0 = un_0; u_p = un_p;
    v_m = vn_m; v_0 = vn_0; v_p = vn_p;
    f_m = fn_m; f_0 = fn_0; f_p = fn_p;
    w_m = wn_m; w_0 = wn_0; w_p = wn_p;
    y_0 = yn_0; x_0 = xn_0; x_p = xn_p; z_0 = zn_0;
  }
#undef P0
#undef P1
}

}  // namespace

#endif  // DIFF_UVW_FLUX_CUH
