/*
 * family_ref.c — plain-C restatement of the rest of the MicroHH stencil family
 * (advec_v, advec_w, advec_s, diff_c, evisc_smag) — TEST INFRASTRUCTURE ONLY.
 *
 * The same formulas as oracle/family_oracle.py (NumPy), in float64, cell by
 * cell over a k-range, so the GPU kernels of SURVEY §8f row 2 can be checked
 * against every cell of their benchmarked 512^3 grids in seconds
 * (tests/stencil_helpers.cref_chunks); tests/test_oracle.py
 * (test_cref_chunks_cover_the_grid_like_the_numpy_oracle) checks the two
 * restatements agree.  Parity with upstream MicroHH is UNPINNED (a
 * third-party dependency absent from /root/reference — see oracle/__init__.py).
 *
 * Layout as in stencil_ref.c: C-order [k][j][i], row pitch jj, plane pitch
 * kk (elements), ghost cells around [istart,iend) x [jstart,jend) x
 * [kstart,kend).  Staggering (Arakawa C): u at (i-1/2, j, k), v at
 * (i, j-1/2, k), w at (i, j, k-1/2), scalars / evisc / rhoref at centres,
 * rhorefh and dzhi at k-1/2.
 */
#include <math.h>
#include <stddef.h>

static inline double i6(double a, double b, double c, double d, double e, double f) {
  return (37.0 * (c + d) - 8.0 * (b + e) + (a + f)) / 60.0;
}
static inline double i5(double a, double b, double c, double d, double e, double f) {
  return (10.0 * (d - c) - 5.0 * (e - b) + (f - a)) / 60.0;
}
static inline double fl(double vel, const double* p, ptrdiff_t s) {
  /* 5th-order upwind flux through the face between p[0] and p[s] */
  const double a = p[-2 * s], b = p[-s], c = p[0], d = p[s], e = p[2 * s], f = p[3 * s];
  return vel * i6(a, b, c, d, e, f) - fabs(vel) * i5(a, b, c, d, e, f);
}
/* -(divergence of the upwind fluxes of phi at n): face velocities west/east,
 * south/north, bottom/top; rh_* weight the z faces, fac the z metric */
static inline double advect(const double* phi, ptrdiff_t n, ptrdiff_t J, ptrdiff_t K, double vw, double ve,
                            double vs, double vn, double vb, double vt, double rh_bot, double rh_top, double fac,
                            double dxi, double dyi) {
  const double* c = phi + n;
  const double fx = fl(ve, c, 1) - fl(vw, c - 1, 1);
  const double fy = fl(vn, c, J) - fl(vs, c - J, J);
  const double fz = rh_top * fl(vt, c, K) - rh_bot * fl(vb, c - K, K);
  return -fx * dxi - fy * dyi - fz * fac;
}

#define LOOP                                       \
  const ptrdiff_t I = 1, J = jj, K = kk;           \
  (void)I;                                         \
  for (int k = kstart; k < kend; ++k)              \
    for (int j = jstart; j < jend; ++j)            \
      for (int i = istart; i < iend; ++i)

#define BOUNDS int jj, ptrdiff_t kk, int istart, int iend, int jstart, int jend, int kstart, int kend

void advec_v_f64(double* vt, const double* u, const double* v, const double* w, const double* rhoref,
                 const double* rhorefh, const double* dzi, double dxi, double dyi, BOUNDS) {
  LOOP {
    const ptrdiff_t n = i + j * J + k * K;
    vt[n] += advect(v, n, J, K, 0.5 * (u[n - J] + u[n]), 0.5 * (u[n + I - J] + u[n + I]),
                    0.5 * (v[n - J] + v[n]), 0.5 * (v[n] + v[n + J]), 0.5 * (w[n - J] + w[n]),
                    0.5 * (w[n - J + K] + w[n + K]), rhorefh[k], rhorefh[k + 1], dzi[k] / rhoref[k], dxi, dyi);
  }
}

void advec_w_f64(double* wt, const double* u, const double* v, const double* w, const double* rhoref,
                 const double* rhorefh, const double* dzhi, double dxi, double dyi, BOUNDS) {
  LOOP {
    const ptrdiff_t n = i + j * J + k * K;
    wt[n] += advect(w, n, J, K, 0.5 * (u[n - K] + u[n]), 0.5 * (u[n + I - K] + u[n + I]),
                    0.5 * (v[n - K] + v[n]), 0.5 * (v[n + J - K] + v[n + J]), 0.5 * (w[n - K] + w[n]),
                    0.5 * (w[n] + w[n + K]), rhoref[k - 1], rhoref[k], dzhi[k] / rhorefh[k], dxi, dyi);
  }
}

void advec_s_f64(double* st, const double* s, const double* u, const double* v, const double* w,
                 const double* rhoref, const double* rhorefh, const double* dzi, double dxi, double dyi, BOUNDS) {
  LOOP {
    const ptrdiff_t n = i + j * J + k * K;
    st[n] += advect(s, n, J, K, u[n], u[n + I], v[n], v[n + J], w[n], w[n + K], rhorefh[k], rhorefh[k + 1],
                    dzi[k] / rhoref[k], dxi, dyi);
  }
}

void diff_c_f64(double* st, const double* s, const double* e, const double* dzi, const double* dzhi,
                const double* rhoref, const double* rhorefh, double dxi, double dyi, double tpri, BOUNDS) {
  LOOP {
    const ptrdiff_t n = i + j * J + k * K;
    const double s0 = s[n], e0 = e[n];
    const double ee = 0.5 * (e0 + e[n + I]) * tpri, ew = 0.5 * (e[n - I] + e0) * tpri;
    const double en = 0.5 * (e0 + e[n + J]) * tpri, es = 0.5 * (e[n - J] + e0) * tpri;
    const double et = 0.5 * (e0 + e[n + K]) * tpri, eb = 0.5 * (e[n - K] + e0) * tpri;
    st[n] += (ee * (s[n + I] - s0) - ew * (s0 - s[n - I])) * dxi * dxi +
             (en * (s[n + J] - s0) - es * (s0 - s[n - J])) * dyi * dyi +
             (rhorefh[k + 1] * et * (s[n + K] - s0) * dzhi[k + 1] - rhorefh[k] * eb * (s0 - s[n - K]) * dzhi[k]) /
                 rhoref[k] * dzi[k];
  }
}

static inline double sq(double x) { return x * x; }

/* squared strain rate 2 S_ij S_ij at the centre of cell n (family_oracle.strain2) */
static inline double strain2(const double* u, const double* v, const double* w, ptrdiff_t n, ptrdiff_t J,
                             ptrdiff_t K, double dxi, double dyi, double dz, double dzh, double dzh1) {
  const ptrdiff_t I = 1;
  const double diag = 2.0 * (sq((u[n + I] - u[n]) * dxi) + sq((v[n + J] - v[n]) * dyi) + sq((w[n + K] - w[n]) * dz));
#define SXY(di, dj)                                                                                              \
  sq((u[n + (di) * I + (dj) * J] - u[n + (di) * I + ((dj) - 1) * J]) * dyi +                                    \
     (v[n + (di) * I + (dj) * J] - v[n + ((di) - 1) * I + (dj) * J]) * dxi)
#define SXZ(di, dk, h)                                                                                           \
  sq((u[n + (di) * I + (dk) * K] - u[n + (di) * I + ((dk) - 1) * K]) * (h) +                                    \
     (w[n + (di) * I + (dk) * K] - w[n + ((di) - 1) * I + (dk) * K]) * dxi)
#define SYZ(dj, dk, h)                                                                                           \
  sq((v[n + (dj) * J + (dk) * K] - v[n + (dj) * J + ((dk) - 1) * K]) * (h) +                                    \
     (w[n + (dj) * J + (dk) * K] - w[n + ((dj) - 1) * J + (dk) * K]) * dyi)
  const double off = 0.25 * (SXY(0, 0) + SXY(0, 1) + SXY(1, 0) + SXY(1, 1) + SXZ(0, 0, dzh) + SXZ(0, 1, dzh1) +
                              SXZ(1, 0, dzh) + SXZ(1, 1, dzh1) + SYZ(0, 0, dzh) + SYZ(0, 1, dzh1) + SYZ(1, 0, dzh) +
                              SYZ(1, 1, dzh1));
#undef SXY
#undef SXZ
#undef SYZ
  return diag + off;
}

void evisc_smag_f64(double* evisc, const double* u, const double* v, const double* w, const double* dzi,
                    const double* dzhi, double dxi, double dyi, double cs, BOUNDS) {
  LOOP {
    const ptrdiff_t n = i + j * J + k * K;
    const double mlen = cbrt(1.0 / (dxi * dyi * dzi[k]));
    const double s2 = strain2(u, v, w, n, J, K, dxi, dyi, dzi[k], dzhi[k], dzhi[k + 1]);
    evisc[n] = sq(cs * mlen) * sqrt(s2);
  }
}
