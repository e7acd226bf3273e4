/*
 * stencil_ref.c — plain-C restatement of the MicroHH interior stencils
 * (SURVEY.md Appendix A.2 advec_u, A.3 diff_uvw) — TEST INFRASTRUCTURE ONLY.
 *
 * Second, independent CPU restatement next to oracle/stencil_oracle.py (NumPy):
 * tests/test_oracle.py checks the two agree; bench.py times this one (all host
 * threads, each on a z-chunk; ctypes drops the GIL) as the CPU baseline.  Parity
 * with upstream MicroHH is UNPINNED (the kernels are a third-party dependency
 * absent from /root/reference — see oracle/__init__.py).
 *
 * Arrays are C-order [k][j][i] with a row pitch `jj` and plane pitch `kk`
 * (elements) and ghost cells around the interior [istart,iend) x
 * [jstart,jend) x [kstart,kend) — the same layout the GPU kernels use.
 * Built by oracle/Makefile into oracle/_build/libstencil_ref.so (gcc -O3) and
 * bound with ctypes in oracle/cref.py.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

#define IDX(i, j, k) ((i) + (ptrdiff_t)(j) * jj + (ptrdiff_t)(k) * kk)

#define DEFINE_KERNELS(T, SUFFIX)                                                                              \
  static inline T i6_##SUFFIX(T a, T b, T c, T d, T e, T f) { return ((T)37 * (c + d) - (T)8 * (b + e) + (a + f)) / (T)60; } \
  static inline T i5_##SUFFIX(T a, T b, T c, T d, T e, T f) { return ((T)10 * (d - c) - (T)5 * (e - b) + (f - a)) / (T)60; } \
  static inline T fl_##SUFFIX(T vel, T a, T b, T c, T d, T e, T f) {                                           \
    return vel * i6_##SUFFIX(a, b, c, d, e, f) - (T)fabs((double)vel) * i5_##SUFFIX(a, b, c, d, e, f);        \
  }                                                                                                            \
                                                                                                               \
  void advec_u_##SUFFIX(T* ut, const T* u, const T* v, const T* w, const T* rhoref, const T* rhorefh,         \
                        const T* dzi, T dxi, T dyi, int jj, ptrdiff_t kk, int istart, int iend, int jstart,   \
                        int jend, int kstart, int kend) {                                                      \
    const ptrdiff_t I = 1, J = jj, K = kk;                                                                     \
                                                                                                               \
    for (int k = kstart; k < kend; ++k)                                                                        \
      for (int j = jstart; j < jend; ++j)                                                                      \
        for (int i = istart; i < iend; ++i) {                                                                  \
          const ptrdiff_t n = IDX(i, j, k);                                                                    \
          const T* c = u + n;                                                                                  \
          const T ue = (T)0.5 * (c[0] + c[I]), uw = (T)0.5 * (c[-I] + c[0]);                                   \
          const T fx = fl_##SUFFIX(ue, c[-2 * I], c[-I], c[0], c[I], c[2 * I], c[3 * I]) -                     \
                       fl_##SUFFIX(uw, c[-3 * I], c[-2 * I], c[-I], c[0], c[I], c[2 * I]);                     \
          const T vn = (T)0.5 * (v[n - I + J] + v[n + J]), vs = (T)0.5 * (v[n - I] + v[n]);                    \
          const T fy = fl_##SUFFIX(vn, c[-2 * J], c[-J], c[0], c[J], c[2 * J], c[3 * J]) -                     \
                       fl_##SUFFIX(vs, c[-3 * J], c[-2 * J], c[-J], c[0], c[J], c[2 * J]);                     \
          const T wt = (T)0.5 * (w[n - I + K] + w[n + K]), wb = (T)0.5 * (w[n - I] + w[n]);                    \
          const T fz = rhorefh[k + 1] * fl_##SUFFIX(wt, c[-2 * K], c[-K], c[0], c[K], c[2 * K], c[3 * K]) -     \
                       rhorefh[k] * fl_##SUFFIX(wb, c[-3 * K], c[-2 * K], c[-K], c[0], c[K], c[2 * K]);         \
          ut[n] += -fx * dxi - fy * dyi - fz / rhoref[k] * dzi[k];                                             \
        }                                                                                                      \
  }                                                                                                            \
                                                                                                               \
  void diff_uvw_##SUFFIX(T* ut, T* vt, T* wt, const T* e, const T* u, const T* v, const T* w, const T* dzi,    \
                         const T* dzhi, const T* rhoref, const T* rhorefh, T dxi, T dyi, int jj, ptrdiff_t kk, \
                         int istart, int iend, int jstart, int jend, int kstart, int kend) {                  \
    const ptrdiff_t I = 1, J = jj, K = kk;                                                                     \
    const T q = (T)0.25;                                                                                       \
                                                                                                               \
    for (int k = kstart; k < kend; ++k)                                                                        \
      for (int j = jstart; j < jend; ++j)                                                                      \
        for (int i = istart; i < iend; ++i) {                                                                  \
          const ptrdiff_t n = IDX(i, j, k);                                                                    \
          const T* E = e + n;                                                                                  \
          const T* U = u + n;                                                                                  \
          const T* V = v + n;                                                                                  \
          const T* W = w + n;                                                                                  \
          const T e0 = E[0];                                                                                   \
          {                                                                                                    \
            const T en = q * (E[-I] + e0 + E[-I + J] + E[J]), es = q * (E[-I - J] + E[-J] + E[-I] + e0);      \
            const T et = q * (E[-I] + e0 + E[-I + K] + E[K]), eb = q * (E[-I - K] + E[-K] + E[-I] + e0);      \
            ut[n] += (e0 * (U[I] - U[0]) * dxi - E[-I] * (U[0] - U[-I]) * dxi) * (T)2 * dxi +                  \
                     (en * ((U[J] - U[0]) * dyi + (V[J] - V[-I + J]) * dxi) -                                  \
                      es * ((U[0] - U[-J]) * dyi + (V[0] - V[-I]) * dxi)) * dyi +                              \
                     (rhorefh[k + 1] * et * ((U[K] - U[0]) * dzhi[k + 1] + (W[K] - W[-I + K]) * dxi) -         \
                      rhorefh[k] * eb * ((U[0] - U[-K]) * dzhi[k] + (W[0] - W[-I]) * dxi)) / rhoref[k] * dzi[k]; \
          }                                                                                                    \
          {                                                                                                    \
            const T ee = q * (E[-J] + e0 + E[I - J] + E[I]), ew = q * (E[-I - J] + E[-I] + E[-J] + e0);        \
            const T et = q * (E[-J] + e0 + E[-J + K] + E[K]), eb = q * (E[-J - K] + E[-K] + E[-J] + e0);      \
            vt[n] += (ee * ((V[I] - V[0]) * dxi + (U[I] - U[I - J]) * dyi) -                                   \
                      ew * ((V[0] - V[-I]) * dxi + (U[0] - U[-J]) * dyi)) * dxi +                              \
                     (e0 * (V[J] - V[0]) * dyi - E[-J] * (V[0] - V[-J]) * dyi) * (T)2 * dyi +                  \
                     (rhorefh[k + 1] * et * ((V[K] - V[0]) * dzhi[k + 1] + (W[K] - W[-J + K]) * dyi) -         \
                      rhorefh[k] * eb * ((V[0] - V[-K]) * dzhi[k] + (W[0] - W[-J]) * dyi)) / rhoref[k] * dzi[k]; \
          }                                                                                                    \
          {                                                                                                    \
            const T ee = q * (E[-K] + e0 + E[I - K] + E[I]), ew = q * (E[-I - K] + E[-I] + E[-K] + e0);        \
            const T en = q * (E[-K] + e0 + E[J - K] + E[J]), es = q * (E[-J - K] + E[-J] + E[-K] + e0);        \
            wt[n] += (ee * ((W[I] - W[0]) * dxi + (U[I] - U[I - K]) * dzhi[k]) -                               \
                      ew * ((W[0] - W[-I]) * dxi + (U[0] - U[-K]) * dzhi[k])) * dxi +                          \
                     (en * ((W[J] - W[0]) * dyi + (V[J] - V[J - K]) * dzhi[k]) -                               \
                      es * ((W[0] - W[-J]) * dyi + (V[0] - V[-K]) * dzhi[k])) * dyi +                          \
                     (rhoref[k] * e0 * (W[K] - W[0]) * dzi[k] -                                                \
                      rhoref[k - 1] * E[-K] * (W[0] - W[-K]) * dzi[k - 1]) / rhorefh[k] * (T)2 * dzhi[k];       \
          }                                                                                                    \
        }                                                                                                      \
  }

DEFINE_KERNELS(double, f64)
DEFINE_KERNELS(float, f32)

/* Synthetic input fields, bit-exact with oracle/synth.py and the device
 * generator klb_synth_field (value of element (i,j,k) = draw n+1 of
 * SplitMix64(seed), n the global logical index with periodic x/y ghosts,
 * mapped to [lo, hi) by two IEEE double ops — no FMA contraction: -std=c11).
 * Fills planes [k0, k1) of a contiguous (kcells, jcells, icells) array whose
 * plane 0 is global plane k_offset; the CPU reference arm fills whole 1024^3
 * grids with it, one z-chunk per host thread. */
static inline uint64_t synth_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

#define DEFINE_SYNTH(T, SUFFIX)                                                                          \
  void synth_field_##SUFFIX(T* out, uint64_t seed, double lo, double hi, int icells, int jcells, int igc, \
                            int jgc, int k_offset, int k0, int k1) {                                      \
    const int itot = icells - 2 * igc, jtot = jcells - 2 * jgc;                                           \
    const double span = hi - lo;                                                                          \
    for (int k = k0; k < k1; ++k)                                                                         \
      for (int j = 0; j < jcells; ++j) {                                                                  \
        const int js = jgc + ((j - jgc) % jtot + jtot) % jtot;                                            \
        T* row = out + ((ptrdiff_t)k * jcells + j) * icells;                                              \
        for (int i = 0; i < icells; ++i) {                                                                \
          const int is = igc + ((i - igc) % itot + itot) % itot;                                          \
          const uint64_t n = ((uint64_t)(k + k_offset) * jcells + js) * icells + is;                      \
          const uint64_t h = synth_mix64(seed + (n + 1ull) * 0x9E3779B97F4A7C15ull);                      \
          const double x = (double)(h >> 11) * 0x1.0p-53;                                                 \
          row[i] = (T)(lo + span * x);                                                                    \
        }                                                                                                 \
      }                                                                                                   \
  }

DEFINE_SYNTH(float, f32)
DEFINE_SYNTH(double, f64)
