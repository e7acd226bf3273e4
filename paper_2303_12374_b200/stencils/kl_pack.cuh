// kl_pack.cuh — packed fp32 pairs for the runtime-compiled stencils.
//
// sm_100 issues FADD2 / FMUL2 / FFMA2: one instruction operates on a pair of
// fp32 values held in an aligned register pair (NVRTC builtins __fadd2_rn,
// __fmul2_rn, __ffma2_rn; operand negation and |x| fold into modifiers and a
// broadcast constant into an immediate).  The fp32 flux-form stencils are
// issue-bound, so evaluating the arithmetic of two neighbouring columns per
// instruction halves their FP instruction count.  `f2` is that pair; the
// _rn intrinsics are never contracted, so every FMA is written explicitly.

#ifndef KL_PACK_CUH
#define KL_PACK_CUH

namespace kl {

struct f2 {
  float2 v;
  __device__ __forceinline__ f2() {}
  __device__ __forceinline__ f2(float a, float b) : v(make_float2(a, b)) {}
  __device__ __forceinline__ explicit f2(float a) : v(make_float2(a, a)) {}
  __device__ __forceinline__ float lo() const { return v.x; }
  __device__ __forceinline__ float hi() const { return v.y; }
};

__device__ __forceinline__ f2 mk2(float2 v) {
  f2 r;
  r.v = v;
  return r;
}
__device__ __forceinline__ f2 operator+(f2 a, f2 b) { return mk2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator-(f2 a, f2 b) { return mk2(__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))); }
__device__ __forceinline__ f2 operator*(f2 a, f2 b) { return mk2(__fmul2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return mk2(__ffma2_rn(a.v, b.v, c.v)); }
__device__ __forceinline__ f2 nabs2(f2 a) { return mk2(make_float2(-fabsf(a.v.x), -fabsf(a.v.y))); }

// 60 x the 5th-order upwind flux of two faces from the first-level operand
// sums / differences: s_cd = c+d, s_be = b+e, s_af = a+f, d_dc = d-c,
// d_eb = e-b, d_fa = f-a (see kl_common.cuh flux5x60).
__device__ __forceinline__ f2 flux5x60_sd(f2 vel, f2 s_cd, f2 s_be, f2 s_af, f2 d_dc, f2 d_eb, f2 d_fa) {
  const f2 i6 = fma2(f2(37.f), s_cd, fma2(f2(-8.f), s_be, s_af));
  const f2 i5 = fma2(f2(10.f), d_dc, fma2(f2(-5.f), d_eb, d_fa));
  return fma2(nabs2(vel), i5, vel * i6);
}

// The same from the six operands of both faces (already paired).
__device__ __forceinline__ f2 flux5x60(f2 vel, f2 a, f2 b, f2 c, f2 d, f2 e, f2 f) {
  return flux5x60_sd(vel, c + d, b + e, a + f, d - c, e - b, f - a);
}

// fp64 has no packed instructions: d2 is the same interface over two doubles
// (two scalar instructions per operation), so pair-structured kernels serve
// both precisions from one source.
struct d2 {
  double x, y;
  __device__ __forceinline__ d2() {}
  __device__ __forceinline__ d2(double a, double b) : x(a), y(b) {}
  __device__ __forceinline__ explicit d2(double a) : x(a), y(a) {}
  __device__ __forceinline__ double lo() const { return x; }
  __device__ __forceinline__ double hi() const { return y; }
};
__device__ __forceinline__ d2 operator+(d2 a, d2 b) { return d2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ d2 operator-(d2 a, d2 b) { return d2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ d2 operator*(d2 a, d2 b) { return d2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ d2 fma2(d2 a, d2 b, d2 c) { return d2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y)); }
__device__ __forceinline__ d2 nabs2(d2 a) { return d2(-fabs(a.x), -fabs(a.y)); }
__device__ __forceinline__ d2 flux5x60_sd(d2 vel, d2 s_cd, d2 s_be, d2 s_af, d2 d_dc, d2 d_eb, d2 d_fa) {
  const d2 i6 = fma2(d2(37.0), s_cd, fma2(d2(-8.0), s_be, s_af));
  const d2 i5 = fma2(d2(10.0), d_dc, fma2(d2(-5.0), d_eb, d_fa));
  return fma2(nabs2(vel), i5, vel * i6);
}
__device__ __forceinline__ d2 flux5x60(d2 vel, d2 a, d2 b, d2 c, d2 d, d2 e, d2 f) {
  return flux5x60_sd(vel, c + d, b + e, a + f, d - c, e - b, f - a);
}

// square roots: fp32 uses the hardware approximation (sqrt.approx, max
// relative error 2^-23 — far inside the 1e-5 parity bar, and one MUFU instead
// of the IEEE-rounded sequence with its special-case branch); fp64 stays exact
__device__ __forceinline__ float sqrt_fast(float a) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double sqrt_fast(double a) { return sqrt(a); }
__device__ __forceinline__ f2 sqrt2(f2 a) { return f2(sqrt_fast(a.v.x), sqrt_fast(a.v.y)); }
__device__ __forceinline__ d2 sqrt2(d2 a) { return d2(sqrt(a.x), sqrt(a.y)); }
__device__ __forceinline__ float sqrt2(float a) { return sqrt_fast(a); }
__device__ __forceinline__ double sqrt2(double a) { return sqrt(a); }

// the pair type of a precision
template <class T>
struct pair_of;
template <>
struct pair_of<float> {
  using type = f2;
};
template <>
struct pair_of<double> {
  using type = d2;
};

}  // namespace kl

#endif  // KL_PACK_CUH
