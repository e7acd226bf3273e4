// kl_common.cuh — shared prelude of the runtime-compiled MicroHH stencils.
//
// Every tunable parameter of the selected configuration arrives as a -D
// define rendered by KernelDefinition.render_compile_request (reference
// kerneldef.py:188-211): ints verbatim, bools as true/false, strings bare
// (so UNRAVEL=ZYX names one of the macros below).  The Table-2 knobs
// map to code as follows:
//   BLOCK_{X,Y,Z}     blockDim
//   TILE_{X,Y,Z}      cells per thread along each axis
//   UNROLL_{X,Y,Z}    #pragma unroll (full) vs #pragma unroll 1 on the tile loop
//   CONTIG_{X,Y,Z}    true: a thread's cells are consecutive (x, x+1, ...);
//                     false: block-strided (x, x+BLOCK_X, ...)
//   UNRAVEL           order in which the 1-D block id is unravelled into
//                     (bx, by, bz); first letter varies fastest
//   MIN_BLOCKS        second argument of __launch_bounds__
// Problem-shape constants (KL_JJ, KL_KK: row / plane pitch in elements) are
// specialised at compile time from the launch's scalar arguments, so every
// neighbour offset becomes an immediate in the SASS addressing mode.

#ifndef KL_COMMON_CUH
#define KL_COMMON_CUH

#ifndef KL_REAL
#error "KL_REAL (float|double) must be defined"
#endif
typedef KL_REAL real;

#define XYZ 0
#define XZY 1
#define YXZ 2
#define YZX 3
#define ZXY 4
#define ZYX 5

#define KL_STR(x) #x
#define KL_PRAGMA(x) _Pragma(KL_STR(x))

#if UNROLL_X
#define KL_UNROLL_X KL_PRAGMA(unroll)
#else
#define KL_UNROLL_X KL_PRAGMA(unroll 1)
#endif
#if UNROLL_Y
#define KL_UNROLL_Y KL_PRAGMA(unroll)
#else
#define KL_UNROLL_Y KL_PRAGMA(unroll 1)
#endif
#if UNROLL_Z
#define KL_UNROLL_Z KL_PRAGMA(unroll)
#else
#define KL_UNROLL_Z KL_PRAGMA(unroll 1)
#endif

#define KL_THREADS (BLOCK_X * BLOCK_Y * BLOCK_Z)

namespace kl {

// Programmatic dependent launch (sm_90+; klb_launch_ex KLB_LAUNCH_PDL): a
// kernel launched with the attribute may be scheduled while the previous
// kernel on the stream drains.  pdl_wait() blocks until that kernel has
// completed and its writes are visible — every stencil calls it before its
// first global read; pdl_trigger() as a block leaves (PdlTriggerAtExit)
// lets the next kernel's blocks launch into the slots this grid's finishing
// blocks free, before the grid's completion is signalled.  Both are no-ops for a
// kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Triggers when the block leaves the kernel (every return path): triggering
// at entry let the next kernel's blocks occupy SM slots while this grid still
// had blocks to schedule — measured slower (bench ``graph`` rows, r02f).
struct PdlTriggerAtExit {
  __device__ __forceinline__ ~PdlTriggerAtExit() { pdl_trigger(); }
};

// 1-D block id -> 3-D block coordinates; the first letter of UNRAVEL is the
// fastest-varying axis (PAPER.md: "for (Z,X,Y) ... first along Z, then X, then Y").
__device__ __forceinline__ void unravel(unsigned b, unsigned nbx, unsigned nby, unsigned nbz,
                                        int& bx, int& by, int& bz) {
#if UNRAVEL == XYZ
  bx = b % nbx; b /= nbx; by = b % nby; bz = b / nby;
#elif UNRAVEL == XZY
  bx = b % nbx; b /= nbx; bz = b % nbz; by = b / nbz;
#elif UNRAVEL == YXZ
  by = b % nby; b /= nby; bx = b % nbx; bz = b / nbx;
#elif UNRAVEL == YZX
  by = b % nby; b /= nby; bz = b % nbz; bx = b / nbz;
#elif UNRAVEL == ZXY
  bz = b % nbz; b /= nbz; bx = b % nbx; by = b / nbx;
#elif UNRAVEL == ZYX
  bz = b % nbz; b /= nbz; by = b % nby; bx = b / nby;
#else
#error "UNRAVEL must be one of XYZ XZY YXZ YZX ZXY ZYX"
#endif
}

// Global index of tile item t of thread `tid` in block `b` along one axis.
template <int BLOCK, int TILE, bool CONTIG>
__device__ __forceinline__ int tile_index(int b, int tid, int t) {
  return CONTIG ? (b * BLOCK + tid) * TILE + t : b * BLOCK * TILE + t * BLOCK + tid;
}

__device__ __forceinline__ unsigned ceil_div(unsigned a, unsigned b) { return (a + b - 1) / b; }

// MicroHH finite-difference helpers (restated in oracle/stencil_oracle.py).
template <typename T>
__device__ __forceinline__ T interp2(T a, T b) { return T(0.5) * (a + b); }

__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
// 60 * interp6_ws(a..f): 6th-order centred face value, unscaled
// (pair sums, then two FMAs: 37 (c+d) - 8 (b+e) + (a+f)).
template <typename T>
__device__ __forceinline__ T i6x60(T a, T b, T c, T d, T e, T f) {
  return fma_(T(37), c + d, fma_(T(-8), b + e, a + f));
}
// 60 * interp5_ws(a..f): the odd (upwind-correction) part, unscaled
// (10 (d-c) - 5 (e-b) + (f-a)).
template <typename T>
__device__ __forceinline__ T i5x60(T a, T b, T c, T d, T e, T f) {
  return fma_(T(10), d - c, fma_(T(-5), e - b, f - a));
}
// 60 * (vel * interp6_ws - |vel| * interp5_ws): 5th-order upwind flux.
// Called with vel = interp2(...) it is 60x the MicroHH face flux; the
// flux-form kernels pass the un-halved velocity SUM and fold the 1/2 into
// their final scale (120 instead of 60).
template <typename T>
__device__ __forceinline__ T flux5x60(T vel, T a, T b, T c, T d, T e, T f) {
  return vel * i6x60(a, b, c, d, e, f) - fabs(vel) * i5x60(a, b, c, d, e, f);
}
}  // namespace kl

#endif  // KL_COMMON_CUH
