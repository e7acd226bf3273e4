// kl_tma.cuh — TMA (cp.async.bulk.tensor) + mbarrier helpers for the
// runtime-compiled stencils (sm_90+/sm_100a PTX; NVRTC has no CUDA headers,
// so the few instructions are written inline).
//
// Host protocol (paper_2303_12374_b200/cuda/compiler.py): a kernel that wants
// tensor maps exports
//   extern "C" __device__ const int kl_tma_spec[1 + 5*N]
//       = {N, ptr_arg, jj_arg, kk_arg, box_w, box_h, ...};
// and takes one extra, trailing kernel parameter
//   const __grid_constant__ KlTmaParams tma      // { TmaDesc map[N]; }
// After loading the module the executable reads kl_tma_spec; when it packs
// the launch parameters it encodes one 3-D tensor map per entry (dims {jj,
// kk/jj, planes}, box {box_w, box_h, 1}, no swizzle, zero OOB fill) over the
// 16-byte-aligned base of the pointer argument and appends them.  The kernel
// adds kl::tma_xoff(ptr) to its x coordinates to undo the alignment shift.
// (Descriptors live in the parameter space, as __grid_constant__ — the TMA
// unit reads them without any generic-proxy fence.)

#ifndef KL_TMA_CUH
#define KL_TMA_CUH

struct __align__(64) TmaDesc {
  unsigned long long raw[16];
};

namespace kl {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <typename T>
__device__ __forceinline__ int tma_xoff(const T* p) {
  return static_cast<int>((reinterpret_cast<unsigned long long>(p) & 15ull) / sizeof(T));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "KL_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra KL_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Order this thread's earlier generic-proxy shared-memory accesses before
// subsequent async-proxy (TMA) writes to the same memory.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const TmaDesc* map, unsigned long long* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// L2 eviction-priority policies (createpolicy) for the .L2::cache_hint forms
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_3d_hint(void* dst, const TmaDesc* map, unsigned long long* bar, int x,
                                                 int y, int z, unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// L2 prefetch of a 3-D box (no shared memory, no barrier): the box's DRAM
// reads start now, and a later tma_load_3d of it hits L2
__device__ __forceinline__ void tma_prefetch_3d(const TmaDesc* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

}  // namespace kl

#endif  // KL_TMA_CUH
