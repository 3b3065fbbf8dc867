// hx_async.cuh -- asynchronous-copy primitives for sm_100a: mbarriers, 1D bulk copies
// (cp.async.bulk, the TMA engine's non-tensor mode) and 3D tensor tiles.
#pragma once

#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched from the runtime)

namespace hx {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// 3D tensor tile -> shared memory, completion on an mbarrier
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// contiguous global span -> shared memory (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared memory -> contiguous global span (bulk-group completion)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (bulk store source)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// contiguous span of n doubles -> shared memory through the bulk-copy engine: thread 0
// issues one cp.async.bulk of the 16-byte-aligned body (span_bulk_bytes of it must have
// been announced on the mbarrier with mbar_expect_tx first), an odd trailing double goes
// by cp.async (the caller's commit group).  A source that is not 16-byte aligned falls
// back to per-thread cp.async (0 bulk bytes).  dst must be 16-byte aligned.
__device__ __forceinline__ void cp_async8_(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ unsigned span_bulk_bytes(const double* src, int n) {
  return ((reinterpret_cast<unsigned long long>(src) & 15ull) == 0) ? (unsigned)(n & ~1) * 8u : 0u;
}
template <int NT>
__device__ __forceinline__ void span_bulk(double* dst, const double* src, int n, int t, unsigned long long* bar) {
  if ((reinterpret_cast<unsigned long long>(src) & 15ull) == 0) {
    if (t == 0) {
      if (n > 1) bulk_load(dst, src, (unsigned)(n & ~1) * 8u, bar);
      if (n & 1) cp_async8_(dst + n - 1, src + n - 1);
    }
  } else {
    for (int i = t; i < n; i += NT) cp_async8_(dst + i, src + i);
  }
}

}  // namespace hx
