// Distributed-shared-memory idioms shared by the cluster kernels (plan.cu,
// shard.cu): cluster barriers, DSMEM pushes that complete a receiver-side
// mbarrier transaction (st.async ... complete_tx), and mbarrier waits.
#pragma once

#include <cuda_runtime.h>

namespace dp {

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_sync() {
  cl_arrive();
  cl_wait();
}

// DSMEM pushes that signal the receiver's mbarrier (st.async ... complete_tx):
// the receiver waits for exactly the bytes it expects, the sender never
// waits (no cluster-wide barrier, no release fence on the sender's side)
__device__ __forceinline__ unsigned cl_map(const void* p, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void push_f64(const double* dst, int rank, double v, const unsigned long long* bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(cl_map(dst, rank)),
               "l"(__double_as_longlong(v)), "r"(cl_map(bar, rank))
               : "memory");
}
__device__ __forceinline__ void push_u32(const void* dst, int rank, unsigned v, const unsigned long long* bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(cl_map(dst, rank)),
               "r"(v), "r"(cl_map(bar, rank))
               : "memory");
}
__device__ __forceinline__ void push_v4(const void* dst, int rank, int a, int b, int c, int e,
                                        const unsigned long long* bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(
                   cl_map(dst, rank)),
               "r"(a), "r"(b), "r"(c), "r"(e), "r"(cl_map(bar, rank))
               : "memory");
}
__device__ __forceinline__ void mb_expect(const unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait0(const unsigned long long* bar) {  // phase 0 complete (acquire, cluster)
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a)
        : "memory");
}
__device__ __forceinline__ void push_u64(const void* dst, int rank, unsigned long long v,
                                         const unsigned long long* bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(cl_map(dst, rank)),
               "l"(v), "r"(cl_map(bar, rank))
               : "memory");
}
__device__ __forceinline__ void push_v2u64(const void* dst, int rank, unsigned long long a, unsigned long long b,
                                           const unsigned long long* bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];\n" ::"r"(
                   cl_map(dst, rank)),
               "l"(a), "l"(b), "r"(cl_map(bar, rank))
               : "memory");
}
__device__ __forceinline__ void mb_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)));
}

}  // namespace dp
