// Shared device helpers for the Double-P sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "doublep_b200.h"

// Timing-experiment switches (dp_debug_set 0 / 10: skip a phase, drop P's low
// half, ...) are compiled in only with -DDP_AB_KNOBS
// (DP_EXTRA_FLAGS=-DDP_AB_KNOBS python -m paper_2602_05191_b200.build; the A/B
// tools need it).  The product build carries none of their branches: runtime
// mode checks in the plan cost ~0.27 us per layer at 32K (measured).
#ifdef DP_AB_KNOBS
#define DP_AB(dbg, mask) (((dbg) & (mask)) != 0)
#else
#define DP_AB(dbg, mask) (false)
#endif

namespace dp {

constexpr int kMaxGroup = 8;  // GQA group sizes the decode kernels are built for

__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float to_float(float x) { return x; }
__device__ __forceinline__ float to_float(__nv_bfloat16 x) { return __bfloat162float(x); }

// Element loads from a raw pointer of runtime dtype (DP_F32 / DP_BF16).
__device__ __forceinline__ double load_elem_d(const void* p, int dtype, size_t i) {
  return dtype == DP_F32 ? (double)reinterpret_cast<const float*>(p)[i]
                         : (double)bf2f(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ float load_elem_f(const void* p, int dtype, size_t i) {
  return dtype == DP_F32 ? reinterpret_cast<const float*>(p)[i]
                         : bf2f(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reductions; every thread receives the result.  `red` needs
// 32 slots of T in shared memory.  Must be called by all threads.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = lane < nw ? red[lane] : T(0);
  r = warp_sum(r);
  return r;
}
template <typename T>
__device__ __forceinline__ T block_max(T v, T* red, T ident) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = lane < nw ? red[lane] : ident;
  r = warp_max(r);
  return r;
}

// Reference max (nats) of the tensor-core attention's shared accumulators:
// the larger of the head's top cluster log-mass and its sink/window logits
// (always-exact rows the plan never scores otherwise), plus a margin, so an
// exact row up to ~70 nats above it cannot overflow the fp32 sums.  The top
// cluster is always exact and carries >= e^(top log-mass) (Jensen), so the
// margin costs nothing at the low end.
constexpr double kRefMargin = 11.0;
__device__ __forceinline__ double ref_max(double top, double sw) {
  const double m = fmax(top, sw);  // fmax drops a NaN operand
  return (m == -CUDART_INF || m != m) ? 0.0 : fmin(m, 1e30) + kRefMargin;
}

// Block-wide exclusive scan (fixed association order, so deterministic).
// Returns the exclusive prefix; *total receives the block total.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* red, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  __syncthreads();
  if (lane == 31) red[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? red[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    red[lane] = wi - w;  // exclusive prefix of warp totals
    if (lane == 31) red[32] = wi;
  }
  __syncthreads();
  T res = red[warp] + inc - v;
  *total = red[32];
  __syncthreads();
  return res;
}

}  // namespace dp

