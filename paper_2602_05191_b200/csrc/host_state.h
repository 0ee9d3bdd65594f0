// Host-side per-device state shared by the launchers: the SM count and the
// dynamic shared-memory attribute each kernel was raised to, keyed by the
// CURRENT device (cudaFuncSetAttribute applies per device context), behind
// one process-wide lock so launches from several host threads are safe.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

namespace dp {

constexpr int kMaxDevices = 64;

inline std::recursive_mutex& host_mutex() {
  static std::recursive_mutex m;
  return m;
}

inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0) d = 0;
  return d < kMaxDevices ? d : kMaxDevices - 1;
}

inline int sm_count() {
  static int sms[kMaxDevices] = {};
  const int d = current_device();
  std::lock_guard<std::recursive_mutex> g(host_mutex());
  if (!sms[d]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    sms[d] = n > 0 ? n : 148;
  }
  return sms[d];
}

// Raise fn's dynamic shared-memory limit to at least `bytes` on the current
// device (only ever raised: a later, smaller query must not lower it under a
// larger launch).  `nonportable` also allows cluster sizes above 8.
inline cudaError_t ensure_smem(const void* fn, size_t bytes, bool nonportable = false) {
  static std::map<std::pair<int, const void*>, size_t> cur;
  const int d = current_device();
  std::lock_guard<std::recursive_mutex> g(host_mutex());
  size_t& c = cur[{d, fn}];
  if (c >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && nonportable) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) c = bytes;
  return e;
}

}  // namespace dp
