// The reference's per-query kernel plugin seam (kernels.py:47-96) as
// host-pointer C entry points: the same eight operations, the same contract
// (float32 or float64 matrices, float64 accumulation, lowest-index ties,
// ValueError on an unsorted prefix scan), computed on the GPU.
//
// This is the seam a maintainer binds when they want the reference's own
// dispatcher (DOUBLEP_KERNELS) to pick a B200 backend without touching the
// layers above it.  It is NOT the product decode path -- that is the batched,
// device-pointer, graph-capturable API in doublep_b200.h -- and it is not
// fast at the reference's per-query granularity, where the PCIe copies of a
// host array dominate.  What it gives is interchangeability with the
// Cython backend (_kernels_cy.pyx:21-157):
//   - scaled_logits / gather_scaled_logits and nearest_centroid evaluate the
//     Cython loops in the Cython order (one thread per row, sequential over
//     the head dimension, explicit round-to-nearest multiply/add so nvcc
//     cannot contract them into FMAs), so their results are BIT-IDENTICAL
//     to the compiled reference backend;
//   - sorted_prefix_count is the Cython scan verbatim (one thread, sequential
//     fp64 running sum, the ascent check before each add), staged through
//     shared memory in 4096-entry chunks -- an index result, bit-exact;
//   - logsumexp, softmax and weighted_sum are reductions: tree-ordered fp64
//     sums (deterministic, within 1e-12 relative of the sequential sums --
//     the tolerance the reference's own backend-parity test uses,
//     tests/test_kernels.py:30-67).
//
// Device state: one non-blocking stream and one growable staging buffer per
// device, behind a per-device mutex (calls from several host threads
// serialise per GPU).
#include <cuda_runtime.h>
#include <math_constants.h>

#include <mutex>
#include <string>

#include "common.cuh"
#include "host_state.h"

namespace dp {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
}  // namespace dp

namespace {

using dp::set_cuda_error;
using dp::set_error;

// ---------------------------------------------------------------- kernels

constexpr int kLogitRows = 128;  // rows per CTA (one per thread)
constexpr int kLogitCols = 32;   // head-dim slice staged per pass

// scaled_logits / gather_scaled_logits (_kernels_cy.pyx:21-50): a CTA stages
// a [128 rows x 32 cols] slice (warp-coalesced row segments), then each
// thread continues its row's sequential dot product over the slice.
template <typename T>
__global__ void __launch_bounds__(kLogitRows) kn_logits_kernel(const T* __restrict__ keys,
                                                               const int64_t* __restrict__ idx, long long n, int d,
                                                               const double* __restrict__ q, double scale,
                                                               double* __restrict__ out) {
  __shared__ double qs[kLogitCols];
  __shared__ T tile[kLogitRows][kLogitCols + 1];
  const int t = threadIdx.x;
  const long long r0 = (long long)blockIdx.x * kLogitRows;
  double acc = 0.0;
  for (int c0 = 0; c0 < d; c0 += kLogitCols) {
    const int w = min(kLogitCols, d - c0);
    __syncthreads();
    if (t < w) qs[t] = q[c0 + t];
    for (int e = t; e < kLogitRows * kLogitCols; e += kLogitRows) {
      const int r = e / kLogitCols, c = e % kLogitCols;
      const long long i = r0 + r;
      if (i < n && c < w) {
        const long long row = idx ? idx[i] : i;
        tile[r][c] = keys[row * d + c0 + c];
      }
    }
    __syncthreads();
    for (int j = 0; j < w; ++j) acc = __dadd_rn(acc, __dmul_rn((double)tile[t][j], qs[j]));
  }
  if (r0 + t < n) out[r0 + t] = __dmul_rn(acc, scale);
}

// nearest_centroid (_kernels_cy.pyx:115-140): one thread per point, the point
// held in shared memory as fp64, centroids read as warp-uniform (broadcast)
// loads; direct difference, strict '<' so the lowest index keeps a tie.
template <typename T>
__global__ void kn_nearest_kernel(const T* __restrict__ pts, long long n, int d, const double* __restrict__ cents,
                                  int k, int64_t* __restrict__ assign, double* __restrict__ best) {
  extern __shared__ double xs[];
  const int rb = blockDim.x, t = threadIdx.x, ld = d + 1;
  const long long p0 = (long long)blockIdx.x * rb;
  for (long long e = t; e < (long long)rb * d; e += rb) {
    const int r = (int)(e / d), c = (int)(e % d);
    const long long i = p0 + r;
    xs[r * ld + c] = i < n ? (double)pts[i * d + c] : 0.0;
  }
  __syncthreads();
  if (p0 + t >= n) return;
  const double* x = xs + t * ld;
  double bd = CUDART_INF;
  int64_t bc = 0;
  for (int c = 0; c < k; ++c) {
    const double* cv = cents + (size_t)c * d;
    double dist = 0.0;
    for (int j = 0; j < d; ++j) {
      const double diff = __dsub_rn(x[j], __ldg(cv + j));
      dist = __dadd_rn(dist, __dmul_rn(diff, diff));
    }
    if (dist < bd) {
      bd = dist;
      bc = c;
    }
  }
  assign[p0 + t] = bc;
  best[p0 + t] = bd;
}

constexpr int kRedThreads = 1024;

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// max under the Cython rule (m = x[0]; m = x[i] if x[i] > m): NaN only when
// x[0] is NaN, later NaNs never win a '>' comparison.
__device__ __forceinline__ double cy_max(const double* x, long long n, double* red) {
  double m = -CUDART_INF;
  for (long long i = 1 + threadIdx.x; i < n; i += blockDim.x)
    if (x[i] > m) m = x[i];
  for (int o = 16; o; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, m, o);
    if (y > m) m = y;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = -CUDART_INF;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
      if (red[i] > r) r = red[i];
    const double x0 = x[0];
    red[32] = (x0 != x0) ? x0 : (r > x0 ? r : x0);
  }
  __syncthreads();
  return red[32];
}

// logsumexp (_kernels_cy.pyx:53-65, exact for one element) and softmax
// (:68-83): one CTA, max then tree-ordered sum of exp(x - m).
__global__ void __launch_bounds__(kRedThreads) kn_lse_kernel(const double* __restrict__ x, long long n, int softmax,
                                                             double* __restrict__ out) {
  __shared__ double red[33];
  const double m = cy_max(x, n, red);
  if (!softmax && n == 1) {
    if (threadIdx.x == 0) out[0] = m;
    return;
  }
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = exp(x[i] - m);
    if (softmax) out[i] = e;
    s += e;
  }
  s = block_sum(s, red);
  if (!softmax) {
    if (threadIdx.x == 0) out[0] = m + log(s);
    return;
  }
  for (long long i = threadIdx.x; i < n; i += blockDim.x) out[i] = out[i] / s;
}

constexpr int kWsRows = 256;  // rows per CTA
constexpr int kWsY = 8;       // row lanes per CTA (x = 32 columns)

// weighted_sum / gather_weighted_sum (_kernels_cy.pyx:86-112): each CTA sums
// 256 rows into a per-CTA partial (columns across the warp, so every row
// segment is one coalesced load), kn_wsum_final adds the partials in CTA
// order -- deterministic.
template <typename T>
__global__ void __launch_bounds__(32 * kWsY) kn_wsum_kernel(const double* __restrict__ w, const T* __restrict__ mat,
                                                            const int64_t* __restrict__ idx, long long n, int d,
                                                            double* __restrict__ partial) {
  __shared__ double red[kWsY][33];
  const long long r0 = (long long)blockIdx.x * kWsRows;
  for (int c0 = 0; c0 < d; c0 += 32) {
    const int c = c0 + threadIdx.x;
    double acc = 0.0;
    if (c < d)
      for (int r = threadIdx.y; r < kWsRows; r += kWsY) {
        const long long i = r0 + r;
        if (i >= n) break;
        const long long row = idx ? idx[i] : i;
        acc = __dadd_rn(acc, __dmul_rn(w[i], (double)mat[row * d + c]));
      }
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && c < d) {
      double s = red[0][threadIdx.x];
      for (int y = 1; y < kWsY; ++y) s += red[y][threadIdx.x];
      partial[(size_t)blockIdx.x * d + c] = s;
    }
    __syncthreads();
  }
}

__global__ void kn_wsum_final(const double* __restrict__ partial, int parts, int d, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  double s = 0.0;
  for (int b = 0; b < parts; ++b) s += partial[(size_t)b * d + c];
  out[c] = s;
}

constexpr int kPrefixChunk = 4096;

// sorted_prefix_count (_kernels_cy.pyx:143-157): the scan itself is
// inherently sequential (an early-stopping fp64 running sum whose rounding
// decides the count), so one thread runs it over 32 KB shared-memory chunks
// the CTA loads cooperatively.  out = count, or -1 on an ascent.
__global__ void __launch_bounds__(256) kn_prefix_kernel(const double* __restrict__ x, long long n, double p,
                                                        long long* __restrict__ out) {
  __shared__ double buf[kPrefixChunk];
  __shared__ long long res;
  double total = 0.0, prev = CUDART_INF;
  if (threadIdx.x == 0) res = -2;
  for (long long c0 = 0; c0 < n; c0 += kPrefixChunk) {
    const int w = n - c0 < kPrefixChunk ? (int)(n - c0) : kPrefixChunk;
    for (int j = threadIdx.x; j < w; j += blockDim.x) buf[j] = x[c0 + j];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int j = 0; j < w; ++j) {
        const double v = buf[j];
        if (v > prev) {
          res = -1;
          break;
        }
        prev = v;
        total = __dadd_rn(total, v);
        if (total >= p) {
          res = c0 + j + 1;
          break;
        }
      }
    }
    __syncthreads();
    if (res != -2) break;
  }
  if (threadIdx.x == 0) out[0] = res == -2 ? n : res;
}

// ------------------------------------------------------------ host state

struct SeamDevice {
  std::mutex m;
  cudaStream_t stream = nullptr;
  char* buf = nullptr;
  size_t cap = 0;
};

SeamDevice& seam_device() {
  static SeamDevice devs[dp::kMaxDevices];
  return devs[dp::current_device()];
}

// Bump allocator over the device's staging buffer (256-B aligned slices).
struct Arena {
  size_t need = 0;
  char* base = nullptr;
  size_t add(size_t bytes) {
    const size_t off = need;
    need += (bytes + 255) & ~size_t(255);
    return off;
  }
  template <typename P>
  P* at(size_t off) const {
    return reinterpret_cast<P*>(base + off);
  }
};

// Locks the device's seam state, makes sure the stream exists and the buffer
// holds `a.need` bytes; returns DP_OK or an error code.
int acquire(SeamDevice& s, Arena& a) {
  cudaError_t e = cudaSuccess;
  if (!s.stream) e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return set_cuda_error(e, "seam stream");
  if (a.need > s.cap) {
    if (s.buf) {
      cudaStreamSynchronize(s.stream);
      cudaFree(s.buf);
      s.buf = nullptr;
      s.cap = 0;
    }
    const size_t cap = a.need > (1u << 20) ? a.need : (1u << 20);
    e = cudaMalloc(&s.buf, cap);
    if (e != cudaSuccess) return set_cuda_error(e, "seam staging buffer");
    s.cap = cap;
  }
  a.base = s.buf;
  return DP_OK;
}

int finish(SeamDevice& s, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s.stream);
  return e == cudaSuccess ? DP_OK : set_cuda_error(e, where);
}

size_t elem_size(int dtype) { return dtype == DP_F64 ? 8 : 4; }

int check_mat(int dtype, long long rows, int d) {
  if (dtype != DP_F32 && dtype != DP_F64) return set_error(DP_ERR_INVALID, "matrix dtype must be float32 or float64");
  if (rows < 0 || d < 0) return set_error(DP_ERR_INVALID, "negative matrix shape");
  return DP_OK;
}

int check_idx(const int64_t* idx, long long n_idx, long long rows) {
  if (n_idx < 0) return set_error(DP_ERR_INVALID, "negative index count");
  for (long long i = 0; i < n_idx; ++i)
    if (idx[i] < 0 || idx[i] >= rows) return set_error(DP_ERR_INVALID, "index out of range");
  return DP_OK;
}

unsigned blocks_for(long long n, int per) { return (unsigned)((n + per - 1) / per); }

}  // namespace

extern "C" {

int dp_kn_scaled_logits(const void* keys, int32_t dtype, int64_t rows, int32_t d, const int64_t* idx, int64_t n_idx,
                        const double* q, double scale, double* out) {
  int rc = check_mat(dtype, rows, d);
  if (rc) return rc;
  if (idx && (rc = check_idx(idx, n_idx, rows))) return rc;
  const long long n = idx ? n_idx : rows;
  if (n == 0) return DP_OK;
  SeamDevice& s = seam_device();
  std::lock_guard<std::mutex> g(s.m);
  Arena a;
  const size_t o_k = a.add((size_t)rows * d * elem_size(dtype)), o_i = a.add(idx ? n * 8 : 0),
               o_q = a.add((size_t)d * 8), o_out = a.add(n * 8);
  if ((rc = acquire(s, a))) return rc;
  cudaMemcpyAsync(a.at<char>(o_k), keys, (size_t)rows * d * elem_size(dtype), cudaMemcpyHostToDevice, s.stream);
  if (idx) cudaMemcpyAsync(a.at<char>(o_i), idx, n * 8, cudaMemcpyHostToDevice, s.stream);
  cudaMemcpyAsync(a.at<char>(o_q), q, (size_t)d * 8, cudaMemcpyHostToDevice, s.stream);
  const int64_t* di = idx ? a.at<int64_t>(o_i) : nullptr;
  if (dtype == DP_F32)
    kn_logits_kernel<float><<<blocks_for(n, kLogitRows), kLogitRows, 0, s.stream>>>(
        a.at<float>(o_k), di, n, d, a.at<double>(o_q), scale, a.at<double>(o_out));
  else
    kn_logits_kernel<double><<<blocks_for(n, kLogitRows), kLogitRows, 0, s.stream>>>(
        a.at<double>(o_k), di, n, d, a.at<double>(o_q), scale, a.at<double>(o_out));
  cudaMemcpyAsync(out, a.at<double>(o_out), n * 8, cudaMemcpyDeviceToHost, s.stream);
  return finish(s, "dp_kn_scaled_logits");
}

static int lse_or_softmax(const double* x, int64_t n, int softmax, double* out, const char* where) {
  if (n < 1) return set_error(DP_ERR_INVALID, "zero-size array");
  SeamDevice& s = seam_device();
  std::lock_guard<std::mutex> g(s.m);
  Arena a;
  const size_t o_x = a.add(n * 8), o_out = a.add(softmax ? n * 8 : 8);
  int rc = acquire(s, a);
  if (rc) return rc;
  cudaMemcpyAsync(a.at<char>(o_x), x, n * 8, cudaMemcpyHostToDevice, s.stream);
  kn_lse_kernel<<<1, kRedThreads, 0, s.stream>>>(a.at<double>(o_x), n, softmax, a.at<double>(o_out));
  cudaMemcpyAsync(out, a.at<double>(o_out), softmax ? n * 8 : 8, cudaMemcpyDeviceToHost, s.stream);
  return finish(s, where);
}

int dp_kn_logsumexp(const double* x, int64_t n, double* out) { return lse_or_softmax(x, n, 0, out, "dp_kn_logsumexp"); }

int dp_kn_softmax(const double* x, int64_t n, double* out) { return lse_or_softmax(x, n, 1, out, "dp_kn_softmax"); }

int dp_kn_weighted_sum(const double* w, const void* mat, int32_t dtype, int64_t rows, int32_t d, const int64_t* idx,
                       int64_t n_idx, double* out) {
  int rc = check_mat(dtype, rows, d);
  if (rc) return rc;
  if (idx && (rc = check_idx(idx, n_idx, rows))) return rc;
  const long long n = idx ? n_idx : rows;
  if (d == 0) return DP_OK;
  if (n == 0) {
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    return DP_OK;
  }
  const unsigned parts = blocks_for(n, kWsRows);
  SeamDevice& s = seam_device();
  std::lock_guard<std::mutex> g(s.m);
  Arena a;
  const size_t o_m = a.add((size_t)rows * d * elem_size(dtype)), o_i = a.add(idx ? n * 8 : 0), o_w = a.add(n * 8),
               o_p = a.add((size_t)parts * d * 8), o_out = a.add((size_t)d * 8);
  if ((rc = acquire(s, a))) return rc;
  cudaMemcpyAsync(a.at<char>(o_m), mat, (size_t)rows * d * elem_size(dtype), cudaMemcpyHostToDevice, s.stream);
  if (idx) cudaMemcpyAsync(a.at<char>(o_i), idx, n * 8, cudaMemcpyHostToDevice, s.stream);
  cudaMemcpyAsync(a.at<char>(o_w), w, n * 8, cudaMemcpyHostToDevice, s.stream);
  const int64_t* di = idx ? a.at<int64_t>(o_i) : nullptr;
  const dim3 blk(32, kWsY);
  if (dtype == DP_F32)
    kn_wsum_kernel<float><<<parts, blk, 0, s.stream>>>(a.at<double>(o_w), a.at<float>(o_m), di, n, d,
                                                       a.at<double>(o_p));
  else
    kn_wsum_kernel<double><<<parts, blk, 0, s.stream>>>(a.at<double>(o_w), a.at<double>(o_m), di, n, d,
                                                        a.at<double>(o_p));
  kn_wsum_final<<<blocks_for(d, 128), 128, 0, s.stream>>>(a.at<double>(o_p), (int)parts, d, a.at<double>(o_out));
  cudaMemcpyAsync(out, a.at<double>(o_out), (size_t)d * 8, cudaMemcpyDeviceToHost, s.stream);
  return finish(s, "dp_kn_weighted_sum");
}

int dp_kn_nearest_centroid(const void* points, int32_t dtype, int64_t n, int32_t d, const double* centroids,
                           int32_t k, int64_t* assign, double* sqdist) {
  int rc = check_mat(dtype, n, d);
  if (rc) return rc;
  if (k < 1) return set_error(DP_ERR_INVALID, "attempt to get argmin of an empty sequence");
  if (n == 0) return DP_OK;
  // points staged as fp64 rows of d+1 (odd stride) in the 48 KB static budget
  int rb = 128;
  while (rb > 1 && (size_t)rb * (d + 1) * 8 > 48 * 1024) rb >>= 1;
  if ((size_t)rb * (d + 1) * 8 > 48 * 1024) return set_error(DP_ERR_UNSUPPORTED, "head dimension too large");
  SeamDevice& s = seam_device();
  std::lock_guard<std::mutex> g(s.m);
  Arena a;
  const size_t o_p = a.add((size_t)n * d * elem_size(dtype)), o_c = a.add((size_t)k * d * 8), o_a = a.add(n * 8),
               o_b = a.add(n * 8);
  if ((rc = acquire(s, a))) return rc;
  cudaMemcpyAsync(a.at<char>(o_p), points, (size_t)n * d * elem_size(dtype), cudaMemcpyHostToDevice, s.stream);
  cudaMemcpyAsync(a.at<char>(o_c), centroids, (size_t)k * d * 8, cudaMemcpyHostToDevice, s.stream);
  const size_t smem = (size_t)rb * (d + 1) * 8;
  if (dtype == DP_F32)
    kn_nearest_kernel<float><<<blocks_for(n, rb), rb, smem, s.stream>>>(
        a.at<float>(o_p), n, d, a.at<double>(o_c), k, a.at<int64_t>(o_a), a.at<double>(o_b));
  else
    kn_nearest_kernel<double><<<blocks_for(n, rb), rb, smem, s.stream>>>(
        a.at<double>(o_p), n, d, a.at<double>(o_c), k, a.at<int64_t>(o_a), a.at<double>(o_b));
  cudaMemcpyAsync(assign, a.at<int64_t>(o_a), n * 8, cudaMemcpyDeviceToHost, s.stream);
  cudaMemcpyAsync(sqdist, a.at<double>(o_b), n * 8, cudaMemcpyDeviceToHost, s.stream);
  return finish(s, "dp_kn_nearest_centroid");
}

int dp_kn_sorted_prefix_count(const double* sorted_probs, int64_t n, double p, int64_t* count) {
  if (n < 0) return set_error(DP_ERR_INVALID, "negative length");
  if (n == 0) {
    *count = 0;
    return DP_OK;
  }
  SeamDevice& s = seam_device();
  std::lock_guard<std::mutex> g(s.m);
  Arena a;
  const size_t o_x = a.add(n * 8), o_c = a.add(8);
  int rc = acquire(s, a);
  if (rc) return rc;
  long long res = 0;
  cudaMemcpyAsync(a.at<char>(o_x), sorted_probs, n * 8, cudaMemcpyHostToDevice, s.stream);
  kn_prefix_kernel<<<1, 256, 0, s.stream>>>(a.at<double>(o_x), n, p, a.at<long long>(o_c));
  cudaMemcpyAsync(&res, a.at<long long>(o_c), 8, cudaMemcpyDeviceToHost, s.stream);
  if ((rc = finish(s, "dp_kn_sorted_prefix_count"))) return rc;
  if (res < 0) return set_error(DP_ERR_INVALID, "input not sorted");
  *count = res;
  return DP_OK;
}

}  // extern "C"
