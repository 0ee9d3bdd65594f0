// Measurement-side quantities of the reference on the GPU (SURVEY.md §8f
// row 3): the true token distribution, the idealised token top-k baseline
// and the metrics.py statistics that compare a plan against it.
//
//   token_weights        engine.py:122-132 full_attention_weights /
//                        engine.py:147-155 true_token_weights
//                        (logits = (k . q) * scale in fp64, lse =
//                        m + log(sum(exp(x - m))), weights = exp(x - lse))
//   token_topk           engine.py:293-315 baseline_token_topk +
//                        selection.py:85-92 top_k_select (k largest weights,
//                        ties -> lower token position)
//   recovered_mass       metrics.py:26-39
//   adaptive_budget      metrics.py:41-50
//   cluster_approx_error metrics.py:61-76
//   mixed_f64            engine.py:216-252 mixed_attention in fp64 (deterministic
//                        evaluation path for the experiment runner)
//
// All of these read the fp64 weight rows [B, Hq, row_cap] written by
// token_weights (physical row order of the clustered layout; `perm` maps a
// clustered row back to its token position where order matters).  They are
// one-CTA-per-q-head kernels: selection is a bisection over the IEEE bits of
// the non-negative fp64 weights (monotone as unsigned integers), each probe a
// block-wide count/mass over the head's rows, which keeps every decision
// exact (no histogram rounding) at the price of ~63 L2-resident passes -- the
// quantities are evaluation metrics, not the decode hot path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "host_state.h"
#include "decode_internal.h"

namespace dp {

constexpr int kWRows = 64;      // rows per token_weights CTA (8 warps x 8 rows)
constexpr int kMetThreads = 1024;

// ---------------------------------------------------------------------------
// logits in fp64: warp per row, lanes over the head dim; G q heads at once
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) token_logits_kernel(dp_cache_view v, const void* __restrict__ q, int qdt,
                                                           int G, double scale, double* __restrict__ w) {
  const int bh = blockIdx.y, H = v.kv_heads, b = bh / H, h = bh - b * H, d = v.head_dim;
  const int Hq = H * G;
  __shared__ double qs[kMaxGroup][256];
  for (int i = threadIdx.x; i < G * d; i += blockDim.x) {
    const int g = i / d, j = i - g * d;
    qs[g][j] = load_elem_d(q, qdt, ((size_t)b * Hq + h * G + g) * d + j);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t kb = (size_t)bh * v.row_cap * d;
  for (int i = 0; i < kWRows / 8; ++i) {
    const int r = blockIdx.x * kWRows + warp * (kWRows / 8) + i;
    if (r >= v.n_tokens) break;
    double acc[kMaxGroup];
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) acc[g] = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double x = load_elem_d(v.keys, v.dtype, kb + (size_t)r * d + j);
#pragma unroll
      for (int g = 0; g < kMaxGroup; ++g)
        if (g < G) acc[g] = fma(x, qs[g][j], acc[g]);
    }
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
      if (g < G) {
        const double s = warp_sum(acc[g]);
        if (lane == 0) w[((size_t)b * Hq + h * G + g) * v.row_cap + r] = s * scale;
      }
    }
  }
}

// lse (logsumexp, _kernels_py.py logsumexp) and weights = exp(x - lse), in place
__global__ void __launch_bounds__(kMetThreads) token_normalize_kernel(dp_cache_view v, double* __restrict__ w,
                                                                      double* __restrict__ lse) {
  __shared__ double red[33];
  const int n = v.n_tokens;
  double* x = w + (size_t)blockIdx.x * v.row_cap;
  double m = -CUDART_INF;
  for (int r = threadIdx.x; r < n; r += blockDim.x) m = fmax(m, x[r]);
  m = block_max(m, red, -CUDART_INF);
  double s = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) s += exp(x[r] - m);
  s = block_sum(s, red);
  const double z = n == 1 ? m : m + log(s);
  for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = exp(x[r] - z);
  if (threadIdx.x == 0) lse[blockIdx.x] = z;
}

__device__ __forceinline__ unsigned long long wkey(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));  // x >= 0: bits are monotone
}

__device__ __forceinline__ int row_position(int r, const int* perm, int perm_rows) {
  return (perm && r < perm_rows) ? perm[r] : r;
}

// Largest key T with count(key >= T) >= k (so T is the k-th largest key).
__device__ unsigned long long kth_largest_key(const double* x, int n, int k, int* red) {
  unsigned long long t = 0;
  for (int bit = 62; bit >= 0; --bit) {
    const unsigned long long cand = t | (1ull << bit);
    int c = 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) c += wkey(x[r]) >= cand;
    if (block_sum(c, red) >= k) t = cand;
  }
  return t;
}

// ---------------------------------------------------------------------------
// token top-k: select, captured mass, renormalised output (fp64)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kMetThreads) token_topk_kernel(dp_cache_view v, const int* __restrict__ perm,
                                                                 int perm_rows, int G, int budget,
                                                                 const int* __restrict__ budgets,
                                                                 const double* __restrict__ w,
                                                                 double* __restrict__ out,
                                                                 double* __restrict__ captured,
                                                                 uint8_t* __restrict__ selected) {
  extern __shared__ double part[];  // [32 warps][d]
  __shared__ int ired[33];
  __shared__ double dred[33];
  const int hq = blockIdx.x, Hq = v.kv_heads * G, b = hq / Hq, h = (hq - b * Hq) / G;
  const int n = v.n_tokens, d = v.head_dim;
  const int k = max(1, min(min(budget, n), budgets ? budgets[hq] : n));
  const double* x = w + (size_t)hq * v.row_cap;
  const int* pm = perm ? perm + (size_t)(b * v.kv_heads + h) * v.row_cap : nullptr;
  const unsigned long long T = kth_largest_key(x, n, k, ired);
  int gt = 0, eq = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const unsigned long long key = wkey(x[r]);
    gt += key > T;
    eq += key == T;
  }
  gt = block_sum(gt, ired);
  eq = block_sum(eq, ired);
  const int need = k - gt;  // in [1, eq]
  // ties at the threshold: keep the `need` lowest token positions
  int pcut = 0x7fffffff;
  if (need < eq) {
    int lo = 0;  // largest P with count(key == T && pos < P) < need (= the need-th smallest tied position)
    for (int bit = 30; bit >= 0; --bit) {
      const int cand = lo | (1 << bit);
      int c = 0;
      for (int r = threadIdx.x; r < n; r += blockDim.x)
        c += (wkey(x[r]) == T && row_position(r, pm, perm_rows) < cand);
      if (block_sum(c, ired) < need) lo = cand;
    }
    pcut = lo;
  }
  auto is_sel = [&](int r) {
    const unsigned long long key = wkey(x[r]);
    return key > T || (key == T && row_position(r, pm, perm_rows) <= pcut);
  };
  double cap = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const bool s = is_sel(r);
    if (s) cap += x[r];
    if (selected) selected[(size_t)hq * v.row_cap + r] = s;
  }
  cap = block_sum(cap, dred);
  // out = sum_sel (w / captured) v   (gather_weighted_sum of the renormalised weights)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  const size_t vb = (size_t)(b * v.kv_heads + h) * v.row_cap * d;
  for (int r = warp; r < n; r += nw) {
    if (!is_sel(r)) continue;
    const double c = x[r] / cap;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = lane + 32 * e;
      if (j < d) acc[e] = fma(c, load_elem_d(v.values, v.dtype, vb + (size_t)r * d + j), acc[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int j = lane + 32 * e;
    if (j < d) part[warp * d + j] = acc[e];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += part[i * d + j];
    out[(size_t)hq * d + j] = s;
  }
  if (threadIdx.x == 0) captured[hq] = cap;
}

// ---------------------------------------------------------------------------
// recovered mass of a plan: sink + window + members of state==2 clusters
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) recovered_mass_kernel(dp_cache_view v, int G, const double* __restrict__ w,
                                                             const uint8_t* __restrict__ state,
                                                             double* __restrict__ recovered) {
  __shared__ double red[33];
  const int hq = blockIdx.x, Hq = v.kv_heads * G, b = hq / Hq, h = (hq - b * Hq) / G;
  const int bh = b * v.kv_heads + h, n = v.n_tokens;
  const double* x = w + (size_t)hq * v.row_cap;
  const int* offs = v.offs + (size_t)bh * (v.cluster_cap + 1);
  const int K = v.nclusters[bh];
  const uint8_t* st = state + (size_t)hq * v.cluster_cap;
  double s = 0.0;
  for (int r = threadIdx.x; r < v.sink; r += blockDim.x) s += x[r];
  for (int r = n - v.window + threadIdx.x; r < n; r += blockDim.x) s += x[r];
  for (int c = threadIdx.x; c < K; c += blockDim.x)
    if (st[c] == 2)
      for (int r = offs[c]; r < offs[c + 1]; ++r) s += x[r];
  s = block_sum(s, red);
  if (threadIdx.x == 0) recovered[hq] = s;
}

// ---------------------------------------------------------------------------
// per-cluster |true mass - estimated mass|, in estimated-rank order
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) cluster_error_kernel(dp_cache_view v, int G, const double* __restrict__ w,
                                                            const double* __restrict__ lse,
                                                            const double* __restrict__ lm,
                                                            const int* __restrict__ order,
                                                            double* __restrict__ errors) {
  const int hq = blockIdx.x, Hq = v.kv_heads * G, b = hq / Hq, h = (hq - b * Hq) / G;
  const int bh = b * v.kv_heads + h;
  const double* x = w + (size_t)hq * v.row_cap;
  const int* offs = v.offs + (size_t)bh * (v.cluster_cap + 1);
  const int K = v.nclusters[bh];
  const size_t base = (size_t)hq * v.cluster_cap;
  const double z = lse[hq];
  for (int rank = threadIdx.x; rank < K; rank += blockDim.x) {
    const int c = order[base + rank];
    double m = 0.0;
    for (int r = offs[c]; r < offs[c + 1]; ++r) m += x[r];
    errors[base + rank] = fabs(m - exp(lm[base + c] - z));
  }
}

// ---------------------------------------------------------------------------
// minimal token count whose true mass reaches p (cumsum of the descending
// weights, searchsorted(side='left') + 1)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kMetThreads) adaptive_budget_kernel(dp_cache_view v, const double* __restrict__ w,
                                                                      double p, int* __restrict__ budget) {
  __shared__ double dred[33];
  __shared__ int ired[33];
  const int n = v.n_tokens;
  const double* x = w + (size_t)blockIdx.x * v.row_cap;
  double tot = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) tot += x[r];
  tot = block_sum(tot, dred);
  if (!(tot >= p)) {  // never reached: searchsorted returns n
    if (threadIdx.x == 0) budget[blockIdx.x] = n + 1;
    return;
  }
  unsigned long long t = 0;  // largest key with mass(key >= T) >= p
  for (int bit = 62; bit >= 0; --bit) {
    const unsigned long long cand = t | (1ull << bit);
    double s = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      if (wkey(x[r]) >= cand) s += x[r];
    if (block_sum(s, dred) >= p) t = cand;
  }
  double mgt = 0.0;
  int cgt = 0, ceq = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const unsigned long long key = wkey(x[r]);
    if (key > t) {
      mgt += x[r];
      ++cgt;
    }
    ceq += key == t;
  }
  mgt = block_sum(mgt, dred);
  cgt = block_sum(cgt, ired);
  ceq = block_sum(ceq, ired);
  if (threadIdx.x == 0) {
    const double wt = __longlong_as_double((long long)t);
    int j = 0;
    double acc = mgt;
    while (j < ceq) {
      acc += wt;
      ++j;
      if (acc >= p) break;
    }
    budget[blockIdx.x] = cgt + j;
  }
}

// ---------------------------------------------------------------------------
// mixed exact/approximate attention in fp64, one CTA per q head
// (mixed_attention, engine.py:216-252): exact rows = sink + window + rows of
// state==2 clusters, approx pseudo-rows = (log_mass, value_mean) of state==1
// clusters; state == NULL makes every cluster exact (full_attention over the
// clustered rows).  Deterministic (fixed work split and combine order), so
// experiment tables reproduce byte for byte; the decode hot path is the
// fp32 attn_tc_kernel.
// ---------------------------------------------------------------------------
constexpr int kMixWarps = 8;

__global__ void __launch_bounds__(kMixWarps * 32) mixed_f64_kernel(dp_cache_view v, const void* __restrict__ q,
                                                                   int qdt, int G, double scale,
                                                                   const double* __restrict__ lm,
                                                                   const uint8_t* __restrict__ state,
                                                                   double* __restrict__ out, double* __restrict__ lse) {
  __shared__ double sm[kMixWarps], sl[kMixWarps];
  __shared__ double so[kMixWarps][256];
  const int hq = blockIdx.x, Hq = v.kv_heads * G, b = hq / Hq, h = (hq - b * Hq) / G;
  const int bh = b * v.kv_heads + h, n = v.n_tokens, d = v.head_dim;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ne = d / 32 + (d % 32 ? 1 : 0);  // elements per lane (<= 8)
  double qr[8], o[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int j = lane + 32 * e;
    qr[e] = (e < ne && j < d) ? load_elem_d(q, qdt, (size_t)hq * d + j) : 0.0;
    o[e] = 0.0;
  }
  double m = -CUDART_INF, l = 0.0;
  const size_t rb = (size_t)bh * v.row_cap * d;
  auto fold = [&](double x, const double* vv) {  // online softmax update with one (logit, value row)
    const double mn = fmax(m, x);
    const double a = exp(m - mn), p = exp(x - mn);
    l = l * a + p;
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = o[e] * a + p * vv[e];
    m = mn;
  };
  auto row = [&](int r) {
    double s = 0.0, vv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = lane + 32 * e;
      const bool ok = e < ne && j < d;
      s = fma(ok ? load_elem_d(v.keys, v.dtype, rb + (size_t)r * d + j) : 0.0, qr[e], s);
      vv[e] = ok ? load_elem_d(v.values, v.dtype, rb + (size_t)r * d + j) : 0.0;
    }
    fold(warp_sum(s) * scale, vv);
  };
  for (int r = warp; r < v.sink; r += kMixWarps) row(r);
  for (int r = n - v.window + warp; r < n; r += kMixWarps) row(r);
  const int K = v.nclusters[bh];
  const int* offs = v.offs + (size_t)bh * (v.cluster_cap + 1);
  const size_t cb = (size_t)hq * v.cluster_cap;
  for (int c = warp; c < K; c += kMixWarps) {
    const int st = state ? state[cb + c] : 2;
    if (st == 2) {
      for (int r = offs[c]; r < offs[c + 1]; ++r) row(r);
    } else if (st == 1) {
      double vv[8];
      const float* vm = v.value_means + ((size_t)bh * v.cluster_cap + c) * d;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = lane + 32 * e;
        vv[e] = (e < ne && j < d) ? (double)vm[j] : 0.0;
      }
      fold(lm[cb + c], vv);
    }
  }
  if (lane == 0) {
    sm[warp] = m;
    sl[warp] = l;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int j = lane + 32 * e;
    if (e < ne && j < d) so[warp][j] = o[e];
  }
  __syncthreads();
  double M = -CUDART_INF;
  for (int i = 0; i < kMixWarps; ++i) M = fmax(M, sm[i]);
  double L = 0.0;
  for (int i = 0; i < kMixWarps; ++i) L += sm[i] == -CUDART_INF ? 0.0 : sl[i] * exp(sm[i] - M);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < kMixWarps; ++i)
      if (sm[i] != -CUDART_INF) acc += so[i][j] * exp(sm[i] - M);
    out[(size_t)hq * d + j] = L > 0.0 ? acc / L : 0.0;
  }
  if (threadIdx.x == 0 && lse) lse[hq] = L > 0.0 ? M + log(L) : -CUDART_INF;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
cudaError_t launch_token_weights(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double* w,
                                 double* lse, cudaStream_t st) {
  const int BH = v.batch * v.kv_heads;
  token_logits_kernel<<<dim3((v.n_tokens + kWRows - 1) / kWRows, BH), 256, 0, st>>>(v, q, qdt, G, scale, w);
  token_normalize_kernel<<<BH * G, kMetThreads, 0, st>>>(v, w, lse);
  return cudaGetLastError();
}

cudaError_t launch_token_topk(const dp_cache_view& v, const int* perm, int perm_rows, int G, int budget,
                              const int* budgets, const double* w, double* out, double* captured, uint8_t* selected, cudaStream_t st) {
  const int HQ = v.batch * v.kv_heads * G;
  const size_t smem = (size_t)(kMetThreads / 32) * v.head_dim * sizeof(double);
  cudaFuncSetAttribute(token_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  token_topk_kernel<<<HQ, kMetThreads, smem, st>>>(v, perm, perm_rows, G, budget, budgets, w, out, captured,
                                                          selected);
  return cudaGetLastError();
}

cudaError_t launch_recovered_mass(const dp_cache_view& v, int G, const double* w, const uint8_t* state,
                                  double* recovered, cudaStream_t st) {
  recovered_mass_kernel<<<v.batch * v.kv_heads * G, 256, 0, st>>>(v, G, w, state, recovered);
  return cudaGetLastError();
}

cudaError_t launch_cluster_error(const dp_cache_view& v, int G, const double* w, const double* lse,
                                 const double* lm, const int* order, double* errors, cudaStream_t st) {
  cluster_error_kernel<<<v.batch * v.kv_heads * G, 256, 0, st>>>(v, G, w, lse, lm, order, errors);
  return cudaGetLastError();
}

cudaError_t launch_mixed_f64(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                             const uint8_t* state, double* out, double* lse, cudaStream_t st) {
  mixed_f64_kernel<<<v.batch * v.kv_heads * G, kMixWarps * 32, 0, st>>>(v, q, qdt, G, scale, lm, state, out, lse);
  return cudaGetLastError();
}

cudaError_t launch_adaptive_budget(const dp_cache_view& v, int G, const double* w, double p, int* budget,
                                   cudaStream_t st) {
  adaptive_budget_kernel<<<v.batch * v.kv_heads * G, kMetThreads, 0, st>>>(v, w, p, budget);
  return cudaGetLastError();
}

}  // namespace dp
