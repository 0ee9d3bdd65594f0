// Prefill k-means clustering of the keys on sm_100a (build_clustered_cache,
// /root/reference/pkg/src/doublep/clustering.py:266-314).
//
//   kmeanspp   clustering.py:36-55   k-means++ seeding, replaying the host RNG
//                                    stream (first pick + one uniform per centre,
//                                    cdf = cumsum(dsq/total)/cdf[-1],
//                                    searchsorted(side='right')), fp64 dsq
//   assign     _kernels_py.py:58-77  |x|^2 - 2x.c + |c|^2 argmin, ties -> lowest id
//   update     clustering.py:86-98   objective, empty-cluster drop with ascending
//                                    remap (np.unique), convergence test, stable
//                                    counting sort of members (ascending positions)
//   means      clustering.py:100-106 fp64 means summed in member order
//   finalize   clustering.py:298-311 cluster-contiguous rows, fp32 tables
//
// All heads (B*H) are processed by every launch; per-head convergence flags
// let finished heads skip work, so the host loop never synchronises.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cooperative_groups.h>
#include <cuda.h>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "host_state.h"
#include "doublep_b200.h"

namespace cg = cooperative_groups;

namespace dp {

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);

struct KmWs {
  double* dsq;    // [BH][M]
  double* xnorm;  // [BH][M]
  double* cent;   // [BH][k][d]
  double* cnorm;  // [BH][k]
  double* sqd;    // [BH][M]
  int* assign;    // [BH][M]
  int* prev;      // [BH][M]
  int* sorted;    // [BH][M] member point ids, cluster-major, ascending within
  int* counts;    // [BH][k]
  int* remap;     // [BH][k]
  int* start;     // [BH][k+1]
  int* cursor;    // [BH][k]
  int* knum;      // [BH]
  int* done;      // [BH]
  __nv_bfloat16* csplit;  // [3][BH][k][d] centroids as bf16 hi + mid + lo (tensor-core assignment)
};

static size_t km_layout(const dp_cluster_params* p, KmWs* w, char* base) {
  const size_t BH = (size_t)p->batch * p->kv_heads;
  const size_t M = (size_t)p->n_tokens - p->sink - p->window;
  const size_t k = p->k, d = p->head_dim;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return base ? base + o : nullptr;
  };
  KmWs t;
  t.dsq = (double*)take(BH * M * 8);
  t.xnorm = (double*)take(BH * M * 8);
  t.cent = (double*)take(BH * k * d * 8);
  t.cnorm = (double*)take(BH * k * 8);
  t.sqd = (double*)take(BH * M * 8);
  t.assign = (int*)take(BH * M * 4);
  t.prev = (int*)take(BH * M * 4);
  t.sorted = (int*)take(BH * M * 4);
  t.counts = (int*)take(BH * k * 4);
  t.remap = (int*)take(BH * k * 4);
  t.start = (int*)take(BH * (k + 1) * 4);
  t.cursor = (int*)take(BH * k * 4);
  t.knum = (int*)take(BH * 4);
  t.done = (int*)take(BH * 4);
  // >= 128 rows so the tensor map's 128-row boxes never exceed it (rows past
  // 3*BH*k only feed centroid columns >= k, which the argmin masks)
  t.csplit = (__nv_bfloat16*)take(p->fp64_assign == 2 ? std::max<size_t>(3 * BH * k, 128) * d * 2 : 0);
  if (w) *w = t;
  return off;
}

// -------------------------------------------------------------------------
// |x|^2 of every middle point (fp64)
// -------------------------------------------------------------------------
__global__ void xnorm_kernel(dp_cluster_params p, const void* __restrict__ src, KmWs w) {
  const int bh = blockIdx.y;
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= M) return;
  const size_t base = ((size_t)bh * p.n_tokens + p.sink + warp) * d;
  double a = 0.0;
  for (int j = lane; j < d; j += 32) {
    const double x = load_elem_d(src, p.dtype, base + j);
    a = fma(x, x, a);
  }
  a = warp_sum(a);
  if (lane == 0) w.xnorm[(size_t)bh * M + warp] = a;
}

// -------------------------------------------------------------------------
// k-means++ seeding: one CTA per head, all k-1 sequential steps in-kernel.
// Each step streams the head's middle points through shared memory in
// 256-point tiles (coalesced cp.async, double-buffered for bf16), computes
// |x - c|^2 = |x|^2 - 2 x.c + |c|^2 in fp64 (products of bf16/fp32 inputs
// are exact in fp64), folds it into dsq (global, L2-resident), then draws
// the next centre: idx = first j with cdf_j / cdf_last > u, cdf = cumsum of
// dsq/total over contiguous per-thread segments (Generator.choice).
// -------------------------------------------------------------------------
constexpr int kPPThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kPPThreads) kmeanspp_kernel(dp_cluster_params p, const T* __restrict__ src,
                                                            const int* __restrict__ first_pick,
                                                            const double* __restrict__ uniforms,
                                                            const int* __restrict__ alt_picks,
                                                            int* __restrict__ degenerate_from, int* __restrict__ picks,
                                                            KmWs w) {
  constexpr int kStages = sizeof(T) == 2 ? 2 : 1;
  const int bh = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim, k = p.k;
  const int rowb = d * (int)sizeof(T) + 16;  // padded row (bytes): conflict-free 16B LDS
  const int chunks = d * (int)sizeof(T) / 16;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* c = reinterpret_cast<double*>(smem_raw);              // [d]
  unsigned char* tiles = smem_raw + ((d * 8 + 127) / 128) * 128;  // kStages x [256][rowb]
  __shared__ double red[33];
  __shared__ double s_cn;
  __shared__ int s_idx, s_degen;
  const T* X = src + ((size_t)bh * p.n_tokens + p.sink) * d;
  const double* xn = w.xnorm + (size_t)bh * M;
  double* dsq = w.dsq + (size_t)bh * M;
  const int degen_in = degenerate_from ? degenerate_from[bh] : k;
  const int ntiles = (M + kPPThreads - 1) / kPPThreads;
  const int per = (M + nt - 1) / nt;
  const int beg = min(M, tid * per), end = min(M, beg + per);
  if (tid == 0) {
    s_degen = k;
    s_idx = first_pick[bh];
  }
  __syncthreads();

  auto issue_tile = [&](int t, int buf) {
    unsigned char* dst = tiles + (size_t)buf * kPPThreads * rowb;
    const int p0 = t * kPPThreads;
    const int np = min(kPPThreads, M - p0);
    const unsigned char* g = reinterpret_cast<const unsigned char*>(X + (size_t)p0 * d);
    for (int i = tid; i < np * chunks; i += nt) {
      const int r = i / chunks, cc = i - r * chunks;
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + r * rowb + cc * 16));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g + (size_t)r * d * sizeof(T) + cc * 16));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  for (int i = 0; i < k; ++i) {
    const int idx = s_idx;
    if (tid == 0) picks[(size_t)bh * k + i] = idx;
    for (int j = tid; j < d; j += nt) {
      const double x = (double)to_float(X[(size_t)idx * d + j]);
      c[j] = x;
      w.cent[((size_t)bh * k + i) * d + j] = x;
    }
    __syncthreads();
    if (tid < 32) {
      double a = 0.0;
      for (int j = tid; j < d; j += 32) a = fma(c[j], c[j], a);
      a = warp_sum(a);
      if (tid == 0) s_cn = a;
    }
    // ---- dsq update over all tiles -------------------------------------
    issue_tile(0, 0);
    for (int t = 0; t < ntiles; ++t) {
      const int buf = kStages == 2 ? (t & 1) : 0;
      if (kStages == 2 && t + 1 < ntiles) {
        issue_tile(t + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        if (kStages == 1 && t > 0) issue_tile(t, 0);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      __syncthreads();
      const int pt = t * kPPThreads + tid;
      if (pt < M) {
        const unsigned char* row = tiles + (size_t)buf * kPPThreads * rowb + tid * rowb;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int cc = 0; cc < chunks; ++cc) {
          const int4 raw = *reinterpret_cast<const int4*>(row + cc * 16);
          if constexpr (sizeof(T) == 2) {
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
            const double* cj = c + cc * 8;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              if (e & 1) {
                a2 = fma((double)f.x, cj[2 * e], a2);
                a3 = fma((double)f.y, cj[2 * e + 1], a3);
              } else {
                a0 = fma((double)f.x, cj[2 * e], a0);
                a1 = fma((double)f.y, cj[2 * e + 1], a1);
              }
            }
          } else {
            const float* f = reinterpret_cast<const float*>(&raw);
            const double* cj = c + cc * 4;
            a0 = fma((double)f[0], cj[0], a0);
            a1 = fma((double)f[1], cj[1], a1);
            a2 = fma((double)f[2], cj[2], a2);
            a3 = fma((double)f[3], cj[3], a3);
          }
        }
        const double dist = fmax(xn[pt] - 2.0 * ((a0 + a1) + (a2 + a3)) + s_cn, 0.0);
        dsq[pt] = (i == 0) ? dist : fmin(dsq[pt], dist);
      }
      __syncthreads();  // buffer reuse
    }
    if (i + 1 == k) break;
    // ---- draw centre i+1 -------------------------------------------------
    double loc = 0.0;
    for (int j = beg; j < end; ++j) loc += dsq[j];
    const double total = block_sum(loc, red);
    const int step = i + 1;
    if (total > 0.0 && step < degen_in) {
      double lp = 0.0;
      for (int j = beg; j < end; ++j) lp += dsq[j] / total;
      double last;
      const double off = block_exclusive_scan(lp, red, &last);
      const double u = uniforms[(size_t)bh * (k - 1) + (step - 1)];
      if (tid == 0) s_idx = M;
      __syncthreads();
      {  // every segment reports its first crossing; the min is the pick (robust to
         // the scan's rounding at segment edges)
        double run = off;
        for (int j = beg; j < end; ++j) {
          run += dsq[j] / total;
          if (run / last > u) {
            atomicMin(&s_idx, j);
            break;
          }
        }
      }
      __syncthreads();
      if (tid == 0 && s_idx >= M) s_idx = M - 1;
    } else if (tid == 0) {
      if (step >= degen_in && alt_picks) {
        s_idx = alt_picks[(size_t)bh * (k - 1) + (step - 1)];
      } else {
        if (s_degen == k) s_degen = step;
        s_idx = 0;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (degenerate_from) degenerate_from[bh] = s_degen;
    w.knum[bh] = k;
    w.done[bh] = 0;
  }
}

// -------------------------------------------------------------------------
// k-means++ seeding with one 8-CTA thread-block cluster per head: CTA r owns
// a contiguous chunk of the points, each thread a contiguous segment of it.
// Per step: dsq update of my segment (16-B key loads, the single-CTA
// kernel's fp64 arithmetic), CTA sums pushed to every CTA over DSMEM
// (barrier 1, everybody forms the same total T in the same order), then the
// first point whose running dsq sum exceeds u * T -- the sampling draw of
// Generator.choice(p = dsq / T) in unnormalised form -- found per CTA and
// pushed (barrier 2); the minimum is the next centre.  ~2 cluster barriers
// per centre instead of one SM streaming every point.
// -------------------------------------------------------------------------
constexpr int kPPCL = 8;           // CTAs per head (16-CTA clusters: only 7 co-resident on B200)
constexpr int kPPCThreads = 1024;

template <typename T>
__global__ void __launch_bounds__(kPPCThreads) kmeanspp_cluster_kernel(
    dp_cluster_params p, const T* __restrict__ src, const int* __restrict__ first_pick,
    const double* __restrict__ uniforms, const int* __restrict__ alt_picks, int* __restrict__ degenerate_from,
    int* __restrict__ picks, KmWs w, int use_smem) {
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int bh = blockIdx.x / kPPCL;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim, k = p.k;
  const int chunk = (M + kPPCL - 1) / kPPCL;
  const int c0 = min(M, r * chunk), c1 = min(M, c0 + chunk);
  const int per = (c1 - c0 + nt - 1) / nt;
  const int beg = min(c1, c0 + tid * per), end = min(c1, beg + per);
  const int chunks = d * (int)sizeof(T) / 16;
  __shared__ double c[256];
  __shared__ double red[33];
  __shared__ double s_sum[kPPCL];
  __shared__ int s_cand[kPPCL];
  __shared__ double s_cn;
  __shared__ int s_idx, s_degen, s_mine;
  const T* X = src + ((size_t)bh * p.n_tokens + p.sink) * d;
  const double* xn = w.xnorm + (size_t)bh * M;
  // the chunk's dsq lives in shared memory when it fits (no global round trip
  // per point per centre), else in the workspace
  extern __shared__ double sdsq[];
  double* D = use_smem ? sdsq : w.dsq + (size_t)bh * M + c0;  // indexed by pt - c0
  const int degen_in = degenerate_from ? degenerate_from[bh] : k;
  if (tid == 0) {
    s_degen = k;
    s_idx = first_pick[bh];
  }
  __syncthreads();
  for (int i = 0; i < k; ++i) {
    const int idx = s_idx;
    // this step's uniform, loaded while the centre row and the dsq update are in flight
    const double u_next = i + 1 < k ? __ldg(&uniforms[(size_t)bh * (k - 1) + i]) : 0.0;
    if (r == 0 && tid == 0) picks[(size_t)bh * k + i] = idx;
    for (int j = tid; j < d; j += nt) {
      const double x = (double)to_float(X[(size_t)idx * d + j]);
      c[j] = x;
      if (r == 0) w.cent[((size_t)bh * k + i) * d + j] = x;
    }
    __syncthreads();
    if (tid < 32) {
      double a = 0.0;
      for (int j = tid; j < d; j += 32) a = fma(c[j], c[j], a);
      a = warp_sum(a);
      if (tid == 0) s_cn = a;
    }
    __syncthreads();
    const double cn = s_cn;
    double loc = 0.0;
#pragma unroll 1
    for (int pt = beg; pt < end; ++pt) {
      const int4* row = reinterpret_cast<const int4*>(X + (size_t)pt * d);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 4
      for (int cc = 0; cc < chunks; ++cc) {
        const int4 raw = __ldg(row + cc);
        if constexpr (sizeof(T) == 2) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
          const double* cj = c + cc * 8;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            if (e & 1) {
              a2 = fma((double)f.x, cj[2 * e], a2);
              a3 = fma((double)f.y, cj[2 * e + 1], a3);
            } else {
              a0 = fma((double)f.x, cj[2 * e], a0);
              a1 = fma((double)f.y, cj[2 * e + 1], a1);
            }
          }
        } else {
          const float* f = reinterpret_cast<const float*>(&raw);
          const double* cj = c + cc * 4;
          a0 = fma((double)f[0], cj[0], a0);
          a1 = fma((double)f[1], cj[1], a1);
          a2 = fma((double)f[2], cj[2], a2);
          a3 = fma((double)f[3], cj[3], a3);
        }
      }
      const double dist = fmax(xn[pt] - 2.0 * ((a0 + a1) + (a2 + a3)) + cn, 0.0);
      const double nd = (i == 0) ? dist : fmin(D[pt - c0], dist);
      D[pt - c0] = nd;
      loc += nd;
    }
    if (i + 1 == k) break;
    // ---- draw centre i+1 ------------------------------------------------
    const double mine = block_sum(loc, red);
    if (tid < kPPCL) *cluster.map_shared_rank(&s_sum[r], tid) = mine;
    cluster.sync();  // (1) every CTA holds every chunk sum
    double total = 0.0, before = 0.0;
    for (int q = 0; q < kPPCL; ++q) {
      if (q < r) before += s_sum[q];
      total += s_sum[q];
    }
    const int step = i + 1;
    if (total > 0.0 && step < degen_in) {
      double last;
      const double off = block_exclusive_scan(loc, red, &last);
      const double thr = u_next * total;
      if (tid == 0) s_mine = M;
      __syncthreads();
      double run = before + off;
      for (int j = beg; j < end; ++j) {
        run += D[j - c0];
        if (run > thr) {
          atomicMin(&s_mine, j);
          break;
        }
      }
      __syncthreads();
      if (tid < kPPCL) *cluster.map_shared_rank(&s_cand[r], tid) = s_mine;
      cluster.sync();  // (2) every CTA's first crossing
      if (tid == 0) {
        int pick = M;
        for (int q = 0; q < kPPCL; ++q) pick = min(pick, s_cand[q]);
        s_idx = pick >= M ? M - 1 : pick;
      }
    } else if (tid == 0) {
      if (step >= degen_in && alt_picks) {
        s_idx = alt_picks[(size_t)bh * (k - 1) + (step - 1)];
      } else {
        if (s_degen == k) s_degen = step;
        s_idx = 0;
      }
    }
    __syncthreads();
  }
  if (r == 0 && tid == 0) {
    if (degenerate_from) degenerate_from[bh] = s_degen;
    w.knum[bh] = k;
    w.done[bh] = 0;
  }
  cluster.sync();  // no CTA exits while a peer may still push into its shared memory
}

static size_t pp_smem(const dp_cluster_params* p) {
  const int es = p->dtype == DP_F32 ? 4 : 2;
  const int stages = p->dtype == DP_F32 ? 1 : 2;
  return ((p->head_dim * 8 + 127) / 128) * 128 + (size_t)stages * kPPThreads * (p->head_dim * es + 16);
}

int g_pp_single = 0;  // 1: the one-CTA-per-head seeding kernel (dp_debug_set(3, 1))

template <typename T>
static cudaError_t launch_pp_cluster(const dp_cluster_params* p, const T* src, const int* first, const double* u,
                                     const int* alt, int* degen, int* picks, KmWs w, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p->batch * p->kv_heads * kPPCL));
  cfg.blockDim = dim3(kPPCThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kPPCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int M = p->n_tokens - p->sink - p->window;
  const size_t dbytes = (size_t)((M + kPPCL - 1) / kPPCL) * sizeof(double);
  const int use_smem = dbytes <= 200 * 1024;
  cfg.dynamicSmemBytes = use_smem ? dbytes : 0;
  if (use_smem)
    cudaFuncSetAttribute(kmeanspp_cluster_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dbytes);
  return cudaLaunchKernelEx(&cfg, kmeanspp_cluster_kernel<T>, *p, src, first, u, alt, degen, picks, w, use_smem);
}

static cudaError_t launch_kmeanspp(const dp_cluster_params* p, const void* src, const int* first,
                                   const double* u, const int* alt, int* degen, int* picks, KmWs w,
                                   cudaStream_t st) {
  const int BH = p->batch * p->kv_heads;
  if (!g_pp_single && p->head_dim <= 256) {
    if (p->dtype == DP_F32) return launch_pp_cluster(p, (const float*)src, first, u, alt, degen, picks, w, st);
    return launch_pp_cluster(p, (const __nv_bfloat16*)src, first, u, alt, degen, picks, w, st);
  }
  const size_t smem = pp_smem(p);
  if (p->dtype == DP_F32) {
    cudaFuncSetAttribute(kmeanspp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kmeanspp_kernel<float><<<BH, kPPThreads, smem, st>>>(*p, (const float*)src, first, u, alt, degen, picks, w);
  } else {
    cudaFuncSetAttribute(kmeanspp_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kmeanspp_kernel<__nv_bfloat16><<<BH, kPPThreads, smem, st>>>(*p, (const __nv_bfloat16*)src, first, u, alt,
                                                                  degen, picks, w);
  }
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// centroid norms (warp per centroid)
// -------------------------------------------------------------------------
__global__ void cnorm_kernel(dp_cluster_params p, KmWs w) {
  const int bh = blockIdx.y;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= w.knum[bh] || w.done[bh]) return;
  const double* cr = w.cent + ((size_t)bh * p.k + c) * p.head_dim;
  double a = 0.0;
  for (int j = lane; j < p.head_dim; j += 32) a = fma(cr[j], cr[j], a);
  a = warp_sum(a);
  if (lane == 0) w.cnorm[(size_t)bh * p.k + c] = a;
}

// -------------------------------------------------------------------------
// assignment: 64 points x 64 centroids register-tiled "GEMM + argmin".
// dist = |x|^2 - 2 x.c + |c|^2 (the NumPy backend's expansion), clamped at 0.
// -------------------------------------------------------------------------
constexpr int kAP = 64, kAC = 64, kAK = 32;

template <typename Acc>
__global__ void __launch_bounds__(256) assign_kernel(dp_cluster_params p, const void* __restrict__ src, KmWs w) {
  const int bh = blockIdx.y;
  if (w.done[bh]) return;
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim;
  const int kc = w.knum[bh];
  const int p0 = blockIdx.x * kAP;
  if (p0 >= M) return;
  __shared__ Acc xs[kAK][kAP + 1];
  __shared__ Acc cs[kAK][kAC + 1];
  __shared__ Acc cn[kAC];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const size_t xbase = ((size_t)bh * p.n_tokens + p.sink) * d;
  const double* cent = w.cent + (size_t)bh * p.k * d;
  double best[4];
  int bidx[4];
  Acc xn[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    best[i] = CUDART_INF;
    bidx[i] = 0;
    const int pt = p0 + ty * 4 + i;
    xn[i] = pt < M ? (Acc)w.xnorm[(size_t)bh * M + pt] : Acc(0);
  }
  for (int c0 = 0; c0 < kc; c0 += kAC) {
    Acc acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    for (int k0 = 0; k0 < d; k0 += kAK) {
      for (int e = tid; e < kAP * kAK; e += 256) {
        const int r = e / kAK, kk = e - r * kAK;
        const int pt = p0 + r;
        xs[kk][r] = (pt < M && k0 + kk < d) ? (Acc)load_elem_d(src, p.dtype, xbase + (size_t)pt * d + k0 + kk) : Acc(0);
        const int cc = c0 + r;
        cs[kk][r] = (cc < kc && k0 + kk < d) ? (Acc)cent[(size_t)cc * d + k0 + kk] : Acc(0);
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < kAK; ++kk) {
        Acc a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = xs[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = cs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
    for (int e = tid; e < kAC; e += 256) cn[e] = (c0 + e < kc) ? (Acc)w.cnorm[(size_t)bh * p.k + c0 + e] : Acc(0);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c0 + tx * 4 + j;
      if (cc < kc) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double dist = (double)(xn[i] - Acc(2) * acc[i][j] + cn[tx * 4 + j]);
          if (dist < best[i]) {  // strict: lowest index wins ties
            best[i] = dist;
            bidx[i] = cc;
          }
        }
      }
    }
    __syncthreads();
  }
  // reduce across the 16 tx lanes sharing a point row (lowest index on ties)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double b = best[i];
    int bi = bidx[i];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < b || (ob == b && oi < bi)) {
        b = ob;
        bi = oi;
      }
    }
    const int pt = p0 + ty * 4 + i;
    if (tx == 0 && pt < M) {
      w.assign[(size_t)bh * M + pt] = bi;
      w.sqd[(size_t)bh * M + pt] = fmax(b, 0.0);
    }
  }
}

// -------------------------------------------------------------------------
// assignment on the 5th-gen tensor cores (fp64_assign == 2; bf16 keys,
// d in {64, 128}, k <= kTcMaxK).  dot(x, c) for 128 points x 128 centroids
// per accumulator tile with tcgen05.mma (kind::f16, bf16 in, fp32 in TMEM):
// the keys are exact in bf16 and every centroid is split into three bf16
// terms (hi + mid + lo carry 24 mantissa bits, i.e. the fp32 path's
// precision), accumulated into the same TMEM tile.  Warp roles: warp 0 issues
// TMA (keys tile once, then one (centroid tile, split term) per ring stage),
// warp 1 owns TMEM and issues the MMAs from one lane, warps 4-7 drain the
// double-buffered accumulator with tcgen05.ld and keep the running argmin
// (dist = |x|^2 - 2 x.c + |c|^2, ties -> lowest index) for their 32 points;
// when the runner-up is within the tensor-core error band the two candidates
// are re-scored in fp64, so near-ties resolve like the fp64 path.
// -------------------------------------------------------------------------
constexpr int kTcRows = 128;                   // points per CTA = centroids per tile = TMEM lanes
constexpr int kTcStages = 2;                   // ring of (tile, term) stages (2 CTAs per SM hide each other's tails)
constexpr int kTcHalf = kTcRows * 128;         // one 64-column swizzle half: 128 rows x 128 B
constexpr int kTcMaxK = 4096;
constexpr int kTcThreads = 256;  // warp 0 TMA, warp 1 MMA, warps 4-7 epilogue (one per TMEM lane quarter)

__device__ __forceinline__ unsigned tc_smem(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tc_bar_init(unsigned b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void tc_bar_tx(unsigned b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_bar_arrive(unsigned b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
}
__device__ __forceinline__ void tc_bar_wait(unsigned b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TCW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra TCW_%=;\n}\n" ::"r"(b), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_tma2d(unsigned dst, const CUtensorMap* m, int x, int y, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<unsigned long long>(m)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart
__device__ __forceinline__ unsigned long long tc_desc(unsigned saddr) {
  return (unsigned long long)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((unsigned long long)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

__global__ void __launch_bounds__(kTcThreads, 2)
    assign_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmC,
                     dp_cluster_params p, KmWs w, const __nv_bfloat16* __restrict__ tc_keys) {
  const int bh = blockIdx.y;
  if (w.done[bh]) return;
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim;
  const int p0 = blockIdx.x * kTcRows;
  if (p0 >= M) return;
  const int kc = w.knum[bh];
  const int halves = d / 64;
  const int ntile = (kc + kTcRows - 1) / kTcRows, nsteps = ntile * 3;
  const unsigned stage_bytes = (unsigned)halves * kTcHalf;
  extern __shared__ unsigned char tc_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* As = base;                                      // keys tile [halves][128 x 128 B]
  unsigned char* Bs = As + 2 * kTcHalf;                          // ring [stages][halves][128 x 128 B]
  float* cn = reinterpret_cast<float*>(Bs + kTcStages * 2 * kTcHalf);  // [kpad] centroid norms
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(cn + ((p.k + 31) & ~31));
  // bars: full[4], empty[4], afull, accf[2], acce[2]
  unsigned* tslot = reinterpret_cast<unsigned*>(bars + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned b0 = tc_smem(bars);
  auto FULL = [&](int s) { return b0 + 8u * s; };
  auto EMPTY = [&](int s) { return b0 + 8u * (kTcStages + s); };
  const unsigned AFULL = b0 + 8u * (2 * kTcStages);
  auto ACCF = [&](int b) { return b0 + 8u * (2 * kTcStages + 1 + b); };
  auto ACCE = [&](int b) { return b0 + 8u * (2 * kTcStages + 3 + b); };
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      tc_bar_init(FULL(s), 1);
      tc_bar_init(EMPTY(s), 1);
    }
    tc_bar_init(AFULL, 1);
    for (int b = 0; b < 2; ++b) {
      tc_bar_init(ACCF(b), 1);
      tc_bar_init(ACCE(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // 2 x 128 fp32 accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(tc_smem(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid >= 128)
    for (int c = tid - 128; c < kc; c += 128) cn[c] = (float)w.cnorm[(size_t)bh * p.k + c];
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const unsigned tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      const int xrow = bh * p.n_tokens + p.sink + p0;
      tc_bar_tx(AFULL, (unsigned)halves * kTcHalf);
      for (int hf = 0; hf < halves; ++hf) tc_tma2d(tc_smem(As + hf * kTcHalf), &tmX, hf * 64, xrow, AFULL);
      const int BHk = p.batch * p.kv_heads * p.k;
      for (int i = 0; i < nsteps; ++i) {
        const int s = i % kTcStages, j = i / 3, t = i - 3 * j;
        if (i >= kTcStages) tc_bar_wait(EMPTY(s), ((i / kTcStages) - 1) & 1);
        const int crow = t * BHk + bh * p.k + j * kTcRows;
        tc_bar_tx(FULL(s), stage_bytes);
        for (int hf = 0; hf < halves; ++hf)
          tc_tma2d(tc_smem(Bs + (s * 2 + hf) * kTcHalf), &tmC, hf * 64, crow, FULL(s));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: D[128 x 128] (+)= A[128 x 16] . B[128 x 16]^T per instruction
      const unsigned idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(kTcRows >> 3) << 17) |
                             ((unsigned)(kTcRows >> 4) << 24);
      tc_bar_wait(AFULL, 0);
      for (int i = 0; i < nsteps; ++i) {
        const int s = i % kTcStages, j = i / 3, t = i - 3 * j, b = j & 1;
        if (t == 0 && j >= 2) tc_bar_wait(ACCE(b), ((j >> 1) - 1) & 1);
        tc_bar_wait(FULL(s), (i / kTcStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const unsigned dt = tmem + (unsigned)(b * kTcRows);
        for (int kk = 0; kk < halves * 4; ++kk) {
          const unsigned off = (unsigned)((kk >> 2) * kTcHalf + (kk & 3) * 32);
          const unsigned long long da = tc_desc(tc_smem(As) + off);
          const unsigned long long db = tc_desc(tc_smem(Bs + s * 2 * kTcHalf) + off);
          const unsigned acc = (t > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(EMPTY(s))
                     : "memory");
        if (t == 2)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(ACCF(b))
                       : "memory");
      }
    }
  } else if (warp >= 4) {  // epilogue: TMEM lane quarter warp % 4 = my 32 points
    const int ew = warp - 4, row = ew * 32 + lane, pt = p0 + row;
    const float xn = pt < M ? (float)w.xnorm[(size_t)bh * M + pt] : 0.f;
    // four independent (best, runner-up) trackers over columns q % 4: the
    // compare chain is the epilogue's critical path, so it gets ILP
    float tb[4], tb2[4];
    int ti[4], ti2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      tb[u] = tb2[u] = CUDART_INF_F;
      ti[u] = 0x7fffffff;
      ti2[u] = -1;
    }
    for (int j = 0; j < ntile; ++j) {
      const int b = j & 1;
      tc_bar_wait(ACCF(b), (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
      for (int c0 = 0; c0 < kTcRows; c0 += 16) {
        unsigned v[16];
        const unsigned ta = tmem + ((unsigned)(ew * 32) << 16) + (unsigned)(b * kTcRows + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int cb = j * kTcRows + c0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int col = cb + q, u = q & 3;
          const float dist = col < kc ? fmaf(-2.f, __uint_as_float(v[q]), xn + cn[col]) : CUDART_INF_F;
          // branch-free (best, runner-up) update; strict: within a tracker the
          // columns arrive in increasing order, so ties keep the lower index
          const bool lt1 = dist < tb[u], lt2 = dist < tb2[u];
          tb2[u] = lt1 ? tb[u] : (lt2 ? dist : tb2[u]);
          ti2[u] = lt1 ? ti[u] : (lt2 ? col : ti2[u]);
          tb[u] = lt1 ? dist : tb[u];
          ti[u] = lt1 ? col : ti[u];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      tc_bar_arrive(ACCE(b));
    }
    // merge the trackers (static indexing only): lowest (dist, index) wins; the
    // runner-up of a merged pair is min(loser's best, winner's runner-up)
    float best = tb[0], best2 = tb2[0];
    int bi = ti[0], bi2 = ti2[0];
#pragma unroll
    for (int u = 1; u < 4; ++u) {
      if (tb[u] < best || (tb[u] == best && ti[u] < bi)) {
        if (best < tb2[u] || (best == tb2[u] && bi < ti2[u])) {
          best2 = best;
          bi2 = bi;
        } else {
          best2 = tb2[u];
          bi2 = ti2[u];
        }
        best = tb[u];
        bi = ti[u];
      } else if (tb[u] < best2 || (tb[u] == best2 && ti[u] < bi2)) {
        best2 = tb[u];
        bi2 = ti[u];
      }
    }
    if (bi == 0x7fffffff) bi = 0;
    if (pt < M) {
      // the winner is re-scored in fp64 (exact objective, the fp64 path's
      // formula); near-ties -- the runner-up within the tensor-core error
      // band (~1e-6 relative) -- are resolved the same way
      const bool tie = bi2 >= 0 && best2 - best <= 2e-5f * (xn + cn[bi]);
      const double* c1 = w.cent + ((size_t)bh * p.k + bi) * d;
      const double* c2 = w.cent + ((size_t)bh * p.k + (tie ? bi2 : bi)) * d;
      const __nv_bfloat16* xrow = tc_keys + ((size_t)bh * p.n_tokens + p.sink + pt) * d;
      double a1 = 0.0, a2 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll 4
      for (int e0 = 0; e0 < d; e0 += 8) {  // 16-B key loads, independent chains (latency, not flops)
        const uint4 raw = *reinterpret_cast<const uint4*>(xrow + e0);
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 xf = __bfloat1622float2(xh[t]);
          const double2 u = *reinterpret_cast<const double2*>(c1 + e0 + 2 * t);
          a1 = fma((double)xf.x, u.x, a1);
          b1 = fma((double)xf.y, u.y, b1);
          if (tie) {
            const double2 z = *reinterpret_cast<const double2*>(c2 + e0 + 2 * t);
            a2 = fma((double)xf.x, z.x, a2);
            b2 = fma((double)xf.y, z.y, b2);
          }
        }
      }
      a1 += b1;
      a2 += b2;
      const double xnd = w.xnorm[(size_t)bh * M + pt];
      double dbest = xnd - 2.0 * a1 + w.cnorm[(size_t)bh * p.k + bi];
      if (tie) {
        const double d2 = xnd - 2.0 * a2 + w.cnorm[(size_t)bh * p.k + bi2];
        if (d2 < dbest || (d2 == dbest && bi2 < bi)) {
          bi = bi2;
          dbest = d2;
        }
      }
      w.assign[(size_t)bh * M + pt] = bi;
      w.sqd[(size_t)bh * M + pt] = fmax(dbest, 0.0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

// centroids (fp64) -> three bf16 terms: hi = bf16(c), mid = bf16(c - hi), lo = bf16(c - hi - mid)
__global__ void csplit_kernel(dp_cluster_params p, KmWs w) {
  const int bh = blockIdx.y;
  if (w.done[bh]) return;
  const int d = p.head_dim, kc = w.knum[bh];
  const size_t BHk = (size_t)p.batch * p.kv_heads * p.k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kc * d; i += gridDim.x * blockDim.x) {
    const size_t o = (size_t)bh * p.k * d + i;
    const double c = w.cent[o];
    const __nv_bfloat16 hi = __double2bfloat16(c);
    const double r1 = c - (double)__bfloat162float(hi);
    const __nv_bfloat16 mid = __double2bfloat16(r1);
    const double r2 = r1 - (double)__bfloat162float(mid);
    w.csplit[o] = hi;
    w.csplit[BHk * d + o] = mid;
    w.csplit[2 * BHk * d + o] = __double2bfloat16(r2);
  }
}

typedef CUresult (*TcEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static cudaError_t tc_map(CUtensorMap* m, const void* ptr, unsigned long long rows, int d) {
  static TcEncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &qr) !=
            cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn)
      return cudaErrorNotSupported;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  if (rows < (unsigned long long)kTcRows) return cudaErrorInvalidValue;  // the kernel expects full 128-row boxes
  const cuuint32_t box[2] = {64, (cuuint32_t)kTcRows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static size_t tc_smem_bytes(int k) {  // ~101 KB at k = 1022: two CTAs per SM
  return 1024 + 2 * kTcHalf + (size_t)kTcStages * 2 * kTcHalf + (size_t)((k + 31) & ~31) * 4 + 16 * 8 + 16;
}

static bool tc_supported(const dp_cluster_params* p) {
  return p->dtype == DP_BF16 && (p->head_dim == 64 || p->head_dim == 128) && p->k <= kTcMaxK &&
         p->n_tokens - p->sink - p->window >= kTcRows;
}

static cudaError_t launch_assign_tc(const dp_cluster_params* p, const void* src, KmWs w, cudaStream_t st) {
  const int BH = p->batch * p->kv_heads;
  const int M = p->n_tokens - p->sink - p->window;
  CUtensorMap mx, mc;
  cudaError_t e = tc_map(&mx, src, (unsigned long long)BH * p->n_tokens, p->head_dim);
  if (e != cudaSuccess) return e;
  e = tc_map(&mc, w.csplit, std::max(3ull * BH * p->k, (unsigned long long)kTcRows), p->head_dim);
  if (e != cudaSuccess) return e;
  csplit_kernel<<<dim3((p->k * p->head_dim + 255) / 256, BH), 256, 0, st>>>(*p, w);
  const size_t smem = tc_smem_bytes(p->k);
  cudaFuncSetAttribute(assign_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  assign_tc_kernel<<<dim3((M + kTcRows - 1) / kTcRows, BH), kTcThreads, smem, st>>>(
      mx, mc, *p, w, static_cast<const __nv_bfloat16*>(src));
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// update: one CTA per head.  objective, counts, drop + ascending remap,
// convergence test, member offsets and a stable counting sort.
// -------------------------------------------------------------------------
constexpr int kUpdThreads = 1024;
constexpr int kSortSeg = 8;  // point segments (warps) of the member sort (fewer when k is large)

__global__ void __launch_bounds__(kUpdThreads) update_kernel(dp_cluster_params p, KmWs w, int it,
                                                           double* __restrict__ objective,
                                                           int* __restrict__ iters, int nseg) {
  const int bh = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  if (w.done[bh]) return;
  const int M = p.n_tokens - p.sink - p.window;
  const int kc = w.knum[bh];
  __shared__ double redd[33];
  __shared__ int redi[33];
  int* assign = w.assign + (size_t)bh * M;
  int* prev = w.prev + (size_t)bh * M;
  int* counts = w.counts + (size_t)bh * p.k;
  int* remap = w.remap + (size_t)bh * p.k;
  int* start = w.start + (size_t)bh * (p.k + 1);
  int* cursor = w.cursor + (size_t)bh * p.k;
  const double* sqd = w.sqd + (size_t)bh * M;

  double loc = 0.0;
  for (int i = tid; i < M; i += nt) loc += sqd[i];
  const double obj = block_sum(loc, redd);
  if (tid == 0) {
    objective[(size_t)bh * p.max_iters + it] = obj;
    iters[bh] = it + 1;
  }
  for (int c = tid; c < kc; c += nt) counts[c] = 0;
  __syncthreads();
  for (int i = tid; i < M; i += nt) atomicAdd(&counts[assign[i]], 1);
  __syncthreads();
  int base = 0, rowbase = 0;
  for (int c0 = 0; c0 < kc; c0 += nt) {
    const int c = c0 + tid;
    const int cnt = c < kc ? counts[c] : 0;
    const int used = cnt > 0;
    int tot, totr;
    const int ex = block_exclusive_scan(used, redi, &tot);
    const int exr = block_exclusive_scan(cnt, redi, &totr);
    if (c < kc) {
      remap[c] = used ? base + ex : -1;
      if (used) {
        start[base + ex] = rowbase + exr;
        cursor[base + ex] = rowbase + exr;
      }
    }
    base += tot;
    rowbase += totr;
  }
  const int knew = base;
  const bool dropped = knew < kc;
  __syncthreads();
  int diff = 0;
  for (int i = tid; i < M; i += nt) {
    const int a = remap[assign[i]];
    assign[i] = a;
    if (it > 0 && a != prev[i]) diff = 1;
  }
  diff = block_sum(diff, redi);
  if (!dropped && it > 0 && diff == 0) {
    if (tid == 0) w.done[bh] = 1;  // sorted/start from the previous iteration stay valid
    return;
  }
  for (int i = tid; i < M; i += nt) prev[i] = assign[i];
  if (tid == 0) {
    w.knum[bh] = knew;
    start[knew] = M;
  }
  __syncthreads();
  // stable counting sort of the members (ascending point index within each
  // cluster): kSortSeg warps each own a contiguous segment of the points;
  // per-segment cluster counts in shared memory, a per-cluster prefix over the
  // segments, then every warp places its points with shared-memory cursors
  // (no global read-modify-write on the dependent path)
  extern __shared__ int segc[];  // [nseg][k]
  int* sorted = w.sorted + (size_t)bh * M;
  const int seg = (M + nseg - 1) / nseg;
  const int warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < nseg * knew; i += nt) segc[i] = 0;
  __syncthreads();
  if (warp < nseg) {
    int* cnt = segc + warp * knew;
    const int s0 = warp * seg, s1 = min(M, s0 + seg);
    for (int b0 = s0; b0 < s1; b0 += 32) {
      const int i = b0 + lane;
      const unsigned act = __ballot_sync(0xffffffffu, i < s1);
      if (i < s1) {
        const int a = assign[i];
        const unsigned peers = __match_any_sync(act, a);
        if (lane == __ffs(peers) - 1) cnt[a] += __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int c = tid; c < knew; c += nt) {
    int run = start[c];
    for (int g = 0; g < nseg; ++g) {
      const int t = segc[g * knew + c];
      segc[g * knew + c] = run;
      run += t;
    }
  }
  __syncthreads();
  if (warp < nseg) {
    int* cur = segc + warp * knew;
    const int s0 = warp * seg, s1 = min(M, s0 + seg);
    for (int b0 = s0; b0 < s1; b0 += 32) {
      const int i = b0 + lane;
      const unsigned act = __ballot_sync(0xffffffffu, i < s1);
      if (i < s1) {
        const int a = assign[i];
        const unsigned peers = __match_any_sync(act, a);
        const int leader = __ffs(peers) - 1;
        const int rank = __popc(peers & ((1u << lane) - 1u));
        int pos = 0;
        if (lane == leader) {
          pos = cur[a];
          cur[a] = pos + __popc(peers);
        }
        pos = __shfl_sync(peers, pos, leader);
        sorted[pos + rank] = i;
      }
      __syncwarp();
    }
  }
}

// -------------------------------------------------------------------------
// means: warp per cluster, fp64 sums in ascending member order (the order of
// x64[assign == c].mean(axis=0)), then |c|^2 for the next assignment.
// -------------------------------------------------------------------------
__global__ void means_kernel(dp_cluster_params p, const void* __restrict__ src, KmWs w) {
  const int bh = blockIdx.y;
  if (w.done[bh]) return;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= w.knum[bh]) return;
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim;
  const int* start = w.start + (size_t)bh * (p.k + 1);
  const int* sorted = w.sorted + (size_t)bh * M;
  const size_t xbase = ((size_t)bh * p.n_tokens + p.sink) * d;
  const int s = start[c], e = start[c + 1];
  double acc[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t] = 0.0;
  for (int m = s; m < e; ++m) {
    const size_t xb = xbase + (size_t)sorted[m] * d;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = lane + 32 * t;
      if (j < d) acc[t] = acc[t] + load_elem_d(src, p.dtype, xb + j);
    }
  }
  const double n = (double)(e - s);
  double nrm = 0.0;
  double* cr = w.cent + ((size_t)bh * p.k + c) * d;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int j = lane + 32 * t;
    if (j < d) {
      const double mu = acc[t] / n;
      cr[j] = mu;
      nrm = fma(mu, mu, nrm);
    }
  }
  nrm = warp_sum(nrm);
  if (lane == 0) w.cnorm[(size_t)bh * p.k + c] = nrm;
}

// -------------------------------------------------------------------------
// finalize: cluster-contiguous rows + tables
// -------------------------------------------------------------------------
template <typename T>
__global__ void permute_rows_kernel(dp_cluster_params p, const T* __restrict__ sk, const T* __restrict__ sv, KmWs w,
                                    T* __restrict__ dk, T* __restrict__ dv, int row_cap, int* __restrict__ perm) {
  const int bh = blockIdx.y;
  const int N = p.n_tokens, M = N - p.sink - p.window, d = p.head_dim;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= N) return;
  int srcpos = row;
  if (row >= p.sink && row < p.sink + M) srcpos = p.sink + w.sorted[(size_t)bh * M + (row - p.sink)];
  const size_t so = ((size_t)bh * N + srcpos) * d, dof = ((size_t)bh * row_cap + row) * d;
  for (int j = lane; j < d; j += 32) {
    dk[dof + j] = sk[so + j];
    dv[dof + j] = sv[so + j];
  }
  if (lane == 0 && perm) perm[(size_t)bh * row_cap + row] = srcpos;
}

__global__ void tables_kernel(dp_cluster_params p, const void* __restrict__ sv, KmWs w, int* __restrict__ offs,
                              int* __restrict__ ncl, float* __restrict__ cent_out, float* __restrict__ vbar,
                              int cluster_cap) {
  const int bh = blockIdx.y;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int kn = w.knum[bh];
  const int M = p.n_tokens - p.sink - p.window, d = p.head_dim;
  const int* start = w.start + (size_t)bh * (p.k + 1);
  if (c == 0 && lane == 0) ncl[bh] = kn;
  if (c > kn) return;
  if (lane == 0) offs[(size_t)bh * (cluster_cap + 1) + c] = p.sink + start[c];
  if (c == kn) return;
  const int* sorted = w.sorted + (size_t)bh * M;
  const size_t vbase = ((size_t)bh * p.n_tokens + p.sink) * d;
  const int s = start[c], e = start[c + 1];
  double acc[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t] = 0.0;
  for (int m = s; m < e; ++m) {
    const size_t vb = vbase + (size_t)sorted[m] * d;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = lane + 32 * t;
      if (j < d) acc[t] = acc[t] + load_elem_d(sv, p.dtype, vb + j);
    }
  }
  const double n = (double)(e - s);
  const double* cr = w.cent + ((size_t)bh * p.k + c) * d;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int j = lane + 32 * t;
    if (j < d) {
      const size_t o = ((size_t)bh * cluster_cap + c) * d + j;
      cent_out[o] = (float)cr[j];
      vbar[o] = (float)(acc[t] / n);
    }
  }
}

// -------------------------------------------------------------------------
// nearest_centroid on arbitrary points (kernel-seam parity helper)
// -------------------------------------------------------------------------
__global__ void nearest_kernel(const void* __restrict__ pts, int dtype, int n, int d, const double* __restrict__ cents,
                               int k, int fp64, int* __restrict__ assign, double* __restrict__ sqdist) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= n) return;
  double xn = 0.0;
  for (int j = lane; j < d; j += 32) {
    const double x = load_elem_d(pts, dtype, (size_t)i * d + j);
    xn = fma(x, x, xn);
  }
  xn = warp_sum(xn);
  double best = CUDART_INF;
  int bi = 0;
  for (int c = 0; c < k; ++c) {
    double dot = 0.0, cn = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double x = load_elem_d(pts, dtype, (size_t)i * d + j);
      const double cv = cents[(size_t)c * d + j];
      if (fp64) dot = fma(x, cv, dot);
      else dot = (double)fmaf((float)x, (float)cv, (float)dot);
      cn = fma(cv, cv, cn);
    }
    dot = warp_sum(dot);
    cn = warp_sum(cn);
    const double dist = xn - 2.0 * dot + cn;
    if (dist < best) {
      best = dist;
      bi = c;
    }
  }
  if (lane == 0) {
    assign[i] = bi;
    sqdist[i] = fmax(best, 0.0);
  }
}

}  // namespace dp

using namespace dp;

extern "C" {

size_t dp_cluster_workspace_bytes(const dp_cluster_params* p) {
  if (!p) return 0;
  return km_layout(p, nullptr, nullptr);
}

static int check_pp(const dp_cluster_params* p) {
  const int es = p->dtype == DP_F32 ? 4 : 2;
  if ((p->head_dim * es) % 16 != 0) return set_error(DP_ERR_UNSUPPORTED, "head_dim * elem must be a multiple of 16");
  if (pp_smem(p) > 227 * 1024) return set_error(DP_ERR_UNSUPPORTED, "head_dim too large for the k-means++ tile");
  return DP_OK;
}

static int check_params(const dp_cluster_params* p) {
  if (!p) return set_error(DP_ERR_INVALID, "null params");
  if (p->sink < 0 || p->window < 0) return set_error(DP_ERR_INVALID, "sink and window must be >= 0");
  const int M = p->n_tokens - p->sink - p->window;
  if (M < 1) return set_error(DP_ERR_INVALID, "no middle tokens to cluster");
  if (p->k < 1) return set_error(DP_ERR_INVALID, "cluster count must be >= 1");
  if (p->k > M) return set_error(DP_ERR_INVALID, "more clusters than points");
  if (p->max_iters < 1) return set_error(DP_ERR_INVALID, "max_iters must be >= 1");
  if (p->head_dim < 1 || p->head_dim > 256) return set_error(DP_ERR_UNSUPPORTED, "head_dim must be in [1, 256]");
  if (p->dtype != DP_F32 && p->dtype != DP_BF16) return set_error(DP_ERR_INVALID, "unknown dtype");
  if (p->fp64_assign == 2 && !tc_supported(p))
    return set_error(DP_ERR_UNSUPPORTED, "tensor-core assignment needs bf16 keys, head_dim 64/128, k <= 4096");
  return DP_OK;
}

int dp_kmeanspp(const dp_cluster_params* p, const void* src_keys, const int32_t* first_pick, const double* uniforms,
                const int32_t* alt_picks, int32_t* degenerate_from, int32_t* picks, void* ws, size_t ws_bytes,
                void* stream) {
  int r = check_params(p);
  if (r) return r;
  if (ws_bytes < dp_cluster_workspace_bytes(p)) return set_error(DP_ERR_INVALID, "workspace too small");
  KmWs w;
  km_layout(p, &w, (char*)ws);
  cudaStream_t st = (cudaStream_t)stream;
  const int BH = p->batch * p->kv_heads;
  if ((r = check_pp(p))) return r;
  xnorm_kernel<<<dim3((p->n_tokens * 32 + 255) / 256, BH), 256, 0, st>>>(*p, src_keys, w);
  cudaError_t e = launch_kmeanspp(p, src_keys, first_pick, uniforms, alt_picks, degenerate_from, picks, w, st);
  return e == cudaSuccess ? DP_OK : set_cuda_error(e, "dp_kmeanspp");
}

int dp_cluster_build(const dp_cluster_params* p, const void* src_keys, const void* src_values,
                     const int32_t* first_pick, const double* uniforms, const int32_t* alt_picks,
                     int32_t* degenerate_from, void* dst_keys, void* dst_values, int32_t row_cap, int32_t* offs,
                     int32_t* nclusters, float* centroids, float* value_means, int32_t cluster_cap, int32_t* perm,
                     double* objective, int32_t* iters, void* ws, size_t ws_bytes, void* stream) {
  int r = check_params(p);
  if (r) return r;
  if (row_cap < p->n_tokens) return set_error(DP_ERR_INVALID, "row_cap < n_tokens");
  if (cluster_cap < p->k) return set_error(DP_ERR_INVALID, "cluster_cap < k");
  if (ws_bytes < dp_cluster_workspace_bytes(p)) return set_error(DP_ERR_INVALID, "workspace too small");
  KmWs w;
  km_layout(p, &w, (char*)ws);
  cudaStream_t st = (cudaStream_t)stream;
  const int BH = p->batch * p->kv_heads;
  const int M = p->n_tokens - p->sink - p->window;
  // picks are a by-product of seeding; park them in the `sorted` scratch
  cudaError_t e0;
  xnorm_kernel<<<dim3((M * 32 + 255) / 256, BH), 256, 0, st>>>(*p, src_keys, w);
  if ((r = check_pp(p))) return r;
  e0 = launch_kmeanspp(p, src_keys, first_pick, uniforms, alt_picks, degenerate_from, w.sorted, w, st);
  if (e0 != cudaSuccess) return set_cuda_error(e0, "dp_cluster_build (kmeans++)");
  cnorm_kernel<<<dim3((p->k * 32 + 255) / 256, BH), 256, 0, st>>>(*p, w);
  const int nseg = std::max(1, std::min(kSortSeg, (int)((200 * 1024) / ((size_t)p->k * sizeof(int)))));
  const size_t upd_smem = (size_t)nseg * p->k * sizeof(int);
  if ((size_t)p->k * sizeof(int) > 200 * 1024)
    return set_error(DP_ERR_UNSUPPORTED, "more than 51200 clusters per head");
  if (upd_smem > 48 * 1024)
    cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem);
  for (int it = 0; it < p->max_iters; ++it) {
    if (p->fp64_assign == 2) {
      const cudaError_t ea = launch_assign_tc(p, src_keys, w, st);
      if (ea != cudaSuccess) return set_cuda_error(ea, "dp_cluster_build (tensor-core assign)");
    } else if (p->fp64_assign)
      assign_kernel<double><<<dim3((M + kAP - 1) / kAP, BH), 256, 0, st>>>(*p, src_keys, w);
    else
      assign_kernel<float><<<dim3((M + kAP - 1) / kAP, BH), 256, 0, st>>>(*p, src_keys, w);
    update_kernel<<<BH, kUpdThreads, upd_smem, st>>>(*p, w, it, objective, iters, nseg);
    means_kernel<<<dim3((p->k * 32 + 255) / 256, BH), 256, 0, st>>>(*p, src_keys, w);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "dp_cluster_build (lloyd)");
  if (p->dtype == DP_F32)
    permute_rows_kernel<float><<<dim3((p->n_tokens + 7) / 8, BH), 256, 0, st>>>(
        *p, (const float*)src_keys, (const float*)src_values, w, (float*)dst_keys, (float*)dst_values, row_cap, perm);
  else
    permute_rows_kernel<__nv_bfloat16><<<dim3((p->n_tokens + 7) / 8, BH), 256, 0, st>>>(
        *p, (const __nv_bfloat16*)src_keys, (const __nv_bfloat16*)src_values, w, (__nv_bfloat16*)dst_keys,
        (__nv_bfloat16*)dst_values, row_cap, perm);
  tables_kernel<<<dim3(((p->k + 1) * 32 + 255) / 256, BH), 256, 0, st>>>(*p, src_values, w, offs, nclusters,
                                                                        centroids, value_means, cluster_cap);
  e = cudaGetLastError();
  return e == cudaSuccess ? DP_OK : set_cuda_error(e, "dp_cluster_build (tables)");
}

int dp_nearest_centroid(const void* points, int32_t dtype, int32_t n, int32_t d, const double* centroids, int32_t k,
                        int32_t fp64, int32_t* assign, double* sqdist, void* stream) {
  if (n < 1 || d < 1 || k < 1) return set_error(DP_ERR_INVALID, "empty input");
  nearest_kernel<<<(n * 32 + 255) / 256, 256, 0, (cudaStream_t)stream>>>(points, dtype, n, d, centroids, k, fp64,
                                                                         assign, sqdist);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DP_OK : set_cuda_error(e, "dp_nearest_centroid");
}

}  // extern "C"
