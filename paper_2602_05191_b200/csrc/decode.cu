// Double-P decode step on sm_100a: score -> select -> worklist -> split-KV
// attention -> LSE merge.  All stages are stream-ordered with no host sync;
// the data-dependent work lists live in device memory.
//
// Reference semantics (file:line into /root/reference/pkg/src/doublep):
//   score     engine.py:158-177   log_mass = C.q * scale + log|c|
//   select    engine.py:180-213, selection.py:36-65
//   attention engine.py:216-252   (exact rows + approx pseudo-rows, one Z)
//   dense     engine.py:122-144
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "host_state.h"
#include "decode_internal.h"

namespace dp {

// ---------------------------------------------------------------------------
// score: one CTA per (tile of 128 clusters, b*h).  Centroid rows are staged
// through shared memory with coalesced float4 loads; each thread owns one
// cluster and accumulates the G dot products in fp64 (products of fp32
// centroids and bf16/fp32 queries are exact in fp64, so the log-masses match
// the fp64 oracle to ~1e-16 and selection ties are only true ties).
// ---------------------------------------------------------------------------
constexpr int kScoreTile = 64;

__global__ void __launch_bounds__(kScoreTile) score_kernel(dp_cache_view v, const void* __restrict__ q,
                                                         int qdt, int G, double scale,
                                                         double* __restrict__ lm) {
  const int bh = blockIdx.y;
  const int K = v.nclusters[bh];
  const int k0 = blockIdx.x * kScoreTile;
  if (k0 >= K) return;
  const int d = v.head_dim, tid = threadIdx.x;
  const int stride = d + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* qs = reinterpret_cast<double*>(smem_raw);
  float* cs = reinterpret_cast<float*>(qs + G * d);
  // stage the raw queries and the centroid tile with cp.async (all loads in
  // flight at once), then widen the queries to fp64 in shared memory
  unsigned char* qraw = smem_raw + (size_t)G * d * 8 + (size_t)kScoreTile * stride * 4;
  const int esz = qdt == DP_F32 ? 4 : 2;
  const int qchunks = G * d * esz / 16;
  const unsigned char* qsrc = reinterpret_cast<const unsigned char*>(q) + (size_t)bh * G * d * esz;
  for (int i = tid; i < qchunks; i += blockDim.x) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(qraw + i * 16));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(qsrc + i * 16));
  }
  const int n = min(kScoreTile, K - k0);
  const int d4 = d >> 2;
  const float4* C4 = reinterpret_cast<const float4*>(v.centroids + ((size_t)bh * v.cluster_cap + k0) * d);
  for (int i = tid; i < n * d4; i += blockDim.x) {
    const int r = i / d4, c = i - r * d4;
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&cs[r * stride + 4 * c]));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(&C4[(size_t)r * d4 + c]));
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int i = tid; i < G * d; i += blockDim.x)
    qs[i] = esz == 4 ? (double)reinterpret_cast<const float*>(qraw)[i]
                     : (double)bf2f(reinterpret_cast<const __nv_bfloat16*>(qraw)[i]);
  __syncthreads();
  if (tid >= n) return;
  double acc[kMaxGroup];
#pragma unroll
  for (int g = 0; g < kMaxGroup; ++g) acc[g] = 0.0;
  const float* row = &cs[tid * stride];
  for (int j = 0; j < d; j += 4) {
    const float4 c4 = *reinterpret_cast<const float4*>(&row[j]);
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
      if (g < G) {
        const double* qg = &qs[g * d + j];
        double a = acc[g];
        a = fma((double)c4.x, qg[0], a);
        a = fma((double)c4.y, qg[1], a);
        a = fma((double)c4.z, qg[2], a);
        a = fma((double)c4.w, qg[3], a);
        acc[g] = a;
      }
    }
  }
  const int k = k0 + tid;
  const int* offs = v.offs + (size_t)bh * (v.cluster_cap + 1);
  const double ls = log((double)(offs[k + 1] - offs[k]));
#pragma unroll
  for (int g = 0; g < kMaxGroup; ++g)
    if (g < G) lm[((size_t)bh * G + g) * v.cluster_cap + k] = acc[g] * scale + ls;
}

// ---------------------------------------------------------------------------
// select: one CTA (1024 threads) per (b, q head).  softmax in fp64, then a
// shared-memory bitonic sort on (prob desc, cluster id asc) -- the exact
// order of the reference's stable argsort -- then one fp64 prefix scan that
// serves both top-p stages (stage 2 is a prefix of the same sorted order,
// engine.py:189-194).
// ---------------------------------------------------------------------------
constexpr int kSelectThreads = 1024;

__device__ __forceinline__ bool sel_before(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}

__global__ void __launch_bounds__(kSelectThreads) select_kernel(dp_cache_view v, int G, double p1,
                                                              double p2, const double* __restrict__ lm,
                                                              uint8_t* __restrict__ state,
                                                              int* __restrict__ counts,
                                                              int* __restrict__ order,
                                                              double* __restrict__ cum_mass,
                                                              double* __restrict__ probs, int Kp) {
  const int bhq = blockIdx.x, bh = bhq / G;
  const int K = v.nclusters[bh];
  const int cap = v.cluster_cap;
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* key = reinterpret_cast<double*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + Kp);
  __shared__ double red[33];
  __shared__ int s_n1, s_n2;
  const double* x = lm + (size_t)bhq * cap;

  double m = -CUDART_INF;
  for (int i = tid; i < K; i += nt) m = fmax(m, x[i]);
  m = block_max(m, red, -CUDART_INF);
  double s = 0.0;
  for (int i = tid; i < K; i += nt) {
    const double e = exp(x[i] - m);
    key[i] = e;
    s += e;
  }
  const double S = block_sum(s, red);
  double t = 0.0;
  for (int i = tid; i < Kp; i += nt) {
    if (i < K) {
      const double p = key[i] / S;
      key[i] = p;
      if (probs) probs[(size_t)bhq * cap + i] = p;
      idx[i] = i;
      t += p;
    } else {
      key[i] = -1.0;
      idx[i] = 0x7fffffff;
    }
  }
  const double total = block_sum(t, red);  // probs.sum(), selection.py:52
  __syncthreads();

  // bitonic sort, "ascending" in the sel_before order
  for (int kk = 2; kk <= Kp; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < Kp; i += nt) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double a = key[i], b = key[ixj];
          const int ia = idx[i], ib = idx[ixj];
          const bool up = (i & kk) == 0;
          const bool sw = up ? sel_before(b, ib, a, ia) : sel_before(a, ia, b, ib);
          if (sw) {
            key[i] = b; key[ixj] = a;
            idx[i] = ib; idx[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }

  // inclusive prefix sums of the sorted probs (overwrites key)
  const int per = (K + nt - 1) / nt;
  const int beg = min(K, tid * per), end = min(K, beg + per);
  double local = 0.0;
  for (int i = beg; i < end; ++i) local += key[i];
  double tot_unused;
  double c = block_exclusive_scan(local, red, &tot_unused);
  for (int i = beg; i < end; ++i) {
    c += key[i];
    key[i] = c;
  }
  if (tid == 0) { s_n1 = K; s_n2 = K; }
  __syncthreads();
  // stage 1: first i with cum_i/total >= p1 (searchsorted left + 1, clamped)
  for (int i0 = 0; i0 < K; i0 += nt) {  // first index per warp only -> <= 32 atomics
    const int i = i0 + tid;
    const unsigned b = __ballot_sync(0xffffffffu, i < K && key[i] / total >= p1);
    if (b && (tid & 31) == __ffs(b) - 1) atomicMin(&s_n1, i + 1);
  }
  __syncthreads();
  const int n1 = s_n1;
  const double sub_total = key[n1 - 1];  // probs[cp].sum(), engine.py:191
  for (int i0 = 0; i0 < n1; i0 += nt) {
    const int i = i0 + tid;
    const unsigned b = __ballot_sync(0xffffffffu, i < n1 && key[i] / sub_total >= p2);
    if (b && (tid & 31) == __ffs(b) - 1) atomicMin(&s_n2, i + 1);
  }
  __syncthreads();
  const int n2 = min(s_n2, n1);
  uint8_t* st = state + (size_t)bhq * cap;
  for (int r = tid; r < K; r += nt) {
    const int k = idx[r];
    st[k] = r < n2 ? 2 : (r < n1 ? 1 : 0);
    if (order) order[(size_t)bhq * cap + r] = k;
  }
  if (tid == 0) {
    counts[2 * bhq] = n1;
    counts[2 * bhq + 1] = n2;
    if (cum_mass) cum_mass[bhq] = key[n1 - 1] / total;
  }
}

// ---------------------------------------------------------------------------
// worklist: one CTA per (b, kv head).  Builds the GQA-union row runs
// (sink, window, then every cluster exact for >= 1 head of the group, in
// ascending cluster id == ascending row order) with a per-run head mask, and
// the union of approximated clusters with their head masks.
// ---------------------------------------------------------------------------
constexpr int kListThreads = 1024;

__global__ void __launch_bounds__(kListThreads) worklist_kernel(dp_cache_view v, int G,
                                                              const uint8_t* __restrict__ state,
                                                              WorkLists wl) {
  const int bh = blockIdx.x;
  const int K = v.nclusters[bh];
  const int cap = v.cluster_cap, tid = threadIdx.x;
  const int* offs = v.offs + (size_t)bh * (cap + 1);
  int4* runs = wl.runs + (size_t)bh * (cap + 2);
  int2* apx = wl.approx + (size_t)bh * cap;
  __shared__ int red[33];
  __shared__ int s_runs, s_rows, s_apx;
  const int full = (1 << G) - 1;
  unsigned* rowidx = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
  const unsigned ftag = (unsigned)full << 24;
  // packed union rows: (head mask << 24) | physical row
  for (int t = tid; t < v.sink; t += blockDim.x) rowidx[t] = ftag | (unsigned)t;
  for (int t = tid; t < v.window; t += blockDim.x) rowidx[v.sink + t] = ftag | (unsigned)(v.n_tokens - v.window + t);
  if (tid == 0) {
    int r = 0, rows = 0;
    if (v.sink > 0) { runs[r++] = make_int4(0, v.sink, full, rows); rows += v.sink; }
    if (v.window > 0) {
      runs[r++] = make_int4(v.n_tokens - v.window, v.window, full, rows);
      rows += v.window;
    }
    s_runs = r; s_rows = rows; s_apx = 0;
  }
  __syncthreads();
  for (int base = 0; base < K; base += blockDim.x) {
    const int k = base + tid;
    int me = 0, ma = 0, len = 0;
    if (k < K) {
      for (int g = 0; g < G; ++g) {
        const uint8_t s = state[((size_t)bh * G + g) * cap + k];
        me |= (s == 2) << g;
        ma |= (s == 1) << g;
      }
      if (me) len = offs[k + 1] - offs[k];
    }
    int tot_e, tot_a, tot_l;
    const int pe = block_exclusive_scan<int>(me != 0, red, &tot_e);
    const int pa = block_exclusive_scan<int>(ma != 0, red, &tot_a);
    const int pl = block_exclusive_scan<int>(len, red, &tot_l);
    const int rb = s_runs, rowb = s_rows, ab = s_apx;
    const int st0 = me ? offs[k] : 0;
    if (me) runs[rb + pe] = make_int4(st0, len, me, rowb + pl);
    if (ma) apx[ab + pa] = make_int2(k, ma);
    {  // warp-cooperative expansion of the warp's clusters: lanes write consecutive rows
      const int lane = tid & 31;
      unsigned todo = __ballot_sync(0xffffffffu, len > 0);
      while (todo) {
        const int t = __ffs(todo) - 1;
        todo &= todo - 1;
        const int tl = __shfl_sync(0xffffffffu, len, t);
        const int to = __shfl_sync(0xffffffffu, rowb + pl, t);
        const unsigned tag = (unsigned)__shfl_sync(0xffffffffu, me, t) << 24;
        const int ts = __shfl_sync(0xffffffffu, st0, t);
        for (int x = lane; x < tl; x += 32) rowidx[to + x] = tag | (unsigned)(ts + x);
      }
    }
    __syncthreads();
    if (tid == 0) { s_runs = rb + tot_e; s_rows = rowb + tot_l; s_apx = ab + tot_a; }
    __syncthreads();
  }
  if (tid == 0) {
    wl.nruns[bh] = s_runs;
    wl.nrows[bh] = s_rows;
    wl.napprox[bh] = s_apx;
    wl.nchunks[bh] = (s_rows + kChunkRows - 1) / kChunkRows;
    if (wl.stats) {
      wl.stats[4 * bh + 0] = s_rows;
      wl.stats[4 * bh + 1] = s_apx;
      wl.stats[4 * bh + 2] = (s_rows + kChunkRows - 1) / kChunkRows;
      wl.stats[4 * bh + 3] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// attention (generic CUDA-core path): one CTA per (row chunk, b*h).  The
// chunk's rows are gathered from the run list (cluster runs are contiguous
// in HBM, so the 16-byte cp.async copies coalesce), logits for all G heads
// are computed once per row and masked per head, and the chunk emits an
// unnormalised partial (m, l, o) per head.  T = storage type, Acc = fp64 for
// fp32 caches (1e-5 parity bar), fp32 for bf16.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

template <typename T, typename Acc, bool kDense>
__global__ void __launch_bounds__(kAttnThreads) attn_chunk_kernel(dp_cache_view v, const void* __restrict__ q,
                                                                 int qdt, int G, double scale, WorkLists wl,
                                                                 Partials<Acc> pt) {
  const int bh = blockIdx.y, c = blockIdx.x;
  const int rows_total = kDense ? v.n_tokens : wl.nrows[bh];
  const int nchunk = (rows_total + kChunkRows - 1) / kChunkRows;
  if (c >= nchunk) return;
  const int d = v.head_dim, tid = threadIdx.x, nt = blockDim.x;
  const int v0 = c * kChunkRows;
  const int nr = min(kChunkRows, rows_total - v0);
  const int rowb = d * (int)sizeof(T) + 16;  // padded row stride (bytes)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Acc* qs = reinterpret_cast<Acc*>(smem_raw);
  Acc* sc = qs + G * d;                                   // [G][R]
  // ONE row buffer: K, then (once the logits are taken) V -- half the shared memory, so two or
  // three CTAs share an SM and one's loads overlap another's arithmetic
  unsigned char* ks = reinterpret_cast<unsigned char*>(sc + G * kChunkRows);
  unsigned char* vs = ks;
  int* rphys = reinterpret_cast<int*>(ks + kChunkRows * rowb);
  int* rmask = rphys + kChunkRows;

  for (int i = tid; i < G * d; i += nt) qs[i] = (Acc)load_elem_d(q, qdt, (size_t)bh * G * d + i);
  const int full = (1 << G) - 1;
  for (int r = tid; r < kChunkRows; r += nt) {
    int phys = -1, mask = 0;
    if (r < nr) {
      const int vr = v0 + r;
      if (kDense) {
        phys = vr; mask = full;
      } else {
        const unsigned e = reinterpret_cast<const unsigned*>(wl.rowidx)[(size_t)bh * v.row_cap + vr];
        phys = (int)(e & 0xFFFFFFu);
        mask = (int)(e >> 24);
      }
    }
    rphys[r] = phys;
    rmask[r] = mask;
  }
  __syncthreads();
  const size_t head_off = (size_t)bh * v.row_cap * d;
  const T* Kg = reinterpret_cast<const T*>(v.keys) + head_off;
  const T* Vg = reinterpret_cast<const T*>(v.values) + head_off;
  const int ch = d * (int)sizeof(T) / 16;
  auto load_rows = [&](const T* G0, unsigned char* dst) {
    for (int i = tid; i < kChunkRows * ch; i += nt) {
      const int r = i / ch, cc = i - r * ch;
      const int phys = rphys[r];
      unsigned char* kd = dst + r * rowb + cc * 16;
      if (phys >= 0)
        cp_async16<T>(kd, reinterpret_cast<const unsigned char*>(G0 + (size_t)phys * d) + cc * 16);
      else
        *reinterpret_cast<int4*>(kd) = make_int4(0, 0, 0, 0);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  };
  load_rows(Kg, ks);

  // logits: thread per (head, row); lanes share the head -> q broadcast
  const Acc sc_scale = (Acc)scale;
  for (int i = tid; i < G * kChunkRows; i += nt) {
    const int g = i / kChunkRows, r = i - g * kChunkRows;
    Acc s = -INFINITY;
    if ((rmask[r] >> g) & 1) {
      const T* kr = reinterpret_cast<const T*>(ks + r * rowb);
      const Acc* qg = qs + g * d;
      Acc a[4] = {0, 0, 0, 0};  // four independent chains (d % 8 == 0): latency / 4
      for (int j = 0; j < d; j += 4) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if constexpr (sizeof(T) == 4) a[t] = fma((Acc)kr[j + t], qg[j + t], a[t]);
          else a[t] = fma((Acc)bf2f(kr[j + t]), qg[j + t], a[t]);
        }
      }
      s = ((a[0] + a[1]) + (a[2] + a[3])) * sc_scale;
    }
    sc[g * kChunkRows + r] = s;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int g = warp; g < G; g += nw) {
    Acc m = -INFINITY;
    for (int r = lane; r < kChunkRows; r += 32) m = max(m, sc[g * kChunkRows + r]);
    m = warp_max(m);
    Acc l = 0;
    for (int r = lane; r < kChunkRows; r += 32) {
      const Acc s = sc[g * kChunkRows + r];
      const Acc p = (m == -INFINITY || s == -INFINITY) ? Acc(0) : exp(s - m);
      sc[g * kChunkRows + r] = p;
      l += p;
    }
    l = warp_sum(l);
    if (lane == 0) {
      const size_t pi = ((size_t)bh * pt.max_chunks + c) * G + g;
      pt.m[pi] = m;
      pt.l[pi] = l;
    }
  }
  load_rows(Vg, vs);  // (the softmax barrier above: every logit read of K is done)
  for (int i = tid; i < G * d; i += nt) {
    const int g = i / d, j = i - g * d;
    const Acc* pg = sc + g * kChunkRows;
    Acc o[4] = {0, 0, 0, 0};  // four independent chains over the rows
    int r = 0;
    for (; r + 4 <= nr; r += 4) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const T* vr = reinterpret_cast<const T*>(vs + (r + t) * rowb);
        Acc val;
        if constexpr (sizeof(T) == 4) val = (Acc)vr[j];
        else val = (Acc)bf2f(vr[j]);
        o[t] = fma(pg[r + t], val, o[t]);
      }
    }
    for (; r < nr; ++r) {
      const T* vr = reinterpret_cast<const T*>(vs + r * rowb);
      Acc val;
      if constexpr (sizeof(T) == 4) val = (Acc)vr[j];
      else val = (Acc)bf2f(vr[j]);
      o[0] = fma(pg[r], val, o[0]);
    }
    pt.o[(((size_t)bh * pt.max_chunks + c) * G + g) * d + j] = (o[0] + o[1]) + (o[2] + o[3]);
  }
}

// ---------------------------------------------------------------------------
// merge: one CTA (8 warps) per (q head, b*h).  Combines the chunk partials
// with the approx pseudo-rows (logit = log_mass, value = value mean,
// engine.py:231-246) under one normaliser.  Chunks/approx rows are spread
// over threads/warps so every global load is issued in parallel.
// ---------------------------------------------------------------------------
constexpr int kMergeThreads = 256;

template <typename Acc, bool kDense>
__global__ void __launch_bounds__(kMergeThreads) merge_kernel(dp_cache_view v, int G, const double* __restrict__ lm,
                                                             WorkLists wl, Partials<Acc> pt, float* __restrict__ out,
                                                             float* __restrict__ lse) {
  const int g = blockIdx.x, bh = blockIdx.y, hq = bh * G + g;
  const int d = v.head_dim, tid = threadIdx.x, nt = blockDim.x, cap = v.cluster_cap;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int rows_total = kDense ? v.n_tokens : wl.nrows[bh];
  const int nch = (rows_total + kChunkRows - 1) / kChunkRows;
  const int na = kDense ? 0 : wl.napprox[bh];
  const int2* apx = wl.approx + (size_t)bh * cap;
  const float* vbar = v.value_means + (size_t)bh * cap * d;
  const double* lmh = lm ? lm + (size_t)hq * cap : nullptr;
  const size_t pbase = (size_t)bh * pt.max_chunks * G;
  __shared__ double red[33];
  __shared__ double oacc[8][256];

  double mloc = -CUDART_INF;
  for (int c = tid; c < nch; c += nt) mloc = fmax(mloc, (double)pt.m[pbase + (size_t)c * G + g]);
  for (int a = tid; a < na; a += nt) {
    const int2 e = apx[a];
    if ((e.y >> g) & 1) mloc = fmax(mloc, lmh[e.x]);
  }
  const double M = block_max(mloc, red, -CUDART_INF);
  double lloc = 0.0;
  for (int c = tid; c < nch; c += nt) {
    const double mc = pt.m[pbase + (size_t)c * G + g];
    if (mc != -CUDART_INF) lloc += (double)pt.l[pbase + (size_t)c * G + g] * exp(mc - M);
  }
  for (int a = tid; a < na; a += nt) {
    const int2 e = apx[a];
    if ((e.y >> g) & 1) lloc += exp(lmh[e.x] - M);
  }
  const double L = block_sum(lloc, red);

  double acc[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t] = 0.0;
  for (int c = warp; c < nch; c += nw) {
    const double mc = pt.m[pbase + (size_t)c * G + g];
    if (mc == -CUDART_INF) continue;
    const double w = exp(mc - M);
    const Acc* oc = pt.o + (pbase + (size_t)c * G + g) * d;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = lane + 32 * t;
      if (j < d) acc[t] += w * (double)oc[j];
    }
  }
  for (int a = warp; a < na; a += nw) {
    const int2 e = apx[a];
    if (!((e.y >> g) & 1)) continue;
    const double w = exp(lmh[e.x] - M);
    const float* vb = vbar + (size_t)e.x * d;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = lane + 32 * t;
      if (j < d) acc[t] += w * (double)vb[j];
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int j = lane + 32 * t;
    if (j < d) oacc[warp][j] = acc[t];
  }
  __syncthreads();
  for (int j = tid; j < d; j += nt) {
    double o = 0.0;
    for (int w = 0; w < nw; ++w) o += oacc[w][j];
    out[(size_t)hq * d + j] = (float)(o / L);
  }
  if (tid == 0) lse[hq] = (float)(M + log(L));
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
size_t attn_smem_bytes(int d, int G, int elem, int acc) {
  const int rowb = d * elem + 16;
  return (size_t)acc * (G * d + G * kChunkRows) + (size_t)kChunkRows * rowb + 2 * kChunkRows * 4;
}

int select_padded(int K) {
  int kp = 1;
  while (kp < K) kp <<= 1;
  return kp;
}

size_t decode_ws_layout(const dp_cache_view* v, int G, WorkLists* wl, void** parts, size_t* part_bytes,
                        char* base) {
  const size_t BH = (size_t)v->batch * v->kv_heads;
  const int cap = v->cluster_cap;
  // partial slots per head: one per 128-row chunk (generic kernel) or one
  // per CTA touching the head (persistent tensor-core kernel, grid <= kMaxPartSlots)
  const int max_chunks = std::max((v->row_cap + kChunkRows - 1) / kChunkRows, kMaxPartSlots);
  const size_t acc = v->dtype == DP_F32 ? 8 : 4;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return base ? base + o : nullptr;
  };
  char* runs = take(BH * (cap + 2) * sizeof(int4));
  char* apx = take(BH * cap * sizeof(int2));
  char* cnt = take(BH * 4 * sizeof(int));
  char* crun = take(BH * (size_t)v->row_cap * sizeof(int));
  char* ctr = take(BH * sizeof(int));
  char* cpre = take((BH + 1) * sizeof(int));
  char* dn = take(sizeof(int));
  char* ap = take(BH * (size_t)G * (4 + (size_t)v->head_dim) * sizeof(float));  // [m, l, -, -, o]
  char* ac = take(BH * (size_t)G * acc_stride(v->head_dim) * sizeof(float));  // (o, o, l, count) vectors
  char* rm = take(BH * (size_t)G * sizeof(float));
  const size_t pbytes = BH * max_chunks * G * (2 + (size_t)v->head_dim) * acc;
  char* p = take(pbytes);
  char* wlp = take(BH * (size_t)kWlMaxChunks * 4 * sizeof(int));  // split worklist: per-chunk totals
  char* wkey = take(BH * (size_t)G * 2 * sizeof(unsigned long long));  // per q head: lm max key, sink/window max
  if (wl) {
    wl->runs = reinterpret_cast<int4*>(runs);
    wl->approx = reinterpret_cast<int2*>(apx);
    int* c = reinterpret_cast<int*>(cnt);
    wl->nruns = c;
    wl->nrows = c + BH;
    wl->napprox = c + 2 * BH;
    wl->nchunks = c + 3 * BH;
    wl->stats = nullptr;
    wl->rowidx = reinterpret_cast<int*>(crun);
    wl->counters = reinterpret_cast<int*>(ctr);
    wl->chunk_prefix = reinterpret_cast<int*>(cpre);
    wl->done = reinterpret_cast<int*>(dn);
    wl->apart = reinterpret_cast<float*>(ap);
    wl->acc = reinterpret_cast<float*>(ac);
    wl->refm = reinterpret_cast<float*>(rm);
    wl->wlp = reinterpret_cast<int*>(wlp);
    wl->wkey = reinterpret_cast<unsigned long long*>(wkey);
    wl->max_chunks = max_chunks;
  }
  if (parts) *parts = p;
  if (part_bytes) *part_bytes = pbytes;
  return off;
}

template <typename Acc>
Partials<Acc> carve_partials(void* p, size_t BH, int max_chunks, int G, int d) {
  Partials<Acc> pt;
  pt.max_chunks = max_chunks;
  pt.m = reinterpret_cast<Acc*>(p);
  pt.l = pt.m + BH * max_chunks * G;
  pt.o = pt.l + BH * max_chunks * G;
  return pt;
}

cudaError_t launch_score(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double* lm,
                         cudaStream_t st) {
  const size_t smem = (size_t)G * v.head_dim * 8 + (size_t)kScoreTile * (v.head_dim + 4) * 4 +
                      (size_t)G * v.head_dim * 4;
  ensure_smem(reinterpret_cast<const void*>(score_kernel), 200 * 1024);
  dim3 grid((v.cluster_cap + kScoreTile - 1) / kScoreTile, v.batch * v.kv_heads);
  score_kernel<<<grid, kScoreTile, smem, st>>>(v, q, qdt, G, scale, lm);
  return cudaGetLastError();
}

// Fixed cluster-budget baseline (engine.py:318-338, RetroInfer-style): the
// `budget` clusters of largest estimated mass (the select kernel's full
// descending order) are exact, every other cluster is approximated; nothing
// is dropped.  Heads with fewer clusters keep all of them exact.
__global__ void __launch_bounds__(256) topk_state_kernel(dp_cache_view v, int G, int budget,
                                                         const int* __restrict__ order, uint8_t* __restrict__ state,
                                                         int* __restrict__ counts) {
  const int hq = blockIdx.x, bh = hq / G;
  const int K = v.nclusters[bh], cap = v.cluster_cap;
  const int k = budget < K ? budget : K;
  for (int i = threadIdx.x; i < K; i += blockDim.x)
    state[(size_t)hq * cap + order[(size_t)hq * cap + i]] = (uint8_t)(i < k ? 2 : 1);
  if (threadIdx.x == 0 && counts) {
    counts[2 * hq] = K;
    counts[2 * hq + 1] = k;
  }
}

cudaError_t launch_topk_state(const dp_cache_view& v, int G, int budget, const int* order, uint8_t* state,
                              int* counts, cudaStream_t st) {
  topk_state_kernel<<<v.batch * v.kv_heads * G, 256, 0, st>>>(v, G, budget, order, state, counts);
  return cudaGetLastError();
}

cudaError_t launch_select(const dp_cache_view& v, int G, double p1, double p2, const double* lm,
                          uint8_t* state, int* counts, int* order, double* cum, double* probs,
                          cudaStream_t st) {
  const int Kp = select_padded(std::max(1, v.cluster_cap));
  const size_t smem = (size_t)Kp * 12;
  ensure_smem(reinterpret_cast<const void*>(select_kernel), 200 * 1024);
  select_kernel<<<v.batch * v.kv_heads * G, kSelectThreads, smem, st>>>(v, G, p1, p2, lm, state, counts,
                                                                       order, cum, probs, Kp);
  return cudaGetLastError();
}

template <typename T, typename Acc, bool kDense>
cudaError_t launch_attn_t(const dp_cache_view& v, const void* q, int qdt, int G, double scale,
                          const double* lm, WorkLists wl, void* parts, float* out, float* lse,
                          cudaStream_t st) {
  const size_t BH = (size_t)v.batch * v.kv_heads;
  Partials<Acc> pt = carve_partials<Acc>(parts, BH, wl.max_chunks, G, v.head_dim);
  const size_t smem = attn_smem_bytes(v.head_dim, G, sizeof(T), sizeof(Acc));
  ensure_smem(reinterpret_cast<const void*>(attn_chunk_kernel<T, Acc, kDense>), 200 * 1024);
  const int rows = kDense ? v.n_tokens : v.row_cap;
  dim3 grid((rows + kChunkRows - 1) / kChunkRows, (unsigned)BH);
  cudaError_t e;
  if constexpr (sizeof(T) == 2 && sizeof(Acc) == 4) {
    if (v.head_dim == 128) {  // tensor-core kernel with the merge fused in (last CTA per head)
      return launch_attn_tc(v, q, qdt, G, scale, lm, wl, *reinterpret_cast<Partials<float>*>(&pt), out, lse,
                            kDense, st);
    } else {
      attn_chunk_kernel<T, Acc, kDense><<<grid, kAttnThreads, smem, st>>>(v, q, qdt, G, scale, wl, pt);
      e = cudaGetLastError();
    }
  } else {
    attn_chunk_kernel<T, Acc, kDense><<<grid, kAttnThreads, smem, st>>>(v, q, qdt, G, scale, wl, pt);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  merge_kernel<Acc, kDense><<<dim3(G, (unsigned)BH), kMergeThreads, 0, st>>>(v, G, lm, wl, pt, out, lse);
  return cudaGetLastError();
}

// approx partial per q head for the separate-kernel path (the fused plan
// computes it in-cluster): over state==1 clusters, m = max log-mass,
// l = sum e^(lm - m), o = sum e^(lm - m) * value_mean (engine.py:231-246)
__global__ void __launch_bounds__(256) approx_partial_kernel(dp_cache_view v, int G, const double* __restrict__ lm,
                                                            const uint8_t* __restrict__ state, WorkLists wl,
                                                            const void* __restrict__ q, int qdt, double scale,
                                                            int need_partial) {
  const int hq = blockIdx.x, bh = hq / G, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = v.nclusters[bh], cap = v.cluster_cap, d = v.head_dim;
  const double* x = lm + (size_t)hq * cap;
  const uint8_t* st = state + (size_t)hq * cap;
  __shared__ double red[33];
  __shared__ float part[8][256];
  double m = -CUDART_INF, mall = -CUDART_INF;
  for (int k0 = tid; k0 < K; k0 += blockDim.x * 8) {  // 8 loads in flight per thread
    double xv[8];
    uint8_t sv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = k0 + j * blockDim.x;
      xv[j] = k < K ? x[k] : -CUDART_INF;
      sv[j] = k < K ? st[k] : 0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (sv[j] == 1) m = fmax(m, xv[j]);
      mall = fmax(mall, xv[j]);
    }
  }
  // sink/window rows are always exact: their logits join the reference max
  // (q nullable: the dp_build_worklist entry point has no query)
  double sw = -CUDART_INF;
  if (q) {  // one warp per row, lanes over the dims (coalesced)
    const int nsw = v.sink + v.window;
    for (int t = warp; t < nsw; t += blockDim.x / 32) {
      const int row = t < v.sink ? t : v.n_tokens - v.window + (t - v.sink);
      double acc = 0.0;
      for (int c = lane; c < d; c += 32)
        acc += load_elem_d(v.keys, v.dtype, ((size_t)bh * v.row_cap + row) * d + c) *
               load_elem_d(q, qdt, (size_t)hq * d + c);
      acc = warp_sum(acc);
      if (acc == acc) sw = fmax(sw, acc * scale);
    }
  }
  const double M = block_max(m, red, -CUDART_INF);
  const double Mall = block_max(mall, red, -CUDART_INF);
  const double SW = block_max(sw, red, -CUDART_INF);
  // reference max of the tensor-core attention's accumulators (log2 units), as dp_plan writes it
  if (tid == 0) wl.refm[hq] = (float)(ref_max(Mall, SW) * 1.4426950408889634);
  if (!need_partial) return;  // the tensor-core attention folds the approximated clusters itself
  const float* vbar = v.value_means + (size_t)bh * cap * d;
  float acc[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t] = 0.f;
  double l = 0.0;
  for (int k = warp; k < K; k += blockDim.x / 32) {
    if (st[k] != 1) continue;
    const double e = exp(x[k] - M);
    if (lane == 0) l += e;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t < d) acc[t] += (float)e * vbar[(size_t)k * d + lane + 32 * t];
  }
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (lane + 32 * t < d) part[warp][lane + 32 * t] = acc[t];
  const double L = block_sum(l, red);
  float* ap = wl.apart + (size_t)hq * (4 + d);
  for (int c = tid; c < d; c += blockDim.x) {
    float sum = 0.f;
    for (int w = 0; w < 8; ++w) sum += part[w][c];
    ap[4 + c] = sum;
  }
  if (tid == 0) {
    ap[0] = M == -CUDART_INF ? -INFINITY : (float)M;
    ap[1] = (float)L;
  }
}

// ---------------------------------------------------------------------------
// Split worklist for the tensor-core attention (bf16, d = 128): the one-CTA-
// per-head worklist_kernel + approx_partial_kernel take ~35 us at K ~ 4K
// (8 CTAs).  Two launches over (256-cluster chunk, kv head) CTAs instead:
// wl_count (union lengths, chunk totals, the q heads' log-mass maxima and the
// sink/window logit maxima) and wl_write (chunk bases from the totals, the
// packed union rows, runs and approx lists; chunk 0 writes the head's
// counts and the accumulators' reference maxima).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long wl_dkey(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double wl_dfromkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

__device__ __forceinline__ void wl_masks(const uint8_t* __restrict__ state, int bh, int G, int cap, int k, int K,
                                         const int* __restrict__ offs, int& me, int& ma, int& len) {
  me = ma = len = 0;
  if (k < K) {
    for (int g = 0; g < G; ++g) {
      const uint8_t st = state[((size_t)bh * G + g) * cap + k];
      me |= (st == 2) << g;
      ma |= (st == 1) << g;
    }
    if (me) len = offs[k + 1] - offs[k];
  }
}

__global__ void __launch_bounds__(kWlThreads) wl_count_kernel(dp_cache_view v, int G, const uint8_t* __restrict__ state,
                                                             const double* __restrict__ lm, const void* __restrict__ q,
                                                             int qdt, double scale, WorkLists wl) {
  const int ch = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = v.nclusters[bh], cap = v.cluster_cap, d = v.head_dim;
  const int* offs = v.offs + (size_t)bh * (cap + 1);
  const int k = ch * kWlThreads + tid;
  int me, ma, len;
  wl_masks(state, bh, G, cap, k, K, offs, me, ma, len);
  __shared__ int red[3][kWlThreads / 32];
  const int r0 = warp_sum(len), r1 = warp_sum(ma != 0 ? 1 : 0), r2 = warp_sum(me != 0 ? 1 : 0);
  if (lane == 0) {
    red[0][warp] = r0;
    red[1][warp] = r1;
    red[2][warp] = r2;
  }
  // the q heads' log-mass maxima over my clusters (reference max of the attention accumulators)
  for (int g = 0; g < G; ++g) {
    double x = k < K ? lm[((size_t)bh * G + g) * cap + k] : -CUDART_INF;
    x = x != x ? -CUDART_INF : x;
    x = warp_max(x);
    if (lane == 0 && x != -CUDART_INF) atomicMax(&wl.wkey[((size_t)bh * G + g) * 2], wl_dkey(x));
  }
  __syncthreads();
  if (tid < 3) {
    int t = 0;
    for (int w = 0; w < kWlThreads / 32; ++w) t += red[tid][w];
    wl.wlp[((size_t)bh * kWlMaxChunks + ch) * 4 + tid] = t;
  }
  if (ch == 0 && q) {  // sink/window logits (always exact rows): one warp per row, lanes over dims
    const int nsw = v.sink + v.window;
    for (int g = 0; g < G; ++g) {
      double sw = -CUDART_INF;
      for (int t = warp; t < nsw; t += kWlThreads / 32) {
        const int row = t < v.sink ? t : v.n_tokens - v.window + (t - v.sink);
        double acc = 0.0;
        for (int c = lane; c < d; c += 32)
          acc += load_elem_d(v.keys, v.dtype, ((size_t)bh * v.row_cap + row) * d + c) *
                 load_elem_d(q, qdt, ((size_t)bh * G + g) * d + c);
        acc = warp_sum(acc);
        if (acc == acc) sw = fmax(sw, acc * scale);
      }
      if (lane == 0 && sw != -CUDART_INF) atomicMax(&wl.wkey[((size_t)bh * G + g) * 2 + 1], wl_dkey(sw));
    }
  }
}

__global__ void __launch_bounds__(kWlThreads) wl_write_kernel(dp_cache_view v, int G, const uint8_t* __restrict__ state,
                                                             WorkLists wl, int nch) {
  const int ch = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int K = v.nclusters[bh], cap = v.cluster_cap;
  const int* offs = v.offs + (size_t)bh * (cap + 1);
  __shared__ int s_base[3], s_tot[3];
  __shared__ int red[33];
  if (tid < 3) {  // my chunk's bases: the totals of the chunks before it
    int b = 0, t = 0;
    for (int c = 0; c < nch; ++c) {
      const int x = wl.wlp[((size_t)bh * kWlMaxChunks + c) * 4 + tid];
      if (c < ch) b += x;
      t += x;
    }
    s_base[tid] = b;
    s_tot[tid] = t;
  }
  const int k = ch * kWlThreads + tid;
  int me, ma, len;
  wl_masks(state, bh, G, cap, k, K, offs, me, ma, len);
  const int full = (1 << G) - 1;
  const int nsw_runs = (v.sink > 0) + (v.window > 0), sw_rows = v.sink + v.window;
  int tl, ta, te;
  const int pl = block_exclusive_scan<int>(len, red, &tl);
  const int pa = block_exclusive_scan<int>(ma != 0, red, &ta);
  const int pe = block_exclusive_scan<int>(me != 0, red, &te);
  const int rowb = sw_rows + s_base[0] + pl;
  unsigned* rowidx = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
  if (ma) wl.approx[(size_t)bh * cap + s_base[1] + pa] = make_int2(k, ma);
  const int st0 = me ? offs[k] : 0;
  if (me) wl.runs[(size_t)bh * (cap + 2) + nsw_runs + s_base[2] + pe] = make_int4(st0, len, me, rowb);
  unsigned todo = __ballot_sync(0xffffffffu, len > 0);
  while (todo) {  // warp-cooperative expansion: lanes write consecutive rows
    const int t = __ffs(todo) - 1;
    todo &= todo - 1;
    const int tlen = __shfl_sync(0xffffffffu, len, t);
    const int to = __shfl_sync(0xffffffffu, rowb, t);
    const unsigned tag = (unsigned)__shfl_sync(0xffffffffu, me, t) << 24;
    const int ts = __shfl_sync(0xffffffffu, st0, t);
    for (int x = lane; x < tlen; x += 32) rowidx[to + x] = tag | (unsigned)(ts + x);
  }
  if (ch == 0) {
    const unsigned ftag = (unsigned)full << 24;
    for (int t = tid; t < v.sink; t += kWlThreads) rowidx[t] = ftag | (unsigned)t;
    for (int t = tid; t < v.window; t += kWlThreads) rowidx[v.sink + t] = ftag | (unsigned)(v.n_tokens - v.window + t);
    if (tid == 0) {
      int r = 0;
      if (v.sink > 0) wl.runs[(size_t)bh * (cap + 2) + r++] = make_int4(0, v.sink, full, 0);
      if (v.window > 0) wl.runs[(size_t)bh * (cap + 2) + r++] = make_int4(v.n_tokens - v.window, v.window, full, v.sink);
      const int all_r = sw_rows + s_tot[0];
      wl.nrows[bh] = all_r;
      wl.napprox[bh] = s_tot[1];
      wl.nruns[bh] = nsw_runs + s_tot[2];
      wl.nchunks[bh] = (all_r + kChunkRows - 1) / kChunkRows;
      if (wl.stats) {
        wl.stats[4 * bh + 0] = all_r;
        wl.stats[4 * bh + 1] = s_tot[1];
        wl.stats[4 * bh + 2] = (all_r + kChunkRows - 1) / kChunkRows;
        wl.stats[4 * bh + 3] = s_tot[2];
      }
    }
    if (tid < G) {  // reference max (log2 units) as dp_plan writes it; keys re-armed for the next call
      unsigned long long* kk = wl.wkey + ((size_t)bh * G + tid) * 2;
      const double M = kk[0] ? wl_dfromkey(kk[0]) : -CUDART_INF;
      const double SW = kk[1] ? wl_dfromkey(kk[1]) : -CUDART_INF;
      wl.refm[(size_t)bh * G + tid] = (float)(ref_max(M, SW) * 1.4426950408889634);
      kk[0] = 0ull;
      kk[1] = 0ull;
    }
  }
}

cudaError_t launch_worklist(const dp_cache_view& v, int G, const uint8_t* state, int* stats, void* ws,
                            cudaStream_t st, const double* lm, const void* q, int qdt, double scale) {
  WorkLists wl;
  decode_ws_layout(&v, G, &wl, nullptr, nullptr, reinterpret_cast<char*>(ws));
  wl.stats = stats;
  const int nch = (v.cluster_cap + kWlThreads - 1) / kWlThreads;
  if (lm && v.dtype == DP_BF16 && v.head_dim == 128 && nch <= kWlMaxChunks) {
    // the tensor-core attention folds the approximated clusters itself: the
    // split two-launch worklist (no per-q-head approx partial needed)
    const dim3 g((unsigned)nch, (unsigned)(v.batch * v.kv_heads));
    wl_count_kernel<<<g, kWlThreads, 0, st>>>(v, G, state, lm, q, qdt, scale, wl);
    wl_write_kernel<<<g, kWlThreads, 0, st>>>(v, G, state, wl, nch);
    return cudaGetLastError();
  }
  worklist_kernel<<<v.batch * v.kv_heads, kListThreads, 0, st>>>(v, G, state, wl);
  if (lm && v.head_dim <= 256)
    approx_partial_kernel<<<v.batch * v.kv_heads * G, 256, 0, st>>>(v, G, lm, state, wl, q, qdt, scale,
                                                                    !(v.dtype == DP_BF16 && v.head_dim == 128));
  return cudaGetLastError();
}

cudaError_t launch_attend(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                          float* out, float* lse, void* ws, bool dense, cudaStream_t st) {
  WorkLists wl;
  void* parts = nullptr;
  decode_ws_layout(&v, G, &wl, &parts, nullptr, reinterpret_cast<char*>(ws));
  if (v.dtype == DP_F32) {
    return dense ? launch_attn_t<float, double, true>(v, q, qdt, G, scale, lm, wl, parts, out, lse, st)
                 : launch_attn_t<float, double, false>(v, q, qdt, G, scale, lm, wl, parts, out, lse, st);
  }
  return dense ? launch_attn_t<__nv_bfloat16, float, true>(v, q, qdt, G, scale, lm, wl, parts, out, lse, st)
               : launch_attn_t<__nv_bfloat16, float, false>(v, q, qdt, G, scale, lm, wl, parts, out, lse, st);
}

// ---------------------------------------------------------------------------
// decode-time growth (clustering.py:178-229): the new token lands at row
// n_tokens; the row that leaves the window (n_tokens - window) becomes a
// residual singleton cluster appended to the tables.  With the
// [sink | clusters | window] row layout this is an O(d) in-place update.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void append_kernel(dp_cache_view v, const T* __restrict__ nk, const T* __restrict__ nv) {
  const int bh = blockIdx.x, d = v.head_dim, tid = threadIdx.x;
  const int n = v.n_tokens, leave = n - v.window;
  T* K = const_cast<T*>(reinterpret_cast<const T*>(v.keys)) + (size_t)bh * v.row_cap * d;
  T* V = const_cast<T*>(reinterpret_cast<const T*>(v.values)) + (size_t)bh * v.row_cap * d;
  for (int j = tid; j < d; j += blockDim.x) {
    K[(size_t)n * d + j] = nk[(size_t)bh * d + j];
    V[(size_t)n * d + j] = nv[(size_t)bh * d + j];
  }
  int* ncl = const_cast<int*>(v.nclusters);
  const int kc = ncl[bh];
  __syncthreads();
  if (kc >= v.cluster_cap || leave < v.sink) return;
  float* C = const_cast<float*>(v.centroids) + ((size_t)bh * v.cluster_cap + kc) * d;
  float* Vb = const_cast<float*>(v.value_means) + ((size_t)bh * v.cluster_cap + kc) * d;
  for (int j = tid; j < d; j += blockDim.x) {
    if constexpr (sizeof(T) == 4) {
      C[j] = K[(size_t)leave * d + j];
      Vb[j] = V[(size_t)leave * d + j];
    } else {
      C[j] = bf2f(K[(size_t)leave * d + j]);
      Vb[j] = bf2f(V[(size_t)leave * d + j]);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int* offs = const_cast<int*>(v.offs) + (size_t)bh * (v.cluster_cap + 1);
    offs[kc] = leave;
    offs[kc + 1] = leave + 1;
    ncl[bh] = kc + 1;
  }
}

cudaError_t launch_append(const dp_cache_view& v, const void* nk, const void* nv, cudaStream_t st) {
  const int BH = v.batch * v.kv_heads;
  if (v.dtype == DP_F32)
    append_kernel<float><<<BH, 128, 0, st>>>(v, (const float*)nk, (const float*)nv);
  else
    append_kernel<__nv_bfloat16><<<BH, 128, 0, st>>>(v, (const __nv_bfloat16*)nk, (const __nv_bfloat16*)nv);
  return cudaGetLastError();
}

}  // namespace dp
