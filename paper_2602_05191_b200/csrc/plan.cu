// Fused per-layer "plan": size-weighted centroid scoring + two-stage top-p +
// approx partial + GQA-union work list, one launch, one 8-CTA thread-block
// cluster per (sequence, kv head); stages hand data over through distributed
// shared memory instead of HBM round trips.
//
//   phase 1  score   (engine.py:158-177)  CTA r scores clusters [r*per, (r+1)*per)
//                    for every q head of the group: 8 lanes per centroid row,
//                    fp32 query/centroid products accumulated in fp64 (exact
//                    products, so log-masses match the fp64 oracle to ~1e-15).
//   phase 2  select  (engine.py:180-213, selection.py:36-65)  CTA g (g < G) owns
//                    q head g: gathers its K log-masses over DSMEM, e = exp(lm -
//                    max), a mass histogram over 1/16-nat log bins finds the bin
//                    where the cumulative mass crosses p1 (then p2 of the
//                    retained mass); only those boundary bins are sorted (prob
//                    desc, cluster id asc == the stable argsort order) to place
//                    the exact cuts.  It then folds the head's approximated
//                    clusters (logit = log-mass, value = value mean,
//                    engine.py:231-246) into one (m, l, o) partial.
//   phase 3  worklist  every CTA reads all head states over DSMEM, computes
//                    the GQA-union prefix itself (no extra cluster barrier) and
//                    writes its slice's packed row entries (head mask << 24 |
//                    physical row) and (cluster, mask) approx entries.
//
// Cut semantics follow the reference: the first prefix whose cumsum/total
// >= p (searchsorted left + 1, clamped to n); ties -> lower cluster id.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode_internal.h"

namespace cg = cooperative_groups;

namespace dp {

constexpr int kCl = 8;         // CTAs per cluster (portable size)
constexpr int kPT = 256;       // threads per CTA
constexpr int kBins = 1024;    // log-mass bins of width 1/16 nat (span 64 nats)
constexpr float kBinScale = 16.f;
constexpr int kTile = 32;      // centroid rows per score tile (8 lanes per row)
constexpr int kPlanMaxCap = 4096;

// phase timestamps (%globaltimer, ns) of cluster 0: [rank][event]; read with
// dp_debug_plan_timing() -- profiling aid only
__device__ unsigned long long g_plan_ts[kCl][16];
__device__ __forceinline__ void stamp(int r, int ev) {
  if (blockIdx.x < kCl && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_plan_ts[r][ev] = t;
  }
}

__device__ __forceinline__ bool before(double pa, int ia, double pb, int ib) {
  return pa > pb || (pa == pb && ia < ib);
}

struct PlanLayout {
  int per;
  size_t qf, lmS, full, bin, st, bins, cand, ctile, offs, total;
};

__host__ __device__ inline PlanLayout plan_layout(int d, int cap) {
  PlanLayout L;
  L.per = (cap + kCl - 1) / kCl;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += (bytes + 15) & ~size_t(15);
    return r;
  };
  L.qf = take((size_t)kMaxGroup * d * 4);
  L.lmS = take((size_t)kMaxGroup * L.per * 8);
  L.full = take((size_t)cap * 8);
  L.bin = take((size_t)cap * 2);
  L.st = take((size_t)cap);
  L.bins = take((size_t)kBins * 12 > (size_t)cap * 4 ? (size_t)kBins * 12 : (size_t)cap * 4);  // bins | approx ids
  const size_t capP = (size_t)(cap + 15) & ~size_t(15);  // 16-B aligned state rows
  L.cand = take((size_t)cap * 16 > (size_t)kMaxGroup * capP ? (size_t)cap * 16 : (size_t)kMaxGroup * capP);
  L.ctile = take((size_t)2 * kTile * (d + 4) * 4 > (size_t)8 * 256 * 4 ? (size_t)2 * kTile * (d + 4) * 4
                                                                        : (size_t)8 * 256 * 4);
  L.offs = take((size_t)(cap + 1) * 4);  // the head's cluster row offsets
  L.total = o;
  return L;
}

// warp-level search over the bins: first non-empty bin b < limit at which
// the running mass reaches thresh; *before_mass / *before_cnt receive the mass
// and count of the bins before it (limit if never reached)
__device__ int bin_search(const double* bmass, const int* bcnt, int limit, double thresh, double* before_mass,
                          int* before_cnt) {
  const int lane = threadIdx.x & 31;
  constexpr int per = kBins / 32;
  double ms = 0.0;
  int cs = 0;
#pragma unroll 8
  for (int j = 0; j < per; ++j) {
    const int b = lane * per + j;
    if (b < limit) {
      ms += bmass[b];
      cs += bcnt[b];
    }
  }
  double inc = ms;
  int ci = cs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, inc, o);
    const int tc = __shfl_up_sync(0xffffffffu, ci, o);
    if (lane >= o) {
      inc += t;
      ci += tc;
    }
  }
  const unsigned hit = __ballot_sync(0xffffffffu, inc >= thresh && cs > 0);
  if (!hit) {
    *before_mass = __shfl_sync(0xffffffffu, inc, 31);
    *before_cnt = __shfl_sync(0xffffffffu, ci, 31);
    return limit;
  }
  const int f = __ffs(hit) - 1;
  double run = __shfl_sync(0xffffffffu, inc - ms, f);
  int crun = __shfl_sync(0xffffffffu, ci - cs, f);
  int res = limit;
  if (lane == f) {
    // the crossing lies in lane f's bins; if its sequential re-sum rounds
    // below thresh, fall back to its last non-empty bin (a threshold tie)
    int last = -1;
    double run_last = run;
    int crun_last = crun;
    for (int j = 0; j < per; ++j) {
      const int b = f * per + j;
      if (b >= limit) break;
      if (bcnt[b] > 0) {
        if (run + bmass[b] >= thresh) {
          res = b;
          break;
        }
        last = b;
        run_last = run;
        crun_last = crun;
      }
      run += bmass[b];
      crun += bcnt[b];
    }
    if (res == limit && last >= 0) {
      res = last;
      run = run_last;
      crun = crun_last;
    }
  }
  res = __shfl_sync(0xffffffffu, res, f);
  *before_mass = __shfl_sync(0xffffffffu, run, f);
  *before_cnt = __shfl_sync(0xffffffffu, crun, f);
  return res;
}

// warp: first j in [0, n) with (base + sum_{t<=j} p[order[t]]) >= thresh
// (n if never); *at receives the inclusive sum at the cut (or the full sum)
__device__ int warp_cut(const double* cp, const int* order, int n, double base, double thresh, double* at) {
  const int lane = threadIdx.x & 31;
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    const double val = j < n ? cp[order[j]] : 0.0;
    double inc = val;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const double cum = base + inc;
    const unsigned hit = __ballot_sync(0xffffffffu, j < n && cum >= thresh);
    if (hit) {
      const int f = __ffs(hit) - 1;
      *at = __shfl_sync(0xffffffffu, cum, f);
      return j0 + f;
    }
    base += __shfl_sync(0xffffffffu, inc, 31);
  }
  *at = base;
  return n;
}

template <int kG>  // compile-time bound on the GQA group (G <= kG), keeps the head loops branch-free
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kPT, 1)
    plan_kernel(dp_cache_view v, const void* __restrict__ q, int qdt, int G, double scale, double p1, double p2,
                double* __restrict__ lm_out, uint8_t* __restrict__ state_out, int* __restrict__ counts,
                WorkLists wl) {
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int bh = blockIdx.x / kCl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = v.head_dim, cap = v.cluster_cap;
  const int K = v.nclusters[bh];
  const PlanLayout L = plan_layout(d, cap);
  const int per = L.per;
  const int k0 = r * per;
  const int nloc = max(0, min(per, K - k0));
  extern __shared__ __align__(16) unsigned char smem[];
  int* offs = reinterpret_cast<int*>(smem + L.offs);  // staged copy of v.offs[bh]
  float* qf = reinterpret_cast<float*>(smem + L.qf);       // [8][d]
  double* lmS = reinterpret_cast<double*>(smem + L.lmS);  // [8][per]
  double* full = reinterpret_cast<double*>(smem + L.full);
  uint16_t* bin16 = reinterpret_cast<uint16_t*>(smem + L.bin);
  uint8_t* stS = reinterpret_cast<uint8_t*>(smem + L.st);
  double* bmass = reinterpret_cast<double*>(smem + L.bins);
  int* bcnt = reinterpret_cast<int*>(bmass + kBins);
  int* alist = reinterpret_cast<int*>(smem + L.bins);      // phase 2 tail: approx ids
  double* cp_ = reinterpret_cast<double*>(smem + L.cand);  // candidate probs
  int* cid = reinterpret_cast<int*>(cp_ + cap);             // candidate ids
  int* cord = cid + cap;                                    // sorted order (slots)
  uint8_t* stall = reinterpret_cast<uint8_t*>(smem + L.cand);  // phase 3: [G][K] states
  float* ctile = reinterpret_cast<float*>(smem + L.ctile);
  float* ared = ctile;                                      // phase 2 tail: [8 warps][256]
  __shared__ double red[33];
  __shared__ int redi[33];
  __shared__ double s_lmax[kMaxGroup];
  __shared__ int s_b1, s_b2, s_nc, s_c1, s_c2;
  __shared__ double s_sub;

  stamp(r, 0);
  // ---------------- phase 1: score my slice for all G heads ---------------
  // 8 lanes per centroid row (a warp reads 4 rows = 2 KB contiguous with
  // float4 loads straight into registers, one tile of 32 rows ahead); each
  // lane runs G independent fp64 chains over its d/8 dims, then the 8 lanes
  // combine with shuffles.  No shared-memory staging, no barriers.
  const int part = tid & 7, row = tid >> 3;
  const int dpp = d / 8;       // dims per lane (16 at d = 128)
  const int nv = dpp / 4;      // float4 per lane per row (<= 4)
  const float4* C4 = reinterpret_cast<const float4*>(v.centroids + ((size_t)bh * cap + k0) * d);
  const int ntiles = (nloc + kTile - 1) / kTile;
  float4 cur[4], nxt[4];
  // lane `part` of a row reads float4 j*8 + part (j < nv): 8 lanes cover
  // 128 contiguous bytes per step
  auto load_row = [&](int t, float4 (&dst)[4]) {
    const int rr = t * kTile + row;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      dst[j] = (rr < nloc && j < nv) ? __ldg(&C4[(size_t)rr * (d / 4) + j * 8 + part]) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  if (ntiles > 0) load_row(0, cur);
  {
    const int* goffs = v.offs + (size_t)bh * (cap + 1);
    for (int i = tid; i <= K; i += kPT) offs[i] = __ldg(&goffs[i]);
    for (int i = tid; i < kG * d; i += kPT) qf[i] = i < G * d ? load_elem_f(q, qdt, (size_t)bh * G * d + i) : 0.f;
  }
  __syncthreads();
  stamp(r, 12);
  double lmax[kG];
#pragma unroll
  for (int g = 0; g < kG; ++g) lmax[g] = -CUDART_INF;
  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) load_row(t + 1, nxt);
    double acc[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) acc[g] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < nv) {
        const float4 c4 = cur[j];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const float4 q4 = *reinterpret_cast<const float4*>(qf + g * d + 4 * (j * 8 + part));
          acc[g] = fma((double)c4.x, (double)q4.x, acc[g]);
          acc[g] = fma((double)c4.y, (double)q4.y, acc[g]);
          acc[g] = fma((double)c4.z, (double)q4.z, acc[g]);
          acc[g] = fma((double)c4.w, (double)q4.w, acc[g]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], 1);
      acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], 2);
      acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], 4);
    }
    const int rr = t * kTile + row;
    if (rr < nloc) {
      const int k = k0 + rr;
      const double ls = log((double)(offs[k + 1] - offs[k]));
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        if (g < G && part == g) {
          const double val = acc[g] * scale + ls;
          lmS[g * per + rr] = val;
          lm_out[((size_t)bh * G + g) * cap + k] = val;
          lmax[g] = fmax(lmax[g], val);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) cur[j] = nxt[j];
  }
  stamp(r, 13);
  {  // per-head max of my slice: one barrier
    __shared__ double s_wm[kPT / 32][kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      const double m = warp_max(lmax[g]);
      if (lane == 0) s_wm[warp][g] = m;
    }
    __syncthreads();
    if (tid < G) {
      double mm = -CUDART_INF;
#pragma unroll
      for (int w = 0; w < kPT / 32; ++w) mm = fmax(mm, s_wm[w][tid]);
      s_lmax[tid] = mm;
    }
  }
  stamp(r, 1);
  cluster.sync();  // (A) every slice scored
  stamp(r, 2);

  // ---------------- phase 2: two-stage top-p for q head g = r --------------
  if (r < G) {
    const int g = r;
    double M = -CUDART_INF;
    for (int rr = 0; rr < kCl; ++rr) M = fmax(M, cluster.map_shared_rank(s_lmax, rr)[g]);
    for (int b = tid; b < kBins; b += kPT) {
      bmass[b] = 0.0;
      bcnt[b] = 0;
    }
    __syncthreads();
    double s = 0.0;
    for (int i = tid; i < K; i += kPT) {
      const int rr = i / per;
      const double lmv = cluster.map_shared_rank(lmS, rr)[g * per + (i - rr * per)];
      const double e = exp(lmv - M);  // unnormalised softmax (engine.py:168); ratios are scale-free
      int b = (int)((float)(M - lmv) * kBinScale);
      b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
      full[i] = e;
      bin16[i] = (uint16_t)b;
      atomicAdd(&bmass[b], e);
      atomicAdd(&bcnt[b], 1);
      s += e;
    }
    const double total = block_sum(s, red);  // also orders the histogram
    stamp(r, 8);
    // gather + rank-sort the elements of bin `bin` into candidate slots [base, base+n)
    auto sort_bin = [&](int bin, int base) -> int {
      if (tid == 0) s_nc = 0;
      __syncthreads();
      for (int i = tid; i < K; i += kPT) {
        if (bin16[i] == bin) {
          const int slot = atomicAdd(&s_nc, 1);
          cp_[base + slot] = full[i];
          cid[base + slot] = i;
        }
      }
      __syncthreads();
      const int n = s_nc;
      for (int a = tid; a < n; a += kPT) {
        const double pa = cp_[base + a];
        const int ia = cid[base + a];
        int rk = 0;
        for (int j = 0; j < n; ++j) rk += before(cp_[base + j], cid[base + j], pa, ia);
        cord[base + rk] = base + a;
      }
      __syncthreads();
      return n;
    };
    // stage 1: bin holding the crossing of p1 * total
    if (warp == 0) {
      double bm;
      int bc;
      const int b1 = bin_search(bmass, bcnt, kBins, p1 * total, &bm, &bc);
      if (lane == 0) {
        s_b1 = b1;
        s_c1 = bc;
        red[1] = bm;
      }
    }
    __syncthreads();
    const int b1 = s_b1, c1 = s_c1;
    const double before1 = red[1];
    stamp(r, 9);
    int n1c = 0, cut1 = 0;
    if (b1 < kBins) {
      n1c = sort_bin(b1, 0);
      if (warp == 0) {
        double at;
        const int j = warp_cut(cp_, cord, n1c, before1, p1 * total, &at);
        if (lane == 0) {
          s_nc = j < n1c ? j + 1 : n1c;
          s_sub = j < n1c ? at : before1 + bmass[b1];
        }
      }
    } else if (tid == 0) {
      s_sub = before1;  // p1 never reached (rounding at p1 = 1): keep everything
    }
    __syncthreads();
    if (b1 < kBins) cut1 = s_nc;
    const double sub = s_sub;  // retained mass, probs[cp].sum() (engine.py:191)
    stamp(r, 10);
    // stage 2 (engine.py:191-194): same descending order, threshold p2 * sub
    if (warp == 0) {
      double bm;
      int bc;
      const int b2 = bin_search(bmass, bcnt, b1 < kBins ? b1 : kBins, p2 * sub, &bm, &bc);
      if (lane == 0) {
        s_b2 = b2;
        s_c2 = bc;
        red[2] = bm;
      }
    }
    __syncthreads();
    const int b2 = s_b2 < b1 ? s_b2 : b1;
    const int c2 = s_b2 < b1 ? s_c2 : c1;
    const double before2 = s_b2 < b1 ? red[2] : before1;
    int cut2 = 0, n2c = 0;
    const int base2 = n1c;
    if (b2 < b1) {
      n2c = sort_bin(b2, base2);
      if (warp == 0) {
        double at;
        const int j = warp_cut(cp_, cord + base2, n2c, before2, p2 * sub, &at);
        if (lane == 0) s_nc = j < n2c ? j + 1 : n2c;
      }
      __syncthreads();
      cut2 = s_nc;
    } else if (b1 < kBins) {
      if (warp == 0) {
        double at;
        const int j = warp_cut(cp_, cord, cut1, before1, p2 * sub, &at);
        if (lane == 0) s_nc = j < cut1 ? j + 1 : cut1;
      }
      __syncthreads();
      cut2 = s_nc;
    }
    stamp(r, 11);
    // states: 2 exact, 1 approx, 0 dropped
    for (int i = tid; i < K; i += kPT) {
      const int b = bin16[i];
      stS[i] = (uint8_t)(b < b2 ? 2 : (b < b1 ? 1 : 0));
    }
    __syncthreads();
    if (b1 < kBins)
      for (int j = tid; j < n1c; j += kPT)
        stS[cid[cord[j]]] = (uint8_t)(j < cut1 ? (b2 == b1 && j < cut2 ? 2 : 1) : 0);
    if (b2 < b1)
      for (int j = tid; j < n2c; j += kPT) stS[cid[cord[base2 + j]]] = (uint8_t)(j < cut2 ? 2 : 1);
    __syncthreads();
    const int hq = bh * G + g;
    {  // counts straight from the states, so they can never disagree
      int n1 = 0, n2 = 0;
      for (int i = tid; i < K; i += kPT) {
        n1 += stS[i] >= 1;
        n2 += stS[i] == 2;
      }
      n1 = block_sum(n1, redi);
      n2 = block_sum(n2, redi);
      if (tid == 0) {
        counts[2 * hq] = n1;
        counts[2 * hq + 1] = n2;
      }
    }
    (void)c1;
    (void)c2;
    if (state_out)
      for (int i = tid; i < K; i += kPT) state_out[(size_t)hq * cap + i] = stS[i];
    // approx partial: m = M, l = sum e, o = sum e * value_mean over state==1
    int na = 0;
    {
      int cnt = 0;
      const int per_t = (K + kPT - 1) / kPT;
      const int beg = min(K, tid * per_t), end = min(K, beg + per_t);
      for (int i = beg; i < end; ++i) cnt += stS[i] == 1;
      int tot;
      int off = block_exclusive_scan(cnt, redi, &tot);
      for (int i = beg; i < end; ++i)
        if (stS[i] == 1) alist[off++] = i;
      na = tot;
      __syncthreads();
    }
    const float* vbar = v.value_means + (size_t)bh * cap * d;
    const int nq = d / 4;  // float4 columns (d <= 128 -> at most one per lane)
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    double lsum = 0.0;
    for (int a0 = warp; a0 < na; a0 += 4 * (kPT / 32)) {
      float4 vb[4];
      float wt[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int a = a0 + u * (kPT / 32);
        const int k = a < na ? alist[a] : 0;
        wt[u] = a < na ? (float)full[k] : 0.f;
        vb[u] = (a < na && lane < nq) ? *(reinterpret_cast<const float4*>(vbar + (size_t)k * d) + lane)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        if (lane == 0 && a < na) lsum += full[k];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += wt[u] * vb[u].x; acc.y += wt[u] * vb[u].y; acc.z += wt[u] * vb[u].z; acc.w += wt[u] * vb[u].w;
      }
    }
    reinterpret_cast<float4*>(ared + warp * 256)[lane] = acc;
    if (lane == 0) red[warp] = lsum;
    __syncthreads();
    float* ap = wl.apart + (size_t)hq * (4 + d);
    for (int c = tid; c < d; c += kPT) {
      float sum = 0.f;
      for (int w = 0; w < kPT / 32; ++w) sum += ared[w * 256 + c];
      ap[4 + c] = sum;
    }
    if (tid == 0) {
      double l = 0.0;
      for (int w = 0; w < kPT / 32; ++w) l += red[w];
      ap[0] = na > 0 ? (float)M : -INFINITY;  // natural-log domain, like the attention partials
      ap[1] = (float)l;
    }
  }
  stamp(r, 4);
  cluster.sync();  // (C) all head states ready
  stamp(r, 5);

  // ---------------- phase 3: GQA-union work list --------------------------
  // every CTA copies all G state arrays (16-byte DSMEM loads), computes the
  // union prefix over all clusters itself and writes its own slice
  const int capP = (cap + 15) & ~15;
  {
    const int kq = (K + 15) / 16;
    for (int i = tid; i < G * kq; i += kPT) {
      const int gg = i / kq, c = i - gg * kq;
      *reinterpret_cast<int4*>(stall + (size_t)gg * capP + c * 16) =
          *reinterpret_cast<const int4*>(cluster.map_shared_rank(stS, gg) + c * 16);
    }
  }
  // done with remote smem: arrive now, wait at the very end
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  __syncthreads();
  const int full_mask = (1 << G) - 1;
  const int sw_rows = v.sink + v.window;
  const int per_t = (K + kPT - 1) / kPT;
  const int beg = min(K, tid * per_t), end = min(K, beg + per_t);
  int e_cnt = 0, a_cnt = 0, r_cnt = 0;
  for (int k = beg; k < end; ++k) {
    int me = 0, ma = 0;
    for (int gg = 0; gg < G; ++gg) {
      const uint8_t s = stall[(size_t)gg * capP + k];
      me |= (s == 2) << gg;
      ma |= (s == 1) << gg;
    }
    e_cnt += me != 0;
    a_cnt += ma != 0;
    if (me) r_cnt += offs[k + 1] - offs[k];
  }
  int tot_a, tot_r, tot_e;
  int off_a = block_exclusive_scan(a_cnt, redi, &tot_a);
  int off_r = block_exclusive_scan(r_cnt, redi, &tot_r) + sw_rows;
  (void)block_exclusive_scan(e_cnt, redi, &tot_e);
  unsigned* rowidx = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
  int2* apx = wl.approx + (size_t)bh * cap;
  // entries of my cluster slice [k0, k0 + nloc) only
  for (int k = beg; k < end; ++k) {
    int me = 0, ma = 0;
    for (int gg = 0; gg < G; ++gg) {
      const uint8_t s = stall[(size_t)gg * capP + k];
      me |= (s == 2) << gg;
      ma |= (s == 1) << gg;
    }
    const int len = me ? offs[k + 1] - offs[k] : 0;
    if (k >= k0 && k < k0 + nloc) {
      if (ma) apx[off_a] = make_int2(k, ma);
      if (me) {
        const unsigned tag = (unsigned)me << 24;
        const int o0 = offs[k];
        for (int t = 0; t < len; ++t) rowidx[off_r + t] = tag | (unsigned)(o0 + t);
      }
    }
    off_a += ma != 0;
    off_r += len;
  }
  if (r == 0) {
    const unsigned tag = (unsigned)full_mask << 24;
    for (int t = tid; t < v.sink; t += kPT) rowidx[t] = tag | (unsigned)t;
    for (int t = tid; t < v.window; t += kPT) rowidx[v.sink + t] = tag | (unsigned)(v.n_tokens - v.window + t);
    if (tid == 0) {
      const int all_r = tot_r + sw_rows;
      wl.nrows[bh] = all_r;
      wl.napprox[bh] = tot_a;
      wl.nruns[bh] = tot_e + (v.sink > 0) + (v.window > 0);
      wl.nchunks[bh] = (all_r + kChunkRows - 1) / kChunkRows;
      if (wl.stats) {
        wl.stats[4 * bh + 0] = all_r;
        wl.stats[4 * bh + 1] = tot_a;
        wl.stats[4 * bh + 2] = (all_r + kChunkRows - 1) / kChunkRows;
        wl.stats[4 * bh + 3] = tot_e;
      }
    }
  }
  stamp(r, 6);
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");  // (E) remote smem lifetime
  stamp(r, 7);
}

size_t plan_smem_bytes(int d, int cap) { return plan_layout(d, cap).total; }

bool plan_supported(const dp_cache_view& v, int G) {
  return v.cluster_cap <= kPlanMaxCap && G <= kCl && v.head_dim <= 128 && v.head_dim % 32 == 0 &&
         v.row_cap < (1 << 24) && plan_smem_bytes(v.head_dim, v.cluster_cap) <= 227 * 1024;
}

cudaError_t launch_plan(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, void* ws, cudaStream_t st) {
  WorkLists wl;
  decode_ws_layout(&v, G, &wl, nullptr, nullptr, reinterpret_cast<char*>(ws));
  wl.stats = stats;
  const size_t smem = plan_smem_bytes(v.head_dim, v.cluster_cap);
  const int grid = v.batch * v.kv_heads * kCl;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, kPT, smem, st>>>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl);
  };
  if (G <= 1) go(plan_kernel<1>);
  else if (G <= 2) go(plan_kernel<2>);
  else if (G <= 4) go(plan_kernel<4>);
  else go(plan_kernel<8>);
  return cudaGetLastError();
}

}  // namespace dp

extern "C" int dp_debug_plan_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_plan_ts, sizeof(dp::g_plan_ts)) == cudaSuccess ? 0 : 2;  // [8][16]
}
