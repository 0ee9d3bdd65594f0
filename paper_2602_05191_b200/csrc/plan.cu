// Fused per-layer "plan": size-weighted centroid scoring + two-stage top-p +
// GQA-union work list, one launch, one 8-CTA thread-block cluster per
// (sequence, kv head); stages hand data over through distributed shared
// memory instead of HBM round trips.
//
//   phase 1  score   (engine.py:158-177)  CTA r scores clusters [r*per, (r+1)*per)
//                    for every q head of the group: fp64 dot of fp32 centroids
//                    with the query, + log|c|.
//   phase 2  select  (engine.py:180-213, selection.py:36-65)  CTA g (g < G) owns
//                    q head g: gathers its K log-masses over DSMEM, softmax in
//                    fp64, then a mass histogram over 1/16-nat log bins finds the
//                    bin where the cumulative mass crosses p1 (and p2 of the
//                    retained mass); only those boundary bins are sorted (prob
//                    desc, cluster id asc == the stable argsort order) to place
//                    the exact cuts.  No full sort.
//   phase 3  worklist  every CTA turns its cluster slice into GQA-union rows:
//                    packed row entries (head mask << 24 | physical row) for
//                    sink, window and members of clusters exact for >= 1 head,
//                    and (cluster, mask) entries for approximated clusters.
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
constexpr int kPlanTile = 64;  // centroid rows staged per score tile
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
  size_t qd, lmS, full, bin, st, bins, cand, ctile, total;
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
  L.qd = take((size_t)kMaxGroup * d * 8);
  L.lmS = take((size_t)kMaxGroup * L.per * 8);
  L.full = take((size_t)cap * 8);
  L.bin = take((size_t)cap * 2);
  L.st = take((size_t)cap);
  L.bins = take((size_t)kBins * 20);
  L.cand = take((size_t)cap * 16);  // (prob f64, id i32, sorted slot i32)
  L.ctile = take((size_t)kPlanTile * (d + 4) * 4);
  L.total = o;
  return L;
}

// warp 0: first j in [0, n) with (base + sum_{t<=j} p[order[t]]) / denom >= pthr
// (n if never); *at receives the inclusive sum at the cut (or the full sum).
__device__ int warp_cut(const double* cp, const int* order, int n, double base, double denom, double pthr,
                        double* at) {
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
    const unsigned hit = __ballot_sync(0xffffffffu, j < n && cum / denom >= pthr);
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

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kPT)
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
  const int* offs = v.offs + (size_t)bh * (cap + 1);

  extern __shared__ __align__(16) unsigned char smem[];
  double* qd = reinterpret_cast<double*>(smem + L.qd);
  double* lmS = reinterpret_cast<double*>(smem + L.lmS);  // [kMaxGroup][per]
  double* full = reinterpret_cast<double*>(smem + L.full);
  uint16_t* bin16 = reinterpret_cast<uint16_t*>(smem + L.bin);
  uint8_t* stS = reinterpret_cast<uint8_t*>(smem + L.st);
  double* bmass = reinterpret_cast<double*>(smem + L.bins);
  double* bcum = bmass + kBins;
  int* bcnt = reinterpret_cast<int*>(bcum + kBins);
  double* cp_ = reinterpret_cast<double*>(smem + L.cand);  // candidate probs
  int* cid = reinterpret_cast<int*>(cp_ + cap);             // candidate ids
  int* cord = cid + cap;                                    // sorted order (slots)
  float* ctile = reinterpret_cast<float*>(smem + L.ctile);
  __shared__ double red[33];
  __shared__ int redi[33];
  __shared__ double s_lmax[kMaxGroup];
  __shared__ int s_b1, s_b2, s_nc, s_tot[3];

  stamp(r, 0);
  // ---------------- phase 1: score my slice for all G heads ---------------
  for (int i = tid; i < G * d; i += kPT) qd[i] = load_elem_d(q, qdt, (size_t)bh * G * d + i);
  {
    double lmax0 = -CUDART_INF, lmax1 = -CUDART_INF;
    const float4* C4 = reinterpret_cast<const float4*>(v.centroids + ((size_t)bh * cap + k0) * d);
    const int d4 = d >> 2, stride = d + 4;
    const int row = tid & (kPlanTile - 1), slot = tid >> 6;  // 64 rows x 4 head slots
    for (int t0 = 0; t0 < nloc; t0 += kPlanTile) {
      const int n = min(kPlanTile, nloc - t0);
      __syncthreads();
      for (int i = tid; i < n * d4; i += kPT) {
        const int rr = i / d4, c = i - rr * d4;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&ctile[rr * stride + 4 * c]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(&C4[(size_t)(t0 + rr) * d4 + c]));
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      if (row < n) {
        const int k = k0 + t0 + row;
        const double ls = log((double)(offs[k + 1] - offs[k]));
        const float* crow = &ctile[row * stride];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int g = slot + 4 * hh;
          if (g < G) {
            const double* qg = qd + g * d;
            double a0 = 0.0, a1 = 0.0;
            for (int j = 0; j < d; j += 4) {
              const float4 c4 = *reinterpret_cast<const float4*>(&crow[j]);
              a0 = fma((double)c4.x, qg[j], a0);
              a1 = fma((double)c4.y, qg[j + 1], a1);
              a0 = fma((double)c4.z, qg[j + 2], a0);
              a1 = fma((double)c4.w, qg[j + 3], a1);
            }
            const double val = (a0 + a1) * scale + ls;
            lmS[g * per + t0 + row] = val;
            if (hh == 0) lmax0 = fmax(lmax0, val); else lmax1 = fmax(lmax1, val);
            lm_out[((size_t)bh * G + g) * cap + k] = val;
          }
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const double m = warp_max(hh == 0 ? lmax0 : lmax1);
      __syncthreads();
      if (lane == 0) red[warp] = m;
      __syncthreads();
      if (tid < 4 && tid + 4 * hh < G) s_lmax[tid + 4 * hh] = fmax(red[2 * tid], red[2 * tid + 1]);
    }
  }
  stamp(r, 1);
  cluster.sync();  // (A) every slice scored
  stamp(r, 2);

  // ---------------- phase 2: two-stage top-p for q head g = r --------------
  const bool sel = r < G;
  double M = -CUDART_INF;
  if (sel) {
    for (int rr = 0; rr < kCl; ++rr) M = fmax(M, cluster.map_shared_rank(s_lmax, rr)[r]);
    for (int i = tid; i < K; i += kPT) {
      const int rr = i / per;
      full[i] = cluster.map_shared_rank(lmS, rr)[r * per + (i - rr * per)];
    }
  }
  cluster.sync();  // (B) gathers done (lmS no longer read remotely)
  stamp(r, 3);
  if (sel) {
    const int g = r;
    for (int b = tid; b < kBins; b += kPT) {
      bmass[b] = 0.0;
      bcnt[b] = 0;
    }
    double s = 0.0;
    for (int i = tid; i < K; i += kPT) s += exp(full[i] - M);
    const double S = block_sum(s, red);  // also orders the bin zeroing
    double t = 0.0;
    for (int i = tid; i < K; i += kPT) {
      const double lmv = full[i];
      const double p = exp(lmv - M) / S;  // softmax, engine.py:168
      int b = (int)((float)(M - lmv) * kBinScale);
      b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
      full[i] = p;
      bin16[i] = (uint16_t)b;
      atomicAdd(&bmass[b], p);
      atomicAdd(&bcnt[b], 1);
      t += p;
    }
    const double total = block_sum(t, red);  // probs.sum(), selection.py:52
    stamp(r, 8);
    {
      constexpr int bp = kBins / kPT;
      double loc = 0.0;
      for (int j = 0; j < bp; ++j) loc += bmass[tid * bp + j];
      double tot;
      double off = block_exclusive_scan(loc, red, &tot);
      for (int j = 0; j < bp; ++j) {
        bcum[tid * bp + j] = off;
        off += bmass[tid * bp + j];
      }
    }
    if (tid == 0) s_b1 = kBins;
    __syncthreads();
    for (int b0 = 0; b0 < kBins; b0 += kPT) {
      const int b = b0 + tid;
      const bool hit = bcnt[b] > 0 && (bcum[b] + bmass[b]) / total >= p1;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit && lane == __ffs(bal) - 1) atomicMin(&s_b1, b);
    }
    __syncthreads();
    const int b1 = s_b1;  // kBins: p1 never reached (rounding at p1 = 1) -> keep all
    stamp(r, 9);

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

    int n1c = 0, cut1 = 0;
    double sub = total;  // retained (stage-1) mass = probs[cp].sum(), engine.py:191
    if (b1 < kBins) {
      n1c = sort_bin(b1, 0);
      if (warp == 0) {
        double at;
        const int j = warp_cut(cp_, cord, n1c, bcum[b1], total, p1, &at);
        if (lane == 0) {
          s_nc = j < n1c ? j + 1 : n1c;  // cut inside the boundary bin
          red[0] = j < n1c ? at : bcum[b1] + bmass[b1];
        }
      }
      __syncthreads();
      cut1 = s_nc;
      sub = red[0];
    } else {
      double loc = 0.0;  // every bin retained
      if (tid == 0) red[0] = bcum[kBins - 1] + bmass[kBins - 1];
      __syncthreads();
      sub = red[0];
      (void)loc;
    }
    __syncthreads();
    stamp(r, 10);
    // stage 2 (engine.py:191-194): same descending order, denominator = sub
    if (tid == 0) s_b2 = b1;
    __syncthreads();
    for (int b0 = 0; b0 < kBins; b0 += kPT) {  // uniform trip count: full-warp ballots
      const int b = b0 + tid;
      const bool hit = b < b1 && bcnt[b] > 0 && (bcum[b] + bmass[b]) / sub >= p2;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit && lane == __ffs(bal) - 1) atomicMin(&s_b2, b);
    }
    __syncthreads();
    const int b2 = s_b2;
    int cut2 = 0, n2c = 0, base2 = 0;
    if (b2 < b1) {
      base2 = n1c;
      n2c = sort_bin(b2, base2);
      if (warp == 0) {
        double at;
        const int j = warp_cut(cp_, cord + base2, n2c, bcum[b2], sub, p2, &at);
        if (lane == 0) s_nc = j < n2c ? j + 1 : n2c;
      }
      __syncthreads();
      cut2 = s_nc;
    } else if (b1 < kBins) {
      if (warp == 0) {
        double at;
        const int j = warp_cut(cp_, cord, cut1, bcum[b1], sub, p2, &at);
        if (lane == 0) s_nc = j < cut1 ? j + 1 : cut1;
      }
      __syncthreads();
      cut2 = s_nc;
    }
    __syncthreads();
    stamp(r, 11);
    // states: 2 exact, 1 approx, 0 dropped
    for (int i = tid; i < K; i += kPT) {
      const int b = bin16[i];
      stS[i] = (uint8_t)(b < b2 ? 2 : (b < b1 ? 1 : 0));
    }
    __syncthreads();
    if (b1 < kBins) {
      for (int j = tid; j < n1c; j += kPT) {
        const int id = cid[cord[j]];
        stS[id] = (uint8_t)(j < cut1 ? (b2 == b1 && j < cut2 ? 2 : 1) : 0);
      }
    }
    if (b2 < b1) {
      for (int j = tid; j < n2c; j += kPT) stS[cid[cord[base2 + j]]] = (uint8_t)(j < cut2 ? 2 : 1);
    }
    // counts: elements of bins strictly above the boundary + the cuts
    int c1 = 0, c2 = 0;
    for (int b = tid; b < kBins; b += kPT) {
      if (b < b1) c1 += bcnt[b];
      if (b < b2) c2 += bcnt[b];
    }
    c1 = block_sum(c1, redi);
    c2 = block_sum(c2, redi);
    if (tid == 0) {
      const int hq = bh * G + g;
      counts[2 * hq] = b1 < kBins ? c1 + cut1 : K;
      counts[2 * hq + 1] = c2 + cut2;
    }
    __syncthreads();
    if (state_out)
      for (int i = tid; i < K; i += kPT) state_out[((size_t)bh * G + g) * cap + i] = stS[i];
  }
  stamp(r, 4);
  cluster.sync();  // (C) all head states ready
  stamp(r, 5);

  // ---------------- phase 3: GQA-union work list for my slice ------------
  const int full_mask = (1 << G) - 1;
  const int sw_rows = v.sink + v.window;
  int me_l[2] = {0, 0}, ma_l[2] = {0, 0}, len_l[2] = {0, 0};
  int e_loc = 0, a_loc = 0, r_loc = 0;
#pragma unroll
  for (int u = 0; u < 2; ++u) {  // per <= 512 -> 2 clusters per thread
    const int li = tid * 2 + u;
    if (li < nloc) {
      const int k = k0 + li;
      int me = 0, ma = 0;
      for (int gg = 0; gg < G; ++gg) {
        const uint8_t s = cluster.map_shared_rank(stS, gg)[k];
        me |= (s == 2) << gg;
        ma |= (s == 1) << gg;
      }
      me_l[u] = me;
      ma_l[u] = ma;
      len_l[u] = me ? offs[k + 1] - offs[k] : 0;
      e_loc += me != 0;
      a_loc += ma != 0;
      r_loc += len_l[u];
    }
  }
  int tot_e, tot_a, tot_r;
  const int pe = block_exclusive_scan(e_loc, redi, &tot_e);
  const int pa = block_exclusive_scan(a_loc, redi, &tot_a);
  const int pr = block_exclusive_scan(r_loc, redi, &tot_r);
  if (tid == 0) {
    s_tot[0] = tot_e;
    s_tot[1] = tot_a;
    s_tot[2] = tot_r;
  }
  stamp(r, 12);
  cluster.sync();  // (D) slice totals visible
  stamp(r, 13);
  int off_e = 0, off_a = 0, off_r = sw_rows, all_e = 0, all_a = 0, all_r = sw_rows;
  for (int rr = 0; rr < kCl; ++rr) {
    const int* t3 = cluster.map_shared_rank(s_tot, rr);
    if (rr < r) {
      off_e += t3[0];
      off_a += t3[1];
      off_r += t3[2];
    }
    all_e += t3[0];
    all_a += t3[1];
    all_r += t3[2];
  }
  unsigned* rowidx = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
  int2* apx = wl.approx + (size_t)bh * cap;
  {
    int ea = off_a + pa, er = off_r + pr;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid * 2 + u;
      if (li < nloc) {
        const int k = k0 + li;
        if (ma_l[u]) apx[ea++] = make_int2(k, ma_l[u]);
        if (me_l[u]) {
          const unsigned tag = (unsigned)me_l[u] << 24;
          const int o0 = offs[k];
          for (int t = 0; t < len_l[u]; ++t) rowidx[er + t] = tag | (unsigned)(o0 + t);
          er += len_l[u];
        }
      }
    }
  }
  (void)pe;
  if (r == 0) {
    const unsigned tag = (unsigned)full_mask << 24;
    for (int t = tid; t < v.sink; t += kPT) rowidx[t] = tag | (unsigned)t;
    for (int t = tid; t < v.window; t += kPT) rowidx[v.sink + t] = tag | (unsigned)(v.n_tokens - v.window + t);
  }
  if (r == kCl - 1 && tid == 0) {
    wl.nrows[bh] = all_r;
    wl.napprox[bh] = all_a;
    wl.nruns[bh] = all_e + (v.sink > 0) + (v.window > 0);
    wl.nchunks[bh] = (all_r + kChunkRows - 1) / kChunkRows;
    publish_chunk_prefix(wl, v.batch * v.kv_heads);
    if (wl.stats) {
      wl.stats[4 * bh + 0] = all_r;
      wl.stats[4 * bh + 1] = all_a;
      wl.stats[4 * bh + 2] = (all_r + kChunkRows - 1) / kChunkRows;
      wl.stats[4 * bh + 3] = all_e;
    }
  }
  stamp(r, 6);
  cluster.sync();  // (E) keep smem alive until every remote read is done
  stamp(r, 7);
}

}  // namespace dp

extern "C" int dp_debug_plan_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_plan_ts, sizeof(dp::g_plan_ts)) == cudaSuccess ? 0 : 2;  // [8][16]
}

namespace dp {

size_t plan_smem_bytes(int d, int cap) { return plan_layout(d, cap).total; }

bool plan_supported(const dp_cache_view& v, int G) {
  return v.cluster_cap <= kPlanMaxCap && G <= kCl && v.head_dim <= 256 && v.row_cap < (1 << 24) &&
         plan_smem_bytes(v.head_dim, v.cluster_cap) <= 227 * 1024;
}

cudaError_t launch_plan(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, void* ws, cudaStream_t st) {
  WorkLists wl;
  decode_ws_layout(&v, G, &wl, nullptr, nullptr, reinterpret_cast<char*>(ws));
  wl.stats = stats;
  const size_t smem = plan_smem_bytes(v.head_dim, v.cluster_cap);
  static size_t attr = 0;
  if (attr < smem) {
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  plan_kernel<<<v.batch * v.kv_heads * kCl, kPT, smem, st>>>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl);
  return cudaGetLastError();
}

}  // namespace dp
