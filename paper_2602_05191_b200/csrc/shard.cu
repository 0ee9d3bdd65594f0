// Sequence-sharded Double-P with the reference's GLOBAL semantics (SURVEY.md
// section 8e, config 5): the per-rank device pieces.  The host layer
// (paper_2602_05191_b200/seqshard.py) strings them together with
// torch.distributed collectives (NCCL over NVLink; gloo in the tests).
//
//   * global k-means++ (clustering.py:36-55) over position-sharded points:
//     kmpp_dsq_kernel folds the newest centre into every local point's
//     squared distance and reduces the local sum; after an all-gather of the
//     P local sums, kmpp_pick_kernel finds whether this rank owns the point
//     where the GLOBAL running sum first exceeds u * total (the reference's
//     Generator.choice(p = dsq / total) in unnormalised form, the same rule
//     as the single-GPU seeding kernel) and writes that row; an all-reduce
//     of the (owner row, zeros elsewhere) buffer hands the centre to all.
//   * global Lloyd (clustering.py:58-107): nearest-centroid assignment of
//     the local points (dp_nearest_centroid), then lloyd_sums_kernel -- fp64
//     per-cluster sums of the local members in ascending position order
//     (deterministic) -- whose [K, d + 1] results are all-reduced.
//   * global two-stage top-p (engine.py:180-213) over the all-gathered
//     per-shard log-mass slices: select_global_kernel, one CTA per q head,
//     any cluster count (the 1M-token config has K = 32,766): the same
//     histogram / boundary-candidate algorithm as the fused plan's select
//     (select.cuh), with per-element data recomputed from the log-masses or
//     kept in global scratch instead of registers.
//   * lse_merge_kernel: the exchange step's log-sum-exp merge of the P
//     partial (out, lse) (engine.py:234-246 across shards).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "common.cuh"
#include "decode_internal.h"
#include "host_state.h"
#include "select.cuh"
#include "dsmem.cuh"

namespace cg = cooperative_groups;

namespace dp {

// ---------------------------------------------------------------------------
// global k-means++
// ---------------------------------------------------------------------------
constexpr int kKT = 256;

// dsq[u, i] = |x_i - c_u|^2 (first) or min(dsq, |x_i - c_u|^2); sums[u] =
// sum_i dsq[u, i] in a fixed association order (thread segments, then a
// fixed tree), fp64 throughout (clustering.py:45,53)
__global__ void __launch_bounds__(kKT) kmpp_dsq_kernel(const void* __restrict__ pts, int dtype, int n, int d,
                                                      const double* __restrict__ centre, int first,
                                                      double* __restrict__ dsq, double* __restrict__ sums) {
  const int u = blockIdx.x, tid = threadIdx.x;
  extern __shared__ double s_c[];  // [d] the centre
  __shared__ double s_red[kKT];
  for (int j = tid; j < d; j += kKT) s_c[j] = centre[(size_t)u * d + j];
  __syncthreads();
  const int per = (n + kKT - 1) / kKT, i0 = min(n, tid * per), i1 = min(n, i0 + per);
  double acc = 0.0;
  for (int i = i0; i < i1; ++i) {
    const size_t base = ((size_t)u * n + i) * d;
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      const double x = load_elem_d(pts, dtype, base + j) - s_c[j];
      s += x * x;
    }
    double* p = dsq + (size_t)u * n + i;
    const double v = first ? s : fmin(*p, s);
    *p = v;
    acc += v;
  }
  s_red[tid] = acc;
  __syncthreads();
  for (int w = kKT / 2; w > 0; w >>= 1) {
    if (tid < w) s_red[tid] += s_red[tid + w];
    __syncthreads();
  }
  if (tid == 0) sums[u] = s_red[0];
}

// Centre pick of one step.  all_sums [P, U] (rank order); u_draw [U]; an
// explicit global index (pick_in[u] >= 0: the first centre, or an
// rng.integers draw once the mass is zero) takes precedence.  This rank owns
// global middle indices [gbase, gbase + n).  Writes centre_out[u] (the row
// in fp64 on the owner, zeros elsewhere) and pick_out[u] (global index on
// the owner, -1 elsewhere).  One CTA per unit.
__global__ void __launch_bounds__(kKT) kmpp_pick_kernel(const void* __restrict__ pts, int dtype, int n, int d,
                                                       const double* __restrict__ dsq,
                                                       const double* __restrict__ all_sums, int P, int rank,
                                                       const double* __restrict__ u_draw,
                                                       const int* __restrict__ pick_in, long long gbase,
                                                       double* __restrict__ centre_out, int* __restrict__ pick_out) {
  const int u = blockIdx.x, U = gridDim.x, tid = threadIdx.x;
  __shared__ double s_part[kKT];
  __shared__ int s_pick;
  if (tid == 0) s_pick = -1;
  long long gpick = pick_in ? pick_in[u] : -1;
  double target = 0.0, before = 0.0, total = 0.0;
  if (gpick < 0) {
    for (int r = 0; r < P; ++r) {
      const double s = all_sums[(size_t)r * U + u];
      if (r < rank) before += s;
      total += s;
    }
    if (!(total > 0.0)) gpick = -2;  // degenerate: the host replays rng.integers (pick_in)
    target = u_draw[u] * total;
  }
  const bool mine_explicit = gpick >= gbase && gpick < gbase + n;
  const double mysum = gpick == -1 ? all_sums[(size_t)rank * U + u] : 0.0;
  const bool owner = gpick >= 0 ? mine_explicit
                                : (gpick == -1 && before <= target && target < before + mysum);
  __syncthreads();
  if (owner) {
    if (gpick >= 0) {
      if (tid == 0) s_pick = (int)(gpick - gbase);
    } else {
      // first local index whose running sum exceeds target - before: thread
      // segments, their sums scanned in a fixed order
      const double t = target - before;
      const int per = (n + kKT - 1) / kKT, i0 = min(n, tid * per), i1 = min(n, i0 + per);
      double acc = 0.0;
      for (int i = i0; i < i1; ++i) acc += dsq[(size_t)u * n + i];
      s_part[tid] = acc;
      __syncthreads();
      if (tid == 0) {
        double run = 0.0;
        int seg = kKT - 1;
        for (int s = 0; s < kKT; ++s) {
          if (run + s_part[s] > t) {
            seg = s;
            break;
          }
          run += s_part[s];
        }
        const int j0 = min(n, seg * per), j1 = min(n, j0 + per);
        int pick = j1 > j0 ? j1 - 1 : n - 1;
        for (int i = j0; i < j1; ++i) {
          run += dsq[(size_t)u * n + i];
          if (run > t) {
            pick = i;
            break;
          }
        }
        s_pick = pick;
      }
    }
  }
  __syncthreads();
  const int lp = s_pick;
  for (int j = tid; j < d; j += kKT)
    centre_out[(size_t)u * d + j] = lp >= 0 ? load_elem_d(pts, dtype, ((size_t)u * n + lp) * d + j) : 0.0;
  if (tid == 0) pick_out[u] = lp >= 0 ? (int)(gbase + lp) : (gpick == -2 ? -2 : -1);
}

// ---------------------------------------------------------------------------
// global Lloyd: local per-cluster sums in ascending position order
// ---------------------------------------------------------------------------
// One CTA per unit: counting sort of the local points by cluster (stable:
// ascending local index), then warp w sums clusters w, w + 8, ... member by
// member (lane j covers dims j, j + 32, ...).  sums [U, k, d] fp64, counts
// [U, k] int64 (a point with assign < 0 is skipped).  Scratch: cnt/cur [U, k]
// int, order [U, n] int.
constexpr int kLT = 256;
__global__ void __launch_bounds__(kLT) lloyd_sums_kernel(const void* __restrict__ pts, int dtype, int n, int d,
                                                        const int* __restrict__ assign, int k,
                                                        double* __restrict__ sums, long long* __restrict__ counts,
                                                        int* __restrict__ cnt, int* __restrict__ order) {
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int* a = assign + (size_t)u * n;
  int* c = cnt + (size_t)u * k;
  int* o = order + (size_t)u * n;
  for (int j = tid; j < k; j += kLT) c[j] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += kLT)
    if (a[i] >= 0 && a[i] < k) atomicAdd(&c[a[i]], 1);
  __syncthreads();
  if (tid == 0) {  // exclusive offsets (serial: prefill-only, k is small per unit)
    int run = 0;
    for (int j = 0; j < k; ++j) {
      const int x = c[j];
      c[j] = run;
      run += x;
    }
  }
  __syncthreads();
  if (tid == 0)  // stable placement (ascending index inside each cluster)
    for (int i = 0; i < n; ++i)
      if (a[i] >= 0 && a[i] < k) o[c[a[i]]++] = i;
  __syncthreads();
  for (int j = warp; j < k; j += kLT / 32) {
    const int e = c[j], s = j == 0 ? 0 : c[j - 1];  // c now holds inclusive ends
    for (int dd = lane; dd < d; dd += 32) {
      double acc = 0.0;
      for (int m = s; m < e; ++m) acc += load_elem_d(pts, dtype, ((size_t)u * n + o[m]) * d + dd);
      sums[((size_t)u * k + j) * d + dd] = acc;
    }
    if (lane == 0) counts[(size_t)u * k + j] = e - s;
  }
}

// ---------------------------------------------------------------------------
// global two-stage top-p over a log-mass row of any length
// ---------------------------------------------------------------------------
constexpr int kGT = 1024;
constexpr int kGB = 2048;
constexpr int kGU = 8;        // element loads in flight per thread
constexpr int kGCand = 4096;  // candidates staged in shared memory (more: the global-scratch path)
constexpr size_t kGDyn = (size_t)kGCand * (8 + 8 + 8 + 4 + 4);

__device__ __forceinline__ double gsel_sanitise(double x) { return x != x ? -CUDART_INF : fmin(x, 1.7976931348623157e308); }

// u = exp(lm - M) as a 2^-38 fixed-point integer and its 1/32-nat bin
__device__ __forceinline__ void gsel_elem(double M, double lm, unsigned long long& u, int& b) {
  const float xf = M == -CUDART_INF ? CUDART_INF_F : (float)(M - lm);
  u = __float2ull_rn(__expf(-xf) * (float)kFixF);
  b = (int)(xf * kBinScale);
  b = b < 0 ? 0 : (b >= kGB ? kGB - 1 : b);
}

// rows: one per (sequence, q head); K[row] clusters at lm + row * ld.
// Scratch per row (ld entries each): pos int, ex u64, cand int.
__global__ void __launch_bounds__(kGT, 1) select_global_kernel(const double* __restrict__ lm_all, int ld,
                                                              const int* __restrict__ Ks, double p1, double p2,
                                                              uint8_t* __restrict__ state_all,
                                                              int* __restrict__ counts, int* __restrict__ pos_ws,
                                                              unsigned long long* __restrict__ ex_ws,
                                                              int* __restrict__ cand_ws,
                                                              unsigned long long* __restrict__ pk_ws) {
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = Ks[row];
  const double* lm = lm_all + (size_t)row * ld;
  uint8_t* state = state_all + (size_t)row * ld;
  int* pos = pos_ws + (size_t)row * ld;
  unsigned long long* ex = ex_ws + (size_t)row * ld;
  int* cand = cand_ws + (size_t)row * ld;
  // (u, bin) of every element, packed once in pass (1) and re-read by the
  // later passes instead of recomputing exp / conversions: u << 11 | bin
  unsigned long long* pk = pk_ws + (size_t)row * ld;
  __shared__ unsigned long long s_hm[kGB];  // exact u64 bin masses (u32 halves overflow on flat rows)
  __shared__ int s_hc[kGB + 1];
  unsigned* s_cur = reinterpret_cast<unsigned*>(s_hm);  // after the bin scan: per-bin cursors of the candidate placement
  __shared__ unsigned long long s_pm[kGB];
  __shared__ unsigned long long s_wm[33];
  __shared__ int s_wc[33];
  __shared__ double s_red[32];
  __shared__ unsigned long long s_before1, s_mass1, s_at1;
  __shared__ int s_b1, s_n1, s_n2, s_blo, s_bhi;
  extern __shared__ __align__(16) unsigned char g_dyn[];  // staged candidates
  unsigned long long* s_cu = reinterpret_cast<unsigned long long*>(g_dyn);
  unsigned long long* s_cex = s_cu + kGCand;
  double* s_clm = reinterpret_cast<double*>(s_cex + kGCand);
  int* s_cid = reinterpret_cast<int*>(s_clm + kGCand);
  int* s_cpos = s_cid + kGCand;
  for (int j = tid; j < kGB; j += kGT) {
    s_hm[j] = 0ull;
    s_hc[j] = 0;
  }
  if (tid == 0) {
    s_b1 = kGB;
    s_n1 = 0;
    s_n2 = 0;
    s_at1 = 0ull;
  }
  // (0) the row's maximum
  // every element loop below issues kGU loads before using any of them
  // (one load per iteration would serialise L2 round trips: 32 per thread)
  double m = -CUDART_INF;
  for (int i0 = tid; i0 < K; i0 += kGT * kGU) {
    double x[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) x[j] = i0 + j * kGT < K ? lm[i0 + j * kGT] : -CUDART_INF;
#pragma unroll
    for (int j = 0; j < kGU; ++j) m = fmax(m, gsel_sanitise(x[j]));
  }
  m = warp_max(m);
  if (lane == 0) s_red[warp] = m;
  __syncthreads();
  double M = -CUDART_INF;
#pragma unroll
  for (int w = 0; w < kGT / 32; ++w) M = fmax(M, s_red[w]);
  // (1) histogram
  for (int i0 = tid; i0 < K; i0 += kGT * kGU) {
    double x[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) x[j] = i0 + j * kGT < K ? lm[i0 + j * kGT] : -CUDART_INF;
#pragma unroll
    for (int j = 0; j < kGU; ++j) {
      const int i = i0 + j * kGT;
      if (i >= K) break;
      unsigned long long u;
      int b;
      gsel_elem(M, gsel_sanitise(x[j]), u, b);
      pk[i] = (u << 11) | (unsigned long long)b;
      if (u) {
        atomicAdd(&s_hm[b], u);
        atomicAdd(&s_hc[b], 1);
      }
    }
  }
  __syncthreads();
  // (2) exclusive bin prefixes (2 bins per thread), total, stage-1 bin
  constexpr int kBPT = kGB / kGT;
  unsigned long long bm[kBPT], mloc = 0ull;
  int bc[kBPT], cloc = 0;
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    const int b = tid * kBPT + j;
    bm[j] = s_hm[b];
    bc[j] = s_hc[b];
    mloc += bm[j];
    cloc += bc[j];
  }
  unsigned long long mi = mloc;
  int ci = cloc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long tm = __shfl_up_sync(0xffffffffu, mi, o);
    const int tc = __shfl_up_sync(0xffffffffu, ci, o);
    if (lane >= o) {
      mi += tm;
      ci += tc;
    }
  }
  if (lane == 31) {
    s_wm[warp] = mi;
    s_wc[warp] = ci;
  }
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = s_wm[lane];
    const int wc = s_wc[lane];
    unsigned long long wi = w;
    int wci = wc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long tm = __shfl_up_sync(0xffffffffu, wi, o);
      const int tc = __shfl_up_sync(0xffffffffu, wci, o);
      if (lane >= o) {
        wi += tm;
        wci += tc;
      }
    }
    s_wm[lane] = wi - w;
    s_wc[lane] = wci - wc;
    if (lane == 31) {
      s_wm[32] = wi;
      s_wc[32] = wci;
    }
  }
  __syncthreads();
  const unsigned long long T = s_wm[32];
  unsigned long long mex = s_wm[warp] + mi - mloc;
  int cex = s_wc[warp] + ci - cloc;
  const double thr1 = p1 * (double)T;
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    const int b = tid * kBPT + j;
    const unsigned long long inc = mex + bm[j];
    if (bm[j] && (double)mex < thr1 && thr1 <= (double)inc) {
      s_b1 = b;
      s_before1 = mex;
      s_mass1 = bm[j];
    }
    s_pm[b] = mex;
    s_hc[b] = cex;  // -> exclusive count prefix
    s_cur[b] = 0u;
    mex = inc;
    cex += bc[j];
  }
  if (tid == kGT - 1) s_hc[kGB] = s_wc[32];
  __syncthreads();
  const int b1 = s_b1;
  if (T == 0ull || b1 >= kGB) {  // no mass (a non-finite query)
    const uint8_t st = p1 >= 1.0 ? (p2 >= 1.0 ? 2 : 1) : 0;
    for (int i = tid; i < K; i += kGT) state[i] = st;
    if (tid == 0) {
      counts[2 * row] = p1 >= 1.0 ? K : 0;
      counts[2 * row + 1] = p1 >= 1.0 && p2 >= 1.0 ? K : 0;
    }
    return;
  }
  // integer thresholds (a u64 -> fp64 conversion per element costs more than the test)
  const unsigned long long Tlo = ceil_u64(p2 * (double)s_before1), Thi = ceil_u64(p2 * (double)(s_before1 + s_mass1));
  auto is_cand = [&](int b) {
    const unsigned long long inc = b + 1 < kGB ? s_pm[b + 1] : T;
    return b == b1 || (b < b1 && inc >= Tlo && s_pm[b] < Thi);
  };
  // (3) candidates -> their bin segments of the global sorted order; the
  //     candidate bins are [blo, bhi] and b1, i.e. two contiguous slot ranges
  if (tid == 0) {
    s_blo = kGB;
    s_bhi = -1;
  }
  __syncthreads();
  for (int i0 = tid; i0 < K; i0 += kGT * kGU) {
    unsigned long long wv[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) wv[j] = i0 + j * kGT < K ? pk[i0 + j * kGT] : 0ull;
#pragma unroll
    for (int j = 0; j < kGU; ++j) {
      const int i = i0 + j * kGT;
      const unsigned long long u = wv[j] >> 11;
      const int b = (int)(wv[j] & 2047u);
      if (u && b <= b1 && is_cand(b)) {
        cand[s_hc[b] + (int)atomicAdd(&s_cur[b], 1u)] = i;
        if (b < b1) {
          atomicMin(&s_blo, b);
          atomicMax(&s_bhi, b);
        }
      }
    }
  }
  __syncthreads();
  // stage the candidates in shared memory (id, log-mass, mass): slots of
  // [blo, bhi] then those of b1
  const int r1a = s_bhi >= 0 ? s_hc[s_blo] : 0, r1b = s_bhi >= 0 ? s_hc[s_bhi + 1] : 0;
  const int r2a = s_hc[b1], r2b = s_hc[b1 + 1];
  const int n1c = r1b - r1a, nc = n1c + (r2b - r2a);
  const bool staged = nc <= kGCand;
  auto sidx = [&](int slot) { return slot >= r2a ? n1c + (slot - r2a) : slot - r1a; };
  if (staged) {
    for (int t = tid; t < nc; t += kGT) {
      const int slot = t < n1c ? r1a + t : r2a + (t - n1c);
      const int i = cand[slot];
      s_cid[t] = i;
      s_clm[t] = gsel_sanitise(lm[i]);
      s_cu[t] = pk[i] >> 11;
    }
  }
  __syncthreads();
  // (4) rank inside the bin (log-mass desc, id asc) -> sorted position and
  //     exclusive cumulative mass; the stage-1 crossing element
  if (staged) {
    for (int t = tid; t < nc; t += kGT) {
      const int i = s_cid[t];
      const double la = s_clm[t];
      const unsigned long long u = s_cu[t];
      const int b = (int)(pk[i] & 2047u);
      const int j0 = s_hc[b], j1 = s_hc[b + 1], k0 = sidx(j0);
      int rk = 0;
      unsigned long long pre = 0ull;
      for (int j = 0; j < j1 - j0; ++j) {
        const double lj = s_clm[k0 + j];
        const int ij = s_cid[k0 + j];
        const bool ahead = lj > la || (lj == la && ij < i);
        rk += ahead;
        pre += ahead ? s_cu[k0 + j] : 0ull;
      }
      const int ps = j0 + rk;
      const unsigned long long e0 = s_pm[b] + pre;
      s_cpos[t] = ps;
      s_cex[t] = e0;
      if ((double)e0 < thr1 && thr1 <= (double)(e0 + u)) {
        s_n1 = ps + 1;
        s_at1 = e0 + u;
      }
    }
  } else {  // many candidates (very flat scores): the same from global scratch
    for (int i = tid; i < K; i += kGT) {
      unsigned long long u;
      int b;
      const double la = gsel_sanitise(lm[i]);
      gsel_elem(M, la, u, b);
      if (!(u && b <= b1 && is_cand(b))) continue;
      const int j0 = s_hc[b], j1 = s_hc[b + 1];
      int rk = 0;
      unsigned long long pre = 0ull;
      for (int j = j0; j < j1; ++j) {
        const int ij = cand[j];
        const double lj = gsel_sanitise(lm[ij]);
        const bool ahead = lj > la || (lj == la && ij < i);
        if (ahead) {
          unsigned long long uj;
          int bj;
          gsel_elem(M, lj, uj, bj);
          ++rk;
          pre += uj;
        }
      }
      pos[i] = j0 + rk;
      ex[i] = s_pm[b] + pre;
      const unsigned long long inc = ex[i] + u;
      if ((double)ex[i] < thr1 && thr1 <= (double)inc) {
        s_n1 = j0 + rk + 1;
        s_at1 = inc;
      }
    }
  }
  __syncthreads();
  // (5) stage-2 crossing
  const int n1 = p1 >= 1.0 ? K : s_n1;
  const double thr2 = p2 * (double)s_at1;
  if (staged) {
    for (int t = tid; t < nc; t += kGT)
      if ((double)s_cex[t] < thr2 && thr2 <= (double)(s_cex[t] + s_cu[t])) s_n2 = s_cpos[t] + 1;
  } else {
    for (int i = tid; i < K; i += kGT) {
      unsigned long long u;
      int b;
      gsel_elem(M, gsel_sanitise(lm[i]), u, b);
      if (u && b <= b1 && is_cand(b) && (double)ex[i] < thr2 && thr2 <= (double)(ex[i] + u)) s_n2 = pos[i] + 1;
    }
  }
  __syncthreads();
  const int n2 = p1 >= 1.0 && p2 >= 1.0 ? K : s_n2;
  // (6) states: candidates by position, the rest by bin
  const uint8_t zst = p1 >= 1.0 ? (p2 >= 1.0 ? 2 : 1) : 0;
  for (int i0 = tid; i0 < K; i0 += kGT * kGU) {
    unsigned long long wv[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) wv[j] = i0 + j * kGT < K ? pk[i0 + j * kGT] : 0ull;
#pragma unroll
    for (int j = 0; j < kGU; ++j) {
      const int i = i0 + j * kGT;
      if (i >= K) break;
      const unsigned long long u = wv[j] >> 11;
      const int b = (int)(wv[j] & 2047u);
      uint8_t st;
      if (!u) {
        st = zst;
      } else if (b <= b1 && is_cand(b)) {
        if (staged) continue;  // written from the staged copy below
        st = pos[i] < n2 ? 2 : (pos[i] < n1 ? 1 : 0);
      } else if (b > b1) {
        st = 0;
      } else {
        const unsigned long long inc = b + 1 < kGB ? s_pm[b + 1] : T;
        st = inc < Tlo ? 2 : 1;
      }
      state[i] = st;
    }
  }
  if (staged)
    for (int t = tid; t < nc; t += kGT) state[s_cid[t]] = s_cpos[t] < n2 ? 2 : (s_cpos[t] < n1 ? 1 : 0);
  if (tid == 0) {
    counts[2 * row] = n1;
    counts[2 * row + 1] = n2;
  }
}

// ---------------------------------------------------------------------------
// The same selection split over many CTAs per row (large K: the single-CTA
// kernel is instruction-bound on ONE SM per q head, ~45 us at K = 32,766).
// Five launches: max -> histogram -> bin scan -> candidates/states ->
// candidate ranking; per-row state lives in global scratch (GSelRow).
// ---------------------------------------------------------------------------
struct GSelRow {
  unsigned long long mkey;  // ordered-int max of the row (atomicMax); 0 = unset
  unsigned long long T, before1, mass1, Tlo, Thi;
  int b1, blo, bhi, pad;
};
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dfromkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}
constexpr int kST2 = 256;  // threads of the split kernels

__global__ void __launch_bounds__(kST2) gs_max_kernel(const double* __restrict__ lm, int ld, const int* __restrict__ Ks,
                                                     GSelRow* __restrict__ rd, unsigned long long* __restrict__ hm,
                                                     int* __restrict__ hc, int* __restrict__ cur) {
  const int row = blockIdx.y, S = gridDim.x, sp = blockIdx.x, tid = threadIdx.x;
  const int K = Ks[row];
  // zero my share of the row's histogram, counts and cursors
  for (int b = sp * (kGB / S) + tid; b < (sp + 1) * (kGB / S); b += kST2) {
    hm[(size_t)row * kGB + b] = 0ull;
    hc[(size_t)row * (kGB + 1) + b] = 0;
    cur[(size_t)row * kGB + b] = 0;
  }
  const int i0 = (int)((long long)K * sp / S), i1 = (int)((long long)K * (sp + 1) / S);
  double m = -CUDART_INF;
  for (int i = i0 + tid; i < i1; i += kST2 * kGU) {
    double x[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) x[j] = i + j * kST2 < i1 ? lm[(size_t)row * ld + i + j * kST2] : -CUDART_INF;
#pragma unroll
    for (int j = 0; j < kGU; ++j) m = fmax(m, gsel_sanitise(x[j]));
  }
  m = warp_max(m);
  if ((tid & 31) == 0) atomicMax(&rd[row].mkey, dkey(m));
}

__global__ void __launch_bounds__(kST2) gs_hist_kernel(const double* __restrict__ lm, int ld, const int* __restrict__ Ks,
                                                      const GSelRow* __restrict__ rd,
                                                      unsigned long long* __restrict__ hm, int* __restrict__ hc,
                                                      unsigned long long* __restrict__ pk_ws) {
  const int row = blockIdx.y, S = gridDim.x, sp = blockIdx.x, tid = threadIdx.x;
  const int K = Ks[row];
  __shared__ unsigned long long s_h[kGB];
  __shared__ int s_c[kGB];
  for (int b = tid; b < kGB; b += kST2) {
    s_h[b] = 0ull;
    s_c[b] = 0;
  }
  __syncthreads();
  const double M = dfromkey(rd[row].mkey);
  unsigned long long* pk = pk_ws + (size_t)row * ld;
  const int i0 = (int)((long long)K * sp / S), i1 = (int)((long long)K * (sp + 1) / S);
  for (int i = i0 + tid; i < i1; i += kST2 * kGU) {
    double x[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) x[j] = i + j * kST2 < i1 ? lm[(size_t)row * ld + i + j * kST2] : -CUDART_INF;
#pragma unroll
    for (int j = 0; j < kGU; ++j) {
      const int ii = i + j * kST2;
      if (ii >= i1) break;
      unsigned long long u;
      int b;
      gsel_elem(M, gsel_sanitise(x[j]), u, b);
      pk[ii] = (u << 11) | (unsigned long long)b;
      if (u) {
        atomicAdd(&s_h[b], u);
        atomicAdd(&s_c[b], 1);
      }
    }
  }
  __syncthreads();
  for (int b = tid; b < kGB; b += kST2)
    if (s_c[b]) {
      atomicAdd(&hm[(size_t)row * kGB + b], s_h[b]);
      atomicAdd(&hc[(size_t)row * (kGB + 1) + b], s_c[b]);
    }
}

// one CTA (1024 threads) per row: exclusive bin prefixes (in place: hm -> pm,
// hc -> pc), total, the stage-1 bin and the stage-2 candidate range
__global__ void __launch_bounds__(kGT) gs_scan_kernel(const int* __restrict__ Ks, double p1, double p2,
                                                     GSelRow* __restrict__ rd, unsigned long long* __restrict__ hm,
                                                     int* __restrict__ hc) {
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kBPT = kGB / kGT;
  __shared__ unsigned long long s_wm[33];
  __shared__ int s_wc[33];
  unsigned long long* pm = hm + (size_t)row * kGB;
  int* pc = hc + (size_t)row * (kGB + 1);
  unsigned long long bm[kBPT], mloc = 0ull;
  int bc[kBPT], cloc = 0;
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    bm[j] = pm[tid * kBPT + j];
    bc[j] = pc[tid * kBPT + j];
    mloc += bm[j];
    cloc += bc[j];
  }
  unsigned long long mi = mloc;
  int ci = cloc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long tm = __shfl_up_sync(0xffffffffu, mi, o);
    const int tc = __shfl_up_sync(0xffffffffu, ci, o);
    if (lane >= o) {
      mi += tm;
      ci += tc;
    }
  }
  if (lane == 31) {
    s_wm[warp] = mi;
    s_wc[warp] = ci;
  }
  if (tid == 0) {
    rd[row].b1 = kGB;
    rd[row].blo = kGB;
    rd[row].bhi = -1;
  }
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = s_wm[lane];
    const int wc = s_wc[lane];
    unsigned long long wi = w;
    int wci = wc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long tm = __shfl_up_sync(0xffffffffu, wi, o);
      const int tc = __shfl_up_sync(0xffffffffu, wci, o);
      if (lane >= o) {
        wi += tm;
        wci += tc;
      }
    }
    s_wm[lane] = wi - w;
    s_wc[lane] = wci - wc;
    if (lane == 31) {
      s_wm[32] = wi;
      s_wc[32] = wci;
    }
  }
  __syncthreads();
  const unsigned long long T = s_wm[32];
  unsigned long long mex = s_wm[warp] + mi - mloc;
  int cex = s_wc[warp] + ci - cloc;
  const unsigned long long T1 = ceil_u64(p1 * (double)T);
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    const int b = tid * kBPT + j;
    const unsigned long long inc = mex + bm[j];
    if (bm[j] && mex < T1 && T1 <= inc) {
      rd[row].b1 = b;
      rd[row].before1 = mex;
      rd[row].mass1 = bm[j];
      rd[row].Tlo = ceil_u64(p2 * (double)mex);
      rd[row].Thi = ceil_u64(p2 * (double)inc);
    }
    pm[b] = mex;
    pc[b] = cex;
    mex = inc;
    cex += bc[j];
  }
  if (tid == kGT - 1) pc[kGB] = s_wc[32];
  if (tid == 0) rd[row].T = T;
}

// candidates -> their global slots; every other element's state from its bin
__global__ void __launch_bounds__(kST2) gs_cand_kernel(const int* __restrict__ Ks, int ld, double p1, double p2,
                                                      GSelRow* __restrict__ rd,
                                                      const unsigned long long* __restrict__ hm,
                                                      const int* __restrict__ hc, int* __restrict__ cur,
                                                      const unsigned long long* __restrict__ pk_ws,
                                                      int* __restrict__ cand_ws, uint8_t* __restrict__ state_all) {
  const int row = blockIdx.y, S = gridDim.x, sp = blockIdx.x, tid = threadIdx.x;
  const int K = Ks[row];
  const int b1 = rd[row].b1;
  const unsigned long long T = rd[row].T, Tlo = rd[row].Tlo, Thi = rd[row].Thi;
  const unsigned long long* pm = hm + (size_t)row * kGB;
  const int* pc = hc + (size_t)row * (kGB + 1);
  const unsigned long long* pk = pk_ws + (size_t)row * ld;
  int* cand = cand_ws + (size_t)row * ld;
  uint8_t* state = state_all + (size_t)row * ld;
  const uint8_t zst = p1 >= 1.0 ? (p2 >= 1.0 ? 2 : 1) : 0;
  const bool none = T == 0ull || b1 >= kGB;
  const int i0 = (int)((long long)K * sp / S), i1 = (int)((long long)K * (sp + 1) / S);
  int lo = kGB, hi = -1;
  for (int i = i0 + tid; i < i1; i += kST2 * kGU) {
    unsigned long long wv[kGU];
#pragma unroll
    for (int j = 0; j < kGU; ++j) wv[j] = i + j * kST2 < i1 ? pk[i + j * kST2] : 0ull;
#pragma unroll
    for (int j = 0; j < kGU; ++j) {
      const int ii = i + j * kST2;
      if (ii >= i1) break;
      const unsigned long long u = wv[j] >> 11;
      const int b = (int)(wv[j] & 2047u);
      uint8_t st = 0;
      if (none) {
        st = zst;
      } else if (!u) {
        st = zst;
      } else if (b <= b1) {
        const unsigned long long inc = b + 1 < kGB ? pm[b + 1] : T;
        if (b == b1 || (inc >= Tlo && pm[b] < Thi)) {
          cand[pc[b] + atomicAdd(&cur[(size_t)row * kGB + b], 1)] = ii;
          if (b < b1) {
            lo = min(lo, b);
            hi = max(hi, b);
          }
          continue;  // ranked by the last kernel
        }
        st = inc < Tlo ? 2 : 1;
      }
      state[ii] = st;
    }
  }
  if (hi >= 0) {
    atomicMin(&rd[row].blo, lo);
    atomicMax(&rd[row].bhi, hi);
  }
}

// one CTA per row: stage the candidates, rank them, both cuts, their states
__global__ void __launch_bounds__(kGT, 1) gs_rank_kernel(const double* __restrict__ lm, int ld, const int* __restrict__ Ks,
                                                        double p1, double p2, GSelRow* __restrict__ rd,
                                                        const unsigned long long* __restrict__ hm,
                                                        const int* __restrict__ hc,
                                                        const unsigned long long* __restrict__ pk_ws,
                                                        const int* __restrict__ cand_ws,
                                                        uint8_t* __restrict__ state_all, int* __restrict__ counts,
                                                        int* __restrict__ fail) {
  const int row = blockIdx.x, tid = threadIdx.x;
  const int K = Ks[row];
  extern __shared__ __align__(16) unsigned char g_dyn[];
  unsigned long long* s_cu = reinterpret_cast<unsigned long long*>(g_dyn);
  unsigned long long* s_cex = s_cu + kGCand;
  double* s_clm = reinterpret_cast<double*>(s_cex + kGCand);
  int* s_cid = reinterpret_cast<int*>(s_clm + kGCand);
  int* s_cpos = s_cid + kGCand;
  __shared__ int s_n1, s_n2;
  __shared__ unsigned long long s_at1;
  const unsigned long long* pm = hm + (size_t)row * kGB;
  const int* pc = hc + (size_t)row * (kGB + 1);
  const unsigned long long* pk = pk_ws + (size_t)row * ld;
  const int* cand = cand_ws + (size_t)row * ld;
  uint8_t* state = state_all + (size_t)row * ld;
  const int b1 = rd[row].b1, blo = rd[row].blo, bhi = rd[row].bhi;
  const unsigned long long T = rd[row].T;
  if (tid == 0) {
    s_n1 = 0;
    s_n2 = 0;
    s_at1 = 0ull;
  }
  __syncthreads();
  if (T == 0ull || b1 >= kGB) {
    if (tid == 0) {
      counts[2 * row] = p1 >= 1.0 ? K : 0;
      counts[2 * row + 1] = p1 >= 1.0 && p2 >= 1.0 ? K : 0;
      rd[row].mkey = 0ull;
    }
    return;
  }
  const int r1a = bhi >= 0 ? pc[blo] : 0, r1b = bhi >= 0 ? pc[bhi + 1] : 0;
  const int r2a = pc[b1], r2b = pc[b1 + 1];
  const int n1c = r1b - r1a, nc = n1c + (r2b - r2a);
  const unsigned long long T1 = ceil_u64(p1 * (double)T);
  if (nc > kGCand) {  // very flat rows: rank straight from global scratch (slow, rare)
    if (tid == 0) *fail = 1;
    for (int t = tid; t < nc; t += kGT) {
      const int slot = t < n1c ? r1a + t : r2a + (t - n1c);
      const int i = cand[slot];
      const double la = gsel_sanitise(lm[(size_t)row * ld + i]);
      const unsigned long long u = pk[i] >> 11;
      const int b = (int)(pk[i] & 2047u);
      int rk = 0;
      unsigned long long pre = 0ull;
      for (int j = pc[b]; j < pc[b + 1]; ++j) {
        const int ij = cand[j];
        const double lj = gsel_sanitise(lm[(size_t)row * ld + ij]);
        if (lj > la || (lj == la && ij < i)) {
          ++rk;
          pre += pk[ij] >> 11;
        }
      }
      const unsigned long long e0 = pm[b] + pre;
      if (e0 < T1 && T1 <= e0 + u) {
        s_n1 = pc[b] + rk + 1;
        s_at1 = e0 + u;
      }
    }
    __syncthreads();
    const int n1 = p1 >= 1.0 ? K : s_n1;
    const unsigned long long T2 = ceil_u64(p2 * (double)s_at1);
    for (int pass = 0; pass < 2; ++pass) {  // pass 0: the stage-2 cut; pass 1: states
      const int n2 = p1 >= 1.0 && p2 >= 1.0 ? K : s_n2;
      for (int t = tid; t < nc; t += kGT) {
        const int slot = t < n1c ? r1a + t : r2a + (t - n1c);
        const int i = cand[slot];
        const double la = gsel_sanitise(lm[(size_t)row * ld + i]);
        const unsigned long long u = pk[i] >> 11;
        const int b = (int)(pk[i] & 2047u);
        int rk = 0;
        unsigned long long pre = 0ull;
        for (int j = pc[b]; j < pc[b + 1]; ++j) {
          const int ij = cand[j];
          const double lj = gsel_sanitise(lm[(size_t)row * ld + ij]);
          if (lj > la || (lj == la && ij < i)) {
            ++rk;
            pre += pk[ij] >> 11;
          }
        }
        const int ps = pc[b] + rk;
        const unsigned long long e0 = pm[b] + pre;
        if (pass == 0 && e0 < T2 && T2 <= e0 + u) s_n2 = ps + 1;
        if (pass == 1) state[i] = ps < n2 ? 2 : (ps < n1 ? 1 : 0);
      }
      __syncthreads();
    }
    if (tid == 0) {
      counts[2 * row] = n1;
      counts[2 * row + 1] = p1 >= 1.0 && p2 >= 1.0 ? K : s_n2;
      rd[row].mkey = 0ull;
    }
    return;
  }
  auto sidx = [&](int slot) { return slot >= r2a ? n1c + (slot - r2a) : slot - r1a; };
  for (int t = tid; t < nc; t += kGT) {
    const int slot = t < n1c ? r1a + t : r2a + (t - n1c);
    const int i = cand[slot];
    s_cid[t] = i;
    s_clm[t] = gsel_sanitise(lm[(size_t)row * ld + i]);
    s_cu[t] = pk[i] >> 11;
  }
  __syncthreads();
  for (int t = tid; t < nc; t += kGT) {
    const int i = s_cid[t];
    const double la = s_clm[t];
    const unsigned long long u = s_cu[t];
    const int b = (int)(pk[i] & 2047u);
    const int j0 = pc[b], j1 = pc[b + 1], k0 = sidx(j0);
    int rk = 0;
    unsigned long long pre = 0ull;
    for (int j = 0; j < j1 - j0; ++j) {
      const double lj = s_clm[k0 + j];
      const int ij = s_cid[k0 + j];
      const bool ahead = lj > la || (lj == la && ij < i);
      rk += ahead;
      pre += ahead ? s_cu[k0 + j] : 0ull;
    }
    const unsigned long long e0 = pm[b] + pre;
    s_cpos[t] = j0 + rk;
    s_cex[t] = e0;
    if (e0 < T1 && T1 <= e0 + u) {
      s_n1 = j0 + rk + 1;
      s_at1 = e0 + u;
    }
  }
  __syncthreads();
  const int n1 = p1 >= 1.0 ? K : s_n1;
  const unsigned long long T2 = ceil_u64(p2 * (double)s_at1);
  for (int t = tid; t < nc; t += kGT)
    if (s_cex[t] < T2 && T2 <= s_cex[t] + s_cu[t]) s_n2 = s_cpos[t] + 1;
  __syncthreads();
  const int n2 = p1 >= 1.0 && p2 >= 1.0 ? K : s_n2;
  for (int t = tid; t < nc; t += kGT) state[s_cid[t]] = s_cpos[t] < n2 ? 2 : (s_cpos[t] < n1 ? 1 : 0);
  if (tid == 0) {
    counts[2 * row] = n1;
    counts[2 * row + 1] = n2;
    rd[row].mkey = 0ull;  // ready for the next call
  }
}

// ---------------------------------------------------------------------------
// The same selection in ONE launch: a thread-block cluster of CS CTAs
// (1024 threads each) per row, each CTA holding up to 8192 of the row's
// elements in registers (K <= CS * 8192, CS <= 8).  Every exchange is a
// distributed-shared-memory PUSH that completes a transaction on the
// receiver's mbarrier (st.async, dsmem.cuh) -- no cluster-wide barrier and
// no remote load after the start-up one, the plan kernel's protocol:
//   A  CTA maxima -> every CTA;
//   B  local histograms (1/32-nat bins; masses as three 13-bit pieces so
//      native 32-bit shared atomics stay exact) -> the bin-slice owners
//      (CTA s owns 2048/CS bins);
//   C  owners sum their slice over the sources, push slice totals to every
//      CTA, then (knowing the slice's global offset) push every CTA the
//      slice's exclusive mass / count prefixes and that CTA's own offset
//      inside each bin, plus the stage-1 bin if it lies in the slice;
//   D  every CTA classifies its elements: the candidates (stage-1 bin, the
//      stage-2 range) are pushed to CTA 0 at their bin slots, everything
//      else takes its state from its bin;
//   E  CTA 0 ranks the candidates (log-mass desc, index asc), finds both
//      cuts and writes their states.
// Same arithmetic as select_global_kernel (u, bins, double thresholds), so
// the states are identical (tests/test_gpu_seqshard.py).  More candidates
// than kGCand go through global scratch and one cluster barrier instead.
// ---------------------------------------------------------------------------
__device__ int g_gsel_dbg;  // timing experiments (dp_debug_set(12, .)): exit after phase n
constexpr int kGCT = 1024;  // threads per CTA
constexpr int kGCE = 8;     // elements per thread
constexpr int kGCMaxCS = 8;
struct GcLayout {
  // region 1: local histogram + receive buffer, later (CTA 0) the staged candidates
  static constexpr size_t h0 = 0;                          // u32[kGB] mass bits [0, 13)
  static constexpr size_t h1 = h0 + (size_t)kGB * 4;       // u32[kGB] mass bits [13, 26)
  static constexpr size_t h2 = h1 + (size_t)kGB * 4;       // u32[kGB] mass bits [26, 39)
  static constexpr size_t hc = h2 + (size_t)kGB * 4;       // u32[kGB] counts
  static constexpr size_t recv = hc + (size_t)kGB * 4;     // uint4[kGB]: [source][slice bin] pieces + count
  static constexpr size_t cu = 0;                          // u64[kGCand] staged candidates: mass
  static constexpr size_t clm = cu + (size_t)kGCand * 8;   //   log-mass
  static constexpr size_t cex = clm + (size_t)kGCand * 8;  //   exclusive cumulative mass (CTA 0's ranking)
  static constexpr size_t cid = cex + (size_t)kGCand * 8;  //   index
  static constexpr size_t cpos = cid + (size_t)kGCand * 4; //   sorted position
  static constexpr size_t r1 = cpos + (size_t)kGCand * 4;
  // region 2: the row's bin table (every CTA) and candidate cursors
  static constexpr size_t tab = r1;                        // uint4[kGB]: pm lo, pm hi, pc, my base in the bin
  static constexpr size_t cur = tab + (size_t)kGB * 16;    // int[kGB] local candidate cursors
  static constexpr size_t bytes = cur + (size_t)kGB * 4;
  static_assert(recv + (size_t)kGB * 16 <= r1, "histogram region overlaps the bin table");
};

template <int CS>
__global__ void __launch_bounds__(kGCT, 1)
    gsel_cluster_kernel(const double* __restrict__ lm_all, int ld, int part_len, long long part_stride,
                        const int* __restrict__ Ks, double p1, double p2,
                        uint8_t* __restrict__ state_all, int* __restrict__ counts, int* __restrict__ gcid,
                        double* __restrict__ gclm, unsigned long long* __restrict__ gcu,
                        unsigned long long* __restrict__ gcex, int* __restrict__ gcpos) {
  constexpr int W = kGB / CS;                      // bins per slice owner
  constexpr int BPT = W > kGCT ? W / kGCT : 1;     // slice bins per thread
  constexpr int NT = W / BPT;                      // threads holding slice bins
  const int c = (int)cg::this_cluster().block_rank();
  const int row = blockIdx.x / CS, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = Ks[row];
  // element i of the row: part i / part_len, slot i % part_len (one part: the row itself;
  // several: the all-gathered [parts, rows, part_len] slices read in place)
  const double* lm = lm_all + (size_t)row * (part_stride ? part_len : ld);
  auto lm_at = [&](int i) {
    return part_stride ? lm[(long long)(i / part_len) * part_stride + (i % part_len)] : lm[i];
  };
  uint8_t* state = state_all + (size_t)row * ld;
  extern __shared__ __align__(16) unsigned char g_dyn[];
  unsigned* h0 = reinterpret_cast<unsigned*>(g_dyn + GcLayout::h0);
  unsigned* h1 = reinterpret_cast<unsigned*>(g_dyn + GcLayout::h1);
  unsigned* h2 = reinterpret_cast<unsigned*>(g_dyn + GcLayout::h2);
  unsigned* hc = reinterpret_cast<unsigned*>(g_dyn + GcLayout::hc);
  uint4* recv = reinterpret_cast<uint4*>(g_dyn + GcLayout::recv);
  uint4* tab = reinterpret_cast<uint4*>(g_dyn + GcLayout::tab);
  int* lcur = reinterpret_cast<int*>(g_dyn + GcLayout::cur);
  __shared__ __align__(8) unsigned long long s_mb[5];  // A maxima, B histograms, C slice totals, D table, E candidates
  __shared__ __align__(8) double s_cmax[kGCMaxCS];
  __shared__ __align__(8) unsigned long long s_sm[kGCMaxCS];
  __shared__ unsigned s_sc[kGCMaxCS];
  __shared__ int s_rb1[kGCMaxCS];
  __shared__ __align__(16) unsigned long long s_rbm[kGCMaxCS][2];
  __shared__ double s_red[32];
  __shared__ unsigned long long s_wm[33];
  __shared__ unsigned s_wc[33];
  __shared__ unsigned long long s_at1;
  __shared__ int s_myb1, s_n1, s_n2, s_blo, s_bhi;
  __shared__ __align__(16) unsigned long long s_myb1m[2];
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 5; ++i) mb_init(&s_mb[i]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mb_expect(&s_mb[0], CS * 8);
    mb_expect(&s_mb[1], (unsigned)(CS * W * 16));
    mb_expect(&s_mb[2], CS * 12);
    mb_expect(&s_mb[3], (unsigned)(kGB * 16 + CS * 20));
    s_myb1 = kGB;
    s_n1 = 0;
    s_n2 = 0;
    s_at1 = 0ull;
    s_blo = kGB;
    s_bhi = -1;
  }
  for (int j = tid; j < kGB; j += kGCT) {
    h0[j] = 0u;
    h1[j] = 0u;
    h2[j] = 0u;
    hc[j] = 0u;
    lcur[j] = 0;
  }
  // my elements: [e0, e1), thread tid holds e0 + tid + j * kGCT
  const int per = (K + CS - 1) / CS;
  const int e0 = min(K, c * per), e1 = min(K, e0 + per);
  double x[kGCE];
#pragma unroll
  for (int j = 0; j < kGCE; ++j) {
    const int i = e0 + tid + j * kGCT;
    x[j] = i < e1 ? gsel_sanitise(lm_at(i)) : -CUDART_INF;
  }
  double m = x[0];
#pragma unroll
  for (int j = 1; j < kGCE; ++j) m = fmax(m, x[j]);
  m = warp_max(m);
  if (lane == 0) s_red[warp] = m;
  __syncthreads();  // barrier init, zeroed histogram, warp maxima
  cl_arrive_relaxed();  // (S) every CTA has started and initialised its barriers
  const int dbg = g_gsel_dbg;
  // ---- A: maxima
  double cmax = -CUDART_INF;
  if (tid < CS) {
    double mm[32];
#pragma unroll
    for (int w = 0; w < 32; ++w) mm[w] = s_red[w];
#pragma unroll
    for (int h = 16; h > 0; h >>= 1)
#pragma unroll
      for (int w = 0; w < h; ++w) mm[w] = fmax(mm[w], mm[w + h]);
    cmax = mm[0];
  }
  cl_wait();  // (S) -- .aligned: every thread, outside any divergent branch
  if (tid < CS) push_f64(&s_cmax[c], tid, cmax, &s_mb[0]);
  mb_wait0(&s_mb[0]);
  double M = s_cmax[0];
#pragma unroll
  for (int r = 1; r < CS; ++r) M = fmax(M, s_cmax[r]);
  if (dbg == 1) return;
  // ---- B: local histogram -> the slice owners
  unsigned long long pk[kGCE];
#pragma unroll
  for (int j = 0; j < kGCE; ++j) {
    const int i = e0 + tid + j * kGCT;
    pk[j] = 0ull;
    if (i < e1) {
      unsigned long long u;
      int b;
      gsel_elem(M, x[j], u, b);
      pk[j] = (u << 11) | (unsigned long long)b;
      if (u) {
        atomicAdd(&h0[b], (unsigned)(u & 0x1FFFu));
        if (u >> 13) atomicAdd(&h1[b], (unsigned)((u >> 13) & 0x1FFFu));
        if (u >> 26) atomicAdd(&h2[b], (unsigned)(u >> 26));
        atomicAdd(&hc[b], 1u);
      }
    }
  }
  __syncthreads();
  for (int b = tid; b < kGB; b += kGCT) {
    const int s = b / W;
    push_v4(&recv[c * W + (b - s * W)], s, (int)h0[b], (int)h1[b], (int)h2[b], (int)hc[b], &s_mb[1]);
  }
  mb_wait0(&s_mb[1]);
  if (dbg == 2) return;
  // ---- C: my slice [c W, (c + 1) W): sums over the sources, slice totals
  unsigned long long bm[BPT];
  unsigned bc[BPT];
  unsigned long long mloc = 0ull;
  unsigned cloc = 0u;
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    bm[k] = 0ull;
    bc[k] = 0u;
    if (tid < NT) {
      const int lb = tid * BPT + k;
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        const uint4 v = recv[r * W + lb];
        bm[k] += (unsigned long long)v.x + ((unsigned long long)v.y << 13) + ((unsigned long long)v.z << 26);
        bc[k] += v.w;
      }
    }
    mloc += bm[k];
    cloc += bc[k];
  }
  unsigned long long mi = mloc;
  unsigned ci = cloc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long tm = __shfl_up_sync(0xffffffffu, mi, o);
    const unsigned tc = __shfl_up_sync(0xffffffffu, ci, o);
    if (lane >= o) {
      mi += tm;
      ci += tc;
    }
  }
  if (lane == 31) {
    s_wm[warp] = mi;
    s_wc[warp] = ci;
  }
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = s_wm[lane];
    const unsigned wc = s_wc[lane];
    unsigned long long wi = w;
    unsigned wci = wc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long tm = __shfl_up_sync(0xffffffffu, wi, o);
      const unsigned tc = __shfl_up_sync(0xffffffffu, wci, o);
      if (lane >= o) {
        wi += tm;
        wci += tc;
      }
    }
    s_wm[lane] = wi - w;
    s_wc[lane] = wci - wc;
    if (lane == 31) {
      s_wm[32] = wi;
      s_wc[32] = wci;
    }
  }
  __syncthreads();
  if (tid < CS) {
    push_u64(&s_sm[c], tid, s_wm[32], &s_mb[2]);
    push_u32(&s_sc[c], tid, s_wc[32], &s_mb[2]);
  }
  mb_wait0(&s_mb[2]);
  unsigned long long T = 0ull, before = 0ull;
  unsigned cbefore = 0u, ctot = 0u;
#pragma unroll
  for (int r = 0; r < CS; ++r) {
    if (r < c) {
      before += s_sm[r];
      cbefore += s_sc[r];
    }
    T += s_sm[r];
    ctot += s_sc[r];
  }
  const double thr1 = p1 * (double)T;
  {
    unsigned long long mex = before + s_wm[warp] + mi - mloc;
    unsigned cex = cbefore + s_wc[warp] + ci - cloc;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      if (tid < NT) {
        const int lb = tid * BPT + k, b = c * W + lb;
        const unsigned long long inc = mex + bm[k];
        if (bm[k] && (double)mex < thr1 && thr1 <= (double)inc) {
          s_myb1 = b;
          s_myb1m[0] = mex;
          s_myb1m[1] = bm[k];
        }
        // every CTA: this bin's prefixes and that CTA's offset inside the bin
        unsigned base = 0u;
#pragma unroll
        for (int r = 0; r < CS; ++r) {
          push_v4(&tab[b], r, (int)(unsigned)mex, (int)(unsigned)(mex >> 32), (int)cex, (int)base, &s_mb[3]);
          base += recv[r * W + lb].w;
        }
      }
      mex += bm[k];
      cex += bc[k];
    }
  }
  __syncthreads();
  if (tid < CS) {
    push_u32(&s_rb1[c], tid, (unsigned)s_myb1, &s_mb[3]);
    push_v2u64(&s_rbm[c][0], tid, s_myb1m[0], s_myb1m[1], &s_mb[3]);
  }
  mb_wait0(&s_mb[3]);
  if (dbg == 3) return;
  // ---- D: classify; candidates -> CTA 0
  int b1 = kGB;
  unsigned long long before1 = 0ull, mass1 = 0ull;
#pragma unroll
  for (int r = 0; r < CS; ++r)
    if (s_rb1[r] < b1) {
      b1 = s_rb1[r];
      before1 = s_rbm[r][0];
      mass1 = s_rbm[r][1];
    }
  auto pm_of = [&](int b) {
    const uint4 t = tab[b];
    return (unsigned long long)t.x | ((unsigned long long)t.y << 32);
  };
  auto pc_of = [&](int b) { return b < kGB ? (int)tab[b].z : (int)ctot; };
  const bool none = T == 0ull || b1 >= kGB;  // no mass (a non-finite query)
  const uint8_t zst = p1 >= 1.0 ? (p2 >= 1.0 ? 2 : 1) : 0;
  const unsigned long long Tlo = none ? 0ull : ceil_u64(p2 * (double)before1),
                           Thi = none ? 0ull : ceil_u64(p2 * (double)(before1 + mass1));
  auto is_cand = [&](int b) {
    const unsigned long long inc = b + 1 < kGB ? pm_of(b + 1) : T;
    return b == b1 || (b < b1 && inc >= Tlo && pm_of(b) < Thi);
  };
  if (!none) {  // the stage-2 candidate bins below b1 form one range [blo, bhi] (prefixes are monotone)
    int lo = kGB, hi = -1;
    for (int b = tid; b < b1; b += kGCT)
      if (is_cand(b)) {
        lo = min(lo, b);
        hi = max(hi, b);
      }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0 && hi >= 0) {
      atomicMin(&s_blo, lo);
      atomicMax(&s_bhi, hi);
    }
  }
  __syncthreads();
  const int r1a = s_bhi >= 0 ? pc_of(s_blo) : 0, r1b = s_bhi >= 0 ? pc_of(s_bhi + 1) : 0;
  const int r2a = none ? 0 : pc_of(b1), r2b = none ? 0 : pc_of(b1 + 1);
  const int n1c = r1b - r1a, nc = n1c + (r2b - r2a);
  const bool staged = nc <= kGCand;
  auto sidx = [&](int slot) { return slot >= r2a ? n1c + (slot - r2a) : slot - r1a; };
  if (c == 0 && tid == 0) mb_expect(&s_mb[4], staged ? (unsigned)nc * 20u : 0u);
  unsigned long long* s_cu = reinterpret_cast<unsigned long long*>(g_dyn + GcLayout::cu);
  double* s_clm = reinterpret_cast<double*>(g_dyn + GcLayout::clm);
  int* s_cid = reinterpret_cast<int*>(g_dyn + GcLayout::cid);
#pragma unroll
  for (int j = 0; j < kGCE; ++j) {
    const int i = e0 + tid + j * kGCT;
    if (i >= e1) continue;
    const unsigned long long u = pk[j] >> 11;
    const int b = (int)(pk[j] & 2047u);
    uint8_t st;
    if (none || !u) {
      st = zst;
    } else if (b > b1) {
      st = 0;
    } else if (is_cand(b)) {
      const int t = sidx(pc_of(b) + (int)tab[b].w + atomicAdd(&lcur[b], 1));
      const double li = gsel_sanitise(lm_at(i));  // (re-read: x[] is not kept live across the exchanges)
      if (staged) {
        push_u64(&s_cu[t], 0, u, &s_mb[4]);
        push_f64(&s_clm[t], 0, li, &s_mb[4]);
        push_u32(&s_cid[t], 0, (unsigned)i, &s_mb[4]);
      } else {
        gcu[(size_t)row * ld + t] = u;
        gclm[(size_t)row * ld + t] = li;
        gcid[(size_t)row * ld + t] = i;
      }
      continue;  // ranked by CTA 0
    } else {
      const unsigned long long inc = b + 1 < kGB ? pm_of(b + 1) : T;
      st = inc < Tlo ? 2 : 1;
    }
    state[i] = st;
  }
  if (!staged) cl_sync();  // the global-scratch candidates are visible to CTA 0
  if (c != 0) return;
  if (staged) mb_wait0(&s_mb[4]);  // every candidate push has landed (CTA 0 must not exit before)
  if (dbg == 4) return;
  if (none) {
    if (tid == 0) {
      counts[2 * row] = p1 >= 1.0 ? K : 0;
      counts[2 * row + 1] = p1 >= 1.0 && p2 >= 1.0 ? K : 0;
    }
    return;
  }
  // ---- E: CTA 0 ranks the candidates inside their bins (log-mass desc, index asc)
  unsigned long long* a_cu = s_cu;
  double* a_clm = s_clm;
  int* a_cid = s_cid;
  unsigned long long* a_cex = reinterpret_cast<unsigned long long*>(g_dyn + GcLayout::cex);
  int* a_cpos = reinterpret_cast<int*>(g_dyn + GcLayout::cpos);
  if (!staged) {
    a_cu = gcu + (size_t)row * ld;
    a_clm = gclm + (size_t)row * ld;
    a_cid = gcid + (size_t)row * ld;
    a_cex = gcex + (size_t)row * ld;
    a_cpos = gcpos + (size_t)row * ld;
  }
  for (int t = tid; t < nc; t += kGCT) {
    const int i = a_cid[t];
    const double la = a_clm[t];
    const unsigned long long u = a_cu[t];
    unsigned long long uu;
    int b;
    gsel_elem(M, la, uu, b);
    const int j0 = pc_of(b), j1 = pc_of(b + 1), k0 = sidx(j0);
    int rk = 0;
    unsigned long long pre = 0ull;
    for (int j = 0; j < j1 - j0; ++j) {
      const double lj = a_clm[k0 + j];
      const int ij = a_cid[k0 + j];
      const bool ahead = lj > la || (lj == la && ij < i);
      rk += ahead;
      pre += ahead ? a_cu[k0 + j] : 0ull;
    }
    const int ps = j0 + rk;
    const unsigned long long ex = pm_of(b) + pre;
    a_cpos[t] = ps;
    a_cex[t] = ex;
    if ((double)ex < thr1 && thr1 <= (double)(ex + u)) {
      s_n1 = ps + 1;
      s_at1 = ex + u;
    }
  }
  __syncthreads();
  const int n1 = p1 >= 1.0 ? K : s_n1;
  const double thr2 = p2 * (double)s_at1;
  for (int t = tid; t < nc; t += kGCT)
    if ((double)a_cex[t] < thr2 && thr2 <= (double)(a_cex[t] + a_cu[t])) s_n2 = a_cpos[t] + 1;
  __syncthreads();
  const int n2 = p1 >= 1.0 && p2 >= 1.0 ? K : s_n2;
  for (int t = tid; t < nc; t += kGCT) state[a_cid[t]] = a_cpos[t] < n2 ? 2 : (a_cpos[t] < n1 ? 1 : 0);
  if (tid == 0) {
    counts[2 * row] = n1;
    counts[2 * row + 1] = n2;
  }
}

// ---------------------------------------------------------------------------
// LSE merge of P partials: out_parts [P, rows, d], lse_parts [P, rows]
// ---------------------------------------------------------------------------
__global__ void lse_merge_kernel(const float* __restrict__ out_parts, const float* __restrict__ lse_parts, int P,
                                 int rows, int d, float* __restrict__ out, float* __restrict__ lse) {
  const int row = blockIdx.x, tid = threadIdx.x;
  __shared__ double s_w[64];
  __shared__ double s_L;
  if (tid < 32) {  // the P weights once per row (fp64, one lane per part), then every dim reuses them
    const float l = tid < P ? lse_parts[(size_t)tid * rows + row] : -INFINITY;
    const float l2 = tid + 32 < P ? lse_parts[(size_t)(tid + 32) * rows + row] : -INFINITY;
    float M = fmaxf(l, l2);
#pragma unroll
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const double w = l != -INFINITY ? exp((double)l - (double)M) : 0.0;
    const double w2 = l2 != -INFINITY ? exp((double)l2 - (double)M) : 0.0;
    if (tid < P) s_w[tid] = w;
    if (tid + 32 < P) s_w[tid + 32] = w2;
    double L = w + w2;
#pragma unroll
    for (int o = 16; o; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (tid == 0) {
      s_L = L;
      lse[row] = L > 0.0 ? (float)((double)M + log(L)) : -INFINITY;
    }
  }
  __syncthreads();
  const double L = s_L;
  for (int c = tid; c < d; c += blockDim.x) {
    double acc = 0.0;
#pragma unroll 8
    for (int p = 0; p < P; ++p) {  // (unrolled: the part loads are independent and go out together)
      const float x = out_parts[((size_t)p * rows + row) * d + c];
      const double w = s_w[p];
      if (w > 0.0) acc += w * (double)x;
    }
    out[(size_t)row * d + c] = L > 0.0 ? (float)(acc / L) : 0.f;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_kmpp_dsq(const void* pts, int dtype, int units, int n, int d, const double* centre, int first,
                            double* dsq, double* sums, cudaStream_t st) {
  kmpp_dsq_kernel<<<units, kKT, (size_t)d * sizeof(double), st>>>(pts, dtype, n, d, centre, first, dsq, sums);
  return cudaGetLastError();
}
cudaError_t launch_kmpp_pick(const void* pts, int dtype, int units, int n, int d, const double* dsq,
                             const double* all_sums, int P, int rank, const double* u_draw, const int* pick_in,
                             long long gbase, double* centre_out, int* pick_out, cudaStream_t st) {
  kmpp_pick_kernel<<<units, kKT, 0, st>>>(pts, dtype, n, d, dsq, all_sums, P, rank, u_draw, pick_in, gbase,
                                          centre_out, pick_out);
  return cudaGetLastError();
}
size_t lloyd_sums_ws_bytes(int units, int n, int k) { return ((size_t)units * k + (size_t)units * n) * sizeof(int); }
cudaError_t launch_lloyd_sums(const void* pts, int dtype, int units, int n, int d, const int* assign, int k,
                              double* sums, long long* counts, void* ws, cudaStream_t st) {
  int* cnt = reinterpret_cast<int*>(ws);
  int* order = cnt + (size_t)units * k;
  lloyd_sums_kernel<<<units, kLT, 0, st>>>(pts, dtype, n, d, assign, k, sums, counts, cnt, order);
  return cudaGetLastError();
}
size_t select_global_ws_bytes(int rows, int ld) {
  const size_t split = (size_t)rows * ld * (8 + 8 + 4 + 4) +
                       (size_t)rows * (sizeof(GSelRow) + kGB * 8 + (kGB + 1) * 4 + kGB * 4) + 64;
  const size_t clustered = (size_t)rows * ld * (4 + 8 + 8 + 8 + 4) + 64;  // candidate overflow scratch
  return split > clustered ? split : clustered;
}

int g_gsel_path = 0;
int set_gsel_dbg(int v) { return cudaMemcpyToSymbol(g_gsel_dbg, &v, sizeof(int)) == cudaSuccess ? 0 : 2; }  // dp_debug_set(11, .): 0 auto, 1 split launches, 2 one CTA per row, 3 clustered

// cluster size for the one-launch form: 8192 elements per CTA, power of two <= 8
static int gsel_cluster_size(int ld) {
  int cs = 1;
  while (cs < kGCMaxCS && (long long)cs * kGCT * kGCE < ld) cs <<= 1;
  return (long long)cs * kGCT * kGCE >= ld ? cs : 0;
}
bool select_global_parts_supported(int parts, int part_len) {
  return gsel_cluster_size((int)((long long)parts * part_len)) > 0 && (long long)parts * part_len < (1ll << 31);
}
cudaError_t launch_select_global(const double* lm, int rows, int ld, const int* Ks, double p1, double p2,
                                 uint8_t* state, int* counts, void* ws, cudaStream_t st, int part_len) {
  unsigned long long* ex = reinterpret_cast<unsigned long long*>(ws);
  unsigned long long* pk = ex + (size_t)rows * ld;
  int* pos = reinterpret_cast<int*>(pk + (size_t)rows * ld);
  int* cand = pos + (size_t)rows * ld;
  cudaError_t ea = ensure_smem(reinterpret_cast<const void*>(select_global_kernel), kGDyn);
  if (ea == cudaSuccess) ea = ensure_smem(reinterpret_cast<const void*>(gs_rank_kernel), kGDyn);
  if (ea != cudaSuccess) return ea;
  // part_len > 0: lm is [ld / part_len, rows, part_len] (the one-launch form reads it in place)
  const long long part_stride = part_len > 0 ? (long long)rows * part_len : 0;
  if (part_len <= 0) part_len = ld;
  const int CS = gsel_cluster_size(ld);
  if (part_stride && !(CS > 0)) return cudaErrorInvalidValue;
  if ((g_gsel_path == 0 || g_gsel_path == 3 || part_stride) && CS > 0) {
    const void* fn = CS == 1 ? reinterpret_cast<const void*>(gsel_cluster_kernel<1>)
                     : CS == 2 ? reinterpret_cast<const void*>(gsel_cluster_kernel<2>)
                     : CS == 4 ? reinterpret_cast<const void*>(gsel_cluster_kernel<4>)
                               : reinterpret_cast<const void*>(gsel_cluster_kernel<8>);
    cudaError_t e = ensure_smem(fn, GcLayout::bytes);
    if (e != cudaSuccess) return e;
    int* gcid = reinterpret_cast<int*>(ws);
    double* gclm = reinterpret_cast<double*>(gcid + ((size_t)rows * ld + 1) / 2 * 2);
    unsigned long long* gcu = reinterpret_cast<unsigned long long*>(gclm + (size_t)rows * ld);
    unsigned long long* gcex = gcu + (size_t)rows * ld;
    int* gcpos = reinterpret_cast<int*>(gcex + (size_t)rows * ld);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(rows * CS);
    cfg.blockDim = dim3(kGCT);
    cfg.dynamicSmemBytes = GcLayout::bytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    switch (CS) {
      case 1: return cudaLaunchKernelEx(&cfg, gsel_cluster_kernel<1>, lm, ld, part_len, part_stride, Ks, p1, p2, state, counts, gcid, gclm, gcu, gcex, gcpos);
      case 2: return cudaLaunchKernelEx(&cfg, gsel_cluster_kernel<2>, lm, ld, part_len, part_stride, Ks, p1, p2, state, counts, gcid, gclm, gcu, gcex, gcpos);
      case 4: return cudaLaunchKernelEx(&cfg, gsel_cluster_kernel<4>, lm, ld, part_len, part_stride, Ks, p1, p2, state, counts, gcid, gclm, gcu, gcex, gcpos);
      default: return cudaLaunchKernelEx(&cfg, gsel_cluster_kernel<8>, lm, ld, part_len, part_stride, Ks, p1, p2, state, counts, gcid, gclm, gcu, gcex, gcpos);
    }
  }
  // split over several CTAs per row when one SM per row would be the bound
  const int S = g_gsel_path == 2 ? 1
                : (ld >= 8192 || g_gsel_path == 1)
                    ? (rows * 8 <= 2 * sm_count() ? 8 : (rows * 4 <= 2 * sm_count() ? 4 : 1))
                    : 1;
  if (S > 1) {
    char* x = reinterpret_cast<char*>(cand + (size_t)rows * ld);
    x += (16 - (reinterpret_cast<uintptr_t>(x) & 15)) & 15;
    GSelRow* rd = reinterpret_cast<GSelRow*>(x);
    unsigned long long* hm = reinterpret_cast<unsigned long long*>(rd + rows);
    int* hc = reinterpret_cast<int*>(hm + (size_t)rows * kGB);
    int* cur = hc + (size_t)rows * (kGB + 1);
    int* fail = reinterpret_cast<int*>(&rd[0].pad);  // (row 0's pad word) set when candidates overflow
    const dim3 g(S, rows);
    gs_max_kernel<<<g, kST2, 0, st>>>(lm, ld, Ks, rd, hm, hc, cur);
    gs_hist_kernel<<<g, kST2, 0, st>>>(lm, ld, Ks, rd, hm, hc, pk);
    gs_scan_kernel<<<rows, kGT, 0, st>>>(Ks, p1, p2, rd, hm, hc);
    gs_cand_kernel<<<g, kST2, 0, st>>>(Ks, ld, p1, p2, rd, hm, hc, cur, pk, cand, state);
    gs_rank_kernel<<<rows, kGT, kGDyn, st>>>(lm, ld, Ks, p1, p2, rd, hm, hc, pk, cand, state, counts, fail);
    return cudaGetLastError();
  }
  select_global_kernel<<<rows, kGT, kGDyn, st>>>(lm, ld, Ks, p1, p2, state, counts, pos, ex, cand, pk);
  return cudaGetLastError();
}
cudaError_t launch_lse_merge(const float* out_parts, const float* lse_parts, int P, int rows, int d, float* out,
                             float* lse, cudaStream_t st) {
  lse_merge_kernel<<<rows, 128, 0, st>>>(out_parts, lse_parts, P, rows, d, out, lse);
  return cudaGetLastError();
}

}  // namespace dp
