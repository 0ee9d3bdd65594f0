// Two-stage top-p of one q head on one CTA (engine.py:180-213,
// selection.py:36-65), shared by the plan kernel (plan.cu, 512 threads) and
// the fused decode-step kernel (step.cu, 384 threads).
//
// e_k = exp(lm_k - max) as a 2^-39 fixed-point integer (exact,
// order-independent sums); a mass histogram over 1/32-nat bins finds the bin
// holding the p1 crossing (then p2 of the retained mass); only the boundary
// bins are ranked exactly (log-mass desc, cluster id asc == the reference's
// stable argsort order).  Cut semantics follow the reference: the first
// prefix whose cumsum/total >= p (searchsorted left + 1, clamped to n).
// Masses below 2^-39 of the max round to zero (<= 4096 * 2^-39 < 1e-8 of
// the total): such clusters sit past the stage-1 cut for every p1 < 1.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace dp {

constexpr float kBinScale = 32.f;           // bins of 1/32 nat
constexpr double kFix = 549755813888.0;     // 2^39 fixed-point scale of e = exp(lm - max) <= 1
constexpr int kCandBins = 8;                // stage-2 candidate bins ranked together with the stage-1 bin

// phase stamps of the first 16 CTAs' selections (profiling builds only, -DDP_PROFILE)
static __device__ unsigned long long g_sel_ts[16][8];
static __device__ unsigned long long g_sel_sub[16][8];  // finer stamps inside a phase (profiling builds)
__device__ __forceinline__ void sel_sub(int ev) {
#ifdef DP_PROFILE
  if (blockIdx.x < 16 && threadIdx.x == 0) g_sel_sub[blockIdx.x][ev] = clock64();
#endif
}
__device__ __forceinline__ void sel_stamp(int ev) {
#ifdef DP_PROFILE
  if (blockIdx.x < 16 && threadIdx.x == 0) {
    g_sel_ts[blockIdx.x][ev] = clock64();  // SM cycles
  }
#endif
}

// block-wide exclusive scan of (mass u64, count int) pairs; totals to mt / ct.
// Warp scans, one barrier, then every warp scans the kT / 32 warp totals
// itself with shuffles (no serial warp-0 step, no second barrier).  sm/sc need
// kT / 32 slots; callers separate consecutive uses with a barrier.
template <int kT>
__device__ __forceinline__ void scan_pair(unsigned long long m, int c, unsigned long long* sm, int* sc,
                                          unsigned long long& mex, int& cex, unsigned long long& mt, int& ct) {
  constexpr int kW = kT / 32;
  static_assert(kW <= 32, "warp totals fit one warp");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long mi = m;
  int ci = c;
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
    sm[warp] = mi;
    sc[warp] = ci;
  }
  __syncthreads();
  unsigned long long wi = lane < kW ? sm[lane] : 0ull;
  int wci = lane < kW ? sc[lane] : 0;
#pragma unroll
  for (int o = 1; o < kW; o <<= 1) {
    const unsigned long long tm = __shfl_up_sync(0xffffffffu, wi, o);
    const int tc = __shfl_up_sync(0xffffffffu, wci, o);
    if (lane >= o) {
      wi += tm;
      wci += tc;
    }
  }
  mt = __shfl_sync(0xffffffffu, wi, kW - 1);
  ct = __shfl_sync(0xffffffffu, wci, kW - 1);
  const unsigned long long wex = __shfl_sync(0xffffffffu, wi, warp > 0 ? warp - 1 : 0);
  const int wcex = __shfl_sync(0xffffffffu, wci, warp > 0 ? warp - 1 : 0);
  mex = (warp > 0 ? wex : 0ull) + mi - m;
  cex = (warp > 0 ? wcex : 0) + ci - c;
}

// ---------------------------------------------------------------------------
// P2 pieces, one copy each (__noinline__): this code runs once per launch on
// a cold instruction cache, so its footprint -- not its instruction count --
// is what costs time.  All threads of the CTA call them.
// ---------------------------------------------------------------------------
struct SelShared {
  unsigned long long before, at;
  int b, n, nc, cbefore;
};

// first bin (< limit) whose inclusive mass reaches thr; before / cbefore =
// mass / count of the bins ahead of it.  bm/bc: this thread's (NB / kT) bins.
template <int kT, int NB>
__device__ __noinline__ int sel_find_bin(SelShared* sh, const unsigned long long* bm, const int* bc,
                                         unsigned long long mbase, int cbase, double thr, int limit) {
  const int tid = threadIdx.x;
  if (tid == 0) {  // not found (no mass at all: a non-finite query) -> nothing ahead of the last bin
    sh->b = NB;
    sh->before = 0;
    sh->cbefore = 0;
  }
  __syncthreads();
  unsigned long long m = mbase, hmass = 0;
  int c = cbase, hit = -1, hcnt = 0;
#pragma unroll
  for (int j = 0; j < (NB / kT); ++j) {
    const int b = tid * (NB / kT) + j;
    if (hit < 0 && b < limit && bm[j] && (double)(m + bm[j]) >= thr) {
      hit = b;
      hmass = m;
      hcnt = c;
    }
    m += bm[j];
    c += bc[j];
  }
  if (hit >= 0) atomicMin(&sh->b, hit);
  __syncthreads();
  const int bb = sh->b;
  if (hit == bb) {
    sh->before = hmass;
    sh->cbefore = hcnt;
  }
  __syncthreads();
  return bb;
}

// members of bin b -> clist (any order), then cord[rank] = member with the
// exact (log-mass desc, cluster id asc) rank; returns the member count
template <int kT>
__device__ __noinline__ int sel_rank_bin(SelShared* sh, const uint16_t* binI, const double* lmall, int* clist,
                                         int* cord, int K, int b) {
  const int tid = threadIdx.x;
  if (tid == 0) sh->nc = 0;
  __syncthreads();
#pragma unroll 1
  for (int i = tid; i < K; i += kT)
    if (binI[i] == b) clist[atomicAdd(&sh->nc, 1)] = i;
  __syncthreads();
  const int n = sh->nc;
#pragma unroll 1
  for (int a = tid; a < n; a += kT) {
    const int ia = clist[a];
    const double la = lmall[ia];
    int rk = 0;
#pragma unroll 1
    for (int j = 0; j < n; ++j) {
      const int ij = clist[j];
      const double lj = lmall[ij];
      rk += lj > la || (lj == la && ij < ia);
    }
    cord[rk] = ia;
  }
  __syncthreads();
  return n;
}

// warp 0: first j < n with base + sum_{t<=j} u[cord[t]] >= thr (n if none);
// sh->at = that inclusive sum
static __device__ __noinline__ int sel_cut(SelShared* sh, const unsigned long long* um, const int* cord, int n,
                                    unsigned long long base, double thr) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    int res = n;
    unsigned long long at = base;
#pragma unroll 1
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      unsigned long long inc = j < n ? um[cord[j]] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      const unsigned long long cum = base + inc;
      const unsigned hit = __ballot_sync(0xffffffffu, j < n && (double)cum >= thr);
      if (hit) {
        const int f = __ffs(hit) - 1;
        res = j0 + f;
        at = __shfl_sync(0xffffffffu, cum, f);
        break;
      }
      base += __shfl_sync(0xffffffffu, inc, 31);
      at = base;
    }
    if (lane == 0) {
      sh->n = res;
      sh->at = at;
    }
  }
  __syncthreads();
  return sh->n;
}

template <int kT>
struct SelScratch {
  SelShared sel;
  unsigned long long redu[2 * (kT / 32) + 1];
  int redi[(kT / 32) * 4];
  int lo, hi, bcnt[kCandBins + 1], boff[kCandBins + 1];
  unsigned long long pre_m[kCandBins];
  int pre_c[kCandBins];
};

// zero the [2 * NB] mass halves and [NB] counts (callers do it early, off the
// critical path; every thread of the CTA)
template <int kT, int NB>
__device__ __forceinline__ void select_zero_hist(unsigned* hm, int* hc) {
#pragma unroll
  for (int j = 0; j < NB / kT; ++j) {
    hm[threadIdx.x * (NB / kT) + j] = 0u;
    hm[NB + threadIdx.x * (NB / kT) + j] = 0u;
    hc[threadIdx.x * (NB / kT) + j] = 0;
  }
}

// Selection of one q head: lmall[K] log-masses (shared), M = their max.
// Writes stown[i] = 2 exact / 1 approx / 0 dropped for i < K and returns the
// stage-1 / stage-2 counts.  Scratch arrays (shared): um [K] u64, binI [K],
// hm [2 * NB] (zeroed by select_zero_hist), hc [NB] (zeroed), clist [K],
// cord [K].  Every thread of the CTA calls it.
template <int kT, int NB>
__device__ void select_two_stage(const int K, const double M, const double* lmall, const double p1,
                                 const double p2, unsigned long long* um, uint16_t* binI, unsigned* hmh, int* hc,
                                 int* clist, int* cord, uint8_t* stown, SelScratch<kT>* S, int& n1_out,
                                 int& n2_out) {
  static_assert(NB % kT == 0, "bins per thread");
  const int tid = threadIdx.x;
  unsigned* hml = hmh + NB;  // [NB] low 20 bits of the bin masses (hmh: high 19 bits)
  sel_stamp(0);
#pragma unroll 1
    for (int i = tid; i < K; i += kT) {
      const float xf = M == -CUDART_INF ? CUDART_INF_F : (float)(M - lmall[i]);  // >= 0 (+inf: no mass)
      const unsigned long long u = __float2ull_rn(__expf(-xf) * (float)kFix);
      int b = (int)(xf * kBinScale);
      b = b < 0 ? 0 : (b >= NB ? NB - 1 : b);
      um[i] = u;
      binI[i] = (uint16_t)b;
      if (u) {  // native 32-bit shared atomics (a 64-bit add is a CAS loop)
        atomicAdd(&hmh[b], (unsigned)(u >> 20));
        atomicAdd(&hml[b], (unsigned)(u & 0xFFFFFu));
        atomicAdd(&hc[b], 1);  // zero-mass members only ever sit at or past the stage-1 bin
      }
    }
    __syncthreads();
    sel_stamp(1);
    unsigned long long bm[(NB / kT)];
    int bc[(NB / kT)];
    unsigned long long msum = 0;
    int csum = 0;
#pragma unroll
    for (int j = 0; j < (NB / kT); ++j) {
      bm[j] = ((unsigned long long)hmh[tid * (NB / kT) + j] << 20) + hml[tid * (NB / kT) + j];
      bc[j] = hc[tid * (NB / kT) + j];
      msum += bm[j];
      csum += bc[j];
    }
    unsigned long long mbase, total;
    int cbase, ctot;
    scan_pair<kT>(msum, csum, S->redu, S->redi, mbase, cbase, total, ctot);
    sel_stamp(2);
    int cut1 = 0, cbefore1 = 0, n2 = 0;
    if (K > 0) {
      // stage 1 (selection.py:57-58): the bin where the mass crosses p1 * total
      const double thr1 = p1 * (double)total;
      // always found for finite scores; a non-finite query must not index out of range
      const int b1 = min(sel_find_bin<kT, NB>(&S->sel, bm, bc, mbase, cbase, thr1, NB), NB - 1);
      sel_stamp(3);
      const unsigned long long before1 = S->sel.before;
      cbefore1 = S->sel.cbefore;
      // stage 2 (engine.py:191-194) crosses p2 * sub with sub in [before1, before1 + mass(b1)]:
      // its bin lies in [blo, bhi] (or inside b1), so every candidate bin is ranked in ONE pass
      const unsigned long long mb1 = ((unsigned long long)hmh[b1] << 20) + hml[b1];
      if (tid == 0) {
        S->lo = NB;
        S->hi = NB;
      }
      __syncthreads();
      {
        const double tlo = p2 * (double)before1, thi = p2 * (double)(before1 + mb1);
        unsigned long long m = mbase;
        int hlo = -1, hhi = -1;
#pragma unroll
        for (int j = 0; j < (NB / kT); ++j) {
          const int b = tid * (NB / kT) + j;
          if (b < b1 && bm[j]) {
            if (hlo < 0 && (double)(m + bm[j]) >= tlo) hlo = b;
            if (hhi < 0 && (double)(m + bm[j]) >= thi) hhi = b;
          }
          m += bm[j];
        }
        if (hlo >= 0) atomicMin(&S->lo, hlo);
        if (hhi >= 0) atomicMin(&S->hi, hhi);
      }
      __syncthreads();
      const int blo = S->lo;                              // NB: every stage-2 crossing is inside b1
      const int bhi = min(S->hi, b1 - 1);                 // S->hi = NB: up to the bin before b1
      const int nrange = blo <= bhi ? bhi - blo + 1 : 0;  // candidate bins below b1
      const bool wide = nrange > kCandBins;             // rare: fall back to ranking b2 separately
      const int rlo = wide ? NB : blo, rhi = wide ? -1 : bhi;
      {  // exclusive (mass, count) prefix of the candidate range bins
        unsigned long long m = mbase;
        int c = cbase;
#pragma unroll
        for (int j = 0; j < (NB / kT); ++j) {
          const int b = tid * (NB / kT) + j;
          if (b >= blo && b < blo + kCandBins) {
            S->pre_m[b - blo] = m;
            S->pre_c[b - blo] = c;
          }
          m += bm[j];
          c += bc[j];
        }
      }
      // compaction: members of b1 and of [rlo, rhi]; per-bin counts -> segment offsets
      if (tid <= kCandBins) S->bcnt[tid] = 0;
      if (tid == 0) S->sel.nc = 0;
      __syncthreads();
#pragma unroll 1
      for (int i = tid; i < K; i += kT) {
        const int b = binI[i];
        if (b == b1 || (b >= rlo && b <= rhi)) {
          clist[atomicAdd(&S->sel.nc, 1)] = i;
          atomicAdd(&S->bcnt[b == b1 ? kCandBins : b - rlo], 1);
        }
      }
      __syncthreads();
      sel_stamp(4);
      if (tid == 0) {  // segment offsets in rank order: range bins ascending, then b1
        int o = 0;
        for (int j = 0; j <= kCandBins; ++j) {
          const int c = S->bcnt[j];
          S->boff[j] = o;
          o += c;
        }
      }
      __syncthreads();
      const int ncand = S->sel.nc;
#pragma unroll 1
      for (int a = tid; a < ncand; a += kT) {  // exact rank (log-mass desc, id asc) within the bin
        const int ia = clist[a], ba = binI[ia];
        const double la = lmall[ia];
        int rk = 0;
#pragma unroll 1
        for (int j = 0; j < ncand; ++j) {
          const int ij = clist[j];
          if (binI[ij] != ba) continue;
          const double lj = lmall[ij];
          rk += lj > la || (lj == la && ij < ia);
        }
        cord[S->boff[ba == b1 ? kCandBins : ba - rlo] + rk] = ia;
      }
      __syncthreads();
      sel_stamp(5);
      const int o1 = S->boff[kCandBins], n1c = S->bcnt[kCandBins];
      const int j1 = sel_cut(&S->sel, um, cord + o1, n1c, before1, thr1);
      sel_stamp(6);
      cut1 = j1 < n1c ? j1 + 1 : n1c;
      const double thr2 = p2 * (double)S->sel.at;  // retained mass (engine.py:191)
      int b2 = b1, cut2;
      if ((double)before1 >= thr2 && cbefore1 > 0) {  // crossing strictly below bin b1
        if (!wide) {
          // first range bin whose inclusive mass reaches thr2 (it exists: thr2 in [tlo, thi])
          if (tid == 0) {
            int bb = bhi;
            for (int b = blo; b <= bhi; ++b) {
              const unsigned long long mm = ((unsigned long long)hmh[b] << 20) + hml[b];
              if (mm && (double)(S->pre_m[b - blo] + mm) >= thr2) {
                bb = b;
                break;
              }
            }
            S->lo = bb;
          }
          __syncthreads();
          b2 = S->lo;
          const int n2c = S->bcnt[b2 - rlo], o2 = S->boff[b2 - rlo];
          const int j2 = sel_cut(&S->sel, um, cord + o2, n2c, S->pre_m[b2 - blo], thr2);
          cut2 = j2 < n2c ? j2 + 1 : n2c;
          n2 = S->pre_c[b2 - blo] + cut2;
#pragma unroll 1
          for (int j = tid; j < n2c; j += kT) {
            const int i = cord[o2 + j];
            stown[i] = (uint8_t)(j < cut2 ? 2 : 1);
          }
        } else {  // wide range: rank b2 on its own after emitting b1's states
          b2 = min(sel_find_bin<kT, NB>(&S->sel, bm, bc, mbase, cbase, thr2, b1), b1);
          const unsigned long long before2 = S->sel.before;
          const int cbefore2 = S->sel.cbefore;
#pragma unroll 1
          for (int j = tid; j < n1c; j += kT) {
            const int i = cord[o1 + j];
            stown[i] = (uint8_t)(j < cut1 ? 1 : 0);
          }
          __syncthreads();
          const int n2c = sel_rank_bin<kT>(&S->sel, binI, lmall, clist, cord, K, b2);
          const int j2 = sel_cut(&S->sel, um, cord, n2c, before2, thr2);
          cut2 = j2 < n2c ? j2 + 1 : n2c;
          n2 = cbefore2 + cut2;
#pragma unroll 1
          for (int j = tid; j < n2c; j += kT) {
            const int i = cord[j];
            stown[i] = (uint8_t)(j < cut2 ? 2 : 1);
          }
        }
        if (!wide)
#pragma unroll 1
          for (int j = tid; j < n1c; j += kT) {
            const int i = cord[o1 + j];
            stown[i] = (uint8_t)(j < cut1 ? 1 : 0);
          }
      } else {  // crossing inside b1's ranked prefix
        const int j2 = sel_cut(&S->sel, um, cord + o1, cut1, before1, thr2);
        cut2 = j2 < cut1 ? j2 + 1 : cut1;
        n2 = cbefore1 + cut2;
#pragma unroll 1
        for (int j = tid; j < n1c; j += kT) {
          const int i = cord[o1 + j];
          stown[i] = (uint8_t)(j < cut2 ? 2 : (j < cut1 ? 1 : 0));
        }
      }
      // everything outside the boundary bins: bins < b2 exact, [b2, b1) approx, > b1 dropped
#pragma unroll 1
      for (int i = tid; i < K; i += kT) {
        const int b = binI[i];
        if (b != b1 && b != b2) {
          stown[i] = (uint8_t)(b < b2 ? 2 : (b < b1 ? 1 : 0));
        }
      }
      __syncthreads();
    }
  sel_stamp(7);
  (void)ctot;
  n1_out = K > 0 ? cbefore1 + cut1 : 0;
  n2_out = K > 0 ? n2 : 0;
}

// ---------------------------------------------------------------------------
// select_fast: the same two-stage top-p with a short dependent chain (7 CTA
// barriers, no single-thread loops) and little shared-memory traffic per
// warp (on B200 the shared-memory pipe, not latency, bounds a 512-thread
// CTA doing small per-element steps).  Every element keeps its bin, mass and
// sorted position in registers (kEPT slots per thread, K <= kEPT * kT); the
// per-bin (mass, count) histogram is scanned once into exclusive prefixes
// (pm, pc: in place over the histogram), which gives
//   * the stage-1 boundary bin b1 (the unique bin with excl < p1 T <= incl),
//   * the bins that can hold the stage-2 cut without knowing the exact
//     stage-1 cut: p2 * at1 lies in (p2 * before1, p2 * (before1 + mass b1)],
//     so only the bins whose (excl, incl] meets that range (usually one) and
//     b1 itself need an exact order -- every other element's state follows
//     from its bin alone,
//   * each of those candidates' slot in the global sorted order: pc[b] + its
//     rank inside bin b (log-mass desc, id asc), and its exclusive cumulative
//     mass pm[b] + the masses ranked ahead of it.
// Both cuts are then found by the unique candidate whose (excl, incl] holds
// the threshold: no scan over the sorted order.  Cumulative masses are
// 2^-38 fixed-point integers (exact, order-independent sums); a cluster
// whose mass rounds to zero sits past the stage-1 cut unless p1 >= 1 (then
// everything is kept, as the reference's clamp does).
// ---------------------------------------------------------------------------
constexpr double kFixF = 274877906944.0;  // 2^38

#ifdef SEL_PROBE
__device__ long long g_sel_probe[16];
#define SELP(k, S)                                                   \
  if (threadIdx.x == 0) {                                            \
    volatile int _x = *reinterpret_cast<volatile int*>(&(S)->n1);    \
    (void)_x;                                                        \
    g_sel_probe[k] = clock64();                                      \
  }
#else
#define SELP(k, S)
#endif
struct SelFastShared {
  unsigned long long wm[33], wx[33];  // warp totals of the bin scan (mass); their exclusive prefixes, [kW] = total
  int wc[33], wcx[33];                // (count)
  unsigned long long before1, mass1, at1;
  int b1, n1, n2, pad;
  int ba, bb;  // stage-2 candidate bins [ba, bb]: exact below, approx above (up to b1)
  int pad2[2];
};

// zero the histogram (hm: [2 NB] mass halves, hc: [NB + 1] counts) and the
// shared results; every thread, early, followed by a barrier before use
template <int kT, int NB>
__device__ __forceinline__ void select_fast_zero(unsigned* hm, int* hc, SelFastShared* S) {
  for (int j = threadIdx.x; j < 2 * NB; j += kT) hm[j] = 0u;
  for (int j = threadIdx.x; j <= NB; j += kT) hc[j] = 0;
  if (threadIdx.x == 0) {
    S->b1 = NB;
    S->ba = 0;   // (kept when the stage-2 lower threshold is 0)
    S->bb = -1;  // (kept when the upper one is 0: no candidate range)
    S->n1 = 0;
    S->n2 = 0;
    S->at1 = 0ull;
  }
}

// lmall [K] log-masses, M their max.  Scratch (shared): um [K] u64, hm
// [2 NB] u32 (zeroed), hc [NB + 1] int (zeroed), cur [NB] int, clist [K] int.
// Writes stown[i] (2 exact / 1 approx / 0 dropped).  Every thread calls it.
// smallest integer >= t (t a non-negative double): "x >= t" <=> "x >= ceil_u64(t)"
// for an integer x, so every threshold test below is an integer compare (a
// u64 -> fp64 conversion per bin / element costs more than the rest of the
// phase on sm_100)
__device__ __forceinline__ unsigned long long ceil_u64(double t) {
  if (!(t > 0.0)) return 0ull;
  const double c = ceil(t);
  return c >= 1.8e19 ? ~0ull : (unsigned long long)c;
}

template <int kT, int NB, int kEPT>
__device__ void select_fast(const int K, const double M, const double* lmall, const double p1, const double p2,
                            unsigned long long* um, unsigned* hm, int* hc, int* cur, int* clist, uint8_t* stown,
                            SelFastShared* S, int& n1_out, int& n2_out) {
  static_assert(NB % kT == 0, "bins per thread");
  constexpr int kBPT = NB / kT;
  constexpr int kW = kT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned* hmh = hm;       // high bits (u >> 20) per bin
  unsigned* hml = hm + NB;  // low 20 bits per bin
  unsigned long long* pm = reinterpret_cast<unsigned long long*>(hm);  // after the scan: exclusive mass prefix
  int* pc = hc;                                                         // after the scan: exclusive count prefix
  int eb[kEPT];
  unsigned long long eu[kEPT];
  sel_stamp(0);
  SELP(0, S);
  // (1) masses, bins, histogram
#pragma unroll
  for (int s = 0; s < kEPT; ++s) {
    eb[s] = NB;
    eu[s] = 0ull;
    const int i = tid + s * kT;
    if (i < K) {
      const float xf = M == -CUDART_INF ? CUDART_INF_F : (float)(M - lmall[i]);  // >= 0 (+inf: no mass)
      const unsigned long long u = __float2ull_rn(__expf(-xf) * (float)kFixF);
      int b = (int)(xf * kBinScale);
      b = b < 0 ? 0 : (b >= NB ? NB - 1 : b);
      um[i] = u;
      eb[s] = b;
      eu[s] = u;
      if (u) {  // native 32-bit shared atomics (a 64-bit add is a CAS loop)
        atomicAdd(&hmh[b], (unsigned)(u >> 20));
        atomicAdd(&hml[b], (unsigned)(u & 0xFFFFFu));
        atomicAdd(&hc[b], 1);
      }
    }
  }
  __syncthreads();
  SELP(1, S);
  sel_stamp(1);
  // (2) exclusive bin prefixes, total, the stage-1 boundary bin
  static_assert(kBPT == 4 || kBPT == 2, "bins are read and written as vectors (2 or 4 per thread)");
  unsigned long long bm[kBPT], mloc = 0ull;
  int bc[kBPT], cloc = 0;
  {  // one vector per array per thread: contiguous across the warp, no bank conflicts
    unsigned hh[kBPT], ll[kBPT];
    int cc[kBPT];
    if constexpr (kBPT == 4) {
      const uint4 h4 = *reinterpret_cast<const uint4*>(hmh + tid * kBPT);
      const uint4 l4 = *reinterpret_cast<const uint4*>(hml + tid * kBPT);
      const int4 c4 = *reinterpret_cast<const int4*>(hc + tid * kBPT);
      hh[0] = h4.x; hh[1] = h4.y; hh[2] = h4.z; hh[3] = h4.w;
      ll[0] = l4.x; ll[1] = l4.y; ll[2] = l4.z; ll[3] = l4.w;
      cc[0] = c4.x; cc[1] = c4.y; cc[2] = c4.z; cc[3] = c4.w;
    } else {
      const uint2 h2 = *reinterpret_cast<const uint2*>(hmh + tid * kBPT);
      const uint2 l2 = *reinterpret_cast<const uint2*>(hml + tid * kBPT);
      const int2 c2 = *reinterpret_cast<const int2*>(hc + tid * kBPT);
      hh[0] = h2.x; hh[1] = h2.y;
      ll[0] = l2.x; ll[1] = l2.y;
      cc[0] = c2.x; cc[1] = c2.y;
    }
#pragma unroll
    for (int j = 0; j < kBPT; ++j) {
      bm[j] = ((unsigned long long)hh[j] << 20) + ll[j];
      bc[j] = cc[j];
      mloc += bm[j];
      cloc += bc[j];
    }
  }
  sel_sub(0);
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
  sel_sub(1);
  if (lane == 31) {
    S->wm[warp] = mi;
    S->wc[warp] = ci;
  }
  __syncthreads();  // warp totals in place (and every histogram read is done: the prefixes below overwrite it in place)
  SELP(2, S);
  sel_sub(2);
  // every warp scans the kW warp totals itself (one load per lane + shuffles):
  // no single-warp serial prefix and no second barrier
  static_assert(kW <= 32, "warp totals fit one warp");
  unsigned long long wsum = lane < kW ? S->wm[lane] : 0ull;
  int csum = lane < kW ? S->wc[lane] : 0;
#pragma unroll
  for (int o = 1; o < kW; o <<= 1) {
    const unsigned long long tm = __shfl_up_sync(0xffffffffu, wsum, o);
    const int tc = __shfl_up_sync(0xffffffffu, csum, o);
    if (lane >= o) {
      wsum += tm;
      csum += tc;
    }
  }
  const unsigned long long T = __shfl_sync(0xffffffffu, wsum, kW - 1);  // total mass
  const int CT = __shfl_sync(0xffffffffu, csum, kW - 1);                // total count
  const unsigned long long wex = __shfl_sync(0xffffffffu, wsum, warp > 0 ? warp - 1 : 0);
  const int wcex = __shfl_sync(0xffffffffu, csum, warp > 0 ? warp - 1 : 0);
  sel_sub(3);
  SELP(3, S);
  unsigned long long mex = (warp > 0 ? wex : 0ull) + mi - mloc;
  int cex = (warp > 0 ? wcex : 0) + ci - cloc;
  const double thr1 = p1 * (double)T;
  const unsigned long long T1 = ceil_u64(thr1);
  unsigned long long pmv[kBPT];
  int pcv[kBPT];
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    const int b = tid * kBPT + j;
    const unsigned long long inc = mex + bm[j];
    if (bm[j] && mex < T1 && T1 <= inc) {  // the unique crossing bin
      S->b1 = b;
      S->before1 = mex;
      S->mass1 = bm[j];
    }
    pmv[j] = mex;
    pcv[j] = cex;
    mex = inc;
    cex += bc[j];
  }
  reinterpret_cast<ulonglong2*>(pm + tid * kBPT)[0] = make_ulonglong2(pmv[0], pmv[1]);
  if constexpr (kBPT == 4) {
    reinterpret_cast<ulonglong2*>(pm + tid * kBPT)[1] = make_ulonglong2(pmv[2], pmv[3]);
    *reinterpret_cast<int4*>(pc + tid * kBPT) = make_int4(pcv[0], pcv[1], pcv[2], pcv[3]);
    *reinterpret_cast<int4*>(cur + tid * kBPT) = make_int4(0, 0, 0, 0);
  } else {
    *reinterpret_cast<int2*>(pc + tid * kBPT) = make_int2(pcv[0], pcv[1]);
    *reinterpret_cast<int2*>(cur + tid * kBPT) = make_int2(0, 0);
  }
  if (tid == kT - 1) pc[NB] = CT;
  sel_sub(4);
  __syncthreads();
  SELP(4, S);
  sel_stamp(2);
  const int b1 = S->b1;
  if (T == 0ull || b1 >= NB) {  // no mass at all (a non-finite query)
    const uint8_t st = p1 >= 1.0 ? (p2 >= 1.0 ? 2 : 1) : 0;
    for (int i = tid; i < K; i += kT) stown[i] = st;
    n1_out = p1 >= 1.0 ? K : 0;
    n2_out = p1 >= 1.0 && p2 >= 1.0 ? K : 0;
    __syncthreads();
    return;
  }
  // (3) candidates: b1 and the bins whose (excl, incl] meets (tlo, thi]
  const unsigned long long Tlo = ceil_u64(p2 * (double)S->before1), Thi = ceil_u64(p2 * (double)(S->before1 + S->mass1));
  // the prefix is monotone in the bin, so the bins meeting (Tlo, Thi] are one
  // range [ba, bb]: ba holds the Tlo crossing (first inclusive prefix >= Tlo),
  // bb the Thi crossing (last exclusive prefix < Thi).  Found from this
  // thread's bins (still in registers), so the element pass below compares
  // bin indices instead of loading two prefixes per element
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    const unsigned long long ex = pmv[j], in = pmv[j] + bm[j];
    if (ex < Tlo && Tlo <= in) S->ba = tid * kBPT + j;
    if (ex < Thi && Thi <= in) S->bb = tid * kBPT + j;
  }
  __syncthreads();
  const int ba = S->ba, bb = S->bb;
  // every non-candidate's state follows from its bin and is written now;
  // the later passes touch only this thread's candidates (bit s of cmask)
  const uint8_t zst = p1 >= 1.0 ? (p2 >= 1.0 ? 2 : 1) : 0;
  unsigned cmask = 0u;
#pragma unroll
  for (int s = 0; s < kEPT; ++s) {
    const int i = tid + s * kT;
    if (i >= K) continue;
    const int b = eb[s];
    uint8_t st = 0;
    if (!eu[s]) {
      st = zst;
    } else if (b <= b1) {
      if (b == b1 || (b >= ba && b <= bb)) {
        cmask |= 1u << s;
        clist[pc[b] + atomicAdd(&cur[b], 1)] = i;
      } else {
        st = b < ba ? 2 : 1;  // before the candidate range: exact; between it and b1: approx
      }
    }
    if (!((cmask >> s) & 1u)) stown[i] = st;
  }
  __syncthreads();
  SELP(5, S);
  sel_stamp(3);
  // (4) rank inside the bin -> sorted position and exclusive cumulative mass;
  //     the stage-1 crossing element
  int pos[kEPT];
  unsigned long long ex[kEPT];
#pragma unroll
  for (int s = 0; s < kEPT; ++s) {
    pos[s] = 0;
    ex[s] = 0ull;
    if ((cmask >> s) & 1u) {
      const int ia = tid + s * kT, b = eb[s];
      const double la = lmall[ia];
      const int j0 = pc[b], j1 = pc[b + 1];
      int rk = 0;
      unsigned long long pre = 0ull;
#pragma unroll 4
      for (int j = j0; j < j1; ++j) {
        const int ij = clist[j];
        const double lj = lmall[ij];
        const bool ahead = lj > la || (lj == la && ij < ia);
        rk += ahead;
        pre += ahead ? um[ij] : 0ull;
      }
      pos[s] = j0 + rk;
      ex[s] = pm[b] + pre;
      const unsigned long long inc = ex[s] + eu[s];
      if (ex[s] < T1 && T1 <= inc) {
        S->n1 = pos[s] + 1;
        S->at1 = inc;
      }
    }
  }
  __syncthreads();
  SELP(6, S);
  sel_stamp(4);
  // (5) the stage-2 crossing element (p2 of the retained mass, engine.py:191)
  //     and the candidates' states in one pass: along the sorted order the
  //     exclusive cumulative mass of an element with mass > 0 is strictly
  //     increasing, so "position < n2" is "ex < T2" and "position < n1" is
  //     "ex < T1" -- no barrier between finding the cuts and applying them
  //     (the others' states were written in (3))
  const int n1 = p1 >= 1.0 ? K : S->n1;
  const unsigned long long T2 = ceil_u64(p2 * (double)S->at1);
  const bool all2 = p1 >= 1.0 && p2 >= 1.0;
#pragma unroll
  for (int s = 0; s < kEPT; ++s) {
    if ((cmask >> s) & 1u) {
      if (ex[s] < T2 && T2 <= ex[s] + eu[s]) S->n2 = pos[s] + 1;
      stown[tid + s * kT] = all2 || ex[s] < T2 ? 2 : (p1 >= 1.0 || ex[s] < T1 ? 1 : 0);
    }
  }
  __syncthreads();
  SELP(7, S);
  sel_stamp(5);
  sel_stamp(6);
  const int n2 = all2 ? K : S->n2;
  n1_out = n1;
  n2_out = n2;
}
}  // namespace dp
