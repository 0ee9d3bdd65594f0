// Fused per-layer "plan": size-weighted centroid scoring + two-stage top-p +
// approx partial + GQA-union work list in ONE launch, one CL-CTA thread-block
// cluster (CL = 16, or 8 for tiny tables) per (sequence, kv head).
//
// Every cross-CTA hand-off is a PUSH into the consumer's shared memory
// (fire-and-forget st.shared::cluster) followed by one cluster barrier, so no
// stage waits on a remote load; the only HBM traffic is the centroid slice,
// the value means of approximated clusters and the outputs.  Phases:
//
//   P1 score   (engine.py:158-177)  CTA r streams centroid rows [k0, k0 + nloc)
//              through shared memory and scores them for every q head of the
//              group with fp64 tensor-core MMAs (m8n8k4: 8 rows x 8 heads x 4
//              dims; fp32 centroids and queries are exact in fp64), so
//              log-masses agree with the fp64 oracle to ~1e-15.  Scores go to the owner CTA of their
//              head (CTA g owns q head g).                        -> barrier A
//   P2 select  (engine.py:180-213, selection.py:36-65)  owner CTA g:
//              e_k = exp(lm_k - max) as a 2^-48 fixed-point integer (exact,
//              order-independent sums), a mass histogram over 1/32-nat bins
//              finds the bin holding the p1 crossing (then p2 of the retained
//              mass); only the boundary bins are ranked exactly (log-mass
//              desc, cluster id asc == the reference's stable argsort order).
//              States go back to the CTAs owning each cluster slice.  -> B
//   P3 union   every CTA counts its slice's union rows / clusters and folds
//              its approximated clusters (logit = log-mass, value = value
//              mean, engine.py:231-246) into per-head (l, o) partials, pushed
//              to the head owners; slice counts pushed to all.      -> C
//   P4 lists   exclusive offsets from the pushed counts; coalesced packed
//              row entries ((head mask << 24) | physical row); owners sum the
//              approx partials of their head.  No remote access after C.
//
// Cut semantics follow the reference: the first prefix whose cumsum/total
// >= p (searchsorted left + 1, clamped to n); ties -> lower cluster id.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode_internal.h"

namespace cg = cooperative_groups;

namespace dp {

constexpr int kPT = 512;          // threads per CTA
constexpr int kPW = kPT / 32;     // warps per CTA
constexpr int kBins = 2048;       // log-mass bins of width 1/32 nat (span 64 nats)
constexpr float kBinScale = 32.f;
constexpr int kBinsPT = kBins / kPT;  // 4 bins per thread
constexpr double kFix = 549755813888.0;  // 2^39 fixed-point scale of e = exp(lm - max) <= 1
// (mass below 2^-39 of the max rounds to zero: <= 4096 * 2^-39 < 1e-8 of the total)
constexpr int kPlanMaxCap = 4096;
constexpr int kCh = 128;
constexpr int kTileBytes = kCh * 128 * 4;  // one tile: kCh rows x 128 fp32 (4 swizzled column blocks)
constexpr int kMaxPer = 512;      // clusters per CTA slice (cap 4096 / 8)          // centroid rows per shared-memory tile (P1)

// phase timestamps (%globaltimer, ns) of cluster 0: [rank][event]; read with
// dp_debug_plan_timing() -- profiling aid only
__device__ unsigned long long g_plan_ts[16][24];
__device__ __forceinline__ void stamp(int r, int ev) {
  if (blockIdx.x < 16 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_plan_ts[r][ev] = t;
  }
}

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_sync() {
  cl_arrive();
  cl_wait();
}

struct PlanLayout {
  int per;                 // centroid rows per CTA (capacity)
  size_t cs;               // P1: [per][d + 4] fp32 centroid slice | P2 (owners): select arrays | P3 scratch
  size_t um, bin, hm, hc, clist, cord;  // P2 arrays (inside the cs region)
  size_t lmall;            // [cap] fp64 log-masses of my head (owners; pushed by every CTA)
  size_t lml;              // [kG][per] fp64 log-masses of my slice
  size_t stl;              // [kG][per] u8 states of my slice (pushed by the owners)
  size_t aps;              // [CL][d + 4] fp32 approx partials of my head (owners; pushed by every CTA)
  size_t offs;             // [per + 1] int row offsets of my slice
  size_t total;
};

__host__ __device__ inline PlanLayout plan_layout(int CL, int kG, int d, int cap) {
  PlanLayout L;
  L.per = (cap + CL - 1) / CL;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += (bytes + 1023) & ~size_t(1023);  // 1 KB: TMA 128B-swizzle destinations
    return r;
  };
  size_t p2 = 0;  // the P2 arrays overlay the centroid slice (only needed in P1)
  auto take2 = [&](size_t bytes) {
    const size_t r = p2;
    p2 += (bytes + 127) & ~size_t(127);
    return r;
  };
  L.um = take2((size_t)cap * 8);
  L.bin = take2((size_t)cap * 2);
  L.hm = take2((size_t)kBins * 8);
  L.hc = take2((size_t)kBins * 4);
  L.clist = take2((size_t)cap * 4);
  L.cord = take2((size_t)cap * 4);
  const size_t csb = (size_t)2 * kTileBytes;  // two TMA tiles (128B swizzle) to d + 4 floats (conflict-free A loads)
  const size_t redb = (size_t)kPW * kG * (d + 4) * 4;  // P3 cross-warp scratch
  size_t big = csb > p2 ? csb : p2;
  big = big > redb ? big : redb;
  L.cs = take(big);
  L.um += L.cs; L.bin += L.cs; L.hm += L.cs; L.hc += L.cs; L.clist += L.cs; L.cord += L.cs;
  L.lmall = take((size_t)cap * 8);
  L.lml = take((size_t)kG * L.per * 8 > (size_t)8 * (d + 4) * 4 ? (size_t)kG * L.per * 8 : (size_t)8 * (d + 4) * 4);
  L.stl = take((size_t)kG * L.per);
  L.aps = take((size_t)CL * (d + 4) * 4);
  L.offs = take((size_t)(L.per + 1) * 4);
  L.total = o;
  return L;
}

__device__ __forceinline__ bool before(double la, int ia, double lb, int ib) {
  return la > lb || (la == lb && ia < ib);
}

template <typename T>
__device__ __forceinline__ T* remote(cg::cluster_group& c, T* p, int rank) {
  return c.map_shared_rank(p, rank);
}

// block-wide exclusive scan of (mass u64, count int) pairs; totals to mt / ct.
// Callers separate consecutive uses with a barrier (sm/sc are reused).
__device__ __forceinline__ void scan_pair(unsigned long long m, int c, unsigned long long* sm, int* sc,
                                          unsigned long long& mex, int& cex, unsigned long long& mt, int& ct) {
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
  unsigned long long wb = 0, wt = 0;
  int cb = 0, cbt = 0;
#pragma unroll
  for (int w = 0; w < kPW; ++w) {
    const unsigned long long a = sm[w];
    const int b = sc[w];
    if (w < warp) {
      wb += a;
      cb += b;
    }
    wt += a;
    cbt += b;
  }
  mex = wb + mi - m;
  cex = cb + ci - c;
  mt = wt;
  ct = cbt;
}

template <int CL, int kG>
__global__ void __launch_bounds__(kPT, 1)
    plan_kernel(const __grid_constant__ CUtensorMap tmC, dp_cache_view v, const void* __restrict__ q, int qdt, int G,
                double scale, double p1, double p2, double* __restrict__ lm_out, uint8_t* __restrict__ state_out,
                int* __restrict__ counts, WorkLists wl) {
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int bh = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = v.head_dim, cap = v.cluster_cap;
  const PlanLayout L = plan_layout(CL, kG, d, cap);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1 KB-aligned base (TMA 128B-swizzle destinations); the launch adds the slack
  unsigned char* smem = smem_raw + ((1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  float* Cs = reinterpret_cast<float*>(smem + L.cs);
  double* lmall = reinterpret_cast<double*>(smem + L.lmall);
  double* lml = reinterpret_cast<double*>(smem + L.lml);
  uint8_t* stl = reinterpret_cast<uint8_t*>(smem + L.stl);
  float* aps = reinterpret_cast<float*>(smem + L.aps);
  int* offs = reinterpret_cast<int*>(smem + L.offs);

  __shared__ __align__(8) unsigned long long s_tbar[2];  // TMA tile barriers
  __shared__ double s_max[CL][kG];      // pushed slice maxima (owners)
  __shared__ int s_cnt[CL][4];          // pushed slice counts (rows, exact clusters, approx clusters)
  __shared__ double s_Mg[kG];           // pushed head maxima (every CTA)
  __shared__ double s_wm[kPW][kG];
  __shared__ unsigned long long s_redu[kPW];
  __shared__ int s_redi[kPW * 4];
  __shared__ int s_b, s_n, s_nc;
  __shared__ unsigned long long s_before, s_at;
  __shared__ int s_cbefore;
  __shared__ int s_alist[kMaxPer];          // approx clusters of my slice (local id | head mask << 16), P3
  __shared__ int s_na;

  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // PDL: inputs of the previous grid are visible
  cl_arrive_relaxed();  // (S) every CTA of the cluster has started before DSMEM is touched
  stamp(r, 0);

  const int K = __ldg(&v.nclusters[bh]);
  const int per = (K + CL - 1) / CL;
  const int k0 = min(K, r * per);
  const int nloc = max(0, min(per, K - k0));

  // ---------------- P1: score my centroid slice ---------------------------
  // The slice streams through a shared-memory tile of kCh rows padded to
  // d + 4 floats (conflict-free MMA A-fragment loads) with 128-bit loads;
  // the next tile is fetched into registers while this one is multiplied.
  // S[row, head] = sum_k C[row, k] q[head, k] on the fp64 tensor pipe:
  // mma.m8n8k4.f64 with M = 8 centroid rows, N = 8 heads (G <= 8, the rest
  // zero), K = 4 dims; each lane feeds one fp32 centroid element (exact in
  // fp64) per MMA, the query B-fragments stay in registers.
  const int qP = d + 4;  // padded query rows (conflict-free fragment loads)
  float* qs = reinterpret_cast<float*>(smem + L.lml);  // staging for q (lml is written only after)
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&s_tbar[0]);
  const int ntile = (nloc + kCh - 1) / kCh;
  const int ncb = d / 32;  // 128-B column blocks per row
  // TMA: tile t -> buffer t & 1, one 2-D box (32 floats x kCh rows, 128B
  // swizzle) per column block, completing on s_tbar[t & 1]
  auto issue_tile = [&](int t) {
    const unsigned b = bar0 + (unsigned)(t & 1) * 8;
    const unsigned dst = (unsigned)__cvta_generic_to_shared(Cs) + (unsigned)(t & 1) * kTileBytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"((unsigned)(ncb * kCh * 128))
                 : "memory");
    for (int cb = 0; cb < ncb; ++cb)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
              dst + (unsigned)cb * kCh * 128),
          "l"(reinterpret_cast<unsigned long long>(&tmC)), "r"(cb * 32), "r"(bh * cap + k0 + t * kCh), "r"(b)
          : "memory");
  };
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (ntile > 0) issue_tile(0);
    if (ntile > 1) issue_tile(1);
  }
  {
    const int* goffs = v.offs + (size_t)bh * (cap + 1) + k0;
    for (int i = tid; i <= nloc; i += kPT) offs[i] = __ldg(&goffs[i]);
    for (int i = tid; i < 8 * d; i += kPT) {
      const int h = i / d, c = i - h * d;
      qs[h * qP + c] = h < G ? load_elem_f(q, qdt, ((size_t)bh * G + h) * d + c) : 0.f;
    }
    if (tid == 0) {
      s_nc = 0;
      s_na = 0;
    }
  }
  __syncthreads();  // qs, offs, barrier init
  stamp(r, 1);
  double qreg[32];  // lane l: q[head l/4][4 kk + l%4]
#pragma unroll
  for (int kk = 0; kk < 32; ++kk) qreg[kk] = kk * 4 < d ? (double)qs[(lane >> 2) * qP + kk * 4 + (lane & 3)] : 0.0;
  stamp(r, 2);
  cl_wait();  // (S)
  stamp(r, 12);
  double lmax[2] = {-CUDART_INF, -CUDART_INF};  // heads 2(l%4), 2(l%4)+1
  for (int t = 0; t < ntile; ++t) {
    const int row0 = t * kCh;
    {
      const unsigned b = bar0 + (unsigned)(t & 1) * 8;
      unsigned done = 0;
      while (!done)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(b), "r"((unsigned)((t >> 1) & 1))
            : "memory");
    }
    const unsigned char* tileC = reinterpret_cast<const unsigned char*>(Cs) + (size_t)(t & 1) * kTileBytes;
    const int nrb = (min(kCh, nloc - row0) + 7) >> 3;
    for (int rb = warp; rb < nrb; rb += kPW) {
      // row i = rb*8 + lane/4, dim = 4 kk + lane%4: column block kk/8, 16-B chunk
      // kk%8 stored at chunk (kk%8) ^ (i%8) (128B swizzle) -> 32 distinct banks
      const int ia = rb * 8 + (lane >> 2);
      const unsigned char* arow = tileC + (size_t)ia * 128 + (lane & 3) * 4;
      const int sw = ia & 7;
      double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          if ((kk + tt) * 4 < d) {
            const int kq = kk + tt;
            const double a = (double)*reinterpret_cast<const float*>(
                arow + (size_t)(kq >> 3) * kCh * 128 + (((kq & 7) ^ sw) << 4));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[tt][0]), "+d"(c[tt][1])
                         : "d"(a), "d"(qreg[kk + tt]));
          }
        }
      }
      const int row = row0 + rb * 8 + (lane >> 2);
      if (t == 0 && rb == 0) stamp(r, 14);
      if (row < nloc) {
        const double ls = log((double)(offs[row + 1] - offs[row]));
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int h = 2 * (lane & 3) + e;
          if (h < G) {
            const double val = ((c[0][e] + c[1][e]) + (c[2][e] + c[3][e])) * scale + ls;
            lml[h * L.per + row] = val;
            remote(cluster, lmall, h)[k0 + row] = val;
            lmax[e] = fmax(lmax[e], val);
          }
        }
      }
    }
    if (t + 2 < ntile) {  // refill this buffer once every warp is done with it
      __syncthreads();
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue_tile(t + 2);
      }
    }
  }
  stamp(r, 10);
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    double m = lmax[e];
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 8));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 16));
    const int h = 2 * lane + e;
    if (lane < 4 && h < kG) s_wm[warp][h] = m;
  }
  __syncthreads();
  if (tid < G) {
    double mm = -CUDART_INF;
#pragma unroll
    for (int w = 0; w < kPW; ++w) mm = fmax(mm, s_wm[w][tid]);
    remote(cluster, &s_max[0][0], tid)[r * kG + tid] = mm;
  }
  stamp(r, 3);
  cl_sync();  // (A) every score is in its owner's shared memory
  stamp(r, 4);

  // ---------------- P2: two-stage top-p, owner CTA g = r -------------------
  if (r < G) {
    const int g = r;
    const int hq = bh * G + g;
    unsigned long long* um = reinterpret_cast<unsigned long long*>(smem + L.um);
    uint16_t* binI = reinterpret_cast<uint16_t*>(smem + L.bin);
    unsigned long long* hm = reinterpret_cast<unsigned long long*>(smem + L.hm);
    int* hc = reinterpret_cast<int*>(smem + L.hc);
    int* clist = reinterpret_cast<int*>(smem + L.clist);
    int* cord = reinterpret_cast<int*>(smem + L.cord);
    double M = -CUDART_INF;
#pragma unroll
    for (int rr = 0; rr < CL; ++rr) M = fmax(M, s_max[rr][g]);
    unsigned* hmh = reinterpret_cast<unsigned*>(hm);  // [kBins] high parts
    unsigned* hml = hmh + kBins;                         // [kBins] low parts
#pragma unroll
    for (int j = 0; j < kBinsPT; ++j) {
      hmh[tid * kBinsPT + j] = 0u;
      hml[tid * kBinsPT + j] = 0u;
      hc[tid * kBinsPT + j] = 0;
    }
    __syncthreads();
    for (int i = tid; i < K; i += kPT) {
      const float xf = (float)(M - lmall[i]);  // >= 0
      const unsigned long long u = __float2ull_rn(__expf(-xf) * (float)kFix);
      int b = (int)(xf * kBinScale);
      b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
      um[i] = u;
      binI[i] = (uint16_t)b;
      if (u) {  // native 32-bit shared atomics (a 64-bit add is a CAS loop): 19 + 20 bit halves
        atomicAdd(&hmh[b], (unsigned)(u >> 20));
        atomicAdd(&hml[b], (unsigned)(u & 0xFFFFFu));
      }
      atomicAdd(&hc[b], 1);
    }
    __syncthreads();
    // my 4 bins [4 tid, 4 tid + 4): exclusive (mass, count) bases
    unsigned long long bm[kBinsPT];
    int bc[kBinsPT];
    unsigned long long msum = 0;
    int csum = 0;
#pragma unroll
    for (int j = 0; j < kBinsPT; ++j) {
      bm[j] = ((unsigned long long)hmh[tid * kBinsPT + j] << 20) + hml[tid * kBinsPT + j];
      bc[j] = hc[tid * kBinsPT + j];
      msum += bm[j];
      csum += bc[j];
    }
    unsigned long long mbase, total;
    int cbase, ctot;
    if (tid == 0) s_b = kBins;
    scan_pair(msum, csum, s_redu, s_redi, mbase, cbase, total, ctot);
    // first bin (< limit) whose inclusive mass reaches thr; s_before / s_cbefore
    auto find_bin = [&](double thr, int limit) {
      unsigned long long m = mbase;
      int c = cbase, hit = -1;
      unsigned long long hm_ = 0;
      int hc_ = 0;
#pragma unroll
      for (int j = 0; j < kBinsPT; ++j) {
        const int b = tid * kBinsPT + j;
        if (hit < 0 && b < limit && bm[j] && (double)(m + bm[j]) >= thr) {
          hit = b;
          hm_ = m;
          hc_ = c;
        }
        m += bm[j];
        c += bc[j];
      }
      if (hit >= 0) atomicMin(&s_b, hit);
      __syncthreads();
      const int bb = s_b;
      if (hit == bb) {
        s_before = hm_;
        s_cbefore = hc_;
      }
      __syncthreads();
      return bb;
    };
    // members of bin b (any order) -> clist; exact rank by (lm desc, id asc) -> cord
    auto rank_bin = [&](int b) {
      for (int i = tid; i < K; i += kPT)
        if (binI[i] == b) clist[atomicAdd(&s_nc, 1)] = i;
      __syncthreads();
      const int n = s_nc;
      for (int a = tid; a < n; a += kPT) {
        const int ia = clist[a];
        const double la = lmall[ia];
        int rk = 0;
        for (int j = 0; j < n; ++j) {
          const int ij = clist[j];
          rk += before(lmall[ij], ij, la, ia);
        }
        cord[rk] = ia;
      }
      __syncthreads();
      if (tid == 0) s_nc = 0;  // ready for the next bin (read again only after a barrier)
      return n;
    };
    // warp 0: first j < n with base + sum_{t<=j} u[cord[t]] >= thr (n if none);
    // s_at = that inclusive sum
    auto cut_in = [&](int n, unsigned long long base, double thr) {
      if (warp == 0) {
        int res = n;
        unsigned long long at = base;
        for (int j0 = 0; j0 < n; j0 += 32) {
          const int j = j0 + lane;
          const unsigned long long val = j < n ? um[cord[j]] : 0ull;
          unsigned long long inc = val;
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
          s_n = res;
          s_at = at;
        }
      }
      __syncthreads();
      return s_n;
    };
    // cluster i's state byte goes to the CTA owning its slice
    auto push_state = [&](int i, int s) {
      const int rr = i / per;
      remote(cluster, stl, rr)[g * L.per + (i - rr * per)] = (uint8_t)s;
    };

    if (K > 0) {
      // stage 1 (selection.py:57-58): crossing of p1 * total
      const double thr1 = p1 * (double)total;
      const int b1 = find_bin(thr1, kBins);  // always found: total reaches thr1
      const unsigned long long before1 = s_before;
      const int cbefore1 = s_cbefore;
      stamp(r, 11);
      const int n1c = rank_bin(b1);
      const int j1 = cut_in(n1c, before1, thr1);
      const int cut1 = j1 < n1c ? j1 + 1 : n1c;
      stamp(r, 13);
      const unsigned long long sub = s_at;  // retained mass (engine.py:191); j1 < n1c always
      // stage 2 (engine.py:191-194): same order, threshold p2 * sub
      const double thr2 = p2 * (double)sub;
      int b2 = b1, cut2 = 0, n2 = 0;
      if ((double)before1 >= thr2 && cbefore1 > 0) {  // crossing strictly below bin b1
        if (tid == 0) s_b = kBins;
        __syncthreads();
        b2 = find_bin(thr2, b1);
        const unsigned long long before2 = s_before;
        const int cbefore2 = s_cbefore;
        // bin b1's order lives in cord; emit its states before re-ranking
        for (int j = tid; j < n1c; j += kPT) push_state(cord[j], j < cut1 ? 1 : 0);
        __syncthreads();
        const int n2c = rank_bin(b2);
        const int j2 = cut_in(n2c, before2, thr2);
        cut2 = j2 < n2c ? j2 + 1 : n2c;
        for (int j = tid; j < n2c; j += kPT) push_state(cord[j], j < cut2 ? 2 : 1);
        n2 = cbefore2 + cut2;
      } else {
        const int j2 = cut_in(cut1, before1, thr2);
        cut2 = j2 < cut1 ? j2 + 1 : cut1;
        for (int j = tid; j < n1c; j += kPT) push_state(cord[j], j < cut2 ? 2 : (j < cut1 ? 1 : 0));
        n2 = cbefore1 + cut2;
      }
      // everything outside the boundary bins: bins < b2 exact, [b2, b1) approx, > b1 dropped
      for (int i = tid; i < K; i += kPT) {
        const int b = binI[i];
        if (b != b1 && b != b2) push_state(i, b < b2 ? 2 : (b < b1 ? 1 : 0));
      }
      if (tid == 0) {
        counts[2 * hq] = cbefore1 + cut1;
        counts[2 * hq + 1] = n2;
      }
    } else if (tid == 0) {  // no clusters (engine.py:162 raises on the host side): empty plan
      counts[2 * hq] = 0;
      counts[2 * hq + 1] = 0;
    }
    if (tid < CL) remote(cluster, s_Mg, tid)[g] = K > 0 ? M : 0.0;
  }
  stamp(r, 5);
  cl_sync();  // (B) every cluster state and head max is in place
  stamp(r, 6);

  // ---------------- P3: union counts + approx partial of my slice --------
  int e_rows = 0, e_cl = 0, a_cl = 0;
  for (int i = tid; i < nloc; i += kPT) {
    int me = 0, ma = 0;
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      if (g < G) {
        const uint8_t s = stl[g * L.per + i];
        me |= (s == 2) << g;
        ma |= (s == 1) << g;
      }
    }
    if (me) {
      e_rows += offs[i + 1] - offs[i];
      e_cl += 1;
    }
    if (ma) {
      a_cl += 1;
      const int slot = atomicAdd(&s_na, 1);
      if (slot < kMaxPer) s_alist[slot] = i | (ma << 16);
    }
  }
  {  // (rows, exact clusters, approx clusters) of my slice -> every CTA
    const int v0 = warp_sum(e_rows), v1 = warp_sum(e_cl), v2 = warp_sum(a_cl);
    if (lane == 0) {
      s_redi[warp * 4 + 0] = v0;
      s_redi[warp * 4 + 1] = v1;
      s_redi[warp * 4 + 2] = v2;
    }
  }
  __syncthreads();
  stamp(r, 15);
  if (tid < CL) {
    int t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
    for (int w = 0; w < kPW; ++w) {
      t0 += s_redi[w * 4 + 0];
      t1 += s_redi[w * 4 + 1];
      t2 += s_redi[w * 4 + 2];
    }
    int* dst = remote(cluster, &s_cnt[0][0], tid) + r * 4;
    dst[0] = t0;
    dst[1] = t1;
    dst[2] = t2;
  }
  {
    // warp w folds approx clusters w, w + 16, ...: all the Vbar rows it needs
    // are loaded before any is used (one HBM round trip)
    const int na = min(s_na, kMaxPer);
    const float* vbar = v.value_means + ((size_t)bh * cap + k0) * d;
    constexpr int kU = 4;
    float4 acc[kG];
    float lsum[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
      lsum[g] = 0.f;
    }
    for (int a0 = warp; a0 < na; a0 += kU * kPW) {
      float4 vb[kU];
      int ent[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int a = a0 + u * kPW;
        ent[u] = a < na ? s_alist[a] : -1;
        vb[u] = (ent[u] >= 0 && lane * 4 < d)
                    ? __ldg(reinterpret_cast<const float4*>(vbar + (size_t)(ent[u] & 0xFFFF) * d) + lane)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (ent[u] < 0) continue;
        const int i = ent[u] & 0xFFFF, ma = ent[u] >> 16;
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          if ((ma >> g) & 1) {
            const float w = __expf((float)(lml[g * L.per + i] - s_Mg[g]));
            lsum[g] += w;
            acc[g].x += w * vb[u].x; acc[g].y += w * vb[u].y; acc[g].z += w * vb[u].z; acc[g].w += w * vb[u].w;
          }
        }
      }
    }
    float* red = Cs;  // [warps][kG][d + 4] (the centroid slice is dead)
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      float* rw = red + ((size_t)warp * kG + g) * (d + 4);
      if (lane * 4 < d) reinterpret_cast<float4*>(rw + 4)[lane] = acc[g];
      if (lane == 0) rw[0] = lsum[g];
    }
    __syncthreads();
    // sum over warps; push my slice's (l, o) for head g into owner g's slot r
    for (int i = tid; i < G * (d + 4); i += kPT) {
      const int g = i / (d + 4), c = i - g * (d + 4);
      if (c == 1 || c == 2 || c == 3) continue;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kPW; ++w) s += red[((size_t)w * kG + g) * (d + 4) + c];
      remote(cluster, aps, g)[r * (d + 4) + c] = s;
    }
  }
  stamp(r, 7);
  cl_sync();  // (C) slice counts + approx partials published; no remote access after this
  stamp(r, 8);

  // ---------------- P4: work lists -----------------------------------------
  const int sw_rows = v.sink + v.window;
  int row_base = sw_rows, apx_base = 0, tot_r = 0, tot_e = 0, tot_a = 0;
#pragma unroll
  for (int rr = 0; rr < CL; ++rr) {
    if (rr < r) {
      row_base += s_cnt[rr][0];
      apx_base += s_cnt[rr][2];
    }
    tot_r += s_cnt[rr][0];
    tot_e += s_cnt[rr][1];
    tot_a += s_cnt[rr][2];
  }
  if (r < G) {  // owner: the head's approx partial = sum of the CL slice partials
    const int g = r;
    float* ap = wl.apart + ((size_t)bh * G + g) * (4 + d);
    for (int c = tid; c < d + 4; c += kPT) {
      if (c == 1 || c == 2 || c == 3) continue;
      float s = 0.f;
#pragma unroll
      for (int rr = 0; rr < CL; ++rr) s += aps[rr * (d + 4) + c];
      if (c == 0) {
        ap[0] = s > 0.f ? (float)s_Mg[g] : -INFINITY;  // natural-log domain, like the attention partials
        ap[1] = s;
      } else {
        ap[c] = s;
      }
    }
  }
  stamp(r, 16);
  // debug / parity outputs of my slice (kept off the barrier-release paths above)
  if (lm_out)
    for (int i = tid; i < G * nloc; i += kPT) {
      const int g = i / nloc, k = i - g * nloc;
      lm_out[((size_t)bh * G + g) * cap + k0 + k] = lml[g * L.per + k];
    }
  if (state_out)
    for (int i = tid; i < G * nloc; i += kPT) {
      const int g = i / nloc, k = i - g * nloc;
      state_out[((size_t)bh * G + g) * cap + k0 + k] = stl[g * L.per + k];
    }
  stamp(r, 17);
  unsigned* rowidx = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
  int2* apx = wl.approx + (size_t)bh * cap;
  for (int i0 = 0; i0 < nloc; i0 += kPT) {
    const int i = i0 + tid;
    int me = 0, ma = 0, len = 0, st0 = 0;
    if (i < nloc) {
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        if (g < G) {
          const uint8_t s = stl[g * L.per + i];
          me |= (s == 2) << g;
          ma |= (s == 1) << g;
        }
      }
      st0 = offs[i];
      len = me ? offs[i + 1] - st0 : 0;
    }
    unsigned long long ro64, trr64;
    int ao, taa;
    scan_pair((unsigned long long)len, ma != 0 ? 1 : 0, s_redu, s_redi, ro64, ao, trr64, taa);
    const int ro = (int)ro64 + row_base;
    if (i0 == 0) stamp(r, 18);
    if (ma) apx[ao + apx_base] = make_int2(k0 + i, ma);
    // warp-cooperative expansion of the warp's 32 clusters: lanes write consecutive rows
    unsigned todo = __ballot_sync(0xffffffffu, len > 0);
    while (todo) {
      const int t = __ffs(todo) - 1;
      todo &= todo - 1;
      const int tl = __shfl_sync(0xffffffffu, len, t);
      const int to = __shfl_sync(0xffffffffu, ro, t);
      const unsigned tag = (unsigned)__shfl_sync(0xffffffffu, me, t) << 24;
      const int ts = __shfl_sync(0xffffffffu, st0, t);
      for (int x = lane; x < tl; x += 32) rowidx[to + x] = tag | (unsigned)(ts + x);
    }
    row_base += (int)trr64;
    apx_base += taa;
    if (i0 == 0) stamp(r, 19);
    __syncthreads();  // s_redu / s_redi reuse
  }
  if (r == 0) {
    const unsigned tag = (unsigned)((1 << G) - 1) << 24;
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
  stamp(r, 9);
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

int g_plan_cl = 0;  // 0: auto; 8 / 16 forces the cluster size (dp_debug_set(1, .))
// 8-CTA clusters: on B200 at most 7 sixteen-CTA clusters are co-resident
// (GPC shapes), so 8 kv heads of 16-CTA clusters would run in two waves
static int pick_cl(const dp_cache_view& v) {
  if (g_plan_cl == 8 || g_plan_cl == 16) return g_plan_cl;
  return 8;
}

size_t plan_smem_bytes(int d, int cap, int CL, int kG) { return plan_layout(CL, kG, d, cap).total + 1024; }

// 2-D tensor map over all centroid rows [B*H*cap, d] fp32: 32-float x kCh-row
// boxes, 128B swizzle (conflict-free fp64-MMA fragment loads)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static cudaError_t centroid_tmap(const dp_cache_view& v, CUtensorMap* m) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &qr) !=
            cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn)
      return cudaErrorNotSupported;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)v.head_dim, (cuuint64_t)v.batch * v.kv_heads * v.cluster_cap};
  const cuuint64_t strides[1] = {(cuuint64_t)v.head_dim * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)kCh};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(v.centroids), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static int group_bound(int G) { return G <= 1 ? 1 : (G <= 2 ? 2 : (G <= 4 ? 4 : 8)); }

bool plan_supported(const dp_cache_view& v, int G) {
  const int CL = pick_cl(v);
  const int per = (v.cluster_cap + CL - 1) / CL;
  return v.cluster_cap <= kPlanMaxCap && G <= 8 && G <= CL && v.head_dim <= 128 && v.head_dim % 32 == 0 &&
         per <= kMaxPer && v.row_cap < (1 << 24) &&
         plan_smem_bytes(v.head_dim, v.cluster_cap, CL, group_bound(G)) <= 227 * 1024;
}

template <int CL, int kG>
static cudaError_t launch_plan_t(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1,
                                 double p2, double* lm, uint8_t* state, int* counts, const WorkLists& wl,
                                 cudaStream_t st) {
  auto kern = plan_kernel<CL, kG>;
  const size_t smem = plan_smem_bytes(v.head_dim, v.cluster_cap, CL, kG);
  static size_t attr = 0;
  if (attr < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(v.batch * v.kv_heads * CL));
  cfg.blockDim = dim3(kPT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  CUtensorMap tm;
  const cudaError_t e = centroid_tmap(v, &tm);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, kern, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl);
}

cudaError_t launch_plan(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, void* ws, cudaStream_t st) {
  WorkLists wl;
  decode_ws_layout(&v, G, &wl, nullptr, nullptr, reinterpret_cast<char*>(ws));
  wl.stats = stats;
  const int kG = group_bound(G);
  if (pick_cl(v) == 16) {
    switch (kG) {
      case 1: return launch_plan_t<16, 1>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
      case 2: return launch_plan_t<16, 2>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
      case 4: return launch_plan_t<16, 4>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
      default: return launch_plan_t<16, 8>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
    }
  }
  switch (kG) {
    case 1: return launch_plan_t<8, 1>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
    case 2: return launch_plan_t<8, 2>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
    case 4: return launch_plan_t<8, 4>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
    default: return launch_plan_t<8, 8>(v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, st);
  }
}

}  // namespace dp

extern "C" int dp_debug_plan_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_plan_ts, sizeof(dp::g_plan_ts)) == cudaSuccess ? 0 : 2;  // [16][24]
}

// max co-resident clusters of the plan kernel at this geometry (profiling aid)
extern "C" int dp_debug_plan_occupancy(const dp_cache_view* v, int G, int cl) {
  const int kG = dp::group_bound(G);
  const size_t smem = dp::plan_smem_bytes(v->head_dim, v->cluster_cap, cl, kG);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(v->batch * v->kv_heads * cl));
  cfg.blockDim = dim3(dp::kPT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = -1;
  cudaError_t e;
  if (cl == 16) {
    auto k = dp::plan_kernel<16, 4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
  } else {
    auto k = dp::plan_kernel<8, 4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
  }
  return e == cudaSuccess ? n : -(int)e;
}
