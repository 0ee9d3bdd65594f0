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
//   P3 union   every CTA counts its slice's union rows / exact clusters /
//              approximated clusters and pushes the counts to all.  -> C
//   P4 lists   exclusive offsets from the pushed counts; coalesced packed
//              row entries ((head mask << 24) | physical row), the approx
//              cluster list and the log-masses.  No remote access after C.
//              (The approximated clusters' pseudo-rows -- logit = log-mass,
//              value = value mean, engine.py:231-246 -- are folded in by the
//              attention kernel while its first tiles are in flight.)
//
// Cut semantics follow the reference: the first prefix whose cumsum/total
// >= p (searchsorted left + 1, clamped to n); ties -> lower cluster id.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "host_state.h"
#include "select.cuh"
#include "decode_internal.h"

#include "dsmem.cuh"  // cluster barriers, st.async pushes, mbarrier waits

namespace cg = cooperative_groups;

namespace dp {

// kMode (compile time, so the normal plan carries none of it): 0 the plan; 1 score only
// (log-masses out, then exit); 2 states read from state_out (an outside selection), not selected
constexpr int kModePlan = 0, kModeScore = 1, kModeGiven = 2;
constexpr int kPT = 512;          // threads per CTA
constexpr int kPW = kPT / 32;     // warps per CTA
constexpr int kBins = 1024;       // log-mass bins of width 1/32 nat: span 32 nats, past the 27 nats where a 2^-38 mass rounds to 0
constexpr int kPlanMaxCap = 4096;
constexpr int kCh = 128;          // centroid rows per shared-memory tile (P1)
constexpr int kTileBytes = kCh * 128 * 4;  // one tile: kCh rows x 128 fp32 (4 swizzled column blocks)
constexpr int kMaxPer = 1024;     // clusters per CTA slice (cap 4096 / 4)
constexpr int kMaxCL = 16;

// phase timestamps (%globaltimer, ns) of cluster 0: [rank][event]; read with
// dp_debug_plan_timing() -- profiling aid only
__device__ unsigned long long g_plan_ts[16][24];
__device__ unsigned long long g_plan_clk[16][2];
__device__ unsigned long long g_plan_cyc[16][24];
__device__ unsigned long long g_sel_ts2[16][8];  // DP_SEL_REPEAT: the first pass's select stamps
// (compiled in only with -DDP_PROFILE: DP_PROFILE=1 python -m paper_2602_05191_b200.build)
__device__ __forceinline__ void stamp(int r, int ev) {
#ifdef DP_PROFILE
  if (blockIdx.x < 16 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_plan_ts[r][ev] = t;
    g_plan_cyc[r][ev] = clock64();  // SM cycles: phase durations within one CTA
    if (ev == 0 || ev == 9) g_plan_clk[r][ev == 9] = clock64();
  }
#endif
}

struct PlanLayout {
  int per;                 // centroid rows per CTA (capacity)
  size_t cs;               // P1: [per][d + 4] fp32 centroid slice | P2 (owners): select arrays | P3 scratch
  size_t um, bin, hm, hc, clist, cord, stown;  // P2 arrays (inside the cs region; bin = cursors, cord unused)
  size_t lmall;            // [cap] fp64 log-masses of my head (owners; pushed by every CTA)
  size_t lml;              // [per] fp64 log cluster sizes of my slice (sized kG * per)
  size_t qd;               // [8][d + 4] fp64 queries (padded rows)
  size_t stl;              // [kG][per] u8 states of my slice (pushed by the owners)
  size_t offs;             // [per + 1] int row offsets of my slice
  size_t total;
};

__host__ __device__ inline PlanLayout plan_layout(int CL, int kG, int d, int cap) {
  PlanLayout L;
  L.per = ((cap + CL - 1) / CL + 3) & ~3;  // multiple of 4: states travel as packed words
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
  L.bin = take2((size_t)kBins * 4);  // select_fast: per-bin cursors
  L.hm = take2((size_t)kBins * 8);
  L.hc = take2((size_t)(kBins + 1) * 4);
  L.clist = take2((size_t)cap * 4);
  L.cord = 0;
  L.stown = take2((size_t)cap + 4);
  const size_t csb = (size_t)2 * kTileBytes;  // two TMA tiles (128B swizzle) to d + 4 floats (conflict-free A loads)
  const size_t big = csb > p2 ? csb : p2;
  L.cs = take(big);
  L.um += L.cs; L.bin += L.cs; L.hm += L.cs; L.hc += L.cs; L.clist += L.cs; L.stown += L.cs;
  L.lmall = take((size_t)cap * 8);
  L.lml = take((size_t)kG * L.per * 8);
  L.qd = take((size_t)8 * (d + 4) * 8);
  L.stl = take((size_t)kG * L.per);
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


template <int kG, int kMode>
__global__ void __launch_bounds__(kPT, 1)
    plan_kernel(const __grid_constant__ CUtensorMap tmC, dp_cache_view v, const void* __restrict__ q, int qdt, int G,
                double scale, double p1, double p2, double* __restrict__ lm_out, uint8_t* __restrict__ state_out,
                int* __restrict__ counts, WorkLists wl, int CL, int boxr, int dbg, int sld) {
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
  double* lsz = reinterpret_cast<double*>(smem + L.lml);  // [nloc] log cluster sizes of my slice
  double* qd = reinterpret_cast<double*>(smem + L.qd);
  uint8_t* stl = reinterpret_cast<uint8_t*>(smem + L.stl);
  int* offs = reinterpret_cast<int*>(smem + L.offs);

  __shared__ __align__(8) unsigned long long s_tbar[2];  // TMA tile barriers
  // hand-off barriers: A (owner g <- every slice's scores of head g, maxima),
  // B (slice r <- every owner's states of the slice; CTA 0 also the head
  // maxima and late sink/window maxima), C (every CTA <- every slice's counts)
  __shared__ __align__(8) unsigned long long s_mb[3];
  __shared__ double s_max[kMaxCL][kG];  // pushed slice maxima (owners)
  __shared__ double s_swx[kMaxCL][kG];  // pushed sink/window logit maxima (owners)
  __shared__ double s_sw[kPW][kG];
  __shared__ __align__(16) int s_cnt[kMaxCL][4];  // pushed slice counts (rows, exact clusters, approx clusters)
  __shared__ double s_Mg[kG];           // pushed head maxima (every CTA)
  __shared__ double s_wm[kPW][kG];
  __shared__ SelScratch<kPT> s_selx;
  __shared__ SelFastShared s_self;
  unsigned long long* s_redu = s_selx.redu;
  int* s_redi = s_selx.redi;

  // Before griddepcontrol.wait only the cache tables are touched (centroid
  // tiles, offsets): the previous grid in the stream (the last layer's
  // attention) never writes them, and anything that does (dp_append_token,
  // prefill) completed before that grid started.  So the centroid TMA and the
  // offset loads overlap the previous layer's tail; q and every output wait.
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&s_mb[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cl_arrive_relaxed();  // (S) every CTA of the cluster has started (and initialised its barriers) before DSMEM is touched
  stamp(r, 0);

  const int K = __ldg(&v.nclusters[bh]);
  const int per = ((K + CL - 1) / CL + 3) & ~3;
  const int k0 = min(K, r * per);
  const int nloc = max(0, min(per, K - k0));

  // ---------------- P1: score my centroid slice ---------------------------
  // Tiles of kCh centroid rows arrive by TMA (two in flight, 128B swizzle).
  // S[row, head] = sum_k C[row, k] q[head, k] on the fp64 tensor pipe:
  // mma.m8n8k4.f64 with M = 8 centroid rows, N = 8 heads (G <= 8, the rest
  // zero), K = 4 dims; fp32 centroids and queries are exact in fp64.
  const int qP = d + 2;  // padded fp64 query rows: a row is 16 B past a 128-B multiple -> conflict-free 16-B B-fragment loads
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&s_tbar[0]);
  // given states: the log-masses are already written (dp_plan_score) -- no scoring pass
  const int ntile = kMode == kModeGiven || DP_AB(dbg, 8192) ? 0 : (nloc + kCh - 1) / kCh;
  const int ncb = d / 32;  // 128-B column blocks per row
  if (tid == 0) {
    // bytes each hand-off barrier of this CTA receives
    // (given states: no scores travel, only the slice maxima)
    if (r < G) mb_expect(&s_mb[0], (unsigned)((kMode == kModeGiven ? 0 : K * 8) + CL * 16));
    unsigned eb = (unsigned)(G * 4 * ((nloc + 3) / 4));
    if (r == 0) eb += (unsigned)(G * 8 + (CL > G ? (CL - G) * G * 8 : 0));
    mb_expect(&s_mb[1], eb);
    mb_expect(&s_mb[2], (unsigned)(CL * 16));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // TMA: tile t -> buffer t & 1, one 2-D box (32 floats x kCh rows) per column block
#pragma unroll 1
  for (int t = 0; t < 2 && t < ntile; ++t) {
    if (tid == 0) {
      const unsigned b = bar0 + (unsigned)(t & 1) * 8;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Cs) + (unsigned)(t & 1) * kTileBytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"((unsigned)(ncb * boxr * 128))
                   : "memory");
#pragma unroll 1
      for (int cb = 0; cb < ncb; ++cb)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                dst + (unsigned)cb * kCh * 128),
            "l"(reinterpret_cast<unsigned long long>(&tmC)), "r"(cb * 32), "r"(bh * cap + k0 + t * kCh), "r"(b)
            : "memory");
    }
  }
  // the slice's later tiles (only two fit in shared memory) are requested
  // into L2 now: the centroid tables are layer-static, so this also overlaps
  // the previous grid's tail, and the refills after the wait hit L2
  if (tid == 0 && ntile > 2 && !DP_AB(dbg, 32)) {
    const char* cbase = reinterpret_cast<const char*>(v.centroids) + ((size_t)bh * cap + k0) * d * 4;
    const size_t rest = (size_t)(nloc - 2 * kCh) * d * 4;
    for (size_t o = 0; o < rest; o += 65536)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(cbase + (size_t)2 * kCh * d * 4 + o),
                   "r"((unsigned)(rest - o < 65536 ? rest - o : 65536))
                   : "memory");
  }
  {
    const int* goffs = v.offs + (size_t)bh * (cap + 1) + k0;
#pragma unroll 1
    for (int i = tid; i <= nloc; i += kPT) offs[i] = __ldg(&goffs[i]);
    // log cluster sizes of the slice (engine.py:165, the size weight): layer-static, so
    // they are taken here, overlapping the previous grid, not in P1's epilogue
#pragma unroll 1
    for (int i = tid; i < nloc; i += kPT) lsz[i] = log((double)(__ldg(&goffs[i + 1]) - __ldg(&goffs[i])));
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // PDL: inputs of the previous grid are visible
    // let the attention grid become resident on the SMs this launch leaves free
    // (its CTAs wait for our completion before reading anything we write)
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if DP_AB(dbg, 64) {  // timing experiment: the launch + dependency-wait floor
      cl_wait();
      return;
    }
    if (r == 0) {  // sink and window rows open every head's union list (plan-independent)
      const unsigned tag = (unsigned)((1 << G) - 1) << 24;
      unsigned* rw = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
#pragma unroll 1
      for (int t = tid; t < v.sink + v.window; t += kPT)
        rw[t] = tag | (unsigned)(t < v.sink ? t : v.n_tokens - v.window + (t - v.sink));
    }
    // the group's queries -> fp64 rows: one 16-B load per thread (a single
    // round trip; the scalar loop took two dependent ones per thread)
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) {  // unaligned caller buffer: scalar loads
#pragma unroll 1
      for (int i = tid; i < 8 * d; i += kPT) {
        const int h = i / d, c = i - h * d;
        qd[h * qP + c] = h < G ? (double)load_elem_f(q, qdt, ((size_t)bh * G + h) * d + c) : 0.0;
      }
    } else {
      const int es = qdt == DP_F32 ? 4 : 2, per16 = 16 / es, nchunk = 8 * d / per16;
      for (int i = tid; i < nchunk; i += kPT) {
        const int h = (i * per16) / d, c0 = (i * per16) - h * d;
        if (h < G) {
          const uint4 raw = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(q) +
                                                                 (((size_t)bh * G + h) * d + c0) * es));
          const unsigned w[4] = {raw.x, raw.y, raw.z, raw.w};
          if (es == 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) qd[h * qP + c0 + j] = (double)__uint_as_float(w[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              qd[h * qP + c0 + 2 * j] = (double)__uint_as_float(w[j] << 16);
              qd[h * qP + c0 + 2 * j + 1] = (double)__uint_as_float(w[j] & 0xFFFF0000u);
            }
          }
        } else {
          for (int j = 0; j < per16; ++j) qd[h * qP + c0 + j] = 0.0;
        }
      }
    }
  }
  __syncthreads();  // qd, offs, barrier init
  if DP_AB(dbg, 128) {  // timing experiment: + the query load
    cl_wait();
    return;
  }
  stamp(r, 1);
  cl_wait();  // (S)
  stamp(r, 2);
  double lmax[2] = {-CUDART_INF, -CUDART_INF};  // heads 2(l%4), 2(l%4)+1
  // B fragment (m8n8k4 .col): lane holds q[head l/4][dim]; MMA step 4m + u takes dims
  // 16m + 4(l%4) + u, so a lane's A and B operands of four steps are one 16-B
  // (A: 4 fp32) / two 16-B (B: 4 fp64) shared loads
  const double* qrow = qd + (lane >> 2) * qP + 4 * (lane & 3);
  // DSMEM targets of my two heads' scores (owners h = 2(l%4) + e), mapped once
  unsigned lm_cl[2] = {0u, 0u}, mb_cl[2] = {0u, 0u};
#pragma unroll
  for (int e = 0; e < 2; ++e)
    if (2 * (lane & 3) + e < G) {
      lm_cl[e] = cl_map(lmall + k0, 2 * (lane & 3) + e);
      mb_cl[e] = cl_map(&s_mb[0], 2 * (lane & 3) + e);
    }
  if (kMode == kModeGiven) {  // my slice's maxima from the written log-masses (same lane -> head map as below)
#pragma unroll 1
    for (int row = tid >> 2; row < nloc; row += kPT / 4)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = 2 * (lane & 3) + e;
        if (h < G) lmax[e] = fmax(lmax[e], lm_out[((size_t)bh * G + h) * cap + k0 + row]);
      }
  }
#pragma unroll 1
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
    if (t < 2) stamp(r, t == 0 ? 14 : 21);  // tile arrived (profiling builds)
    if (t == 3) stamp(r, 23);
    const unsigned char* tileC = reinterpret_cast<const unsigned char*>(Cs) + (size_t)(t & 1) * kTileBytes;
    const int nrb = (min(kCh, nloc - row0) + 7) >> 3;
#pragma unroll 1
    for (int rb = warp; rb < nrb; rb += kPW) {
      // MMA row l/4 is tile row ia = rb*8 + perm(l/4), perm = 0,4,1,5,2,6,3,7: the two
      // rows of a quarter-warp then differ in bit 2, so their 128B-swizzled 16-B
      // chunks (logical chunk ^ (row % 8)) fall in disjoint bank groups
      const int mr = lane >> 2;
      const int ia = rb * 8 + (((mr & 1) << 2) | (mr >> 1));
      const unsigned char* arow = tileC + (size_t)ia * 128;
      const int sw = ia & 7;
      if (t == 0 && rb == 0) stamp(r, 22);  // (profiling builds) tile 0, warp 0: row block start
      double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        if (m * 16 >= d) break;
        const int lc = 4 * m + (lane & 3);  // logical 16-B chunk of the row: column block lc / 8
        const float4 a4 = *reinterpret_cast<const float4*>(arow + (size_t)(lc >> 3) * kCh * 128 + (((lc & 7) ^ sw) << 4));
        const double2 b01 = *reinterpret_cast<const double2*>(qrow + 16 * m);
        const double2 b23 = *reinterpret_cast<const double2*>(qrow + 16 * m + 2);
        const double av[4] = {(double)a4.x, (double)a4.y, (double)a4.z, (double)a4.w};
        const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[u][0]), "+d"(c[u][1])
                       : "d"(av[u]), "d"(bv[u]));
      }
      if (t == 0 && rb == 0) stamp(r, 13);  // (profiling builds) tile 0, warp 0: MMA loop done
      const int row = row0 + ia;
      if (row < nloc) {
        const double ls = lsz[row];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int h = 2 * (lane & 3) + e;
          if (h < G) {
            double val = ((c[0][e] + c[1][e]) + (c[2][e] + c[3][e])) * scale + ls;
            // a non-finite query must not break the selection's ordering: NaN
            // ranks last (-inf), +inf first (the largest finite double)
            val = val != val ? -CUDART_INF : fmin(val, 1.7976931348623157e308);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                             lm_cl[e] + (unsigned)row * 8u),
                         "l"(__double_as_longlong(val)), "r"(mb_cl[e])
                         : "memory");
            if (lm_out) lm_out[((size_t)bh * G + h) * cap + k0 + row] = val;  // (read by the attention kernel)
            lmax[e] = fmax(lmax[e], val);
          }
        }
      }
    }
    if (t < 2) stamp(r, t == 0 ? 11 : 12);  // tile computed (warp 0)
    if (t + 2 < ntile) {  // refill this buffer once every warp is done with it
      __syncthreads();
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const unsigned b = bar0 + (unsigned)(t & 1) * 8;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(Cs) + (unsigned)(t & 1) * kTileBytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b),
                     "r"((unsigned)(ncb * boxr * 128))
                     : "memory");
#pragma unroll 1
        for (int cb = 0; cb < ncb; ++cb)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                  dst + (unsigned)cb * kCh * 128),
              "l"(reinterpret_cast<unsigned long long>(&tmC)), "r"(cb * 32), "r"(bh * cap + k0 + (t + 2) * kCh), "r"(b)
              : "memory");
      }
    }
  }
  // sink/window logits of my share of those rows (always exact; never scored
  // otherwise): their max joins the attention's reference max (ref_max)
  {
    double swl[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) swl[g] = -CUDART_INF;
    // with idle CTAs in P2 (CL > G) they take these rows after barrier A
    // (sw_late below); otherwise every CTA takes a share here
    const int nsw = CL > G ? 0 : v.sink + v.window, s0 = r * nsw / CL, s1 = (r + 1) * nsw / CL;
#pragma unroll 1
    for (int t = s0 + warp; t < s1; t += kPW) {
      const int row = t < v.sink ? t : v.n_tokens - v.window + (t - v.sink);
      const size_t kb = ((size_t)bh * v.row_cap + row) * d;
      float kx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) kx[j] = lane + 32 * j < d ? load_elem_f(v.keys, v.dtype, kb + lane + 32 * j) : 0.f;
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane + 32 * j < d) acc += (double)kx[j] * qd[g * qP + lane + 32 * j];
        acc = warp_sum(acc) * scale;
        if (g < G && acc == acc) swl[g] = fmax(swl[g], acc);
      }
    }
    if (lane == 0)
#pragma unroll
      for (int g = 0; g < kG; ++g) s_sw[warp][g] = swl[g];
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
  if (tid < G) {  // (independent loads, then a tree: no serial chain of shared loads)
    double mm[kPW], sm[kPW];
#pragma unroll
    for (int w = 0; w < kPW; ++w) {
      mm[w] = s_wm[w][tid];
      sm[w] = s_sw[w][tid];
    }
#pragma unroll
    for (int h = kPW / 2; h > 0; h >>= 1)
#pragma unroll
      for (int w = 0; w < h; ++w) {
        mm[w] = fmax(mm[w], mm[w + h]);
        sm[w] = fmax(sm[w], sm[w + h]);
      }
    push_f64(&s_max[r][tid], tid, mm[0], &s_mb[0]);
    push_f64(&s_swx[r][tid], tid, sm[0], &s_mb[0]);
  }
  if (r < G) {  // owners: zero the histogram now (the tile buffers it overlays are consumed)
    select_fast_zero<kPT, kBins>(reinterpret_cast<unsigned*>(smem + L.hm), reinterpret_cast<int*>(smem + L.hc), &s_self);
  }
  stamp(r, 3);
  if (r < G) {  // (A) every score of my head is in my shared memory
    mb_wait0(&s_mb[0]);
    __syncthreads();  // (the zeroed histogram too)
  }
  stamp(r, 4);
  if (kMode == kModeScore) {  // log-masses written; every push into an owner has landed (A)
    // slots [K, cap) read -inf (a table of several slices has holes there)
#pragma unroll 1
    for (int i = K + r * kPT + tid; i < cap; i += CL * kPT)
#pragma unroll 1
      for (int h = 0; h < G; ++h) lm_out[((size_t)bh * G + h) * cap + i] = -CUDART_INF;
    return;
  }

  // ---------------- P2: two-stage top-p, owner CTA g = r -------------------
  if (r < G) {
    const int g = r;
    const int hq = bh * G + g;
    unsigned long long* um = reinterpret_cast<unsigned long long*>(smem + L.um);
    uint8_t* stown = reinterpret_cast<uint8_t*>(smem + L.stown);  // this head's states, then packed out
    int* cur = reinterpret_cast<int*>(smem + L.bin);
    unsigned* hm = reinterpret_cast<unsigned*>(smem + L.hm);
    int* hc = reinterpret_cast<int*>(smem + L.hc);
    int* clist = reinterpret_cast<int*>(smem + L.clist);
    double M = -CUDART_INF;
    {  // max of the pushed slice maxima (independent loads, then a tree)
      double mm[kMaxCL];
#pragma unroll
      for (int rr = 0; rr < kMaxCL; ++rr) mm[rr] = rr < CL ? s_max[rr][g] : -CUDART_INF;
#pragma unroll
      for (int w = kMaxCL / 2; w > 0; w >>= 1)
#pragma unroll
        for (int rr = 0; rr < w; ++rr) mm[rr] = fmax(mm[rr], mm[rr + w]);
      M = mm[0];
    }
    stamp(r, 20);
    int n1 = 0, n2 = 0;
    if (kMode == kModeGiven) {  // the states come from outside (a global selection): load them
      const uint8_t* sin = state_out + (size_t)hq * sld;  // row stride sld (>= cap)
      for (int i = tid; i < K; i += kPT) stown[i] = sin[i];
      __syncthreads();
    } else if DP_AB(dbg, 2) {  // timing experiment: no selection (nothing but sink/window selected)
      for (int i = tid; i < K; i += kPT) stown[i] = 0;
      __syncthreads();
    } else {
      // register slots per thread sized to the table: 2 up to 1024 clusters (32K contexts), else 8
      if (K <= 2 * kPT)
        select_fast<kPT, kBins, 2>(K, M, lmall, p1, p2, um, hm, hc, cur, clist, stown, &s_self, n1, n2);
      else
        select_fast<kPT, kBins, kPlanMaxCap / kPT>(K, M, lmall, p1, p2, um, hm, hc, cur, clist, stown, &s_self, n1,
                                                   n2);
    }
#ifdef DP_SEL_REPEAT
    // experiment: the same selection again with a warm instruction cache
    if (blockIdx.x < 16 && tid < 8) g_sel_ts2[blockIdx.x][tid] = g_sel_ts[blockIdx.x][tid];
    select_fast_zero<kPT, kBins>(hm, hc, &s_self);
    __syncthreads();
    select_fast<kPT, kBins, kPlanMaxCap / kPT>(K, M, lmall, p1, p2, um, hm, hc, cur, clist, stown, &s_self, n1, n2);
#endif
    if (K > 0) {
      // states travel to the slice owners as packed 4-byte words (slices are 4-aligned)
#pragma unroll 1
      for (int i = 4 * tid; i < K; i += 4 * kPT) {
        unsigned w = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (i + t < K) w |= (unsigned)stown[i + t] << (8 * t);
        const int rr = i / per;
        push_u32(stl + g * L.per + (i - rr * per), rr, w, &s_mb[1]);
      }
    }
    if (tid == 0 && kMode != kModeGiven) {
      counts[2 * hq] = n1;
      counts[2 * hq + 1] = n2;
    }
    if (tid == 0) {
      double SW = -CUDART_INF;
      if (CL <= G)
#pragma unroll 1
        for (int rr = 0; rr < CL; ++rr) SW = fmax(SW, s_swx[rr][g]);
      push_f64(&s_Mg[g], 0, CL > G ? (K > 0 ? M : -CUDART_INF) : ref_max(K > 0 ? M : -CUDART_INF, SW), &s_mb[1]);
    }
  }
  if (CL > G && r >= G) {  // sw_late: the CTAs idle in P2 score the sink/window rows -> CTA 0
    const int nid = CL - G, nsw = v.sink + v.window;
    const int s0 = (r - G) * nsw / nid, s1 = (r - G + 1) * nsw / nid;
    double swl[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) swl[g] = -CUDART_INF;
#pragma unroll 1
    for (int t = s0 + warp; t < s1; t += kPW) {
      const int row = t < v.sink ? t : v.n_tokens - v.window + (t - v.sink);
      const size_t kb = ((size_t)bh * v.row_cap + row) * d;
      float kx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) kx[j] = lane + 32 * j < d ? load_elem_f(v.keys, v.dtype, kb + lane + 32 * j) : 0.f;
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane + 32 * j < d) acc += (double)kx[j] * qd[g * qP + lane + 32 * j];
        acc = warp_sum(acc) * scale;
        if (g < G && acc == acc) swl[g] = fmax(swl[g], acc);
      }
    }
    if (lane == 0)
#pragma unroll
      for (int g = 0; g < kG; ++g) s_sw[warp][g] = swl[g];
    __syncthreads();
    if (tid < G) {
      double sm[kPW];
#pragma unroll
      for (int w = 0; w < kPW; ++w) sm[w] = s_sw[w][tid];
#pragma unroll
      for (int h = kPW / 2; h > 0; h >>= 1)
#pragma unroll
        for (int w = 0; w < h; ++w) sm[w] = fmax(sm[w], sm[w + h]);
      push_f64(&s_swx[r][tid], 0, sm[0], &s_mb[1]);
    }
  }
  stamp(r, 5);
  mb_wait0(&s_mb[1]);  // (B) every cluster state of my slice (CTA 0: and the head maxima) is in place
  stamp(r, 6);
  if DP_AB(dbg, 4) return;  // timing experiment: no work lists

  // ---------------- P3: union rows of my slice ----------------------------
  // Slice-local exclusive offsets (rows; approx | exact << 16 cluster counts)
  // are scanned BEFORE the count exchange, so only the slice bases remain
  // after it.  Scratch: the P1/P2 region (tiles / selection arrays), free now.
  int* s_ro = reinterpret_cast<int*>(smem + L.cs);   // [per] local row offset
  int* s_ao = s_ro + L.per;                          // [per] local approx offset
  int t_rows = 0, t_pk = 0;
#pragma unroll 1
  for (int i0 = 0; i0 < nloc; i0 += kPT) {
    const int i = i0 + tid;
    int me = 0, ma = 0, len = 0;
    if (i < nloc) {
#pragma unroll 1
      for (int g = 0; g < G; ++g) {
        const uint8_t st = stl[g * L.per + i];
        me |= (st == 2) << g;
        ma |= (st == 1) << g;
      }
      len = me ? offs[i + 1] - offs[i] : 0;
    }
    unsigned long long ro64, trr64;
    int pk, tpk;
    scan_pair<kPT>((unsigned long long)len, (ma != 0) | ((me != 0) << 16), s_redu, s_redi, ro64, pk, trr64, tpk);
    if (i < nloc) {
      s_ro[i] = t_rows + (int)ro64;
      s_ao[i] = (t_pk & 0xFFFF) + (pk & 0xFFFF);
    }
    t_rows += (int)trr64;
    t_pk += tpk;
    __syncthreads();  // s_redu / s_redi reuse
  }
  stamp(r, 15);
  if (tid < CL) push_v4(&s_cnt[r][0], tid, t_rows, t_pk >> 16, t_pk & 0xFFFF, 0, &s_mb[2]);
  stamp(r, 7);
  if (!DP_AB(dbg, 16)) mb_wait0(&s_mb[2]);  // (C) every slice's counts are in place; no remote access after this
  stamp(r, 8);

  // ---------------- P4: work lists -----------------------------------------
  const int sw_rows = v.sink + v.window;
  int row_base = sw_rows, apx_base = 0, tot_r = 0, tot_e = 0, tot_a = 0;
#pragma unroll
  for (int rr = 0; rr < kMaxCL; ++rr) {
    if (rr >= CL) break;
    const int c0 = s_cnt[rr][0], c1 = s_cnt[rr][1], c2 = s_cnt[rr][2];
    if (rr < r) {
      row_base += c0;
      apx_base += c2;
    }
    tot_r += c0;
    tot_e += c1;
    tot_a += c2;
  }
  stamp(r, 16);
  if (state_out && kMode != kModeGiven)  // debug states of my slice
#pragma unroll 1
    for (int i = tid; i < G * nloc; i += kPT) {
      const int g = i / nloc, k = i - g * nloc;
      state_out[((size_t)bh * G + g) * cap + k0 + k] = stl[g * L.per + k];
    }
  stamp(r, 17);
  unsigned* rowidx = reinterpret_cast<unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap;
  int2* apx = wl.approx + (size_t)bh * cap;
#pragma unroll 1
  for (int i0 = 0; i0 < nloc; i0 += kPT) {
    // lane l of warp w takes cluster i0 + l * kPW + w: a slice's clusters
    // spread over all 16 warps (a small slice would otherwise leave most
    // warps idle while 4 of them expand every row)
    const int i = i0 + lane * kPW + warp;
    int me = 0, ma = 0, len = 0, st0 = 0, ro = 0;
    if (i < nloc) {
#pragma unroll 1
      for (int g = 0; g < G; ++g) {
        const uint8_t st = stl[g * L.per + i];
        me |= (st == 2) << g;
        ma |= (st == 1) << g;
      }
      st0 = offs[i];
      len = me ? offs[i + 1] - st0 : 0;
      ro = row_base + s_ro[i];
      if (ma) apx[apx_base + s_ao[i]] = make_int2(k0 + i, ma);
    }
    // warp-cooperative expansion of the warp's 32 clusters: lanes write consecutive rows
    unsigned todo = __ballot_sync(0xffffffffu, len > 0 && !DP_AB(dbg, 8));
#pragma unroll 1
    while (todo) {
      const int t = __ffs(todo) - 1;
      todo &= todo - 1;
      const int tl = __shfl_sync(0xffffffffu, len, t);
      const int to = __shfl_sync(0xffffffffu, ro, t);
      const unsigned tag = (unsigned)__shfl_sync(0xffffffffu, me, t) << 24;
      const int ts = __shfl_sync(0xffffffffu, st0, t);
#pragma unroll 1
      for (int x = lane; x < tl; x += 32) rowidx[to + x] = tag | (unsigned)(ts + x);
    }
  }
  stamp(r, 19);
  if (r == 0) {
    if (tid < G)  // reference max of the attention accumulators: the head's top log-mass (log2 units)
    {
      double Mref = s_Mg[tid];
      if (CL > G) {  // sink/window maxima pushed by the CTAs idle in P2
        double SW = -CUDART_INF;
#pragma unroll 1
        for (int rr = G; rr < CL; ++rr) SW = fmax(SW, s_swx[rr][tid]);
        Mref = ref_max(Mref, SW);
      }
      wl.refm[(size_t)bh * G + tid] = (float)(Mref * 1.4426950408889634);
    }
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
}

int g_plan_cl = 0;  // 0: auto; 2..16 forces the cluster size (dp_debug_set(1, .))
int g_plan_dbg = 0;  // timing experiments (dp_debug_set(10, .)): bit 1 skips the selection, bit 2 the work lists
size_t plan_smem_bytes(int d, int cap, int CL, int kG) { return plan_layout(CL, kG, d, cap).total + 1024; }

// 2-D tensor map over all centroid rows [B*H*cap, d] fp32: 32-float x kCh-row
// boxes, 128B swizzle (conflict-free fp64-MMA fragment loads)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static cudaError_t centroid_tmap_encode(const dp_cache_view& v, CUtensorMap* m);
// a few recent maps, keyed by (centroid pointer, rows, d): encoding costs host
// microseconds on every layer of every step otherwise
cudaError_t centroid_tmap(const dp_cache_view& v, CUtensorMap* m) {
  struct Entry {
    const void* ptr;
    long long rows;
    int d;
    CUtensorMap map;
  };
  static Entry cache[64];
  static int next = 0;
  std::lock_guard<std::recursive_mutex> lock(host_mutex());
  const long long rows = (long long)v.batch * v.kv_heads * v.cluster_cap;
  for (const Entry& e : cache)
    if (e.ptr == v.centroids && e.rows == rows && e.d == v.head_dim) {
      *m = e.map;
      return cudaSuccess;
    }
  const cudaError_t err = centroid_tmap_encode(v, m);
  if (err == cudaSuccess) {
    cache[next] = Entry{v.centroids, rows, v.head_dim, *m};
    next = (next + 1) % 64;
  }
  return err;
}
static cudaError_t centroid_tmap_encode(const dp_cache_view& v, CUtensorMap* m) {
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
  const cuuint64_t rows = (cuuint64_t)v.batch * v.kv_heads * v.cluster_cap;
  const cuuint32_t box[2] = {32, (cuuint32_t)(rows < (cuuint64_t)kCh ? rows : kCh)};  // a box may not exceed the tensor
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(v.centroids), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static int group_bound(int G) { return G <= 1 ? 1 : (G <= 2 ? 2 : (G <= 4 ? 4 : 8)); }

template <int kG>
static void* plan_fn(int mode) {
  return mode == kModeScore ? reinterpret_cast<void*>(plan_kernel<kG, kModeScore>)
         : mode == kModeGiven ? reinterpret_cast<void*>(plan_kernel<kG, kModeGiven>)
                              : reinterpret_cast<void*>(plan_kernel<kG, kModePlan>);
}
static void* plan_fn_for(int kG, int mode = kModePlan) {
  return kG == 1 ? plan_fn<1>(mode) : kG == 2 ? plan_fn<2>(mode) : kG == 4 ? plan_fn<4>(mode) : plan_fn<8>(mode);
}

// the kernel's dynamic shared-memory limit only ever grows (the occupancy
// queries below and the launches share it; lowering it for a query would
// make a later, larger launch fail)
static void ensure_smem_attr(int kG, size_t smem) {
  for (int mode = 0; mode < 3; ++mode) ensure_smem(plan_fn_for(kG, mode), smem, true);
}

// co-resident clusters of size cl at this shared-memory footprint
static int max_active_clusters(int kG, int cl, size_t smem) {
  static int cache[kMaxDevices][9][17] = {};
  static size_t cache_smem[kMaxDevices][9][17] = {};
  const int dev = current_device();
  std::lock_guard<std::recursive_mutex> lock(host_mutex());
  if (cache_smem[dev][kG][cl] == smem) return cache[dev][kG][cl];
  void* fn = plan_fn_for(kG);
  ensure_smem_attr(kG, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cl);
  cfg.blockDim = dim3(kPT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[dev][kG][cl] = n;
  cache_smem[dev][kG][cl] = smem;
  return n;
}

static bool cl_fits(const dp_cache_view& v, int G, int cl) {
  const int per = (v.cluster_cap + cl - 1) / cl;
  return G <= cl && per <= kMaxPer && plan_smem_bytes(v.head_dim, v.cluster_cap, cl, group_bound(G)) <= 227 * 1024;
}

// Cluster size: the widest (<= 16) for which every (sequence, kv head) cluster
// is co-resident in one wave -- more CTAs per head shorten the per-CTA slice;
// a second wave would double the latency.  (B200: 7 sixteen-CTA clusters fit,
// so 8 kv heads use 12-14.)  Batches with more heads than one wave holds at
// any size use 8.
static int pick_cl(const dp_cache_view& v, int G) {
  if (g_plan_cl >= 2 && g_plan_cl <= kMaxCL && cl_fits(v, G, g_plan_cl)) return g_plan_cl;
  const int units = v.batch * v.kv_heads;
  const int kG = group_bound(G);
  // 8 when every cluster fits in one wave: wider clusters shorten the slices
  // but leave fewer SMs for the attention CTAs that become resident during
  // the plan (measured: 8 vs 10 at 32K 25.6 vs 25.8 us per plan + attend; at
  // 128K: 10 is 0.6 us per plan + attend faster, tools/plan_ab.py r2o); wider
  // only when the narrowest does not fit the table
  if (v.cluster_cap > 2048 && cl_fits(v, G, 10) &&
      max_active_clusters(kG, 10, plan_smem_bytes(v.head_dim, v.cluster_cap, 10, kG)) >= units)
    return 10;
  for (int cl = 8; cl <= kMaxCL; ++cl)
    if (cl_fits(v, G, cl) &&
        max_active_clusters(kG, cl, plan_smem_bytes(v.head_dim, v.cluster_cap, cl, kG)) >= units)
      return cl;
  // more heads than one wave holds: the phases are latency-bound, so a CTA's
  // time grows slowly with its slice -- the narrowest cluster costs the
  // fewest SM-microseconds per head
  for (int cl = max(4, G); cl < 8; ++cl)
    if (cl_fits(v, G, cl)) return cl;
  return 8;
}

bool plan_supported(const dp_cache_view& v, int G) {
  return v.cluster_cap <= kPlanMaxCap && G <= 8 && v.head_dim <= 128 && v.head_dim % 32 == 0 &&
         v.row_cap < (1 << 24) && cl_fits(v, G, 8);
}

template <int kG>
static cudaError_t launch_plan_mode(const cudaLaunchConfig_t& cfg, int mode, const CUtensorMap& tm,
                                    const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1,
                                    double p2, double* lm, uint8_t* state, int* counts, WorkLists wl, int CL, int boxr,
                                    int sld) {
  if (mode == kModeScore)
    return cudaLaunchKernelEx(&cfg, plan_kernel<kG, kModeScore>, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl,
                              CL, boxr, g_plan_dbg, sld);
  if (mode == kModeGiven)
    return cudaLaunchKernelEx(&cfg, plan_kernel<kG, kModeGiven>, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl,
                              CL, boxr, g_plan_dbg, sld);
  return cudaLaunchKernelEx(&cfg, plan_kernel<kG, kModePlan>, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, CL,
                            boxr, g_plan_dbg, sld);
}

cudaError_t launch_plan(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, void* ws, cudaStream_t st, int mode,
                        int state_ld) {
  WorkLists wl;
  decode_ws_layout(&v, G, &wl, nullptr, nullptr, reinterpret_cast<char*>(ws));
  wl.stats = stats;
  if (!lm) return cudaErrorInvalidValue;  // the attention kernel reads the approx clusters' log-masses
  const int kG = group_bound(G);
  const int CL = pick_cl(v, G);
  const size_t smem = plan_smem_bytes(v.head_dim, v.cluster_cap, CL, kG);
  ensure_smem_attr(kG, smem);
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
  const long long rows = (long long)v.batch * v.kv_heads * v.cluster_cap;
  const int boxr = rows < kCh ? (int)rows : kCh;  // rows per TMA box (the tile is never fuller than that)
  const int sld = state_ld > 0 ? state_ld : v.cluster_cap;
  switch (kG) {
    case 1: return launch_plan_mode<1>(cfg, mode, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, CL, boxr, sld);
    case 2: return launch_plan_mode<2>(cfg, mode, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, CL, boxr, sld);
    case 4: return launch_plan_mode<4>(cfg, mode, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, CL, boxr, sld);
    default: return launch_plan_mode<8>(cfg, mode, tm, v, q, qdt, G, scale, p1, p2, lm, state, counts, wl, CL, boxr, sld);
  }
}

int plan_cluster_size(const dp_cache_view& v, int G) { return pick_cl(v, G); }

}  // namespace dp

extern "C" int dp_debug_plan_clock(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_plan_clk, sizeof(dp::g_plan_clk)) == cudaSuccess ? 0 : 2;  // [16][2]
}
extern "C" int dp_debug_plan_cycles(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_plan_cyc, sizeof(dp::g_plan_cyc)) == cudaSuccess ? 0 : 2;  // [16][24]
}
extern "C" int dp_debug_plan_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_plan_ts, sizeof(dp::g_plan_ts)) == cudaSuccess ? 0 : 2;  // [16][24]
}

// max co-resident clusters of the plan kernel at this geometry (profiling aid)
namespace dp {
int plan_occupancy(const dp_cache_view& v, int G, int cl) {
  const int kG = group_bound(G);
  return max_active_clusters(kG, cl, plan_smem_bytes(v.head_dim, v.cluster_cap, cl, kG));
}
}  // namespace dp
extern "C" int dp_debug_plan_occupancy(const dp_cache_view* v, int G, int cl) {
  if (cl == 0) return dp::plan_cluster_size(*v, G);  // the size launch_plan picks
  return dp::plan_occupancy(*v, G, cl);
}
extern "C" int dp_debug_sel_sub(unsigned long long* out) {  // [16][8] stamps inside a select phase
  return cudaMemcpyFromSymbol(out, dp::g_sel_sub, sizeof(dp::g_sel_sub)) == cudaSuccess ? 0 : 2;
}
extern "C" int dp_debug_sel_cycles2(unsigned long long* out) {  // [16][8] first pass (DP_SEL_REPEAT builds)
  return cudaMemcpyFromSymbol(out, dp::g_sel_ts2, sizeof(dp::g_sel_ts2)) == cudaSuccess ? 0 : 2;
}
extern "C" int dp_debug_sel_cycles(unsigned long long* out) {  // [16][8] select phase cycles (plan.cu's copy)
  return cudaMemcpyFromSymbol(out, dp::g_sel_ts, sizeof(dp::g_sel_ts)) == cudaSuccess ? 0 : 2;
}
