// One-launch Double-P decode step: score + two-stage top-p + mixed
// exact/approximate attention + LSE merge for every (sequence, kv head) in a
// SINGLE kernel, one CL-CTA thread-block cluster per (sequence, kv head).
// This is the batch-1 latency path (engine.py:267-278 decode_step for a whole
// layer): it is used whenever all B*H clusters are co-resident in one wave;
// larger batches take plan_kernel + attn_tc_kernel (plan.cu, attn_tc.cu).
//
// CTA r of a head's cluster owns the cluster slice [k0, k0 + nloc) of the
// head's table -- which is a set of CONTIGUOUS row runs in the
// cluster-contiguous layout -- and, for r == CL-1, the sink and window rows.
//
//   prologue   (before griddepcontrol.wait: overlaps the previous layer)
//              TMA of the slice's first centroid tiles, the slice offsets
//   P1 score   (engine.py:158-177)  fp64 tensor-core MMAs over fp32
//              centroids; log-masses pushed to the owner CTA of each q head
//              (CTA g owns q head g) and written to lm_out; slice maxima to
//              every CTA                                             -> A
//   prefetch   every CTA issues L2 bulk prefetches of its slice's clusters
//              within tau nats of the head maximum (the likely exact set),
//              so HBM streams while the owners select
//   P2 select  (engine.py:180-213, selection.py:36-65) owner g: select.cuh;
//              states pushed back to the slice owners            -> B
//   lists      each CTA compacts its slice's exact clusters into row runs
//              (mask of the q heads that keep them exact) and its approx
//              clusters into a pseudo-row list -- no global row list
//   attend     (engine.py:216-252) warp-specialised split-KV flash decode over
//              the CTA's runs: 4 producer warps gather rows with 16-B cp.async
//              into a 3-stage swizzled ring, 8 consumer warps run S = K Q^T and
//              O^T += V^T P on mma.sync (bf16 in, fp32 accumulate), an online
//              softmax per warp, approximated clusters folded in as pseudo-rows
//              (logit = log-mass, value = value mean)
//   merge      each CTA's per-head partial (m, l, o) is pushed into the head
//              owner's shared memory                              -> C
//              owner g combines the CL partials: out = o / l, lse.
// Merges use each partial's own maximum, so no reference maximum is needed
// and no logit can overflow the accumulators.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode_internal.h"
#include "host_state.h"
#include "select.cuh"
#include "tc_common.cuh"

namespace cg = cooperative_groups;

namespace dp {

constexpr int kST = 384;                 // threads: 8 consumer warps + 4 producer warps
constexpr int kSW = kST / 32;
constexpr int kCW = 8;                   // consumer (MMA) warps
constexpr int kCons = kCW * 32;
constexpr int kSBins = 1920;             // 1/32-nat selection bins (5 per thread, span 60 nats)
constexpr int kRows = 128;               // attention tile rows (16 per consumer warp)
constexpr int kNStage = 3;
constexpr int kKVTile = kRows * 256;     // one K (or V) tile: two 64-column planes of 128 rows x 128 B (TMA 128B swizzle)
constexpr int kTileGroups = kRows / 8;   // 8-row TMA groups per tile
constexpr int kLRuns = 64;               // clipped runs the producer stages at a time
constexpr int kStageBytes = 2 * kKVTile;
constexpr size_t kRingBytes = (size_t)kNStage * kStageBytes;  // 192 KB
constexpr int kCCh = 128;                // centroid rows per TMA tile
constexpr int kCTile = kCCh * 128 * 4;   // 64 KB
constexpr int kStepMaxPer = 512;         // clusters per CTA slice
constexpr int kStepMaxCL = 16;
constexpr int kStepMaxCap = 4096;
constexpr int kStepMaxSmem = 227 * 1024;

float g_step_tau = 0.f;  // prefetch margin (nats below the head maximum); <= 0 disables (dp_debug_set key 4, x0.1)
int g_step_cl = 0;       // 0: auto; forces the cluster size (dp_debug_set key 5)
int g_step_off = 1;      // 1: never use the one-launch step (dp_debug_set key 6, 0 = allow); default off: slower than plan + attend
int g_step_dbg = 0;      // bit 0: skip the attention math; bit 1: skip the K/V loads (dp_debug_set key 7)

__device__ unsigned long long g_step_ts[16][16];
__device__ __forceinline__ void sstamp(int r, int ev) {
#ifdef DP_PROFILE
  if (blockIdx.x < 16 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_step_ts[r][ev] = t;
  }
#endif
}

__device__ __forceinline__ void sc_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void sc_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void sc_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void sc_sync() {
  sc_arrive();
  sc_wait();
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kCons) : "memory"); }
// one 64-column x 8-row box of a [rows, 128] bf16 tensor -> shared (128B swizzle), completing on bar
__device__ __forceinline__ void tma_box(unsigned dst, const CUtensorMap* map, int c0, int row, unsigned bar,
                                        unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(row), "r"(bar), "l"(pol)
      : "memory");
}


struct StepLayout {
  int per;  // slice capacity (cap / CL rounded up to 4)
  // plan phases (inside the ring region; dead once the ring fills)
  size_t cs, um, bin, hm, hc, clist, cord, stown, p2_end;
  size_t lmall, qd, lml, stl, offs, plan_end;
  // persistent
  size_t runs, lruns, apx, rmask, pbuf, pslot, total;
};

__host__ __device__ inline StepLayout step_layout(int CL, int cap) {
  constexpr int kG = kMaxGroup;
  StepLayout L;
  L.per = ((cap + CL - 1) / CL + 3) & ~3;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t al) {
    o = (o + al - 1) & ~(al - 1);
    const size_t r = o;
    o += bytes;
    return r;
  };
  L.cs = take(2 * (size_t)kCTile, 1024);  // two TMA tiles (128B swizzle: 1 KB aligned)
  size_t p = L.cs;  // the owners' selection arrays overlay the tiles (P1 is done with them)
  auto take2 = [&](size_t bytes) {
    const size_t r = p;
    p += (bytes + 127) & ~size_t(127);
    return r;
  };
  L.um = take2((size_t)cap * 8);
  L.bin = take2((size_t)cap * 2);
  L.hm = take2((size_t)kSBins * 8);
  L.hc = take2((size_t)kSBins * 4);
  L.clist = take2((size_t)cap * 4);
  L.cord = take2((size_t)cap * 4);
  L.stown = take2((size_t)cap + 4);
  L.p2_end = p;
  L.lmall = take((size_t)cap * 8, 128);
  L.qd = take((size_t)8 * (128 + 4) * 8, 128);
  L.lml = take((size_t)kG * L.per * 4, 128);
  L.stl = take((size_t)kG * L.per, 128);
  L.offs = take((size_t)(L.per + 1) * 4, 128);
  L.plan_end = o;
  o = kRingBytes;
  L.runs = take((size_t)(L.per + 2) * 8, 128);
  L.lruns = take((size_t)kLRuns * 8, 128);
  L.apx = take((size_t)L.per * 8, 128);
  L.rmask = take((size_t)kNStage * kRows * 4, 128);
  L.pbuf = take((size_t)kCW * kRows * 4, 128);
  L.pslot = take((size_t)CL * (128 + 4) * 4, 128);
  L.total = o;
  return L;
}

template <int kG>
__global__ void __launch_bounds__(kST, 1)
    step_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmK8,
                const __grid_constant__ CUtensorMap tmK16, const __grid_constant__ CUtensorMap tmK32,
                const __grid_constant__ CUtensorMap tmV8, const __grid_constant__ CUtensorMap tmV16,
                const __grid_constant__ CUtensorMap tmV32, dp_cache_view v, const void* __restrict__ q, int qdt, int G,
                double scale, double p1, double p2, double* __restrict__ lm_out, uint8_t* __restrict__ state_out,
                int* __restrict__ counts, int* __restrict__ stats, float* __restrict__ out, float* __restrict__ lse,
                int CL, int boxr, float tau, int dbg) {
  constexpr int d = 128;
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int bh = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cap = v.cluster_cap;
  const StepLayout L = step_layout(CL, cap);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  float* Cs = reinterpret_cast<float*>(smem + L.cs);
  double* lmall = reinterpret_cast<double*>(smem + L.lmall);
  double* qd = reinterpret_cast<double*>(smem + L.qd);
  float* lml = reinterpret_cast<float*>(smem + L.lml);
  uint8_t* stl = reinterpret_cast<uint8_t*>(smem + L.stl);
  int* offs = reinterpret_cast<int*>(smem + L.offs);
  int2* runs = reinterpret_cast<int2*>(smem + L.runs);
  int2* lruns = reinterpret_cast<int2*>(smem + L.lruns);
  int2* apx = reinterpret_cast<int2*>(smem + L.apx);
  int* rmask = reinterpret_cast<int*>(smem + L.rmask);
  float* Pbuf = reinterpret_cast<float*>(smem + L.pbuf);
  float* pslot = reinterpret_cast<float*>(smem + L.pslot);  // [CL][4 + d]: (m log2, l, -, -, o[d]) of my head
  unsigned char* ring = smem;

  __shared__ __align__(8) unsigned long long s_tbar[2], full_bar[kNStage], empty_bar[kNStage];
  __shared__ double s_max[kStepMaxCL][kG];  // slice maxima of every CTA (pushed)
  __shared__ double s_wmd[kSW][kG];
  __shared__ SelScratch<kST> s_sel;
  __shared__ float s_wm[kCW][8], s_wl[kCW][8];
  __shared__ int s_cnt[kStepMaxCL][4];  // (rows, approx clusters, exact clusters) per CTA (CTA 0)
  __shared__ int2 s_gc[kStepMaxCL];  // (runs, 8-row groups) of every CTA's list (pushed)
  __shared__ int s_napx;

  sc_arrive_relaxed();  // (S) every CTA of the cluster has started before DSMEM is touched
  sstamp(r, 0);
  const int K = __ldg(&v.nclusters[bh]);
  const int perk = ((K + CL - 1) / CL + 3) & ~3;  // balanced slices of the live table
  const int k0 = min(K, r * perk);
  const int nloc = max(0, min(perk, K - k0));
  const int qP = d + 4;
  const unsigned tb0 = smem_u32(&s_tbar[0]);
  const int ntile = (nloc + kCCh - 1) / kCCh;
  if (tid == 0) {
    mbar_init(tb0, 1);
    mbar_init(tb0 + 8, 1);
    for (int s = 0; s < kNStage; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);  // the producer's arrive.expect_tx; TMA bytes complete it
      mbar_init(smem_u32(&empty_bar[s]), kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  auto issue_tile = [&](int t) {  // centroid rows [k0 + t*kCCh, +kCCh) -> buffer t & 1
    const unsigned b = tb0 + (unsigned)(t & 1) * 8;
    const unsigned dst = smem_u32(Cs) + (unsigned)(t & 1) * kCTile;
    mbar_expect_tx(b, (unsigned)(4 * boxr * 128));
#pragma unroll 1
    for (int cb = 0; cb < 4; ++cb)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];\n" ::"r"(dst + (unsigned)cb * kCCh * 128),
          "l"(reinterpret_cast<unsigned long long>(&tmC)), "r"(cb * 32), "r"(bh * cap + k0 + t * kCCh), "r"(b)
          : "memory");
  };
  if (tid == 0)
    for (int t = 0; t < 2 && t < ntile; ++t) issue_tile(t);
  {
    const int* goffs = v.offs + (size_t)bh * (cap + 1) + k0;
#pragma unroll 1
    for (int i = tid; i <= nloc; i += kST) offs[i] = __ldg(&goffs[i]);
  }
  // PDL: nothing above reads what the previous grid writes; q and every output wait
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#pragma unroll 1
  for (int i = tid; i < 8 * d; i += kST) {
    const int h = i / d, c = i - h * d;
    qd[h * qP + c] = h < G ? (double)load_elem_f(q, qdt, ((size_t)bh * G + h) * d + c) : 0.0;
  }
  __syncthreads();
  sc_wait();  // (S)
  sstamp(r, 1);

  // ---------------- P1: score my slice (fp64 tensor pipe) ------------------
  double lmax[2] = {-CUDART_INF, -CUDART_INF};  // heads 2(l%4), 2(l%4)+1
  {
    const double* qrow = qd + (lane >> 2) * qP + (lane & 3);  // B fragment: q[head l/4][4 kk + l%4]
#pragma unroll 1
    for (int t = 0; t < ntile; ++t) {
      const int row0 = t * kCCh;
      mbar_wait(tb0 + (unsigned)(t & 1) * 8, (unsigned)((t >> 1) & 1));
      const unsigned char* tileC = reinterpret_cast<const unsigned char*>(Cs) + (size_t)(t & 1) * kCTile;
      const int nrb = (min(kCCh, nloc - row0) + 7) >> 3;
#pragma unroll 1
      for (int rb = warp; rb < nrb; rb += kSW) {
        const int ia = rb * 8 + (lane >> 2);
        const unsigned char* arow = tileC + (size_t)ia * 128 + (lane & 3) * 4;
        const int sw = ia & 7;
        double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
#pragma unroll
          for (int tt = 0; tt < 4; ++tt) {
            const int kq = kk + tt;
            const double a = (double)*reinterpret_cast<const float*>(arow + (size_t)(kq >> 3) * kCCh * 128 +
                                                                     (((kq & 7) ^ sw) << 4));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[tt][0]), "+d"(c[tt][1])
                         : "d"(a), "d"(qrow[kq * 4]));
          }
        }
        const int row = row0 + ia;
        if (row < nloc) {
          const double ls = log((double)(offs[row + 1] - offs[row]));
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int h = 2 * (lane & 3) + e;
            if (h < G) {
              double val = ((c[0][e] + c[1][e]) + (c[2][e] + c[3][e])) * scale + ls;
              val = val != val ? -CUDART_INF : fmin(val, 1.7976931348623157e308);
              lml[h * L.per + row] = (float)val;
              cluster.map_shared_rank(lmall, h)[k0 + row] = val;
              lm_out[((size_t)bh * G + h) * cap + k0 + row] = val;
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
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    double m = lmax[e];
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 8));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 16));
    const int h = 2 * lane + e;
    if (lane < 4 && h < kG) s_wmd[warp][h] = m;
  }
  __syncthreads();
  if (tid < CL * G) {  // my slice maximum of head g -> every CTA
    const int rr = tid / G, g = tid - rr * G;
    double mm = -CUDART_INF;
#pragma unroll 1
    for (int w = 0; w < kSW; ++w) mm = fmax(mm, s_wmd[w][g]);
    cluster.map_shared_rank(&s_max[0][0], rr)[r * kG + g] = mm;
  }
  if (r < G) select_zero_hist<kST, kSBins>(reinterpret_cast<unsigned*>(smem + L.hm), reinterpret_cast<int*>(smem + L.hc));
  sstamp(r, 2);
  sc_sync();  // (A) every score is in its owner's shared memory, every maximum everywhere
  sstamp(r, 3);

  // ---------------- speculative L2 prefetch of the likely exact clusters ----
  // The CTAs that do not select (r >= G) prefetch, for every slice of the head
  // (reading the slice owners' offsets and log-masses over DSMEM), the rows of
  // clusters within tau nats of the head maximum of some q head, so HBM
  // streams the likely exact set into L2 while the owners select.
  if (tau > 0.f && r >= G) {
    float Mf[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      double m = -CUDART_INF;
      if (g < G)
        for (int rr = 0; rr < CL; ++rr) m = fmax(m, s_max[rr][g]);
      Mf[g] = (float)m - tau;
    }
    const size_t hb = (size_t)bh * v.row_cap * d * 2;
    const char* kb = reinterpret_cast<const char*>(v.keys) + hb;
    const char* vb = reinterpret_cast<const char*>(v.values) + hb;
    const int nno = CL - G;
#pragma unroll 1
    for (int sl = r - G; sl < CL; sl += nno) {
      const int n_sl = max(0, min(perk, K - sl * perk));
      const int* offs_sl = cluster.map_shared_rank(offs, sl);
      const float* lml_sl = cluster.map_shared_rank(lml, sl);
#pragma unroll 1
      for (int i = tid; i < n_sl; i += kST) {
        bool hot = false;
#pragma unroll
        for (int g = 0; g < kG; ++g)
          if (g < G) hot |= lml_sl[g * L.per + i] >= Mf[g];
        if (hot) {
          const int o0 = offs_sl[i], o1 = offs_sl[i + 1];
          const unsigned bytes = (unsigned)(o1 - o0) * (d * 2);
          if (bytes) {
            prefetch_l2(kb + (size_t)o0 * d * 2, bytes);
            prefetch_l2(vb + (size_t)o0 * d * 2, bytes);
          }
        }
      }
    }
  }

  // ---------------- P2: two-stage top-p, owner CTA g = r -------------------
  if (r < G) {
    const int g = r;
    double M = -CUDART_INF;
#pragma unroll 1
    for (int rr = 0; rr < CL; ++rr) M = fmax(M, s_max[rr][g]);
    uint8_t* stown = reinterpret_cast<uint8_t*>(smem + L.stown);
    int n1 = 0, n2 = 0;
    select_two_stage<kST, kSBins>(K, M, lmall, p1, p2, reinterpret_cast<unsigned long long*>(smem + L.um),
                                  reinterpret_cast<uint16_t*>(smem + L.bin), reinterpret_cast<unsigned*>(smem + L.hm),
                                  reinterpret_cast<int*>(smem + L.hc), reinterpret_cast<int*>(smem + L.clist),
                                  reinterpret_cast<int*>(smem + L.cord), stown, &s_sel, n1, n2);
    if (K > 0) {  // states -> the slice owners, packed 4 per word (slices are 4-aligned)
#pragma unroll 1
      for (int i = 4 * tid; i < K; i += 4 * kST) {
        unsigned w = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (i + t < K) w |= (unsigned)stown[i + t] << (8 * t);
        const int rr = i / perk;
        *reinterpret_cast<unsigned*>(cluster.map_shared_rank(stl, rr) + g * L.per + (i - rr * perk)) = w;
      }
    }
    if (tid == 0 && counts) {
      counts[2 * ((size_t)bh * G + g)] = n1;
      counts[2 * ((size_t)bh * G + g) + 1] = n2;
    }
  }
  sstamp(r, 4);
  sc_sync();  // (B) every state of my slice is in place
  sstamp(r, 5);

  // ---------------- my lists: exact row runs + approx pseudo-rows ----------
  // runs[j] = (first row, mask << 24 | len) for my slice's clusters that are
  // exact for >= 1 q head of the group (plus, on the last CTA, the sink and
  // window rows); the attention streams them in 8-row TMA groups
  {
    int row_base = 0, run_base = 0, grp_base = 0, apx_base = 0;
#pragma unroll 1
    for (int i0 = 0; i0 < nloc; i0 += kST) {
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
      // (rows << 40 | groups << 20 | runs) scanned in one pass
      const unsigned long long pk =
          ((unsigned long long)len << 40) | ((unsigned long long)((len + 7) >> 3) << 20) | (unsigned)(me != 0);
      unsigned long long ex, tot;
      int exa, tota;
      scan_pair<kST>(pk, ma != 0, s_sel.redu, s_sel.redi, ex, exa, tot, tota);
      if (me) runs[run_base + (int)(ex & 0xFFFFFu)] = make_int2(st0, (int)(((unsigned)me << 24) | (unsigned)len));
      if (ma) apx[apx_base + exa] = make_int2(k0 + i, ma);
      row_base += (int)(tot >> 40);
      grp_base += (int)((tot >> 20) & 0xFFFFFu);
      run_base += (int)(tot & 0xFFFFFu);
      apx_base += tota;
      __syncthreads();  // scan scratch reuse
    }
    if (tid == 0) {
      const int nexact = run_base;
      if (r == CL - 1) {  // the sink and window rows are exact for every q head
        const unsigned all = ((1u << G) - 1u) << 24;
        if (v.sink > 0) {
          runs[run_base++] = make_int2(0, (int)(all | (unsigned)v.sink));
          row_base += v.sink;
          grp_base += (v.sink + 7) >> 3;
        }
        if (v.window > 0) {
          runs[run_base++] = make_int2(v.n_tokens - v.window, (int)(all | (unsigned)v.window));
          row_base += v.window;
          grp_base += (v.window + 7) >> 3;
        }
      }
      s_napx = apx_base;
      int* dst = cluster.map_shared_rank(&s_cnt[0][0], 0) + r * 4;
      dst[0] = row_base;
      dst[1] = apx_base;
      dst[2] = nexact;
#ifdef DP_PROFILE
      if (blockIdx.x < 16) {
        g_step_ts[r][11] = (unsigned long long)row_base;
        g_step_ts[r][12] = (unsigned long long)run_base;
        g_step_ts[r][13] = (unsigned long long)apx_base;
      }
#endif
      // (runs, groups) of my list -> every CTA of the head
      for (int rr = 0; rr < CL; ++rr) {
        int2* gd = cluster.map_shared_rank(&s_gc[0], rr);
        gd[r] = make_int2(run_base, grp_base);
      }
    }
    if (state_out)
#pragma unroll 1
      for (int i = tid; i < G * nloc; i += kST) {
        const int g = i / nloc, k = i - g * nloc;
        state_out[((size_t)bh * G + g) * cap + k0 + k] = stl[g * L.per + k];
      }
  }
  // the ring overlays the plan arrays: order their generic accesses before the TMA writes
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  sc_sync();  // (B2) every CTA's run list and group count is published; the plan arrays are dead
  sstamp(r, 6);

  // ---------------- attention: the head's row groups balanced over its CTAs ---
  // The head's exact rows are the concatenation of the CTAs' run lists in 8-row
  // groups (runs padded to whole groups); CTA r attends groups [g0, g1).
  int gtot = 0;
#pragma unroll 1
  for (int rr = 0; rr < CL; ++rr) gtot += s_gc[rr].y;
  const int g0 = (int)((long long)gtot * r / CL), g1 = (int)((long long)gtot * (r + 1) / CL);
  const int ngrp = g1 - g0;
  const int ntiles = (ngrp + kTileGroups - 1) / kTileGroups;
  const int napx = s_napx;
  if (warp >= kCW) {
    // ---- producer warp: walks the runs covering groups [g0, g1) of the head's
    // list (reading the other CTAs' lists over DSMEM, kLRuns at a time, clipped
    // to my groups); lane 0 issues the TMA boxes, lanes 0-7 write the row masks
    if (warp == kCW) {
      int p_rr = 0, p_j = 0, p_gb = 0, p_base = 0;  // next run to examine: source CTA, index, groups
      auto pull = [&]() {  // refill lruns with the next clipped runs (warp-uniform)
        int n = 0;
#pragma unroll 1
        while (p_rr < CL && n <= kLRuns - 32) {
          const int2 gc = s_gc[p_rr];
          if (p_j >= gc.x || p_gb + gc.y <= g0 || p_base >= g1) {  // next source list
            if (p_base >= g1) {
              p_rr = CL;
              break;
            }
            p_gb += gc.y;
            ++p_rr;
            p_j = 0;
            p_base = p_gb;
            continue;
          }
          const int2* src = cluster.map_shared_rank(runs, p_rr);
          const int j = p_j + lane;
          const int2 rn = j < gc.x ? src[j] : make_int2(0, 0);
          const int len = j < gc.x ? (rn.y & 0xFFFFFF) : 0;
          const int ng = (len + 7) >> 3;
          int inc = ng;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
          }
          const int lo_g = p_base + inc - ng, hi_g = p_base + inc;  // this run's groups in the head
          const int a = max(lo_g, g0), b = min(hi_g, g1);
          const bool keep = a < b;
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          if (keep) {
            const int skip = (a - lo_g) * 8;
            lruns[n + __popc(bal & ((1u << lane) - 1u))] =
                make_int2(rn.x + skip, (int)(((unsigned)rn.y & 0xFF000000u) | (unsigned)min(len - skip, (b - a) * 8)));
          }
          n += __popc(bal);
          p_j += 32;
          p_base += __shfl_sync(0xffffffffu, inc, 31);
        }
        __syncwarp();
        return n;
      };
      const unsigned long long pol = evict_first_policy();
      const int rowbase = bh * v.row_cap;
      int nl = pull(), li = 0, goff = 0;
#pragma unroll 1
      for (int idx = 0; idx < ntiles; ++idx) {
        const int s = idx % kNStage;
        const int ngt = min(kTileGroups, ngrp - idx * kTileGroups);
        if (idx >= kNStage) mbar_wait(smem_u32(&empty_bar[s]), (unsigned)(((idx / kNStage) + 1) & 1));
        unsigned char* st = ring + (size_t)s * kStageBytes;
        int* rm = rmask + s * kRows;
        const unsigned fb = smem_u32(&full_bar[s]);
        // runs are cut into segments (one run, one tile) of whole 8-row groups;
        // each segment goes out as 32/16/8-row TMA boxes (two 64-column planes
        // of K and of V each), landing at its group slot
        int g = 0;
#pragma unroll 1
        while (g < ngt) {
          if (li == nl) {
            nl = pull();
            li = 0;
          }
          const int2 rn = lruns[li];
          const int len = rn.y & 0xFFFFFF;
          const int m = (int)((unsigned)rn.y >> 24);
          const int ns = min(((len + 7) >> 3) - goff, ngt - g);
#pragma unroll 1
          for (int j = lane; j < 8 * ns; j += 32) rm[8 * g + j] = 8 * goff + j < len ? m : 0;
          if (lane == 0 && !(dbg & 2)) {
            int row = rowbase + rn.x + 8 * goff, slot = g, n = ns;
#pragma unroll 1
            while (n > 0) {
              const int b = n >= 4 ? 4 : (n >= 2 ? 2 : 1);  // groups per box
              const CUtensorMap* km = b == 4 ? &tmK32 : (b == 2 ? &tmK16 : &tmK8);
              const CUtensorMap* vm = b == 4 ? &tmV32 : (b == 2 ? &tmV16 : &tmV8);
              const unsigned kd = smem_u32(st + slot * 1024);
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                tma_box(kd + hf * (kRows * 128), km, hf * 64, row, fb, pol);
                tma_box(kd + kKVTile + hf * (kRows * 128), vm, hf * 64, row, fb, pol);
              }
              slot += b;
              row += 8 * b;
              n -= b;
            }
          }
          g += ns;
          goff += ns;
          if (8 * goff >= len) {
            ++li;
            goff = 0;
          }
        }
#pragma unroll 1
        for (int j = 8 * ngt + lane; j < kRows; j += 32) rm[j] = 0;
        if (ngt & 1) {  // a consumer warp spans two groups: the unfilled one's V rows must be finite (P = 0 there)
          float4* vz = reinterpret_cast<float4*>(st + kKVTile + ngt * 1024);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            vz[t * (kRows * 128 / 16) + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
            vz[t * (kRows * 128 / 16) + 32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        __syncwarp();
        // releases the row masks; the boxes' bytes complete the phase
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb),
                                    "r"((dbg & 2) ? 0u : (unsigned)ngt * 4096u)
                                    : "memory");
      }
    }
  } else {
    // ---- consumers: every warp owns rows [16w, 16w + 16) of each tile
    const int g8 = lane >> 2, tq = lane & 3;
    unsigned qa[8][2], qb[8][2];
    {
      const bool valid = g8 < G;
      const size_t qoff = ((size_t)bh * G + (valid ? g8 : 0)) * d;
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = k * 16 + h * 8 + 2 * tq;
          if (!valid) {
            qa[k][h] = 0u;
            qb[k][h] = 0u;
          } else if (qdt == DP_F32) {
            const float2 f = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(q) + qoff + col);
            split2(f.x, f.y, qa[k][h], qb[k][h]);
          } else {
            qa[k][h] = *reinterpret_cast<const unsigned*>(reinterpret_cast<const __nv_bfloat16*>(q) + qoff + col);
            qb[k][h] = 0u;
          }
        }
    }
    const bool q32 = qdt == DP_F32;
    float o[8][4];
#pragma unroll
    for (int mb = 0; mb < 8; ++mb)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[mb][e] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float* Pw = Pbuf + warp * 128;
    const int r0w = warp * 16;
    // approximated clusters of my slice: pseudo-rows (logit = log-mass, value
    // = value mean), this warp's share folded one per tile, loads a tile ahead
    const int ap_base = napx * warp / kCW, ap_n = napx * (warp + 1) / kCW - ap_base;
    int ap_k = 0;
    bool ap_ready = false;
    float4 ap_v = make_float4(0.f, 0.f, 0.f, 0.f);
    float ap_x = -INFINITY;
    auto ap_issue = [&]() {
      const int2 e = apx[ap_base + ap_k];
      ap_v = __ldg(reinterpret_cast<const float4*>(v.value_means + ((size_t)bh * cap + e.x) * d) + lane);
      ap_x = (lane < G && ((e.y >> lane) & 1))
                 ? (float)(__ldcg(lm_out + ((size_t)bh * G + lane) * cap + e.x) * 1.4426950408889634)
                 : -INFINITY;
      ++ap_k;
      ap_ready = true;
    };
    auto ap_fold = [&]() {
      float x[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) x[hh] = __shfl_sync(0xffffffffu, ap_x, 2 * tq + hh);
      __syncwarp();
      reinterpret_cast<float4*>(Pw)[lane] = ap_v;
      __syncwarp();
      float pa[2], al[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float mn = fmaxf(m_run[hh], x[hh]);
        al[hh] = mn == -INFINITY ? 1.f : exp2f(m_run[hh] - mn);
        pa[hh] = x[hh] == -INFINITY ? 0.f : exp2f(x[hh] - mn);
        m_run[hh] = mn;
        l_run[hh] = l_run[hh] * al[hh] + (g8 == 0 ? pa[hh] : 0.f);  // one lane per head counts it
      }
#pragma unroll
      for (int mb = 0; mb < 8; ++mb) {
        const float v0 = Pw[mb * 16 + g8], v1 = Pw[mb * 16 + g8 + 8];
        o[mb][0] = o[mb][0] * al[0] + pa[0] * v0;
        o[mb][1] = o[mb][1] * al[1] + pa[1] * v0;
        o[mb][2] = o[mb][2] * al[0] + pa[0] * v1;
        o[mb][3] = o[mb][3] * al[1] + pa[1] * v1;
      }
      __syncwarp();
      ap_ready = false;
    };
    if (ap_k < ap_n) ap_issue();
    const float sl2 = (float)(scale * 1.4426950408889634);
#pragma unroll 1
    for (int idx = 0; idx < ntiles; ++idx) {
      const int s = idx % kNStage;
      const int nr = 8 * min(kTileGroups, ngrp - idx * kTileGroups);
      mbar_wait(smem_u32(&full_bar[s]), (unsigned)((idx / kNStage) & 1));
      const unsigned char* Ks = ring + (size_t)s * kStageBytes;
      const unsigned char* Vs = Ks + kKVTile;
      if (!(dbg & 1) && r0w < nr) {
        // ---- S = K Q^T for this warp's 16 rows (two accumulators: short chains)
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
        {
          // K plane k/4 (dims 64(k/4) ..), 16-B chunk (2k + hi) % 8 of the row, 128B swizzle
          const int row = r0w + (lane & 7) + ((lane >> 3) & 1) * 8;
          const unsigned rb = smem_u32(Ks + (size_t)row * 128);
          const int x = row & 7, hi = lane >> 4;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            unsigned a0, a1, a2, a3;
            ldsm_x4(rb + (unsigned)((k >> 2) * (kRows * 128)) + (unsigned)((((2 * k + hi) & 7) ^ x) << 4), a0, a1, a2,
                    a3);
            float* acc = (k & 1) ? sb : sa;
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(qa[k][0]), "r"(qa[k][1]));
            if (q32)
              asm volatile(
                  "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                  "{%0,%1,%2,%3};\n"
                  : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
                  : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(qb[k][0]), "r"(qb[k][1]));
          }
        }
        const int* rm = rmask + s * kRows + r0w + g8;
        const int mlo = rm[0], mhi = rm[8];
        float sc[4], mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = 2 * tq + (e & 1);
          const bool ok = h < G && (((e >> 1) ? mhi : mlo) >> h & 1);
          sc[e] = ok ? (sa[e] + sb[e]) * sl2 : -INFINITY;
          mx[e & 1] = fmaxf(mx[e & 1], sc[e]);
        }
        float alpha[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 4));
          mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 8));
          mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 16));
          const float mn = fmaxf(m_run[hh], mx[hh]);
          alpha[hh] = mn == -INFINITY ? 1.f : exp2f(m_run[hh] - mn);
          m_run[hh] = mn;
          l_run[hh] *= alpha[hh];
        }
        float pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          pv[e] = sc[e] == -INFINITY ? 0.f : exp2f(sc[e] - m_run[e & 1]);
          l_run[e & 1] += pv[e];
        }
#pragma unroll
        for (int mb = 0; mb < 8; ++mb) {
          o[mb][0] *= alpha[0];
          o[mb][1] *= alpha[1];
          o[mb][2] *= alpha[0];
          o[mb][3] *= alpha[1];
        }
        // P (rows x heads) -> B fragment (k = row, n = head) through the warp's buffer
        *reinterpret_cast<float2*>(Pw + g8 * 8 + 2 * tq) = make_float2(pv[0], pv[1]);
        *reinterpret_cast<float2*>(Pw + (g8 + 8) * 8 + 2 * tq) = make_float2(pv[2], pv[3]);
        __syncwarp();
        unsigned bh0, bl0, bh1, bl1;
        split2(Pw[(2 * tq) * 8 + g8], Pw[(2 * tq + 1) * 8 + g8], bh0, bl0);
        split2(Pw[(2 * tq + 8) * 8 + g8], Pw[(2 * tq + 9) * 8 + g8], bh1, bl1);
        __syncwarp();
        // ---- O^T += V^T P over all 128 dims (8 independent m-blocks)
        {
          const int row = r0w + (lane & 7) + ((lane >> 4) & 1) * 8;
          const unsigned rb = smem_u32(Vs + (size_t)row * 128);
          const int x = row & 7, hi = (lane >> 3) & 1;
#pragma unroll
          for (int mb = 0; mb < 8; ++mb) {
            unsigned a0, a1, a2, a3;
            ldsm_x4_t(rb + (unsigned)((mb >> 2) * (kRows * 128)) + (unsigned)((((2 * mb + hi) & 7) ^ x) << 4), a0, a1,
                      a2, a3);
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+f"(o[mb][0]), "+f"(o[mb][1]), "+f"(o[mb][2]), "+f"(o[mb][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bh0), "r"(bh1));
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+f"(o[mb][0]), "+f"(o[mb][1]), "+f"(o[mb][2]), "+f"(o[mb][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bl0), "r"(bl1));
          }
        }
      }
      if (ap_ready) ap_fold();  // one approx pseudo-row per tile, the next one's loads in flight
      if (ap_k < ap_n) ap_issue();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty_bar[s]));
    }
    if (ap_ready) ap_fold();
#pragma unroll 1
    while (ap_k < ap_n) {
      ap_issue();
      ap_fold();
    }
    sstamp(r, 7);
    // ---- combine the 8 warp states -> this CTA's partial per q head -> owner
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 4);
      l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 8);
      l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 16);
    }
    cons_sync();  // every warp is done reading the ring
    float* scratch = reinterpret_cast<float*>(ring);  // [8 warps][8 heads][d]
#pragma unroll
    for (int mb = 0; mb < 8; ++mb)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        scratch[((size_t)warp * 8 + 2 * tq + (e & 1)) * d + mb * 16 + g8 + (e >> 1) * 8] = o[mb][e];
    if (g8 == 0) {
      s_wm[warp][2 * tq] = m_run[0];
      s_wm[warp][2 * tq + 1] = m_run[1];
      s_wl[warp][2 * tq] = l_run[0];
      s_wl[warp][2 * tq + 1] = l_run[1];
    }
    cons_sync();
#pragma unroll 1
    for (int i = tid; i < G * d; i += kCons) {
      const int h = i / d, c = i - h * d;
      float Mw = -INFINITY;
#pragma unroll
      for (int w = 0; w < kCW; ++w) Mw = fmaxf(Mw, s_wm[w][h]);
      float sum = 0.f, Lw = 0.f;
#pragma unroll
      for (int w = 0; w < kCW; ++w) {
        const float wm = s_wm[w][h];
        if (wm != -INFINITY) {
          const float f = exp2f(wm - Mw);
          sum += f * scratch[((size_t)w * 8 + h) * d + c];
          Lw += f * s_wl[w][h];
        }
      }
      float* dst = cluster.map_shared_rank(pslot, h) + (size_t)r * (d + 4);
      dst[4 + c] = sum;
      if (c == 0) {
        dst[0] = Mw;
        dst[1] = Lw;
      }
    }
  }
  sstamp(r, 8);
  sc_sync();  // (C) every partial is in its owner's shared memory; no remote access after this
  sstamp(r, 9);

  // ---------------- merge: owner g combines the CL partials of q head g -----
  if (r < G) {
    const size_t hq = (size_t)bh * G + r;
#pragma unroll 1
    for (int c = tid; c < d; c += kST) {
      float M = -INFINITY;
#pragma unroll 1
      for (int rr = 0; rr < CL; ++rr) M = fmaxf(M, pslot[rr * (d + 4)]);
      float sum = 0.f, Lt = 0.f;
#pragma unroll 1
      for (int rr = 0; rr < CL; ++rr) {
        const float m = pslot[rr * (d + 4)];
        if (m != -INFINITY) {
          const float f = exp2f(m - M);
          sum += f * pslot[rr * (d + 4) + 4 + c];
          Lt += f * pslot[rr * (d + 4) + 1];
        }
      }
      out[hq * d + c] = Lt > 0.f ? sum / Lt : 0.f;
      if (c == 0) lse[hq] = Lt > 0.f ? M * 0.69314718055994531f + logf(Lt) : -INFINITY;
    }
  }
  if (r == 0 && tid == 0 && stats) {
    int rows = 0, na = 0, ne = 0;
    for (int rr = 0; rr < CL; ++rr) {
      rows += s_cnt[rr][0];
      na += s_cnt[rr][1];
      ne += s_cnt[rr][2];
    }
    stats[4 * bh + 0] = rows;
    stats[4 * bh + 1] = na;
    stats[4 * bh + 2] = (rows + kRows - 1) / kRows;
    stats[4 * bh + 3] = ne;
  }
  sstamp(r, 10);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int group_bound8(int G) { return G <= 1 ? 1 : (G <= 2 ? 2 : (G <= 4 ? 4 : 8)); }

static const void* step_fn(int kG) {
  switch (kG) {
    case 1: return reinterpret_cast<const void*>(step_kernel<1>);
    case 2: return reinterpret_cast<const void*>(step_kernel<2>);
    case 4: return reinterpret_cast<const void*>(step_kernel<4>);
    default: return reinterpret_cast<const void*>(step_kernel<8>);
  }
}

static size_t step_static_smem(int kG) {
  static size_t cache[9] = {};
  std::lock_guard<std::recursive_mutex> lock(host_mutex());
  if (!cache[kG]) {
    cudaFuncAttributes a;
    cache[kG] = cudaFuncGetAttributes(&a, step_fn(kG)) == cudaSuccess ? a.sharedSizeBytes + 1 : 8192;
  }
  return cache[kG] - 1;
}

typedef CUresult (*StepEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D map over a bf16 [rows, 128] key or value tensor: 64-column x 8-row boxes,
// 128B swizzle (conflict-free ldmatrix on the staged tiles); a few recent maps cached
static cudaError_t kv_tmap(const void* ptr, long long rows, int boxr, CUtensorMap* m) {
  struct Entry {
    const void* ptr;
    long long rows;
    int boxr;
    CUtensorMap map;
  };
  static Entry cache[48];
  static int next = 0;
  static StepEncodeFn fn = nullptr;
  std::lock_guard<std::recursive_mutex> lock(host_mutex());
  for (const Entry& e : cache)
    if (e.ptr == ptr && e.rows == rows && e.boxr == boxr) {
      *m = e.map;
      return cudaSuccess;
    }
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &qr) !=
            cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn)
      return cudaErrorNotSupported;
  }
  const cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, (cuuint32_t)boxr};
  const cuuint32_t es[2] = {1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  cache[next] = Entry{ptr, rows, boxr, *m};
  next = (next + 1) % 48;
  return cudaSuccess;
}

static size_t step_smem_bytes(int CL, int cap) { return step_layout(CL, cap).total + 1024; }

static bool step_fits(const dp_cache_view& v, int G, int cl) {
  if (G > cl || cl > kStepMaxCL) return false;
  const StepLayout L = step_layout(cl, v.cluster_cap);
  return L.per <= kStepMaxPer && L.plan_end <= kRingBytes && L.p2_end <= L.cs + 2 * (size_t)kCTile &&
         step_smem_bytes(cl, v.cluster_cap) + step_static_smem(group_bound8(G)) <= (size_t)kStepMaxSmem;
}

static int step_max_active(int kG, int cl, size_t smem) {
  static int cache[kMaxDevices][9][kStepMaxCL + 1] = {};
  static size_t cache_smem[kMaxDevices][9][kStepMaxCL + 1] = {};
  const int dev = current_device();
  std::lock_guard<std::recursive_mutex> lock(host_mutex());
  if (cache_smem[dev][kG][cl] == smem) return cache[dev][kG][cl];
  ensure_smem(step_fn(kG), smem, true);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cl);
  cfg.blockDim = dim3(kST);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, step_fn(kG), &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[dev][kG][cl] = n;
  cache_smem[dev][kG][cl] = smem;
  return n;
}

// widest cluster (most SMs per head) for which every (sequence, kv head) is
// co-resident in one wave; 0 if none
static int step_pick_cl(const dp_cache_view& v, int G) {
  const int units = v.batch * v.kv_heads, kG = group_bound8(G);
  if (g_step_cl >= 1 && g_step_cl <= kStepMaxCL)
    return step_fits(v, G, g_step_cl) &&
                   step_max_active(kG, g_step_cl, step_smem_bytes(g_step_cl, v.cluster_cap)) >= units
               ? g_step_cl
               : 0;
  for (int cl = kStepMaxCL; cl >= 2 && cl >= G; --cl)
    if (step_fits(v, G, cl) && step_max_active(kG, cl, step_smem_bytes(cl, v.cluster_cap)) >= units) return cl;
  return 0;
}

bool step_supported(const dp_cache_view& v, int G, int qdt) {
  (void)qdt;
  return !g_step_off && v.dtype == DP_BF16 && v.head_dim == 128 && G >= 1 && G <= kMaxGroup &&
         v.cluster_cap <= kStepMaxCap && v.cluster_cap >= 1 && v.row_cap < (1 << 24) && step_pick_cl(v, G) > 0;
}

int step_cluster_size(const dp_cache_view& v, int G) { return step_pick_cl(v, G); }

cudaError_t launch_step(const dp_cache_view& v, const void* q, int qdt, int G, double scale, double p1, double p2,
                        double* lm, uint8_t* state, int* counts, int* stats, float* out, float* lse, void* ws,
                        cudaStream_t st) {
  (void)ws;
  if (!lm) return cudaErrorInvalidValue;  // the approx pseudo-rows read their log-masses back
  const int CL = step_pick_cl(v, G);
  if (!CL) return cudaErrorInvalidConfiguration;
  const int kG = group_bound8(G);
  const size_t smem = step_smem_bytes(CL, v.cluster_cap);
  ensure_smem(step_fn(kG), smem, true);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(v.batch * v.kv_heads * CL));
  cfg.blockDim = dim3(kST);
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
  CUtensorMap tm, kv[6];
  cudaError_t e = centroid_tmap(v, &tm);
  if (e != cudaSuccess) return e;
  const long long kvrows = (long long)v.batch * v.kv_heads * v.row_cap;
  for (int i = 0; i < 3; ++i)
    if ((e = kv_tmap(v.keys, kvrows, 8 << i, &kv[i])) != cudaSuccess ||
        (e = kv_tmap(v.values, kvrows, 8 << i, &kv[3 + i])) != cudaSuccess)
      return e;
  const long long rows = (long long)v.batch * v.kv_heads * v.cluster_cap;
  const int boxr = rows < kCCh ? (int)rows : kCCh;
  const float tau = g_step_tau;
  switch (kG) {
    case 1: return cudaLaunchKernelEx(&cfg, step_kernel<1>, tm, kv[0], kv[1], kv[2], kv[3], kv[4], kv[5], v, q, qdt, G, scale, p1, p2, lm, state, counts, stats, out, lse, CL, boxr, tau, g_step_dbg);
    case 2: return cudaLaunchKernelEx(&cfg, step_kernel<2>, tm, kv[0], kv[1], kv[2], kv[3], kv[4], kv[5], v, q, qdt, G, scale, p1, p2, lm, state, counts, stats, out, lse, CL, boxr, tau, g_step_dbg);
    case 4: return cudaLaunchKernelEx(&cfg, step_kernel<4>, tm, kv[0], kv[1], kv[2], kv[3], kv[4], kv[5], v, q, qdt, G, scale, p1, p2, lm, state, counts, stats, out, lse, CL, boxr, tau, g_step_dbg);
    default: return cudaLaunchKernelEx(&cfg, step_kernel<8>, tm, kv[0], kv[1], kv[2], kv[3], kv[4], kv[5], v, q, qdt, G, scale, p1, p2, lm, state, counts, stats, out, lse, CL, boxr, tau, g_step_dbg);
  }
}

}  // namespace dp

extern "C" int dp_debug_step_timing(unsigned long long* out) {
  // [16][16] step phases, then [16][8] selection phases (select.cuh) of the same launch
  if (cudaMemcpyFromSymbol(out, dp::g_step_ts, sizeof(dp::g_step_ts)) != cudaSuccess) return 2;
  return cudaMemcpyFromSymbol(out + 256, dp::g_sel_ts, sizeof(dp::g_sel_ts)) == cudaSuccess ? 0 : 2;
}
extern "C" int dp_debug_step_cluster_size(const dp_cache_view* v, int G) { return dp::step_cluster_size(*v, G); }
