// Gathered split-KV decode attention for bf16 caches on tensor cores.
//
// Persistent, warp-specialised: one CTA per SM = 8 compute warps + 1
// producer warp.  The GQA-union rows of every
// (sequence, kv head) form a global sequence of 128-row chunks (the plan /
// worklist kernel publishes the per-head chunk prefix); CTA i owns the
// contiguous range [i*T/grid, (i+1)*T/grid) of it -- balanced to +-1 chunk
// with no atomics -- and runs an online softmax over it, flushing one partial
// (m, l, o) per head it touches.  Rows are gathered through a 3-stage
// TMA-bulk ring (64 KB of K+V per stage, two chunks in flight while one is
// computed): 16-byte cp.async copies, a warp moving 2 rows = 512 contiguous
// bytes per instruction into padded 272-B smem rows (conflict-free ldmatrix).
// (tools/bw_probe.cu: this ring streams at ~5.4 TB/s on B200; per-row
// cp.async.bulk reached 4.6 TB/s.)
//
//   S[row, head]  = K[row, :] . Q[head, :]     mma.m16n8k16 bf16 -> f32, M = 16 rows,
//                                                N = 8 heads (G <= 8), K = 16 dims
//   O^T[d, head] += V^T[d, row] . P[row, head]  M = 16 dims, N = 8 heads, K = 16 rows
// (heads on N keeps M dense: 24 MMAs per warp per 128-row chunk)
//
// P is split hi + lo into two bf16 operands (two MMAs) so the weights keep
// ~2^-16 relative precision; an fp32 query is split the same way.  The last
// CTA to finish a head merges its partials with the approx pseudo-rows
// (logit = log-mass, value = value mean; engine.py:216-252) -- no extra launch.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "host_state.h"
#include "decode_internal.h"
#include "tc_common.cuh"

namespace dp {

constexpr int kTcRows = kChunkRows;  // 128
constexpr int kConsumers = 256;  // 8 compute warps
constexpr int kProducers = 4;  // producer warps, 32 rows each
constexpr int kTcThreads = kConsumers + 32 * kProducers;
constexpr int kRowStride = 136;      // bf16 elements per staged row (272 B: conflict-free ldmatrix)
constexpr int kStages = 3;
int g_seg_cost = 768;  // rows' worth of time a head segment start costs a CTA (range balancing; dp_debug_set(9, .))
constexpr int kStageElems = kTcRows * kRowStride;  // one K (or V) tile
int g_attn_debug = 0;  // profiling switches (dp_debug_set)
// barrier over the 8 compute warps only (the producer warp never joins)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumers) : "memory"); }

// per-CTA phase stamps (%globaltimer ns) of the last launch; profiling aid,
// read with dp_debug_attn_timing()
__device__ unsigned long long g_attn_ts[512][12];

// (compiled in only with -DDP_PROFILE)
__device__ __forceinline__ void astamp(int ev) {
#ifdef DP_PROFILE
  if (threadIdx.x == 0 && blockIdx.x < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_attn_ts[blockIdx.x][ev] = t;
  }
#endif
}
__device__ __forceinline__ void astamp_at(int ev, unsigned long long v) {
#ifdef DP_PROFILE
  if (blockIdx.x < 512) g_attn_ts[blockIdx.x][ev] = v;
#endif
}

// owner CTA of global row j when T rows are split evenly over `grid` CTAs
// as [floor(i*T/grid), floor((i+1)*T/grid))
__device__ __forceinline__ int row_owner(long long j, long long T, int grid) {
  return (int)(((j + 1) * grid - 1) / T);
}

struct TcSmem {
  static constexpr size_t kv = (size_t)kStages * 2 * kStageElems * 2;  // K,V ring
  static constexpr size_t ps = 8 * kTcRows * 4;
  static constexpr size_t rows = (size_t)kStages * kTcRows * 4;         // head mask per stage
  static constexpr size_t fixed = kv + ps + rows;
};

// Walks a CTA's contiguous range [s, end) of the global union-row sequence
// in tiles of <= 128 rows that never straddle two heads.  Producer and
// consumer warps run identical copies, so they agree on every tile.
struct TileWalk {
  long long s, end;
  int bh;
  __device__ __forceinline__ void init(const long long* rp, int BH, long long s0, long long e0) {
    s = s0;
    end = e0;
    int lo = 0, hi = BH - 1;  // last b with rp[b] <= s, then skip empty heads
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= s) lo = mid; else hi = mid - 1;
    }
    bh = lo;
    while (bh < BH - 1 && rp[bh + 1] <= s) ++bh;
  }
  __device__ __forceinline__ bool more() const { return s < end; }
  // current tile: head bh, head-local rows [v0, v0 + nr)
  __device__ __forceinline__ void tile(const long long* rp, int& tb, int& v0, int& nr) const {
    tb = bh;
    v0 = (int)(s - rp[bh]);
    long long lim = rp[bh + 1] < end ? rp[bh + 1] : end;
    nr = (int)((lim - s) < kTcRows ? (lim - s) : kTcRows);
  }
  __device__ __forceinline__ void next(const long long* rp, int BH, int nr) {
    s += nr;
    while (bh < BH - 1 && rp[bh + 1] <= s) ++bh;
  }
};

template <bool kDense, bool kQF32>
__global__ void __launch_bounds__(kTcThreads, 1) attn_tc_kernel(dp_cache_view v, const void* __restrict__ q, int G,
                                                               float scale_log2, const double* __restrict__ lm,
                                                               WorkLists wl, Partials<float> pt,
                                                               float* __restrict__ out, float* __restrict__ lse,
                                                               int dbg, int kSegCost) {
  constexpr int d = 128;
  constexpr int kWarps = kConsumers / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, tq = lane & 3;  // fragment row / column-pair
  const int BH = v.batch * v.kv_heads;
  const int grid = gridDim.x, me = blockIdx.x;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* KV = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [stage][K|V][rows][stride]
  float* Pbuf = reinterpret_cast<float*>(smem_raw + TcSmem::kv);    // [8 warps][16 rows][8 heads]
  int* rmask = reinterpret_cast<int*>(smem_raw + TcSmem::kv + TcSmem::ps);  // [stage][rows]
  long long* rp = reinterpret_cast<long long*>(smem_raw + TcSmem::fixed);    // [BH+1] row prefix
  __shared__ float s_wm[kWarps][8], s_wl[kWarps][8];  // warp states (flush / merge)
  __shared__ int s_merge[32], s_nmerge;
  __shared__ __align__(8) unsigned long long full_bar[kStages], empty_bar[kStages];

  astamp(0);
  if (tid == 0) {
    s_nmerge = 0;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 33 * kProducers);  // per producer warp: 32 async + 1 release
      mbar_init(smem_u32(&empty_bar[i]), kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // PDL: everything above overlapped the plan kernel's tail; its outputs
  // (row lists, counts, approx lists) are visible after the wait.  q is not
  // written by the plan and its producers finished before the plan started,
  // so it is pulled into L2 now (load_q then hits L2 on the critical path).
  {
    const size_t qbytes = (size_t)BH * G * d * (kQF32 ? 4 : 2);
    const char* qc = reinterpret_cast<const char*>(q);
    for (size_t off = (size_t)tid * 128; off < qbytes; off += (size_t)kTcThreads * 128)
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(qc + off));
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  // ---- row prefix over heads (warp 0, 32 heads per step) ------------------
  if (warp == 0) {
    long long base = 0;
    for (int b0 = 0; b0 < BH; b0 += 32) {
      const long long nr = b0 + lane < BH ? (kDense ? v.n_tokens : __ldcg(&wl.nrows[b0 + lane])) : 0;
      long long inc = nr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (b0 + lane < BH) rp[b0 + lane] = base + inc - nr;
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) rp[BH] = base;
  }
  __syncthreads();
  astamp(1);
  // Ranges are balanced in a virtual row space where every head is preceded
  // by kSegCost empty rows: a CTA whose range starts a head segment (q load,
  // approx list, one more flush) gets correspondingly fewer real rows.
  // virtual(j) = j + (b + 1) * kSegCost for real row j of head b.
  const long long TV = rp[BH] + (long long)BH * kSegCost;
  auto real_of = [&](long long vv) {  // first real row at or after virtual row vv
    int lo = 0, hi = BH - 1;           // last head b with rp[b] + b * kSegCost <= vv
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rp[mid] + (long long)mid * kSegCost <= vv) lo = mid; else hi = mid - 1;
    }
    const long long o = vv - (rp[lo] + (long long)(lo + 1) * kSegCost);
    return o <= 0 ? rp[lo] : (rp[lo] + o < rp[lo + 1] ? rp[lo] + o : rp[lo + 1]);
  };
  const long long r0 = real_of(TV * me / grid), r1 = me + 1 == grid ? rp[BH] : real_of(TV * (me + 1) / grid);
  auto owner = [&](long long j, int b) { return row_owner(j + (long long)(b + 1) * kSegCost, TV, grid); };
  auto first_owner = [&](int bh) { return owner(rp[bh], bh); };
  auto head_parts = [&](int bh) { return owner(rp[bh + 1] - 1, bh) - first_owner(bh) + 1; };

  // ---- producer warps (rows [32p, 32p+32) of every tile): run up to kStages
  // tiles ahead; the next tile's row entries are fetched while this tile's
  // copies issue
  if (warp >= kWarps) {
    if (r0 >= r1) return;
    const int ch = lane & 15, pr0 = (warp - kWarps) * 32;
    const unsigned long long pol = evict_first_policy();
    TileWalk w;
    w.init(rp, BH, r0, r1);
    auto fetch = [&](const TileWalk& tw, unsigned& e, int& bh) {
      int v0, nr;
      tw.tile(rp, bh, v0, nr);
      const int row = pr0 + lane;
      e = row < nr ? (kDense ? (((unsigned)((1 << G) - 1)) << 24) | (unsigned)(v0 + row)
                             : __ldg(reinterpret_cast<const unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap + v0 + row))
                   : 0xFFFFFFFFu;
      return nr;
    };
    unsigned e_nx;
    int bh_nx;
    int nr_nx = fetch(w, e_nx, bh_nx);
    for (int idx = 0; w.more(); ++idx) {
      const int s = idx % kStages;
      const unsigned e = e_nx;
      const int bh = bh_nx;
      w.next(rp, BH, nr_nx);
      if (w.more()) nr_nx = fetch(w, e_nx, bh_nx);
      if (idx >= kStages) mbar_wait(smem_u32(&empty_bar[s]), (unsigned)(((idx / kStages) + 1) & 1));
      rmask[s * kTcRows + pr0 + lane] = e == 0xFFFFFFFFu ? 0 : (int)(e >> 24);
#ifdef DP_PROFILE
      if (idx == 0 && warp == kWarps && lane == 0 && blockIdx.x < 512) {  // profiling: first row entries in hand
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "r"(e));
        g_attn_ts[blockIdx.x][9] = t;
      }
#endif
      const size_t head_off = (size_t)bh * v.row_cap * d;
      const __nv_bfloat16* Kg = reinterpret_cast<const __nv_bfloat16*>(v.keys) + head_off;
      const __nv_bfloat16* Vg = reinterpret_cast<const __nv_bfloat16*>(v.values) + head_off;
      __nv_bfloat16* Ks = KV + (size_t)s * 2 * kStageElems;
      __nv_bfloat16* Vs = Ks + kStageElems;
      // lane copies 16-B column `ch` of rows pr0 + (lane >> 4) + 2 r: a warp
      // instruction moves 2 rows = 512 contiguous bytes
#pragma unroll 4
      for (int r = 0; r < 16; ++r) {
        const int row = pr0 + (lane >> 4) + 2 * r;
        const unsigned er = __shfl_sync(0xffffffffu, e, (lane >> 4) + 2 * r);
        const unsigned kd = smem_u32(Ks + row * kRowStride + ch * 8);
        const unsigned vd = smem_u32(Vs + row * kRowStride + ch * 8);
        if (er != 0xFFFFFFFFu) {
          const size_t off = (size_t)(er & 0xFFFFFFu) * d + ch * 8;
          cp16(kd, Kg + off, pol);
          cp16(vd, Vg + off, pol);
        } else {
          cp16_zero(kd, Kg);
          cp16_zero(vd, Vg);
        }
      }
#ifdef DP_PROFILE
      if (idx == 0 && warp == kWarps && lane == 0 && blockIdx.x < 512) {  // profiling: first tile issued
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_attn_ts[blockIdx.x][10] = t;
      }
#endif
      cp_async_arrive(smem_u32(&full_bar[s]));  // completes when this lane's copies land
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full_bar[s]));  // releases the rmask stores
    }
    return;
  }

  // Q^T B-fragments (registers): b0 = Q[head g8][k*16 + 2tq ..], b1 = Q[head g8][k*16 + 8 + 2tq ..]
  unsigned qa[8][2], qb[8][2];  // hi, lo
  // ---- consumer prologue: the first two head segments of this CTA's range get
  // their q staged in shared memory and their approx-list shares computed
  // now, while the producers fetch row entries and the first tiles -- a head
  // switch inside the loop then costs no global round trip
  constexpr int kQes = kQF32 ? 4 : 2;
  __shared__ __align__(16) unsigned char s_qseg[2][8 * d * 4];
  __shared__ float s_refm[2][8];  // the plan's reference maxima of those segments' q heads
  int seg_bh[2] = {-1, -1}, ap_pb[2] = {0, 0}, ap_pn[2] = {0, 0};
  int2 ap_pd[2] = {make_int2(0, 0), make_int2(0, 0)};
  {
    TileWalk w0;
    w0.init(rp, BH, r0, r1);
    if (w0.more()) {
      seg_bh[0] = w0.bh;
      const long long e0 = rp[w0.bh + 1] < r1 ? rp[w0.bh + 1] : r1;
      if (e0 < r1) {
        w0.next(rp, BH, (int)(e0 - w0.s));
        if (w0.more()) seg_bh[1] = w0.bh;
      }
    }
    const int qchunks = G * d * kQes / 16;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (seg_bh[k] >= 0)
        for (int i = tid; i < qchunks; i += kConsumers)
          reinterpret_cast<uint4*>(s_qseg[k])[i] =
              __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(q) + (size_t)seg_bh[k] * G * d * kQes) + i);
    if (!kDense) {
      if (tid < 2 * G && seg_bh[tid / G] >= 0) s_refm[tid / G][tid % G] = __ldcg(&wl.refm[(size_t)seg_bh[tid / G] * G + tid % G]);
      long long na[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) na[k] = seg_bh[k] >= 0 ? __ldcg(&wl.napprox[seg_bh[k]]) : 0;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int bh = seg_bh[k];
        if (bh < 0) continue;
        const long long hr = rp[bh + 1] - rp[bh];
        const long long lo = (r0 > rp[bh] ? r0 : rp[bh]) - rp[bh], hi = (r1 < rp[bh + 1] ? r1 : rp[bh + 1]) - rp[bh];
        const int j0 = hr > 0 ? (int)(na[k] * lo / hr) : 0, j1 = hr > 0 ? (int)(na[k] * hi / hr) : 0;
        ap_pb[k] = j0 + (j1 - j0) * warp / kWarps;
        ap_pn[k] = j0 + (j1 - j0) * (warp + 1) / kWarps - ap_pb[k];
        if (lane < ap_pn[k]) ap_pd[k] = __ldcg(&wl.approx[(size_t)bh * v.cluster_cap + ap_pb[k] + lane]);
      }
    }
    consumers_sync();  // staged q visible to every consumer warp
  }
  auto load_q = [&](int bh) {
    const bool valid = g8 < G;
    const int sk = bh == seg_bh[0] ? 0 : (bh == seg_bh[1] ? 1 : -1);
    const size_t qoff = ((size_t)bh * G + (valid ? g8 : 0)) * d;
    const unsigned char* qs = sk >= 0 ? s_qseg[sk] + (size_t)(valid ? g8 : 0) * d * kQes : nullptr;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = k * 16 + h * 8 + 2 * tq;
        if (!valid) {
          qa[k][h] = 0u;
          qb[k][h] = 0u;
        } else if (kQF32) {
          const float2 f = qs ? *reinterpret_cast<const float2*>(qs + (size_t)col * 4)
                              : *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(q) + qoff + col);
          split2(f.x, f.y, qa[k][h], qb[k][h]);
        } else {
          qa[k][h] = qs ? *reinterpret_cast<const unsigned*>(qs + (size_t)col * 2)
                        : *reinterpret_cast<const unsigned*>(reinterpret_cast<const __nv_bfloat16*>(q) + qoff + col);
          qb[k][h] = 0u;
        }
      }
    }
  };

  // Every consumer warp owns rows [16w, 16w+16) of each tile end to end:
  // S = K Q^T for its rows, its own online softmax, and O^T += V^T P over
  // all 128 dims -- no CTA-wide barrier per tile.  The 8 warp states are
  // combined once per head segment (flush), in the K buffer of the segment's
  // last tile before that stage is released to the producer.
  float o[8][4];       // O^T block mb: dims 16mb + g8 (+8) x heads 2tq, 2tq+1
  float m_run[2];      // running max (log2 units) of heads 2tq + hh over this warp's rows
  float l_run[2];      // this lane's share (rows g8, g8+8) of the running sum of heads 2tq + hh
  float* Pw = Pbuf + warp * 128;  // [16 rows][8 heads] P transpose buffer of this warp
  const int r0w = warp * 16;
  int cur = -1;

  // partial (m, l, o) of a finished head segment; the completion counters are
  // bumped once, after the loop, behind a single fence (no mid-loop stall)
  int flushed[2] = {-1, -1}, nflushed = 0;  // a CTA range touches <= 2 heads unless heads are tiny
  // approx pseudo-row pipeline state (warp-uniform)
  int ap_base = 0, ap_n = 0, ap_k = 0;
  bool ap_ready = false;
  int2 ap_desc = make_int2(0, 0);  // lane i: descriptor of entry ap_base + i (i < 32)
  float4 ap_v = make_float4(0.f, 0.f, 0.f, 0.f);  // value-mean slice [4 lane, 4 lane + 4)
  float ap_x = -INFINITY;          // lanes 0..7: log2-mass of head `lane` (or -inf)
  auto ap_issue = [&](int bh) {    // start the loads of entry ap_k
    int2 e;
    if (ap_k < 32) {
      e.x = __shfl_sync(0xffffffffu, ap_desc.x, ap_k);
      e.y = __shfl_sync(0xffffffffu, ap_desc.y, ap_k);
    } else {
      e = __ldcg(&wl.approx[(size_t)bh * v.cluster_cap + ap_base + ap_k]);
    }
    ap_v = __ldg(reinterpret_cast<const float4*>(v.value_means + ((size_t)bh * v.cluster_cap + e.x) * d) + lane);
    ap_x = (lane < G && ((e.y >> lane) & 1))
               ? (float)(__ldcg(lm + ((size_t)bh * G + lane) * v.cluster_cap + e.x) * 1.4426950408889634)
               : -INFINITY;
    ++ap_k;
    ap_ready = true;
  };
  auto ap_fold = [&]() {  // fold the loaded entry into this warp's online softmax
    float x[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) x[hh] = __shfl_sync(0xffffffffu, ap_x, 2 * tq + hh);
    __syncwarp();
    reinterpret_cast<float4*>(Pw)[lane] = ap_v;  // value row -> fragment layout via the P buffer
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

  auto flush = [&](int bh, float* scratch) {
    if (!kDense && !DP_AB(dbg, 64)) {  // drain this warp's remaining approx entries
      if (ap_ready) ap_fold();
#pragma unroll 1
      while (ap_k < ap_n) {
        ap_issue(bh);
        ap_fold();
      }
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 4);
      l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 8);
      l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 16);
    }
    consumers_sync();  // every warp is done reading this stage
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
    consumers_sync();
    const int slot = me - first_owner(bh);
    const size_t pbase = (size_t)bh * pt.max_chunks * G;
    if (kDense) {
#pragma unroll 1
      for (int i = tid; i < G * d; i += kConsumers) {
        const int h = i / d, c = i - h * d;
        float Mw = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) Mw = fmaxf(Mw, s_wm[ww][h]);
        float sum = 0.f, L = 0.f;
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
          const float wm = s_wm[ww][h];
          if (wm != -INFINITY) {
            const float f = exp2f(wm - Mw);
            sum += f * scratch[((size_t)ww * 8 + h) * d + c];
            L += f * s_wl[ww][h];
          }
        }
        pt.o[(pbase + (size_t)slot * G + h) * d + c] = sum;
        if (c == 0) {
          pt.m[pbase + (size_t)slot * G + h] = Mw == -INFINITY ? -INFINITY : Mw * 0.69314718055994531f;
          pt.l[pbase + (size_t)slot * G + h] = L;
        }
      }
    } else {
      // sparse: scale to the plan's reference max and fold into the head's
      // self-completing accumulators.  Each 16-B vector holds (o[c], o[c+1],
      // l, count); every CTA of the head adds (its o, its l, 1) with ONE
      // returning vector atomic, and the CTA whose add brings the count to
      // the head's CTA total holds the complete sums in the returned value
      // plus its own: it writes out[c..c+1] (and the lse) and clears the
      // vector.  Atomics on one address are totally ordered, so no fence,
      // completion counter or second round trip is needed.
      const int d2 = d >> 1;
      const float parts = (float)head_parts(bh);
#pragma unroll 1
      for (int i = tid; i < G * d2; i += kConsumers) {
        const int h = i / d2, c = (i - h * d2) * 2;
        const float Mr = bh == seg_bh[0] ? s_refm[0][h] : (bh == seg_bh[1] ? s_refm[1][h]
                                                                            : __ldcg(&wl.refm[(size_t)bh * G + h]));
        float o0 = 0.f, o1 = 0.f, L = 0.f;
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
          const float wm = s_wm[ww][h];
          if (wm != -INFINITY) {
            const float f = exp2f(wm - Mr);
            const float2 x = *reinterpret_cast<const float2*>(scratch + ((size_t)ww * 8 + h) * d + c);
            o0 += f * x.x;
            o1 += f * x.y;
            L += f * s_wl[ww][h];
          }
        }
        float* ac = wl.acc + ((size_t)bh * G + h) * acc_stride(d) + 2 * c;
        const float4 old = atom_add_v4(ac, make_float4(o0, o1, L, 1.f));
        if (old.w == parts - 1.f) {  // the last contribution: the sums are complete
          const float lt = old.z + L;
          const float rl = lt > 0.f ? 1.f / lt : 0.f;
          *reinterpret_cast<float2*>(out + ((size_t)bh * G + h) * d + c) = make_float2((old.x + o0) * rl,
                                                                                      (old.y + o1) * rl);
          if (c == 0) lse[(size_t)bh * G + h] = lt > 0.f ? Mr * 0.69314718055994531f + __logf(lt) : -INFINITY;
          *reinterpret_cast<float4*>(ac) = make_float4(0.f, 0.f, 0.f, 0.f);  // zero for the next launch
        }
      }
    }
    // No barrier here: the scratch (this stage's K buffer) is handed back by
    // each warp's empty-barrier arrive after the flush, and the producer
    // refills it only once all 8 warps arrived, i.e. finished reading it;
    // s_wm/s_wl are rewritten only after the next flush's first barrier.
    if (!kDense) return;  // sparse heads complete inside the flush
    consumers_sync();
    if (nflushed < 2) {
      flushed[nflushed++] = bh;
    } else {  // many tiny heads in one range: publish the oldest now
      if (tid == 0)
        if (atom_add_acq_rel(&wl.counters[flushed[0]], 1) == head_parts(flushed[0]) - 1)
          s_merge[s_nmerge++] = flushed[0];
      flushed[0] = flushed[1];
      flushed[1] = bh;
    }
  };

  TileWalk w;
  w.init(rp, BH, r0, r1);
  for (int idx = 0; w.more(); ++idx) {
    const int s = idx % kStages;
    int bh, v0, nr;
    w.tile(rp, bh, v0, nr);
    w.next(rp, BH, nr);
    const bool seg_end = !w.more() || w.bh != bh;
    if (bh != cur) {
      cur = bh;
      load_q(bh);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[mb][e] = 0.f;
      m_run[0] = m_run[1] = -INFINITY;
      l_run[0] = l_run[1] = 0.f;
      // approximated clusters of this head (engine.py:231-246): pseudo-rows
      // with logit = log-mass, value = value mean.  The head's CTAs split the
      // plan's approx list, each warp takes a share and trickles it into its
      // online softmax one entry per tile, loads issued a tile ahead (so the
      // fold never waits on memory); the flush drains what is left.
      if (!kDense && (bh == seg_bh[0] || bh == seg_bh[1])) {  // precomputed in the prologue
        const int sk = bh == seg_bh[0] ? 0 : 1;
        ap_base = ap_pb[sk];
        ap_n = ap_pn[sk];
        ap_desc = ap_pd[sk];
        ap_k = 0;
        ap_ready = false;
      } else if (!kDense) {
        // this CTA's share of the head's approx list is proportional to the
        // rows of the head it covers (a short head segment gets few entries)
        const long long na = __ldcg(&wl.napprox[bh]);
        const long long hr = rp[bh + 1] - rp[bh];
        const long long lo = (r0 > rp[bh] ? r0 : rp[bh]) - rp[bh], hi = (r1 < rp[bh + 1] ? r1 : rp[bh + 1]) - rp[bh];
        const int j0 = (int)(na * lo / hr), j1 = (int)(na * hi / hr);
        ap_base = j0 + (j1 - j0) * warp / kWarps;
        ap_n = j0 + (j1 - j0) * (warp + 1) / kWarps - ap_base;
        ap_desc = lane < ap_n ? __ldcg(&wl.approx[(size_t)bh * v.cluster_cap + ap_base + lane]) : make_int2(0, 0);
        ap_k = 0;
        ap_ready = false;
      }
    }
    mbar_wait(smem_u32(&full_bar[s]), (unsigned)((idx / kStages) & 1));  // stage s landed
    if (idx == 0) astamp(2);
    __nv_bfloat16* Ks = KV + (size_t)s * 2 * kStageElems;
    const __nv_bfloat16* Vs = Ks + kStageElems;
    if (!DP_AB(dbg, 1) && r0w < nr) {
      // ---- S = K Q^T for this warp's 16 rows (two accumulators: short chains)
      float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const unsigned base =
            smem_u32(Ks + (r0w + (lane & 7) + ((lane >> 3) & 1) * 8) * kRowStride + (lane >> 4) * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          unsigned a0, a1, a2, a3;
          ldsm_x4(base + k * 32, a0, a1, a2, a3);
          float* acc = (k & 1) ? sb : sa;
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
              "{%0,%1,%2,%3};\n"
              : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
              : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(qa[k][0]), "r"(qa[k][1]));
          if (kQF32)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(qb[k][0]), "r"(qb[k][1]));
        }
      }
      // sc[e]: row r0w + g8 + (e>>1)*8, head 2tq + (e&1); masked by the row's head set
      const int* rm = rmask + s * kTcRows + r0w + g8;
      const int mlo = rm[0], mhi = rm[8];
      float sc[4], mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = 2 * tq + (e & 1);
        const bool ok = h < G && (((e >> 1) ? mhi : mlo) >> h & 1);
        sc[e] = ok ? (sa[e] + sb[e]) * scale_log2 : -INFINITY;
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
      const unsigned vbase =
          smem_u32(Vs + (r0w + (lane & 7) + ((lane >> 4) & 1) * 8) * kRowStride + ((lane >> 3) & 1) * 8);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb) {
        unsigned a0, a1, a2, a3;
        ldsm_x4_t(vbase + mb * 32, a0, a1, a2, a3);
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};\n"
            : "+f"(o[mb][0]), "+f"(o[mb][1]), "+f"(o[mb][2]), "+f"(o[mb][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bh0), "r"(bh1));
        if (!DP_AB(dbg, 32))  // (32: timing experiment -- P's low half dropped)
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
              "{%0,%1,%2,%3};\n"
              : "+f"(o[mb][0]), "+f"(o[mb][1]), "+f"(o[mb][2]), "+f"(o[mb][3])
              : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bl0), "r"(bl1));
      }
    }
    if (!kDense && !DP_AB(dbg, 64)) {  // one approx pseudo-row per tile: fold the loaded one, issue the next
      if (ap_ready) ap_fold();       // (64: timing experiment, no approx pseudo-rows)
      if (ap_k < ap_n) ap_issue(bh);
    }
    if (seg_end && !DP_AB(dbg, 2)) flush(bh, reinterpret_cast<float*>(Ks));  // this stage's K buffer is the scratch
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty_bar[s]));  // stage s free for the producer
  }
  astamp(3);
  if DP_AB(dbg, 10) return;  // timing experiments: no flush / merge (2), no counters / merge (8)
  if (tid == 0) {  // profiling: rows and head segments of this CTA
    astamp_at(7, (unsigned long long)(r1 - r0));
    astamp_at(8, (unsigned long long)nflushed);
  }
  consumers_sync();  // every partial of this CTA is written (CTA scope)
  if (tid == 0) {
    // release: this CTA's reductions (observed through the barrier) are visible
    // at gpu scope before its count; acquire: the last CTA's merge reads, ordered
    // after the barrier below, see every other CTA's reductions
    // heads with no rows at all (no sink/window, nothing exact): merged by CTA bh % grid
    if (!kDense)
      for (int bh = me; bh < BH; bh += grid)
        if (rp[bh + 1] == rp[bh]) s_merge[atomicAdd(&s_nmerge, 1)] = bh;
  }
  if (kDense && tid < nflushed)  // the (<= 2) completion counters in parallel, one round trip
    if (atom_add_acq_rel(&wl.counters[flushed[tid]], 1) == head_parts(flushed[tid]) - 1)
      s_merge[atomicAdd(&s_nmerge, 1)] = flushed[tid];
  consumers_sync();
  astamp(4);

  // ---- merges of the heads I finished last (engine.py:231-246) ----------
  // partials of every CTA that touched the head + the plan's approx partial
  // (approximated clusters: logit = log-mass, value = value mean).  One
  // round trip: warp w streams partials w, w+8, ... with an online rescale,
  // then the 8 warp states are combined in shared memory.
  const int nm = DP_AB(dbg, 4) ? 0 : s_nmerge;  // (4: timing experiment, no merge)
  if (nm == 0) {
    astamp(5);
    return;
  }
  astamp(6);
  float* ored = reinterpret_cast<float*>(KV);  // [warps][8 heads][d]
  if (tid < nm) wl.counters[s_merge[tid]] = 0;  // self-reset for the next launch
  // (sparse heads with rows completed in their flushes; s_merge holds only
  // the dense heads and the sparse heads without any row)
  const int nm2 = s_nmerge;
  // (merged head, q head) pairs are spread over all 8 warps, so a CTA that
  // closes two heads merges them side by side.  Warp w takes pair
  // w % npr of the round and partials w / npr, + wpp, ...; a head with no rows
  // at all folds its approx list here instead (slow path).
  const int pairs = nm2 * G;
#pragma unroll 1
  for (int base = 0; base < pairs; base += kWarps) {
    const int npr = min(kWarps, pairs - base);
    const int wpp = kWarps / npr;  // warps per pair
    const int pr = warp % npr;
    const int mi = (base + pr) / G, g = (base + pr) % G;
    const int bh = s_merge[mi];
    const bool empty = rp[bh + 1] == rp[bh];
    const int nparts = empty ? 0 : head_parts(bh);
    const size_t pbase = (size_t)bh * pt.max_chunks * G;
    float M = -INFINITY, Lw = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!kDense && empty && warp < npr) {
      const int na = __ldcg(&wl.napprox[bh]);
      const int2* apx = wl.approx + (size_t)bh * v.cluster_cap;
      const float* vbar = v.value_means + (size_t)bh * v.cluster_cap * d;
#pragma unroll 1
      for (int j = 0; j < na; ++j) {
        const int2 e = __ldcg(&apx[j]);
        if (!((e.y >> g) & 1)) continue;
        const float x = (float)__ldcg(lm + ((size_t)bh * G + g) * v.cluster_cap + e.x);
        const float4 vv = __ldg(reinterpret_cast<const float4*>(vbar + (size_t)e.x * d) + lane);
        const float mn = fmaxf(M, x), a = __expf(M - mn), b = __expf(x - mn);
        Lw = Lw * a + b;
        acc.x = acc.x * a + b * vv.x; acc.y = acc.y * a + b * vv.y;
        acc.z = acc.z * a + b * vv.z; acc.w = acc.w * a + b * vv.w;
        M = mn;
      }
    }
    if (warp < wpp * npr) {
      constexpr int kU = 16;
#pragma unroll 1
      for (int p0 = warp / npr; p0 < nparts; p0 += kU * wpp) {
        float pm[kU], pl[kU];
        float4 po[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int p = p0 + u * wpp;
          pm[u] = -INFINITY;
          pl[u] = 0.f;
          po[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p < nparts) {
            pm[u] = __ldcg(pt.m + pbase + (size_t)p * G + g);
            pl[u] = __ldcg(pt.l + pbase + (size_t)p * G + g);
            po[u] = __ldcg(reinterpret_cast<const float4*>(pt.o + (pbase + (size_t)p * G + g) * d) + lane);
          }
        }
        float mx = M;
#pragma unroll
        for (int u = 0; u < kU; ++u) mx = fmaxf(mx, pm[u]);
        if (mx != -INFINITY) {
          const float a = __expf(M - mx);
          Lw *= a;
          acc.x *= a; acc.y *= a; acc.z *= a; acc.w *= a;
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const float b = pm[u] == -INFINITY ? 0.f : __expf(pm[u] - mx);
            Lw += pl[u] * b;
            acc.x += po[u].x * b; acc.y += po[u].y * b; acc.z += po[u].z * b; acc.w += po[u].w * b;
          }
          M = mx;
        }
      }
    }
    reinterpret_cast<float4*>(ored + (size_t)warp * d)[lane] = acc;
    if (lane == 0) {
      s_wm[warp][0] = M;
      s_wl[warp][0] = Lw;
    }
    consumers_sync();
#pragma unroll 1
    for (int i = tid; i < npr * d; i += kConsumers) {
      const int q2 = i / d, c = i - q2 * d;
      const int mi2 = (base + q2) / G, g2 = (base + q2) % G, bh2 = s_merge[mi2];
      float Mx = -INFINITY;
      for (int ww = q2; ww < wpp * npr; ww += npr) Mx = fmaxf(Mx, s_wm[ww][0]);
      float sum = 0.f, L = 0.f;
      for (int ww = q2; ww < wpp * npr; ww += npr) {
        const float wm = s_wm[ww][0];
        if (wm != -INFINITY) {
          const float f = __expf(wm - Mx);
          sum += f * ored[(size_t)ww * d + c];
          L += f * s_wl[ww][0];
        }
      }
      out[((size_t)bh2 * G + g2) * d + c] = L > 0.f ? sum / L : 0.f;
      if (c == 0) lse[(size_t)bh2 * G + g2] = L > 0.f ? Mx + __logf(L) : -INFINITY;
    }
    consumers_sync();
  }
  astamp(5);
}

}  // namespace dp
namespace dp { extern int g_plan_dbg; extern int g_plan_cl, g_pp_single, g_step_cl, g_step_off, g_step_dbg, g_seg_cost; extern float g_step_tau; }
extern "C" int dp_debug_set(int key, int value) {
  if (key == 0) dp::g_attn_debug = value;
  if (key == 1) dp::g_plan_cl = value;
  if (key == 3) dp::g_pp_single = value;
  if (key == 4) dp::g_step_tau = 0.1f * (float)value;
  if (key == 5) dp::g_step_cl = value;
  if (key == 6) dp::g_step_off = value;
  if (key == 7) dp::g_step_dbg = value;
  if (key == 9) dp::g_seg_cost = value;
  if (key == 10) dp::g_plan_dbg = value;
  if (key == 11) dp::g_gsel_path = value;
  if (key == 12) return dp::set_gsel_dbg(value);
  return 0;
}
extern "C" int dp_debug_attn_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_attn_ts, sizeof(dp::g_attn_ts)) == cudaSuccess ? 0 : 2;  // [512][12]
}
namespace dp {


size_t attn_tc_smem_bytes(int BH) { return TcSmem::fixed + (size_t)(BH + 1) * 8; }

template <bool kDense, bool kQF32>
static cudaError_t launch_tc_t(const dp_cache_view& v, const void* q, int G, double scale, const double* lm,
                               WorkLists wl, Partials<float> pt, float* out, float* lse, cudaStream_t st) {
  const int BH = v.batch * v.kv_heads;
  const size_t smem = attn_tc_smem_bytes(BH);
  ensure_smem(reinterpret_cast<const void*>(attn_tc_kernel<kDense, kQF32>), smem);
  const int sms = sm_count();
  // one persistent CTA per SM (row ranges balanced to +-1 row)
  const int grid = sms < kMaxPartSlots ? sms : kMaxPartSlots;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: prologue overlaps the plan
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_tc_kernel<kDense, kQF32>, v, q, G, (float)(scale * 1.4426950408889634), lm,
                            wl, pt, out, lse, g_attn_debug, g_seg_cost);
}

cudaError_t launch_attn_tc(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                           WorkLists wl, Partials<float> pt, float* out, float* lse, bool dense, cudaStream_t st) {
  if (attn_tc_smem_bytes(v.batch * v.kv_heads) > 227 * 1024) return cudaErrorInvalidConfiguration;
  if (qdt == DP_F32)
    return dense ? launch_tc_t<true, true>(v, q, G, scale, lm, wl, pt, out, lse, st)
                 : launch_tc_t<false, true>(v, q, G, scale, lm, wl, pt, out, lse, st);
  return dense ? launch_tc_t<true, false>(v, q, G, scale, lm, wl, pt, out, lse, st)
               : launch_tc_t<false, false>(v, q, G, scale, lm, wl, pt, out, lse, st);
}

}  // namespace dp
