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
#include "decode_internal.h"

namespace dp {

constexpr int kTcRows = kChunkRows;  // 128
constexpr int kConsumers = 256;  // 8 compute warps
constexpr int kProducers = 4;  // producer warps, 32 rows each
constexpr int kTcThreads = kConsumers + 32 * kProducers;
constexpr int kRowStride = 136;      // bf16 elements per staged row (272 B: conflict-free ldmatrix)
constexpr int kStages = 3;
constexpr int kStageElems = kTcRows * kRowStride;  // one K (or V) tile
int g_attn_debug = 0;  // profiling switches (dp_debug_set)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void ldsm_x4(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D += A * B, m16n8k16 bf16 -> f32 (a1 = a3 = 0: rows 8..15 of A are unused heads)
__device__ __forceinline__ void mma_bf16(float (&d)[4], unsigned a0, unsigned a2, unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ unsigned pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<unsigned*>(&v);
}
// split (x, y) into a bf16 hi pair + a bf16 lo pair
__device__ __forceinline__ void split2(float x, float y, unsigned& hi, unsigned& lo) {
  const __nv_bfloat16 hx = __float2bfloat16_rn(x), hy = __float2bfloat16_rn(y);
  __nv_bfloat162 h;
  h.x = hx;
  h.y = hy;
  hi = *reinterpret_cast<unsigned*>(&h);
  lo = pack_bf16(x - __bfloat162float(hx), y - __bfloat162float(hy));
}

// ---- bulk-copy engine (TMA, non-tensor) + mbarrier helpers -------------
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// the mbarrier tracks completion of this thread's prior cp.async copies
__device__ __forceinline__ void cp_async_arrive(unsigned bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
// 16-byte cp.async that writes zeros (src-size 0)
__device__ __forceinline__ void cp16_zero(unsigned dst, const void* any) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;\n" ::"r"(dst), "l"(any));
}
// barrier over the 8 compute warps only (the producer warp never joins)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumers) : "memory"); }

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// one contiguous row (bytes multiple of 16) global -> shared, completing on bar
__device__ __forceinline__ void bulk_row(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// per-CTA phase stamps (%globaltimer ns) of the last launch; profiling aid,
// read with dp_debug_attn_timing()
__device__ unsigned long long g_attn_ts[512][8];
__device__ __forceinline__ void astamp(int ev) {
  if (threadIdx.x == 0 && blockIdx.x < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_attn_ts[blockIdx.x][ev] = t;
  }
}

// owner CTA of global chunk j when T chunks are split evenly over `grid`
// CTAs as [i*T/grid, (i+1)*T/grid)
__device__ __forceinline__ int chunk_owner(long long j, long long T, int grid) {
  return (int)(((j + 1) * grid - 1) / T);
}

struct TcSmem {
  static constexpr size_t kv = (size_t)kStages * 2 * kStageElems * 2;  // K,V ring
  static constexpr size_t ps = 8 * kTcRows * 4;
  static constexpr size_t rows = (size_t)kStages * kTcRows * 4;         // head mask per stage
  static constexpr size_t fixed = kv + ps + rows;
};

template <bool kDense, bool kQF32>
__global__ void __launch_bounds__(kTcThreads, 1) attn_tc_kernel(dp_cache_view v, const void* __restrict__ q, int G,
                                                               float scale_log2, const double* __restrict__ lm,
                                                               WorkLists wl, Partials<float> pt,
                                                               float* __restrict__ out, float* __restrict__ lse,
                                                               int dbg) {
  constexpr int d = 128;
  constexpr int kWarps = kConsumers / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, tq = lane & 3;  // fragment row / column-pair
  const int BH = v.batch * v.kv_heads;
  const int grid = gridDim.x, me = blockIdx.x;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* KV = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [stage][K|V][rows][stride]
  float* Ps = reinterpret_cast<float*>(smem_raw + TcSmem::kv);      // [8 heads][rows]
  int* rmask = reinterpret_cast<int*>(smem_raw + TcSmem::kv + TcSmem::ps);  // [stage][rows]
  int* prefix = reinterpret_cast<int*>(smem_raw + TcSmem::fixed);           // [BH+1]
  __shared__ float red_m[kWarps][8], red_l[kWarps][8];
  __shared__ float s_M[8], s_L[8];
  __shared__ int s_merge[4], s_nmerge;
  __shared__ __align__(8) unsigned long long full_bar[kStages], empty_bar[kStages];

  // ---- chunk prefix over heads, my contiguous chunk range -----------------
  astamp(0);
  const int per_dense = (v.n_tokens + kTcRows - 1) / kTcRows;
  int* nrows_s = prefix + BH + 1;  // [BH] union rows per head (sparse)
  if (kDense) {
    for (int b = tid; b <= BH; b += kTcThreads) prefix[b] = b * per_dense;
  } else {
    // exclusive prefix of the per-head chunk counts (warp 0, 32 heads per step)
    for (int b = tid; b < BH; b += kTcThreads) nrows_s[b] = __ldcg(&wl.nrows[b]);
    if (warp == 0) {
      int base = 0;
      for (int b0 = 0; b0 < BH; b0 += 32) {
        const int nch = b0 + lane < BH ? (__ldcg(&wl.nrows[b0 + lane]) + kTcRows - 1) / kTcRows : 0;
        int inc = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        if (b0 + lane < BH) prefix[b0 + lane] = base + inc - nch;
        base += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) prefix[BH] = base;
    }
  }
  if (tid == 0) {
    s_nmerge = 0;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 33 * kProducers);  // per producer warp: 32 async + 1 release
      mbar_init(smem_u32(&empty_bar[i]), kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  astamp(1);
  const long long T = prefix[BH];
  const int j0 = (int)((long long)me * T / grid), j1 = (int)((long long)(me + 1) * T / grid);
  const int n = j1 - j0;
  if (n <= 0) return;
  // number of partials (CTAs with a non-empty range) of head bh
  auto head_parts = [&](int bh) {
    return T >= grid ? chunk_owner(prefix[bh + 1] - 1, T, grid) - chunk_owner(prefix[bh], T, grid) + 1
                     : prefix[bh + 1] - prefix[bh];
  };
  auto head_of = [&](int j) {  // last b with prefix[b] <= j
    int lo = 0, hi = BH - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
  };

  // ---- producer warps (rows [32p, 32p+32) each): run up to kStages ahead;
  // the next chunk's row entries are fetched while this chunk's copies issue
  if (warp >= kWarps) {
    const int ch = lane & 15, pr0 = (warp - kWarps) * 32;
    auto fetch = [&](int idx, unsigned& e, int& bh, int& v0) {
      const int j = j0 + idx;
      bh = head_of(j);
      v0 = (j - prefix[bh]) * kTcRows;
      const int nr = min(kTcRows, (kDense ? v.n_tokens : nrows_s[bh]) - v0);
      const int row = pr0 + lane;
      e = row < nr ? (kDense ? (((unsigned)((1 << G) - 1)) << 24) | (unsigned)(v0 + row)
                             : __ldg(reinterpret_cast<const unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap + v0 + row))
                   : 0xFFFFFFFFu;
    };
    unsigned e_nx;
    int bh_nx, v0_nx;
    fetch(0, e_nx, bh_nx, v0_nx);
    for (int idx = 0; idx < n; ++idx) {
      const int s = idx % kStages;
      const unsigned e = e_nx;
      const int bh = bh_nx;
      if (idx + 1 < n) fetch(idx + 1, e_nx, bh_nx, v0_nx);
      if (idx >= kStages) mbar_wait(smem_u32(&empty_bar[s]), (unsigned)(((idx / kStages) + 1) & 1));
      rmask[s * kTcRows + pr0 + lane] = e == 0xFFFFFFFFu ? 0 : (int)(e >> 24);
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
          cp16(kd, Kg + off);
          cp16(vd, Vg + off);
        } else {
          cp16_zero(kd, Kg);
          cp16_zero(vd, Vg);
        }
      }
      cp_async_arrive(smem_u32(&full_bar[s]));  // completes when this lane's copies land
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full_bar[s]));  // releases the rmask stores
    }
    return;
  }

  // Q^T B-fragments (registers): b0 = Q[head g8][k*16 + 2tq ..], b1 = Q[head g8][k*16 + 8 + 2tq ..]
  unsigned qa[8][2], qb[8][2];  // hi, lo
  auto load_q = [&](int bh) {
    const bool valid = g8 < G;
    const size_t qoff = ((size_t)bh * G + (valid ? g8 : 0)) * d;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = k * 16 + h * 8 + 2 * tq;
        if (!valid) {
          qa[k][h] = 0u;
          qb[k][h] = 0u;
        } else if (kQF32) {
          const float2 f = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(q) + qoff + col);
          split2(f.x, f.y, qa[k][h], qb[k][h]);
        } else {
          qa[k][h] = *reinterpret_cast<const unsigned*>(reinterpret_cast<const __nv_bfloat16*>(q) + qoff + col);
          qb[k][h] = 0u;
        }
      }
    }
  };

  // O^T accumulator of this warp: dims [16w, 16w+16) x heads; lane holds
  // (dim 16w+g8, heads 2tq, 2tq+1) in o[0..1] and dim +8 in o[2..3]
  float o[4];
  float m_run[2];                       // running max (log2) of heads 2tq, 2tq+1
  float m_t = -INFINITY, l_t = 0.f;     // running max / sum of head `tid` (tid < G)
  const int dim0 = warp * 16;
  int cur = -1;

  auto flush = [&](int bh) {
    const int nparts = head_parts(bh);
    // T >= grid: every CTA owns >= 1 chunk, slot = rank among the head's CTAs;
    // T < grid: non-empty CTAs own exactly one chunk, slot = chunk index
    const int slot = T >= grid ? me - chunk_owner(prefix[bh], T, grid) : j0 - prefix[bh];
    const size_t pbase = (size_t)bh * pt.max_chunks * G;
    if (tid < G) {
      pt.m[pbase + (size_t)slot * G + tid] = m_t == -INFINITY ? -INFINITY : m_t * 0.69314718055994531f;
      pt.l[pbase + (size_t)slot * G + tid] = l_t;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = 2 * tq + (e & 1), dd = dim0 + g8 + (e >> 1) * 8;
      if (h < G) pt.o[(pbase + (size_t)slot * G + h) * d + dd] = o[e];
    }
    __threadfence();
    consumers_sync();
    if (tid == 0 && atomicAdd(&wl.counters[bh], 1) == nparts - 1) s_merge[s_nmerge++] = bh;
  };

  for (int idx = 0; idx < n; ++idx) {
    const int j = j0 + idx, s = idx % kStages;
    const int bh = head_of(j);
    if (bh != cur) {
      if (cur >= 0) flush(cur);
      cur = bh;
      load_q(bh);
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = 0.f;
      m_run[0] = m_run[1] = -INFINITY;
      m_t = -INFINITY;
      l_t = 0.f;
    }
    mbar_wait(smem_u32(&full_bar[s]), (unsigned)((idx / kStages) & 1));  // stage s landed
    if (idx == 0) astamp(2);
    const __nv_bfloat16* Ks = KV + (size_t)s * 2 * kStageElems;
    const __nv_bfloat16* Vs = Ks + kStageElems;
    const int* rm = rmask + s * kTcRows;
    if (dbg & 1) {  // profiling: stream only, no math
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty_bar[s]));
      continue;
    }
    // ---- S = K Q^T for this warp's 16 rows --------------------------------
    const int r0 = warp * 16;
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const unsigned base =
          smem_u32(Ks + (r0 + (lane & 7) + ((lane >> 3) & 1) * 8) * kRowStride + (lane >> 4) * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        unsigned a0, a1, a2, a3;
        ldsm_x4(base + k * 32, a0, a1, a2, a3);
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};\n"
            : "+f"(sc[0]), "+f"(sc[1]), "+f"(sc[2]), "+f"(sc[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(qa[k][0]), "r"(qa[k][1]));
        if (kQF32)
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
              "{%0,%1,%2,%3};\n"
              : "+f"(sc[0]), "+f"(sc[1]), "+f"(sc[2]), "+f"(sc[3])
              : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(qb[k][0]), "r"(qb[k][1]));
      }
    }
    // sc[e]: row r0 + g8 + (e>>1)*8, head 2tq + (e&1)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = 2 * tq + (e & 1), r = r0 + g8 + (e >> 1) * 8;
      const bool ok = h < G && ((rm[r] >> h) & 1);
      const float val = ok ? sc[e] * scale_log2 : -INFINITY;
      sc[e] = val;
      mx[e & 1] = fmaxf(mx[e & 1], val);
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], off));
    }
    if (g8 == 0) {
      red_m[warp][2 * tq] = mx[0];
      red_m[warp][2 * tq + 1] = mx[1];
    }
    consumers_sync();
    float alpha[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float cm = -INFINITY;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) cm = fmaxf(cm, red_m[ww][2 * tq + hh]);
      const float mn = fmaxf(m_run[hh], cm);
      alpha[hh] = mn == -INFINITY ? 1.f : exp2f(m_run[hh] - mn);
      m_run[hh] = mn;
    }
    float ls[2] = {0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = 2 * tq + (e & 1), r = r0 + g8 + (e >> 1) * 8;
      const float pv = sc[e] == -INFINITY ? 0.f : exp2f(sc[e] - m_run[e & 1]);
      ls[e & 1] += pv;
      Ps[h * kTcRows + r] = pv;
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) ls[hh] += __shfl_xor_sync(0xffffffffu, ls[hh], off);
    }
    if (g8 == 0) {
      red_l[warp][2 * tq] = ls[0];
      red_l[warp][2 * tq + 1] = ls[1];
    }
    o[0] *= alpha[0];
    o[1] *= alpha[1];
    o[2] *= alpha[0];
    o[3] *= alpha[1];
    float alpha_t = 1.f;
    if (tid < G) {
      float cmt = -INFINITY;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) cmt = fmaxf(cmt, red_m[ww][tid]);
      const float mtn = fmaxf(m_t, cmt);
      alpha_t = mtn == -INFINITY ? 1.f : exp2f(m_t - mtn);
      m_t = mtn;
    }
    consumers_sync();  // Ps, red_l visible
    if (tid < G) {
      float cl = 0.f;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) cl += red_l[ww][tid];
      l_t = l_t * alpha_t + cl;
    }
    // ---- O^T += V^T P for this warp's 16 dims --------------------------------
    {
      const unsigned vbase =
          smem_u32(Vs + ((lane & 7) + ((lane >> 4) & 1) * 8) * kRowStride + dim0 + ((lane >> 3) & 1) * 8);
#pragma unroll
      for (int ks = 0; ks < kTcRows / 16; ++ks) {
        unsigned a0, a1, a2, a3;
        ldsm_x4_t(vbase + ks * 16 * kRowStride * 2, a0, a1, a2, a3);
        unsigned bh0 = 0u, bl0 = 0u, bh1 = 0u, bl1 = 0u;
        if (g8 < G) {
          const float2 p0 = *reinterpret_cast<const float2*>(Ps + g8 * kTcRows + ks * 16 + 2 * tq);
          const float2 p1 = *reinterpret_cast<const float2*>(Ps + g8 * kTcRows + ks * 16 + 8 + 2 * tq);
          split2(p0.x, p0.y, bh0, bl0);
          split2(p1.x, p1.y, bh1, bl1);
        }
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};\n"
            : "+f"(o[0]), "+f"(o[1]), "+f"(o[2]), "+f"(o[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bh0), "r"(bh1));
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};\n"
            : "+f"(o[0]), "+f"(o[1]), "+f"(o[2]), "+f"(o[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bl0), "r"(bl1));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty_bar[s]));  // stage s free for the producer
  }
  astamp(3);
  flush(cur);
  consumers_sync();
  astamp(4);

  // ---- merges of the heads I finished last (engine.py:231-246) ----------
  // partials of every CTA that touched the head + the plan's approx partial
  // (approximated clusters: logit = log-mass, value = value mean)
  const int nm = s_nmerge;
  if (nm == 0) return;
  __threadfence();
  constexpr int kMaxParts = 256;
  float* ored = reinterpret_cast<float*>(KV);        // [warps][8 heads][d]
  float* s_pm = ored + kWarps * 8 * d;               // [8][kMaxParts] partial m
  float* s_pw = s_pm + 8 * kMaxParts;                // [8][kMaxParts] partial l -> weight
  __shared__ float s_aw[8];
  for (int mi = 0; mi < nm; ++mi) {
    const int bh = s_merge[mi];
    const int nparts = min(kMaxParts, head_parts(bh));
    const size_t pbase = (size_t)bh * pt.max_chunks * G;
    if (tid == 0) wl.counters[bh] = 0;  // self-reset for the next launch
    for (int i = tid; i < G * nparts; i += kConsumers) {
      const int g = i / nparts, p = i - g * nparts;
      s_pm[g * kMaxParts + p] = __ldcg(&pt.m[pbase + (size_t)p * G + g]);
      s_pw[g * kMaxParts + p] = __ldcg(&pt.l[pbase + (size_t)p * G + g]);
    }
    consumers_sync();
    for (int g = warp; g < G; g += kWarps) {
      const float* ap = wl.apart + ((size_t)bh * G + g) * (4 + d);
      const float ma = kDense ? -INFINITY : __ldcg(&ap[0]);
      float mloc = ma;
      for (int p = lane; p < nparts; p += 32) mloc = fmaxf(mloc, s_pm[g * kMaxParts + p]);
      const float M = warp_max(mloc);
      float lloc = 0.f;
      for (int p = lane; p < nparts; p += 32) {
        const float mp = s_pm[g * kMaxParts + p];
        const float w = mp == -INFINITY ? 0.f : __expf(mp - M);
        lloc += s_pw[g * kMaxParts + p] * w;
        s_pw[g * kMaxParts + p] = w;
      }
      lloc = warp_sum(lloc);
      if (lane == 0) {
        const float wa = ma == -INFINITY ? 0.f : __expf(ma - M);
        s_aw[g] = wa;
        s_M[g] = M;
        s_L[g] = lloc + (wa > 0.f ? wa * __ldcg(&ap[1]) : 0.f);
      }
    }
    consumers_sync();
    float4 acc[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!kDense && warp == 0) {  // the approx partial
#pragma unroll
      for (int g = 0; g < 8; ++g)
        if (g < G && s_aw[g] > 0.f) {
          const float4 oa = __ldcg(reinterpret_cast<const float4*>(wl.apart + ((size_t)bh * G + g) * (4 + d) + 4) + lane);
          acc[g].x = s_aw[g] * oa.x; acc[g].y = s_aw[g] * oa.y; acc[g].z = s_aw[g] * oa.z; acc[g].w = s_aw[g] * oa.w;
        }
    }
    // partials: warp-strided, 2 partials (x G heads) in flight per lane
    for (int p0 = warp; p0 < nparts; p0 += 2 * kWarps) {
      float4 op[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int p = p0 + u * kWarps;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          op[u][g] = (p < nparts && g < G)
                         ? __ldcg(reinterpret_cast<const float4*>(pt.o + (pbase + (size_t)p * G + g) * d) + lane)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int p = p0 + u * kWarps;
        if (p < nparts) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (g < G) {
              const float w = s_pw[g * kMaxParts + p];
              acc[g].x += w * op[u][g].x; acc[g].y += w * op[u][g].y;
              acc[g].z += w * op[u][g].z; acc[g].w += w * op[u][g].w;
            }
          }
        }
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (g < G) reinterpret_cast<float4*>(ored + ((size_t)warp * 8 + g) * d)[lane] = acc[g];
    consumers_sync();
    for (int i = tid; i < G * d; i += kConsumers) {
      const int g = i / d, c = i - g * d;
      float sum = 0.f;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) sum += ored[(ww * 8 + g) * d + c];
      out[((size_t)bh * G + g) * d + c] = sum / s_L[g];
    }
    if (tid < G) lse[(size_t)bh * G + tid] = s_M[tid] + __logf(s_L[tid]);
    consumers_sync();
  }
  astamp(5);
}

}  // namespace dp
extern "C" int dp_debug_set(int key, int value) {
  if (key == 0) dp::g_attn_debug = value;
  return 0;
}
extern "C" int dp_debug_attn_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, dp::g_attn_ts, sizeof(dp::g_attn_ts)) == cudaSuccess ? 0 : 2;  // [512][8]
}
namespace dp {


size_t attn_tc_smem_bytes(int BH) { return TcSmem::fixed + (size_t)(2 * BH + 1) * 4; }

template <bool kDense, bool kQF32>
static cudaError_t launch_tc_t(const dp_cache_view& v, const void* q, int G, double scale, const double* lm,
                               WorkLists wl, Partials<float> pt, float* out, float* lse, cudaStream_t st) {
  static size_t attr = 0;
  static int sms = 0;
  const int BH = v.batch * v.kv_heads;
  const size_t smem = attn_tc_smem_bytes(BH);
  if (attr < smem) {
    cudaFuncSetAttribute(attn_tc_kernel<kDense, kQF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // one persistent CTA per SM, capped by the chunk capacity
  const int rows = kDense ? v.n_tokens : v.row_cap;
  const long long cap_chunks = (long long)BH * ((rows + kTcRows - 1) / kTcRows);
  const int grid = (int)(cap_chunks < sms ? cap_chunks : sms);
  attn_tc_kernel<kDense, kQF32><<<grid, kTcThreads, smem, st>>>(v, q, G, (float)(scale * 1.4426950408889634), lm,
                                                               wl, pt, out, lse, g_attn_debug);
  return cudaGetLastError();
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
