// Gathered split-KV decode attention for bf16 caches on tensor cores.
//
// Persistent: one CTA (4 warps) per SM.  The GQA-union rows of every
// (sequence, kv head) form a global sequence of 128-row chunks (the plan /
// worklist kernel publishes the per-head chunk prefix); CTA i owns the
// contiguous range [i*T/grid, (i+1)*T/grid) of it -- balanced to +-1 chunk
// with no atomics -- and runs an online softmax over it, flushing one partial
// (m, l, o) per head it touches.  Rows are gathered through a 3-stage
// TMA-bulk ring (64 KB of K+V per stage, two chunks in flight while one is
// computed).  Rows are moved by the bulk-copy engine (cp.async.bulk, one 256-B
// copy per K/V row into a padded 272-B smem row so ldmatrix stays
// conflict-free) completing on a per-stage mbarrier: the LSU and its
// outstanding-request limit are out of the data path.
//
//   S^T[head, row] = Q[head, :] . K[row, :]     mma.m16n8k16 bf16 -> f32, M = heads
//                                                (G <= 8 of 16), N = 8 rows, K = 16 dims
//   O[head, d]    += P[head, row] . V[row, d]   M = heads, N = 8 dims, K = 16 rows
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
constexpr int kTcThreads = 128;
constexpr int kRowStride = 136;      // bf16 elements per staged row (272 B: conflict-free ldmatrix)
constexpr int kStages = 3;
constexpr int kStageElems = kTcRows * kRowStride;  // one K (or V) tile

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
                                                               float* __restrict__ out, float* __restrict__ lse) {
  constexpr int d = 128;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int BH = v.batch * v.kv_heads;
  const int grid = gridDim.x, me = blockIdx.x;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* KV = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [stage][K|V][rows][stride]
  float* Ps = reinterpret_cast<float*>(smem_raw + TcSmem::kv);      // [8][rows]
  int* rmask = reinterpret_cast<int*>(smem_raw + TcSmem::kv + TcSmem::ps);  // [stage][rows]
  int* prefix = reinterpret_cast<int*>(smem_raw + TcSmem::fixed);           // [BH+1]
  __shared__ float red_m[32], red_l[32];
  __shared__ float s_M[8], s_L[8];
  __shared__ int s_merge[4], s_nmerge;
  __shared__ __align__(8) unsigned long long s_bar[kStages];

  // ---- chunk prefix over heads, my contiguous chunk range -----------------
  const int per_dense = (v.n_tokens + kTcRows - 1) / kTcRows;
  for (int b = tid; b <= BH; b += kTcThreads) prefix[b] = kDense ? b * per_dense : wl.chunk_prefix[b];
  if (tid == 0) {
    s_nmerge = 0;
    for (int i = 0; i < kStages; ++i) mbar_init(smem_u32(&s_bar[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const long long T = prefix[BH];
  const int j0 = (int)((long long)me * T / grid), j1 = (int)((long long)(me + 1) * T / grid);
  const int n = j1 - j0;
  if (n <= 0) return;
  auto head_of = [&](int j) {  // last b with prefix[b] <= j
    int lo = 0, hi = BH - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
  };

  // ---- producer: rows of global chunk j -> stage s through the bulk-copy
  // engine.  Thread 0 posts the stage's byte count (expect_tx) BEFORE the
  // barrier that precedes the copies; thread t then copies row t's K and V
  // (256 B each) and records its head mask.
  auto chunk_rows = [&](int j) {
    const int bh = head_of(j);
    const int rows_total = kDense ? v.n_tokens : __ldg(&wl.nrows[bh]);
    return min(kTcRows, rows_total - (j - prefix[bh]) * kTcRows);
  };
  auto expect_chunk = [&](int j, int s) {  // thread 0 only
    mbar_expect_tx(smem_u32(&s_bar[s]), (unsigned)chunk_rows(j) * (2u * d * 2u));
  };
  auto issue_chunk = [&](int j, int s) {
    const int bh = head_of(j);
    const int c = j - prefix[bh];
    const int rows_total = kDense ? v.n_tokens : __ldg(&wl.nrows[bh]);
    const int v0 = c * kTcRows;
    const int nr = min(kTcRows, rows_total - v0);
    __nv_bfloat16* Ks = KV + (size_t)s * 2 * kStageElems;
    __nv_bfloat16* Vs = Ks + kStageElems;
    int mask = 0;
    if (tid < nr) {
      int phys;
      if (kDense) {
        phys = v0 + tid;
        mask = (1 << G) - 1;
      } else {
        const unsigned e = __ldg(reinterpret_cast<const unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap + v0 + tid);
        phys = (int)(e & 0xFFFFFFu);
        mask = (int)(e >> 24);
      }
      const size_t off = ((size_t)bh * v.row_cap + phys) * d;
      const unsigned bar = smem_u32(&s_bar[s]);
      bulk_row(smem_u32(Ks + tid * kRowStride), reinterpret_cast<const __nv_bfloat16*>(v.keys) + off, d * 2, bar);
      bulk_row(smem_u32(Vs + tid * kRowStride), reinterpret_cast<const __nv_bfloat16*>(v.values) + off, d * 2, bar);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        *reinterpret_cast<int4*>(Ks + tid * kRowStride + i * 8) = make_int4(0, 0, 0, 0);
        *reinterpret_cast<int4*>(Vs + tid * kRowStride + i * 8) = make_int4(0, 0, 0, 0);
      }
    }
    rmask[s * kTcRows + tid] = mask;
  };

  // prologue: fill the ring
  if (tid == 0)
    for (int i = 0; i < kStages && i < n; ++i) expect_chunk(j0 + i, i);
  __syncthreads();
  for (int i = 0; i < kStages && i < n; ++i) issue_chunk(j0 + i, i);

  unsigned qa[8][2], qb[8][2];
  auto load_q = [&](int bh) {
    const bool valid = gq < G;
    const size_t qoff = ((size_t)bh * G + (valid ? gq : 0)) * d;
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

  float o[4][4];
  float m_run = -INFINITY;                // running max (log2 domain) of head gq
  float m_t = -INFINITY, l_t = 0.f;       // running max / sum of head `tid` (tid < G)
  const int n0 = warp * 32;
  int cur = -1;

  // flush the running state of head `bh` as my partial, count it, remember
  // the head if I am its last contributor
  auto flush = [&](int bh) {
    const int first = chunk_owner(prefix[bh], T, grid);
    const int nparts = chunk_owner(prefix[bh + 1] - 1, T, grid) - first + 1;
    const int slot = me - first;
    const size_t pbase = (size_t)bh * pt.max_chunks * G;
    if (tid < G) {
      pt.m[pbase + (size_t)slot * G + tid] = m_t == -INFINITY ? -INFINITY : m_t * 0.69314718055994531f;
      pt.l[pbase + (size_t)slot * G + tid] = l_t;
    }
    if (gq < G) {
      float* dst = pt.o + (pbase + (size_t)slot * G + gq) * d + n0 + 2 * tq;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) *reinterpret_cast<float2*>(dst + nt * 8) = make_float2(o[nt][0], o[nt][1]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0 && atomicAdd(&wl.counters[bh], 1) == nparts - 1) s_merge[s_nmerge++] = bh;
  };

  for (int idx = 0; idx < n; ++idx) {
    const int j = j0 + idx, s = idx % kStages;
    const int bh = head_of(j);
    mbar_wait(smem_u32(&s_bar[s]), (unsigned)((idx / kStages) & 1));  // stage s bytes landed
    if (bh != cur) {
      if (cur >= 0) flush(cur);
      cur = bh;
      load_q(bh);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
      m_run = -INFINITY;
      m_t = -INFINITY;
      l_t = 0.f;
    }
    __syncthreads();  // stage s landed for every thread
    const __nv_bfloat16* Ks = KV + (size_t)s * 2 * kStageElems;
    const __nv_bfloat16* Vs = Ks + kStageElems;
    const int* rm = rmask + s * kTcRows;
    // ---- S^T = Q K^T for this warp's 32 rows ------------------------------
    float sc[4][4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[jj][e] = 0.f;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int rbase = warp * 32 + jj * 8;
      const unsigned base = smem_u32(Ks + (rbase + (lane & 7)) * kRowStride + (lane >> 3) * 8);
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        unsigned b0, b1, b2, b3;
        ldsm_x4(base + kk * 32, b0, b1, b2, b3);
        mma_bf16(sc[jj], qa[kk][0], qa[kk][1], b0, b1);
        mma_bf16(sc[jj], qa[kk + 1][0], qa[kk + 1][1], b2, b3);
        if (kQF32) {
          mma_bf16(sc[jj], qb[kk][0], qb[kk][1], b0, b1);
          mma_bf16(sc[jj], qb[kk + 1][0], qb[kk + 1][1], b2, b3);
        }
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = warp * 32 + jj * 8 + 2 * tq + e;
        const bool ok = gq < G && ((rm[r] >> gq) & 1);
        const float val = ok ? sc[jj][e] * scale_log2 : -INFINITY;
        sc[jj][e] = val;
        mx = fmaxf(mx, val);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    if (tq == 0) red_m[warp * 8 + gq] = mx;
    __syncthreads();
    float cm = -INFINITY;
#pragma unroll
    for (int ww = 0; ww < 4; ++ww) cm = fmaxf(cm, red_m[ww * 8 + gq]);
    const float m_new = fmaxf(m_run, cm);
    const float alpha = m_new == -INFINITY ? 1.f : exp2f(m_run - m_new);
    m_run = m_new;
    float lsum = 0.f;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float pv = (sc[jj][e] == -INFINITY) ? 0.f : exp2f(sc[jj][e] - m_new);
        lsum += pv;
        Ps[gq * kTcRows + warp * 32 + jj * 8 + 2 * tq + e] = pv;
      }
    }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    if (tq == 0) red_l[warp * 8 + gq] = lsum;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      o[nt][0] *= alpha;
      o[nt][1] *= alpha;
    }
    float alpha_t = 1.f;
    if (tid < G) {
      float cmt = -INFINITY;
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) cmt = fmaxf(cmt, red_m[ww * 8 + tid]);
      const float mtn = fmaxf(m_t, cmt);
      alpha_t = mtn == -INFINITY ? 1.f : exp2f(m_t - mtn);
      m_t = mtn;
    }
    __syncthreads();  // Ps, red_l visible
    if (tid < G) {
      float cl = 0.f;
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) cl += red_l[ww * 8 + tid];
      l_t = l_t * alpha_t + cl;
    }
    // ---- O += P V for this warp's 32 head-dim columns ---------------------
#pragma unroll 2
    for (int ks = 0; ks < kTcRows / 16; ++ks) {
      unsigned ah0 = 0u, al0 = 0u, ah2 = 0u, al2 = 0u;
      if (gq < G) {
        const float2 p0 = *reinterpret_cast<const float2*>(Ps + gq * kTcRows + ks * 16 + 2 * tq);
        const float2 p2 = *reinterpret_cast<const float2*>(Ps + gq * kTcRows + ks * 16 + 8 + 2 * tq);
        split2(p0.x, p0.y, ah0, al0);
        split2(p2.x, p2.y, ah2, al2);
      }
      const int vrow = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int np = 0; np < 2; ++np) {
        const unsigned addr = smem_u32(Vs + vrow * kRowStride + n0 + np * 16 + (lane >> 4) * 8);
        unsigned b0, b1, b2, b3;
        ldsm_x4_t(addr, b0, b1, b2, b3);
        mma_bf16(o[2 * np], ah0, ah2, b0, b1);
        mma_bf16(o[2 * np], al0, al2, b0, b1);
        mma_bf16(o[2 * np + 1], ah0, ah2, b2, b3);
        mma_bf16(o[2 * np + 1], al0, al2, b2, b3);
      }
    }
    if (tid == 0 && idx + kStages < n) expect_chunk(j0 + idx + kStages, s);
    __syncthreads();  // stage s and Ps consumed; next expect_tx posted
    if (idx + kStages < n) issue_chunk(j0 + idx + kStages, s);
  }
  flush(cur);
  __syncthreads();
  if (tid < kStages) asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&s_bar[tid])));

  // ---- merges of the heads I finished last (engine.py:231-246) ----------
  const int nm = s_nmerge;
  if (nm == 0) return;
  __threadfence();
  float* ored = reinterpret_cast<float*>(KV);  // [4 warps][8 heads][128] scratch
  for (int mi = 0; mi < nm; ++mi) {
    const int bh = s_merge[mi];
    const int first = chunk_owner(prefix[bh], T, grid);
    const int nparts = chunk_owner(prefix[bh + 1] - 1, T, grid) - first + 1;
    const size_t pbase = (size_t)bh * pt.max_chunks * G;
    const int na = kDense ? 0 : wl.napprox[bh];
    const int2* apx = wl.approx + (size_t)bh * v.cluster_cap;
    const float* vbar = v.value_means + (size_t)bh * v.cluster_cap * d;
    if (tid == 0) wl.counters[bh] = 0;  // self-reset for the next launch
    // (1) per head: max and normaliser over partials + approx pseudo-rows
    for (int g = warp; g < G; g += 4) {
      const double* lmh = kDense ? nullptr : lm + ((size_t)bh * G + g) * v.cluster_cap;
      float mloc = -INFINITY;
      for (int p = lane; p < nparts; p += 32) mloc = fmaxf(mloc, __ldcg(&pt.m[pbase + (size_t)p * G + g]));
      for (int a = lane; a < na; a += 32) {
        const int2 e = apx[a];
        if ((e.y >> g) & 1) mloc = fmaxf(mloc, (float)lmh[e.x]);
      }
      const float M = warp_max(mloc);
      float lloc = 0.f;
      for (int p = lane; p < nparts; p += 32) {
        const float mp = __ldcg(&pt.m[pbase + (size_t)p * G + g]);
        if (mp != -INFINITY) lloc += __ldcg(&pt.l[pbase + (size_t)p * G + g]) * __expf(mp - M);
      }
      for (int a = lane; a < na; a += 32) {
        const int2 e = apx[a];
        if ((e.y >> g) & 1) lloc += __expf((float)lmh[e.x] - M);
      }
      const float L = warp_sum(lloc);
      if (lane == 0) {
        s_M[g] = M;
        s_L[g] = L;
      }
    }
    __syncthreads();
    // (2) weighted sums: warps stride over partials and approx rows, lanes over d
    float4 acc[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = warp; p < nparts; p += 4) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < G) {
          const float mp = __ldcg(&pt.m[pbase + (size_t)p * G + g]);
          const float4 op = __ldcg(reinterpret_cast<const float4*>(pt.o + (pbase + (size_t)p * G + g) * d) + lane);
          const float w = mp == -INFINITY ? 0.f : __expf(mp - s_M[g]);
          acc[g].x += w * op.x; acc[g].y += w * op.y; acc[g].z += w * op.z; acc[g].w += w * op.w;
        }
      }
    }
    for (int a = warp; a < na; a += 4) {
      const int2 e = apx[a];
      const float4 vb = *(reinterpret_cast<const float4*>(vbar + (size_t)e.x * d) + lane);
      float lmv = 0.f;  // lane g fetches head g's log-mass, broadcast below
      if (lane < G && ((e.y >> lane) & 1)) lmv = (float)lm[((size_t)bh * G + lane) * v.cluster_cap + e.x];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float lg = __shfl_sync(0xffffffffu, lmv, g);
        if (g < G && ((e.y >> g) & 1)) {
          const float w = __expf(lg - s_M[g]);
          acc[g].x += w * vb.x; acc[g].y += w * vb.y; acc[g].z += w * vb.z; acc[g].w += w * vb.w;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (g < G) reinterpret_cast<float4*>(ored + ((size_t)warp * 8 + g) * d)[lane] = acc[g];
    __syncthreads();
    for (int i = tid; i < G * d; i += kTcThreads) {
      const int g = i / d, c = i - g * d;
      const float sum = ored[(0 * 8 + g) * d + c] + ored[(1 * 8 + g) * d + c] + ored[(2 * 8 + g) * d + c] +
                        ored[(3 * 8 + g) * d + c];
      out[((size_t)bh * G + g) * d + c] = sum / s_L[g];
    }
    if (tid < G) lse[(size_t)bh * G + tid] = s_M[tid] + __logf(s_L[tid]);
    __syncthreads();
  }
}

size_t attn_tc_smem_bytes(int BH) { return TcSmem::fixed + (size_t)(BH + 1) * 4; }

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
                                                               wl, pt, out, lse);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                           WorkLists wl, Partials<float> pt, float* out, float* lse, bool dense, cudaStream_t st) {
  if ((size_t)(v.batch * v.kv_heads + 1) * 4 + TcSmem::fixed > 227 * 1024) return cudaErrorInvalidConfiguration;
  if (qdt == DP_F32)
    return dense ? launch_tc_t<true, true>(v, q, G, scale, lm, wl, pt, out, lse, st)
                 : launch_tc_t<false, true>(v, q, G, scale, lm, wl, pt, out, lse, st);
  return dense ? launch_tc_t<true, false>(v, q, G, scale, lm, wl, pt, out, lse, st)
               : launch_tc_t<false, false>(v, q, G, scale, lm, wl, pt, out, lse, st);
}

}  // namespace dp
