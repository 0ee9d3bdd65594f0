// Gathered split-KV decode attention for bf16 caches on tensor cores.
//
// Each CTA (4 warps) owns `cpc` consecutive 128-row chunks of one (b, kv
// head) and runs an online softmax over them; the next chunk's K rows are
// fetched while the current chunk's PV runs.  The chunk's rows are the
// GQA-union rows of the head (sink, window, members of clusters exact for
// >= 1 q head of the group); cluster runs are contiguous in HBM, so the
// 16-byte cp.async copies are coalesced.  K then V are staged into padded
// shared memory (272-byte rows: conflict-free ldmatrix), in two cp.async
// groups so V streams in while QK runs.
//
//   S^T[head, row] = Q[head, :] . K[row, :]     mma.m16n8k16 bf16, M = heads (G <= 8
//                                                of 16 used), N = 8 rows, K = 16 dims
//   O[head, d]    += P[head, row] . V[row, d]   M = heads, N = 8 dims, K = 16 rows
//
// P is split hi + lo into two bf16 operands (two MMAs), so the weights keep
// ~2^-16 relative precision; an fp32 query is split the same way.  The chunk
// writes an unnormalised partial (m, l, o) per head; the last chunk of a head
// to finish (atomic counter) folds all partials together with the approx
// pseudo-rows (engine.py:216-252), so no separate merge launch is needed.
// CTAs are indexed by a compact work index (prefix over per-head chunk
// counts), so active chunks are dispatched first.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "decode_internal.h"

namespace dp {

constexpr int kTcRows = kChunkRows;  // 128
constexpr int kTcThreads = 128;
constexpr int kRowStride = 136;      // bf16 elements per staged row (272 B)

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
// split (x, y) into bf16 hi pair + bf16 lo pair
__device__ __forceinline__ void split2(float x, float y, unsigned& hi, unsigned& lo) {
  const __nv_bfloat16 hx = __float2bfloat16_rn(x), hy = __float2bfloat16_rn(y);
  __nv_bfloat162 h;
  h.x = hx;
  h.y = hy;
  hi = *reinterpret_cast<unsigned*>(&h);
  lo = pack_bf16(x - __bfloat162float(hx), y - __bfloat162float(hy));
}

template <bool kDense, bool kQF32>
__global__ void __launch_bounds__(kTcThreads) attn_tc_kernel(dp_cache_view v, const void* __restrict__ q, int G,
                                                            float scale_log2, const double* __restrict__ lm,
                                                            WorkLists wl, Partials<float> pt, float* __restrict__ out,
                                                            float* __restrict__ lse, int cpc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int BH = v.batch * v.kv_heads;
  const int w = blockIdx.x;
  constexpr int d = 128;
  __shared__ int s_bh, s_cta, s_ncta, s_last;
  __shared__ float red_m[32], red_l[32];
  // ---- compact work index -> (head, CTA of that head) ---------------------
  if (kDense) {
    const int per = ((v.n_tokens + kTcRows - 1) / kTcRows + cpc - 1) / cpc;
    if (tid == 0) {
      s_bh = w / per < BH ? w / per : -1;
      s_cta = w % per;
      s_ncta = per;
    }
  } else if (warp == 0) {
    int base = 0, found = 0;
    for (int b0 = 0; b0 < BH && !found; b0 += 32) {
      const int n = b0 + lane < BH ? (wl.nchunks[b0 + lane] + cpc - 1) / cpc : 0;
      int inc = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      const bool hit = b0 + lane < BH && w >= base + inc - n && w < base + inc;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        s_bh = b0 + lane;
        s_cta = w - (base + inc - n);
        s_ncta = n;
      }
      found = bal != 0;
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (!found && lane == 0) s_bh = -1;
  }
  __syncthreads();
  const int bh = s_bh, cta = s_cta, ncta = s_ncta;
  if (bh < 0) return;
  const int rows_total = kDense ? v.n_tokens : wl.nrows[bh];
  const int nch_head = (rows_total + kTcRows - 1) / kTcRows;
  const int c_begin = cta * cpc, c_end = min(c_begin + cpc, nch_head);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* Vs = Ks + kTcRows * kRowStride;
  float* Ps = reinterpret_cast<float*>(Vs + kTcRows * kRowStride);  // [8][kTcRows]
  int* rmask = reinterpret_cast<int*>(Ps + 8 * kTcRows);            // [kTcRows]
  int* rphys = rmask + kTcRows;                                     // [kTcRows]

  const size_t head_off = (size_t)bh * v.row_cap * d;
  const __nv_bfloat16* Kg = reinterpret_cast<const __nv_bfloat16*>(v.keys) + head_off;
  const __nv_bfloat16* Vg = reinterpret_cast<const __nv_bfloat16*>(v.values) + head_off;

  // rows of chunk c -> (physical row, head mask) in smem; ends with a barrier
  auto map_rows = [&](int c) {
    const int v0 = c * kTcRows;
    const int nr = min(kTcRows, rows_total - v0);
    int phys = -1, mask = 0;
    if (kDense) {
      if (tid < nr) {
        phys = v0 + tid;
        mask = (1 << G) - 1;
      }
    } else {
      if (tid < nr) {
        const unsigned e = __ldg(reinterpret_cast<const unsigned*>(wl.rowidx) + (size_t)bh * v.row_cap + v0 + tid);
        phys = (int)(e & 0xFFFFFFu);
        mask = (int)(e >> 24);
      }
    }
    rmask[tid] = mask;
    rphys[tid] = phys;
    __syncthreads();
  };
  // a warp copies 2 rows = 512 contiguous bytes per instruction
  auto issue = [&](const __nv_bfloat16* G0, __nv_bfloat16* S0) {
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int idx = i * kTcThreads + tid;
      const int row = idx >> 4, ch = idx & 15;
      const int pr = rphys[row];
      __nv_bfloat16* dst = S0 + row * kRowStride + ch * 8;
      if (pr >= 0) cp16(smem_u32(dst), G0 + (size_t)pr * d + ch * 8);
      else *reinterpret_cast<int4*>(dst) = make_int4(0, 0, 0, 0);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  map_rows(c_begin);
  issue(Kg, Ks);
  issue(Vg, Vs);

  // ---- Q fragments (registers): a0 = Q[g][k*16 + 2t..], a2 = Q[g][k*16 + 8 + 2t..]
  unsigned qa[8][2], qb[8][2];  // hi, lo
  {
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
  }

  float o[4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
  const int n0 = warp * 32;
  float m_run = -INFINITY;                 // running max (log2 domain) of head gq
  float m_t = -INFINITY, l_t = 0.f;        // running max / sum of head `tid` (tid < G)

  for (int c = c_begin; c < c_end; ++c) {
    const bool has_next = c + 1 < c_end;
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // K_c landed (V_c may still stream)
    __syncthreads();
    // ---- S^T = Q K^T for this warp's 32 rows ----------------------------
    float s[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rbase = warp * 32 + j * 8;
      const unsigned base = smem_u32(Ks + (rbase + (lane & 7)) * kRowStride + (lane >> 3) * 8);
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        unsigned b0, b1, b2, b3;
        ldsm_x4(base + kk * 32, b0, b1, b2, b3);
        mma_bf16(s[j], qa[kk][0], qa[kk][1], b0, b1);
        mma_bf16(s[j], qa[kk + 1][0], qa[kk + 1][1], b2, b3);
        if (kQF32) {
          mma_bf16(s[j], qb[kk][0], qb[kk][1], b0, b1);
          mma_bf16(s[j], qb[kk + 1][0], qb[kk + 1][1], b2, b3);
        }
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = warp * 32 + j * 8 + 2 * tq + e;
        const bool ok = gq < G && ((rmask[r] >> gq) & 1);
        const float val = ok ? s[j][e] * scale_log2 : -INFINITY;
        s[j][e] = val;
        mx = fmaxf(mx, val);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    if (tq == 0) red_m[warp * 8 + gq] = mx;
    __syncthreads();  // Ks, rmask free; chunk maxima visible
    float cm = -INFINITY;
#pragma unroll
    for (int ww = 0; ww < 4; ++ww) cm = fmaxf(cm, red_m[ww * 8 + gq]);
    const float m_new = fmaxf(m_run, cm);
    const float alpha = m_new == -INFINITY ? 1.f : exp2f(m_run - m_new);
    m_run = m_new;
    float lsum = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float pv = (s[j][e] == -INFINITY) ? 0.f : exp2f(s[j][e] - m_new);
        lsum += pv;
        Ps[gq * kTcRows + warp * 32 + j * 8 + 2 * tq + e] = pv;
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
    if (tid < G) {  // running (m, l) of head tid
      float cmt = -INFINITY;
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) cmt = fmaxf(cmt, red_m[ww * 8 + tid]);
      const float mtn = fmaxf(m_t, cmt);
      l_t *= (mtn == -INFINITY ? 1.f : exp2f(m_t - mtn));
      m_t = mtn;
    }
    if (has_next) {  // prefetch the next chunk's K while PV runs
      map_rows(c + 1);
      issue(Kg, Ks);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // V_c landed
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();  // Ps / red_l / V_c visible
    if (tid < G) {
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) l_t += red_l[ww * 8 + tid];
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
    __syncthreads();  // Vs, Ps consumed
    if (has_next) issue(Vg, Vs);
  }

  // ---- this CTA's partial (m natural-log, l, o) ---------------------------
  const size_t pbase = (size_t)bh * pt.max_chunks * G;
  if (tid < G) {
    pt.m[pbase + (size_t)cta * G + tid] = m_t == -INFINITY ? -INFINITY : m_t * 0.69314718055994531f;
    pt.l[pbase + (size_t)cta * G + tid] = l_t;
  }
  if (gq < G) {
    float* dst = pt.o + (pbase + (size_t)cta * G + gq) * d + n0 + 2 * tq;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) *reinterpret_cast<float2*>(dst + nt * 8) = make_float2(o[nt][0], o[nt][1]);
  }

  // ---- fused LSE merge by the last CTA of this head (engine.py:231-246) --
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&wl.counters[bh], 1) == ncta - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) wl.counters[bh] = 0;  // self-reset for the next launch
  const int na = kDense ? 0 : wl.napprox[bh];
  const int2* apx = wl.approx + (size_t)bh * v.cluster_cap;
  const float* vbar = v.value_means + (size_t)bh * v.cluster_cap * d;
  for (int g = warp; g < G; g += kTcThreads / 32) {
    const int hq = bh * G + g;
    const double* lmh = kDense ? nullptr : lm + (size_t)hq * v.cluster_cap;
    float mloc = -INFINITY;
    for (int cc = lane; cc < ncta; cc += 32) mloc = fmaxf(mloc, __ldcg(&pt.m[pbase + (size_t)cc * G + g]));
    for (int a = lane; a < na; a += 32) {
      const int2 e = apx[a];
      if ((e.y >> g) & 1) mloc = fmaxf(mloc, (float)lmh[e.x]);
    }
    const float M = warp_max(mloc);
    float lloc = 0.f;
    for (int cc = lane; cc < ncta; cc += 32) {
      const float mc = __ldcg(&pt.m[pbase + (size_t)cc * G + g]);
      if (mc != -INFINITY) lloc += __ldcg(&pt.l[pbase + (size_t)cc * G + g]) * __expf(mc - M);
    }
    for (int a = lane; a < na; a += 32) {
      const int2 e = apx[a];
      if ((e.y >> g) & 1) lloc += __expf((float)lmh[e.x] - M);
    }
    const float L = warp_sum(lloc);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int cc = 0; cc < ncta; ++cc) {
      const float mc = __ldcg(&pt.m[pbase + (size_t)cc * G + g]);
      const float4 oc = __ldcg(reinterpret_cast<const float4*>(pt.o + (pbase + (size_t)cc * G + g) * d) + lane);
      const float wgt = mc == -INFINITY ? 0.f : __expf(mc - M);
      acc.x += wgt * oc.x; acc.y += wgt * oc.y; acc.z += wgt * oc.z; acc.w += wgt * oc.w;
    }
    // approx pseudo-rows: lanes fetch (cluster, weight) 32 at a time, then the
    // warp streams the value-mean rows with the weights broadcast by shuffle
    for (int a0 = 0; a0 < na; a0 += 32) {
      int k = 0;
      float wgt = 0.f;
      if (a0 + lane < na) {
        const int2 e = apx[a0 + lane];
        k = e.x;
        if ((e.y >> g) & 1) wgt = __expf((float)lmh[e.x] - M);
      }
      const int nb = min(32, na - a0);
#pragma unroll 4
      for (int b = 0; b < nb; ++b) {
        const float wb = __shfl_sync(0xffffffffu, wgt, b);
        const int kb = __shfl_sync(0xffffffffu, k, b);
        if (wb != 0.f) {
          const float4 vb = *(reinterpret_cast<const float4*>(vbar + (size_t)kb * d) + lane);
          acc.x += wb * vb.x; acc.y += wb * vb.y; acc.z += wb * vb.z; acc.w += wb * vb.w;
        }
      }
    }
    const float inv = 1.f / L;
    reinterpret_cast<float4*>(out + (size_t)hq * d)[lane] =
        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (lane == 0) lse[hq] = M + __logf(L);
  }
}

size_t attn_tc_smem_bytes() {
  return (size_t)2 * kTcRows * kRowStride * 2 + 8 * kTcRows * 4 + 2 * kTcRows * 4;
}

template <bool kDense, bool kQF32>
static cudaError_t launch_tc_t(const dp_cache_view& v, const void* q, int G, double scale, const double* lm,
                               WorkLists wl, Partials<float> pt, float* out, float* lse, cudaStream_t st) {
  static bool attr = false;
  static int sms = 148;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel<kDense, kQF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)attn_tc_smem_bytes());
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const int BH = v.batch * v.kv_heads;
  const int rows = kDense ? v.n_tokens : v.row_cap;
  const int max_chunks = (rows + kTcRows - 1) / kTcRows;
  // chunks per CTA: aim for ~3 resident CTAs per SM over the expected work
  // (dense: every row; sparse: ~40% GQA-union rows, SURVEY.md §0 finding 4)
  const double expect = (double)BH * max_chunks * (kDense ? 1.0 : 0.4);
  int cpc = (int)(expect / (3.0 * sms) + 0.5);
  cpc = cpc < 1 ? 1 : (cpc > 16 ? 16 : cpc);
  const int grid = BH * ((max_chunks + cpc - 1) / cpc);  // upper bound; extra CTAs exit
  attn_tc_kernel<kDense, kQF32><<<grid, kTcThreads, attn_tc_smem_bytes(), st>>>(
      v, q, G, (float)(scale * 1.4426950408889634), lm, wl, pt, out, lse, cpc);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const dp_cache_view& v, const void* q, int qdt, int G, double scale, const double* lm,
                           WorkLists wl, Partials<float> pt, float* out, float* lse, bool dense, cudaStream_t st) {
  if (qdt == DP_F32)
    return dense ? launch_tc_t<true, true>(v, q, G, scale, lm, wl, pt, out, lse, st)
                 : launch_tc_t<false, true>(v, q, G, scale, lm, wl, pt, out, lse, st);
  return dense ? launch_tc_t<true, false>(v, q, G, scale, lm, wl, pt, out, lse, st)
               : launch_tc_t<false, false>(v, q, G, scale, lm, wl, pt, out, lse, st);
}

}  // namespace dp
