// Gathered split-KV decode attention for bf16 caches on tensor cores.
//
// One CTA (4 warps) per (row chunk of 128, b*h).  The chunk's rows are the
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
// writes an unnormalised partial (m, l, o) per head that merge_kernel folds
// together with the approx pseudo-rows (engine.py:216-252).
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
                                                            float scale_log2, WorkLists wl, Partials<float> pt) {
  const int bh = blockIdx.y, c = blockIdx.x;
  const int rows_total = kDense ? v.n_tokens : wl.nrows[bh];
  const int nchunk = (rows_total + kTcRows - 1) / kTcRows;
  if (c >= nchunk) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int v0 = c * kTcRows;
  const int nr = min(kTcRows, rows_total - v0);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* Vs = Ks + kTcRows * kRowStride;
  float* Ps = reinterpret_cast<float*>(Vs + kTcRows * kRowStride);  // [8][kTcRows]
  int* rmask = reinterpret_cast<int*>(Ps + 8 * kTcRows);            // [kTcRows]
  float* red = reinterpret_cast<float*>(rmask + kTcRows);           // [4][8] max, [4][8] sum

  // ---- row -> physical row + head mask (thread per row) -----------------
  int phys = -1, mask = 0;
  {
    const int r = tid;
    if (r < nr) {
      const int vr = v0 + r;
      if (kDense) {
        phys = vr;
        mask = (1 << G) - 1;
      } else {
        const int4* runs = wl.runs + (size_t)bh * (v.cluster_cap + 2);
        int lo = 0, hi = wl.nruns[bh] - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (__ldg(&runs[mid].w) <= vr) lo = mid; else hi = mid - 1;
        }
        const int4 ru = runs[lo];
        phys = ru.x + (vr - ru.w);
        mask = ru.z;
      }
    }
    rmask[r] = mask;
  }
  // ---- stage K (group 0) and V (group 1) --------------------------------
  const int d = 128;
  const size_t head_off = (size_t)bh * v.row_cap * d;
  const __nv_bfloat16* Kg = reinterpret_cast<const __nv_bfloat16*>(v.keys) + head_off;
  const __nv_bfloat16* Vg = reinterpret_cast<const __nv_bfloat16*>(v.values) + head_off;
  // each thread copies its own row (16 x 16 B), rows are contiguous runs
  {
    const unsigned kd = smem_u32(Ks + tid * kRowStride);
    if (phys >= 0) {
      const __nv_bfloat16* src = Kg + (size_t)phys * d;
#pragma unroll
      for (int j = 0; j < 16; ++j) cp16(kd + j * 16, src + j * 8);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) *reinterpret_cast<int4*>(Ks + tid * kRowStride + j * 8) = make_int4(0, 0, 0, 0);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const unsigned vd = smem_u32(Vs + tid * kRowStride);
    if (phys >= 0) {
      const __nv_bfloat16* src = Vg + (size_t)phys * d;
#pragma unroll
      for (int j = 0; j < 16; ++j) cp16(vd + j * 16, src + j * 8);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) *reinterpret_cast<int4*>(Vs + tid * kRowStride + j * 8) = make_int4(0, 0, 0, 0);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }

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
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  __syncthreads();

  // ---- S^T = Q K^T for this warp's 32 rows ------------------------------
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
  // scale (log2 domain) + head mask; lane holds head gq, rows warp*32 + j*8 + 2tq + {0,1}
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
  if (tq == 0 && gq < 8) red[warp * 8 + gq] = mx;
  __syncthreads();
  float m = -INFINITY;
  if (gq < 8) {
#pragma unroll
    for (int w = 0; w < 4; ++w) m = fmaxf(m, red[w * 8 + gq]);
  }
  float lsum = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float p = (m == -INFINITY || s[j][e] == -INFINITY) ? 0.f : exp2f(s[j][e] - m);
      lsum += p;
      if (gq < 8) Ps[gq * kTcRows + warp * 32 + j * 8 + 2 * tq + e] = p;
    }
  }
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
  if (tq == 0 && gq < 8) red[32 + warp * 8 + gq] = lsum;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  if (tid < G) {
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) l += red[32 + w * 8 + tid];
    const size_t pi = ((size_t)bh * pt.max_chunks + c) * G + tid;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) mm = fmaxf(mm, red[w * 8 + tid]);
    pt.m[pi] = mm == -INFINITY ? -INFINITY : mm * 0.69314718055994531f;  // back to natural log
    pt.l[pi] = l;
  }

  // ---- O = P V for this warp's 32 head-dim columns ------------------------
  float o[4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
  const int n0 = warp * 32;
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
  if (gq < G) {
    float* dst = pt.o + (((size_t)bh * pt.max_chunks + c) * G + gq) * d + n0 + 2 * tq;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) *reinterpret_cast<float2*>(dst + nt * 8) = make_float2(o[nt][0], o[nt][1]);
  }
}

size_t attn_tc_smem_bytes() {
  return (size_t)2 * kTcRows * kRowStride * 2 + 8 * kTcRows * 4 + kTcRows * 4 + 64 * 4;
}

template <bool kDense, bool kQF32>
static cudaError_t launch_tc_t(const dp_cache_view& v, const void* q, int G, double scale, WorkLists wl,
                               Partials<float> pt, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel<kDense, kQF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)attn_tc_smem_bytes());
    attr = true;
  }
  const int rows = kDense ? v.n_tokens : v.row_cap;
  dim3 grid((rows + kTcRows - 1) / kTcRows, v.batch * v.kv_heads);
  attn_tc_kernel<kDense, kQF32><<<grid, kTcThreads, attn_tc_smem_bytes(), st>>>(
      v, q, G, (float)(scale * 1.4426950408889634), wl, pt);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const dp_cache_view& v, const void* q, int qdt, int G, double scale, WorkLists wl,
                           Partials<float> pt, bool dense, cudaStream_t st) {
  if (qdt == DP_F32)
    return dense ? launch_tc_t<true, true>(v, q, G, scale, wl, pt, st) : launch_tc_t<false, true>(v, q, G, scale, wl, pt, st);
  return dense ? launch_tc_t<true, false>(v, q, G, scale, wl, pt, st) : launch_tc_t<false, false>(v, q, G, scale, wl, pt, st);
}

}  // namespace dp
