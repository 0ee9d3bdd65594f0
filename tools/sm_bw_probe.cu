// Per-SM streaming throughput of the staging methods the one-launch decode
// step can use (profiling aid, not product code).  Each CTA streams its own
// contiguous share of two 2-D bf16 [rows, 128] tensors (K and V) through a
// 3-stage ring of 128-row x 256-B tiles (64 KB per stage, K + V) and only
// releases the stages (no math), at a chosen grid size (e.g. 80 = the step
// kernel's SM count, 148 = every SM):
//   0  cp.async 16 B, 4 warps issue (the first step-kernel producer)
//   1  TMA 2-D box 64 cols x 8 rows   (1 KB, 128B swizzle) x 64 per tile
//   2  TMA 2-D box 64 cols x 64 rows  (8 KB, 128B swizzle) x 8 per tile
//   3  cp.async.bulk 1-D, 8 KB        x 8 per tile
//   4  TMA 2-D box 64 cols x 32 rows  (4 KB) x 16 per tile
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sm_bw_probe tools/sm_bw_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int ROWS = 128, STAGES = 3, TILE = ROWS * 256;

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(unsigned bar, unsigned par) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(bar),
      "r"(par)
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(160, 1) ring(const __grid_constant__ CUtensorMap k8, const __grid_constant__ CUtensorMap v8,
                                               const __grid_constant__ CUtensorMap k64, const __grid_constant__ CUtensorMap v64,
                                               const __grid_constant__ CUtensorMap k32, const __grid_constant__ CUtensorMap v32,
                                               const char* __restrict__ kg, const char* __restrict__ vg, int ntiles_total,
                                               int* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (su(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = (int)((long long)blockIdx.x * ntiles_total / gridDim.x);
  const int t1 = (int)((long long)(blockIdx.x + 1) * ntiles_total / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(MODE == 0 ? 4 * 33 : 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 4) {  // consumer: wait + release
    for (int i = 0; i < t1 - t0; ++i) {
      const int s = i % STAGES;
      wait(su(&full[s]), (i / STAGES) & 1);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
    return;
  }
  for (int i = 0; i < t1 - t0; ++i) {
    const int s = i % STAGES, t = t0 + i;
    if (i >= STAGES) wait(su(&empty[s]), ((i / STAGES) + 1) & 1);
    unsigned char* K = sm + (size_t)s * 2 * TILE;
    unsigned char* V = K + TILE;
    const unsigned fb = su(&full[s]);
    if (MODE == 0) {
      const char* ks = kg + (size_t)t * TILE;
      const char* vs = vg + (size_t)t * TILE;
      for (int j = 0; j < 16; ++j) {
        const int idx = j * 128 + tid, row = idx >> 4, c = idx & 15;
        const unsigned so = row * 256 + ((c ^ (row & 7)) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(K + so)), "l"(ks + row * 256 + c * 16));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(V + so)), "l"(vs + row * 256 + c * 16));
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fb) : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
    } else if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(2 * TILE) : "memory");
      const int row0 = t * ROWS;
      if (MODE == 3) {
        for (int b = 0; b < 4; ++b) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(
                           su(K + b * 8192)),
                       "l"(kg + (size_t)t * TILE + b * 8192), "r"(fb)
                       : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(
                           su(V + b * 8192)),
                       "l"(vg + (size_t)t * TILE + b * 8192), "r"(fb)
                       : "memory");
        }
      } else if (MODE == 5 || MODE == 6) {
        unsigned long long pol = 0;
        if (MODE == 6) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        // runs of 72 rows (9 groups) cut into 32 + 32 + 8 row boxes, 16 groups per tile
        for (int g = 0; g < 16;) {
          const int b = (g % 9) < 8 ? (((g % 9) + 4 <= 8) ? 4 : 1) : 1;
          const int bb = (g + b > 16) ? 16 - g : b;
          const int bx = bb >= 4 ? 4 : (bb >= 2 ? 2 : 1);
          const CUtensorMap* km = bx == 4 ? &k32 : &k8;
          const CUtensorMap* vm = bx == 4 ? &v32 : &v8;
          const int n = bx == 4 ? 1 : bb;
          for (int u = 0; u < n; ++u)
            for (int hf = 0; hf < 2; ++hf) {
              if (MODE == 5) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                        su(K + hf * ROWS * 128 + (g + u) * 1024)),
                    "l"(km), "r"(hf * 64), "r"(row0 + (g + u) * 8), "r"(fb)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                        su(V + hf * ROWS * 128 + (g + u) * 1024)),
                    "l"(vm), "r"(hf * 64), "r"(row0 + (g + u) * 8), "r"(fb)
                    : "memory");
              } else {
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                        su(K + hf * ROWS * 128 + (g + u) * 1024)),
                    "l"(km), "r"(hf * 64), "r"(row0 + (g + u) * 8), "r"(fb), "l"(pol)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                        su(V + hf * ROWS * 128 + (g + u) * 1024)),
                    "l"(vm), "r"(hf * 64), "r"(row0 + (g + u) * 8), "r"(fb), "l"(pol)
                    : "memory");
              }
            }
          g += bx == 4 ? 4 : n;
        }
      } else {
        const int R = MODE == 1 ? 8 : (MODE == 2 ? 64 : 32);
        const CUtensorMap* km = MODE == 1 ? &k8 : (MODE == 2 ? &k64 : &k32);
        const CUtensorMap* vm = MODE == 1 ? &v8 : (MODE == 2 ? &v64 : &v32);
        for (int g = 0; g < ROWS / R; ++g)
          for (int hf = 0; hf < 2; ++hf) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    su(K + hf * ROWS * 128 + g * R * 128)),
                "l"(km), "r"(hf * 64), "r"(row0 + g * R), "r"(fb)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    su(V + hf * ROWS * 128 + g * R * 128)),
                "l"(vm), "r"(hf * 64), "r"(row0 + g * R), "r"(fb)
                : "memory");
          }
      }
    }
  }
  if (tid == 0 && t1 < t0) *sink = 1;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void mk(EncFn fn, CUtensorMap* m, void* p, unsigned long long rows, unsigned R) {
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t str[1] = {256};
  const cuuint32_t box[2] = {64, R};
  const cuuint32_t es[2] = {1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    exit(1);
  }
}

int main(int argc, char** argv) {
  const size_t rows = 8ull * 32768 * 2;  // 2 layers of 8 heads x 32K rows: 134 MB per tensor (> L2)
  char *k, *v;
  int* sink;
  cudaMalloc(&k, rows * 256);
  cudaMalloc(&v, rows * 256);
  cudaMalloc(&sink, 4);
  cudaMemset(k, 1, rows * 256);
  cudaMemset(v, 2, rows * 256);
  EncFn fn;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &qr);
  CUtensorMap k8, v8, k64, v64, k32, v32;
  mk(fn, &k8, k, rows, 8);
  mk(fn, &v8, v, rows, 8);
  mk(fn, &k64, k, rows, 64);
  mk(fn, &v64, v, rows, 64);
  mk(fn, &k32, k, rows, 32);
  mk(fn, &v32, v, rows, 32);
  const int ntiles = (int)(rows / ROWS);
  const size_t smem = (size_t)STAGES * 2 * TILE + 1024;
  void* fns[7] = {(void*)ring<0>, (void*)ring<1>, (void*)ring<2>, (void*)ring<3>, (void*)ring<4>, (void*)ring<5>, (void*)ring<6>};
  for (auto f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[7] = {"cp.async 16B (4 warps)", "TMA 64x8 boxes", "TMA 64x64 boxes", "bulk 1-D 8 KB", "TMA 64x32 boxes",
                          "TMA mixed 32/8 boxes", "TMA mixed + evict_first"};
  int grids[3] = {80, 112, 148};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int m = 0; m < 7; ++m)
    for (int gi = 0; gi < 3; ++gi) {
      const int grid = grids[gi];
      // each CTA streams the same number of tiles regardless of grid: 48 tiles (3 MB)
      const int nt = grid * 48 < ntiles ? grid * 48 : ntiles;
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        switch (m) {
          case 0: ring<0><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
          case 1: ring<1><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
          case 2: ring<2><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
          case 3: ring<3><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
          case 4: ring<4><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
          case 5: ring<5><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
          default: ring<6><<<grid, 160, smem>>>(k8, v8, k64, v64, k32, v32, k, v, nt, sink); break;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double bytes = (double)nt * 2 * TILE;
      printf("%-24s grid %3d: %7.1f GB/s total, %6.1f GB/s per SM  (%s)\n", names[m], grid, bytes / best / 1e6,
             bytes / best / 1e6 / grid, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
