// HBM read-bandwidth probe for K/V staging strategies (profiling aid, not
// product code).  Streams two 67 MB arrays (K and V rows of 256 B, the
// 8-head x 32K bf16 layer of the bench) the ways the attention kernel can:
//   A  LDG.128 into registers               (grid = SMs x 8, 256 thr)
//   B  cp.async 16 B into a 3-stage smem ring  (1 CTA/SM, 128 thr)
//   C  cp.async.bulk per 256-B row, 3 stages   (1 CTA/SM, 128 thr)
//   D  cp.async.bulk per 32-row block (8 KB)   (1 CTA/SM, 128 thr)
//   E  cp.async 16 B, one chunk per CTA, 3 CTAs/SM (the old kernel)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr int ROWB = 256, ROWS_PER_CHUNK = 128, STRIDE = 272, STAGES = 3;

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe_a(const int4* __restrict__ k, const int4* __restrict__ v, size_t n16, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    int4 a = __ldg(&k[i]), b = __ldg(&v[i]);
    acc.x ^= a.x ^ b.x; acc.y ^= a.y ^ b.y; acc.z ^= a.z ^ b.w; acc.w ^= a.w ^ b.z;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345) *sink = 1;
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe_ring(const char* __restrict__ k, const char* __restrict__ v, int nchunks,
                                                     int* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  const int tid = threadIdx.x;
  const int j0 = (int)((long long)blockIdx.x * nchunks / gridDim.x), j1 = (int)((long long)(blockIdx.x + 1) * nchunks / gridDim.x);
  const int n = j1 - j0;
  if (tid == 0)
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
  __syncthreads();
  auto issue = [&](int j, int s) {
    unsigned char* K = sm + (size_t)s * 2 * ROWS_PER_CHUNK * STRIDE;
    unsigned char* V = K + ROWS_PER_CHUNK * STRIDE;
    const char* kg = k + (size_t)j * ROWS_PER_CHUNK * ROWB;
    const char* vg = v + (size_t)j * ROWS_PER_CHUNK * ROWB;
    if (MODE == 0) {  // cp.async 16B, warp copies 2 rows per instr
      for (int i = 0; i < 16; ++i) {
        const int idx = i * 128 + tid, row = idx >> 4, c = idx & 15;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(K + row * STRIDE + c * 16)), "l"(kg + row * ROWB + c * 16));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(V + row * STRIDE + c * 16)), "l"(vg + row * ROWB + c * 16));
      }
      asm volatile("cp.async.commit_group;");
    } else if (MODE == 1) {  // bulk per row
      if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(ROWS_PER_CHUNK * ROWB * 2));
      __syncthreads();
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(su(K + tid * STRIDE)), "l"(kg + tid * ROWB), "r"(su(&bar[s])) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(su(V + tid * STRIDE)), "l"(vg + tid * ROWB), "r"(su(&bar[s])) : "memory");
    } else {  // bulk per 32-row block (unpadded)
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(ROWS_PER_CHUNK * ROWB * 2));
        for (int b = 0; b < 4; ++b) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(su(K + b * 8192)), "l"(kg + b * 8192), "r"(su(&bar[s])) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(su(V + b * 8192)), "l"(vg + b * 8192), "r"(su(&bar[s])) : "memory");
        }
      }
    }
  };
  for (int i = 0; i < STAGES && i < n; ++i) issue(j0 + i, i);
  int acc = 0;
  for (int idx = 0; idx < n; ++idx) {
    const int s = idx % STAGES;
    if (MODE == 0) {
      const int ahead = min(STAGES - 1, n - 1 - idx);
      if (ahead >= 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (ahead == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
      asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(su(&bar[s])), "r"((idx / STAGES) & 1) : "memory");
    }
    __syncthreads();
    acc += sm[(size_t)s * 2 * ROWS_PER_CHUNK * STRIDE + tid * 16];
    __syncthreads();
    if (idx + STAGES < n) issue(j0 + idx + STAGES, s);
  }
  if (acc == 0x7fffffff) *sink = acc;
}

__global__ void __launch_bounds__(128) probe_e(const char* __restrict__ k, const char* __restrict__ v, int nchunks, int* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int j = blockIdx.x, tid = threadIdx.x;
  if (j >= nchunks) return;
  unsigned char* K = sm;
  unsigned char* V = sm + ROWS_PER_CHUNK * STRIDE;
  const char* kg = k + (size_t)j * ROWS_PER_CHUNK * ROWB;
  const char* vg = v + (size_t)j * ROWS_PER_CHUNK * ROWB;
  for (int i = 0; i < 16; ++i) {
    const int idx = i * 128 + tid, row = idx >> 4, c = idx & 15;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(K + row * STRIDE + c * 16)), "l"(kg + row * ROWB + c * 16));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(V + row * STRIDE + c * 16)), "l"(vg + row * ROWB + c * 16));
  }
  asm volatile("cp.async.commit_group; cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (sm[tid * 16] == 0x7f && sm[tid * 16 + 1] == 0x3e) *sink = 1;
}


// TMA tensor probes: 128-row chunks, K and V each split in two 64-column
// (128 B) halves, 128B swizzle.  MODE 3: one box {64,128} per half;
// MODE 4: boxes {64,8}; MODE 5: tile::gather4 with box {64,1}.
template <int MODE>
__global__ void __launch_bounds__(128, 1) probe_tma(const __grid_constant__ CUtensorMap km, const __grid_constant__ CUtensorMap vm,
                                                    int nchunks, int* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  const int tid = threadIdx.x;
  const int j0 = (int)((long long)blockIdx.x * nchunks / gridDim.x), j1 = (int)((long long)(blockIdx.x + 1) * nchunks / gridDim.x);
  const int n = j1 - j0;
  unsigned char* base = sm + ((1024 - (su(sm) & 1023)) & 1023);
  if (tid == 0)
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
  __syncthreads();
  auto issue = [&](int j, int s) {
    if (tid != 0) return;
    const unsigned b = su(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(ROWS_PER_CHUNK * ROWB * 2));
    unsigned char* st = base + (size_t)s * 65536;
    const int row0 = j * ROWS_PER_CHUNK;
    for (int t = 0; t < 2; ++t) {
      const unsigned long long m = t == 0 ? (unsigned long long)&km : (unsigned long long)&vm;
      for (int h = 0; h < 2; ++h) {
        unsigned char* dst = st + t * 32768 + h * 16384;
        if (MODE == 3) {
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(su(dst)), "l"(m), "r"(h * 64), "r"(row0), "r"(b) : "memory");
        } else if (MODE == 4) {
          for (int r = 0; r < ROWS_PER_CHUNK; r += 8)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su(dst + r * 128)), "l"(m), "r"(h * 64), "r"(row0 + r), "r"(b) : "memory");
        } else {
          for (int r = 0; r < ROWS_PER_CHUNK; r += 4)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         ::"r"(su(dst + r * 128)), "l"(m), "r"(h * 64), "r"(row0 + r), "r"(row0 + r + 1), "r"(row0 + r + 2), "r"(row0 + r + 3), "r"(b) : "memory");
        }
      }
    }
  };
  for (int i = 0; i < STAGES && i < n; ++i) issue(j0 + i, i);
  int acc = 0;
  for (int idx = 0; idx < n; ++idx) {
    const int s = idx % STAGES;
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(su(&bar[s])), "r"((idx / STAGES) & 1) : "memory");
    __syncthreads();
    acc += base[(size_t)s * 65536 + tid * 16];
    __syncthreads();
    if (idx + STAGES < n) issue(j0 + idx + STAGES, s);
  }
  if (acc == 0x7fffffff) *sink = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap make_map(const char* p, size_t rows, unsigned boxrows) {
  static EncFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, boxrows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d (box rows %u)\n", (int)r, boxrows);
  return m;
}

int main() {
  const size_t bytes = (size_t)8 * 32768 * ROWB;  // one of K/V per layer
  const int layers = 8;                             // cycle layers so L2 never holds the data
  char *k, *v;
  int* sink;
  cudaMalloc(&k, bytes * layers);
  cudaMalloc(&v, bytes * layers);
  cudaMalloc(&sink, 4);
  cudaMemset(k, 1, bytes * layers);
  cudaMemset(v, 2, bytes * layers);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nchunks = (int)(bytes / (ROWS_PER_CHUNK * ROWB));
  const size_t ring = (size_t)STAGES * 2 * ROWS_PER_CHUNK * STRIDE;
  cudaFuncSetAttribute(probe_ring<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring);
  cudaFuncSetAttribute(probe_ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring);
  cudaFuncSetAttribute(probe_ring<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring);
  cudaFuncSetAttribute(probe_e, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWS_PER_CHUNK * STRIDE);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"A ldg.128 regs (SMs x8 CTAs)", "B cp.async16 ring 1CTA/SM", "C bulk/row ring 1CTA/SM",
                         "D bulk/8KB ring 1CTA/SM", "E cp.async16 1chunk/CTA 3/SM", "A2 ldg.128 (SMs x32 CTAs)",
                         "F TMA box 64x128 swz ring", "G TMA box 64x8 swz ring", "H TMA gather4 swz ring"};
  const size_t tring = (size_t)STAGES * 65536 + 1024;
  cudaFuncSetAttribute(probe_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tring);
  cudaFuncSetAttribute(probe_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tring);
  cudaFuncSetAttribute(probe_tma<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tring);
  const size_t rows = bytes / ROWB;
  CUtensorMap kmF[8], vmF[8], kmG[8], vmG[8], kmH[8], vmH[8];
  for (int l = 0; l < layers; ++l) {
    kmF[l] = make_map(k + l * bytes, rows, 128); vmF[l] = make_map(v + l * bytes, rows, 128);
    kmG[l] = make_map(k + l * bytes, rows, 8); vmG[l] = make_map(v + l * bytes, rows, 8);
    kmH[l] = make_map(k + l * bytes, rows, 1); vmH[l] = make_map(v + l * bytes, rows, 1);
  }
  for (int mode = 0; mode < 9; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      for (int l = 0; l < layers; ++l) {
        const char* kl = k + l * bytes;
        const char* vl = v + l * bytes;
        if (mode == 0) probe_a<<<sms * 8, 256>>>((const int4*)kl, (const int4*)vl, bytes / 16, sink);
        if (mode == 5) probe_a<<<sms * 32, 256>>>((const int4*)kl, (const int4*)vl, bytes / 16, sink);
        if (mode == 1) probe_ring<0><<<sms, 128, ring>>>(kl, vl, nchunks, sink);
        if (mode == 2) probe_ring<1><<<sms, 128, ring>>>(kl, vl, nchunks, sink);
        if (mode == 3) probe_ring<2><<<sms, 128, ring>>>(kl, vl, nchunks, sink);
        if (mode == 4) probe_e<<<nchunks, 128, 2 * ROWS_PER_CHUNK * STRIDE>>>(kl, vl, nchunks, sink);
        if (mode == 6) probe_tma<3><<<sms, 128, tring>>>(kmF[l], vmF[l], nchunks, sink);
        if (mode == 7) probe_tma<4><<<sms, 128, tring>>>(kmG[l], vmG[l], nchunks, sink);
        if (mode == 8) probe_tma<5><<<sms, 128, tring>>>(kmH[l], vmH[l], nchunks, sink);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-34s %8.1f GB/s  (%.1f us per 134 MB layer)\n", names[mode], 2.0 * bytes * layers / (ms * 1e-3) / 1e9, ms * 1e3 / layers);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
